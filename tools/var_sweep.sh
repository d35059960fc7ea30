#!/bin/bash
for v in paper_1811_01110_b200/_lib/var_*.so; do
  echo "== $v"
  GIGAQBX_LIB_PATH=$PWD/$v python tools/sweep.py --lanes 0 --cases c2/dense,c2/literal,c3/dense,c3/literal 2>&1 | grep G=
done
