#!/bin/bash
# near-list build time of each library variant (tools/time_build.py)
CASES=${1:-c2/dense,c2/literal,c4/dense,c5/literal}
for v in paper_1811_01110_b200/_lib/var_*.so; do
  echo "== $v"
  GIGAQBX_LIB_PATH=$PWD/$v python tools/time_build.py $CASES 2>&1 | grep True
done
