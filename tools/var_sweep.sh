#!/bin/bash
# Compare library variants built with different -D flags:
#   tools/var_sweep.sh [case list, default c2/c3 both presets]
CASES=${1:-c2/dense,c2/literal,c3/dense,c3/literal}
for v in paper_1811_01110_b200/_lib/var_*.so; do
  echo "== $v"
  GIGAQBX_LIB_PATH=$PWD/$v python tools/sweep.py --lanes 0 --cases $CASES 2>&1 | grep G=
done
