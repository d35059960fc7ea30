#!/bin/bash
python tools/sweep.py --lanes 0 --cases c2/dense,c2/literal,c3/dense,c3/literal 2>&1 | grep G=
echo "== one target per pass"
GIGAQBX_ONE_TARGET=1 python tools/sweep.py --lanes 0 --cases c2/dense,c2/literal,c3/dense,c3/literal 2>&1 | grep G=
