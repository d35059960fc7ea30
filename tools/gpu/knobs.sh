for v in default gd2 ring2; do
  unset GIGAQBX_LIB_PATH
  if [ $v != default ]; then export GIGAQBX_LIB_PATH=paper_1811_01110_b200/_lib/variants/$v.so; fi
  [ $v != default ] && [ ! -f $GIGAQBX_LIB_PATH ] && continue
  for c in "c5 dense" "c3 dense" "c2 dense" "c4 dense" "c5 literal" "c3 literal"; do
    set -- $c
    echo -n "$v: "; timeout 300 python tools/profile_case.py --case $1 --preset $2 --reps 3 2>&1 | tail -1
  done
done > gpurun_out/knobs.log 2>&1
