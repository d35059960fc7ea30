for v in default helm3 onet; do
  unset GIGAQBX_LIB_PATH GIGAQBX_ONE_TARGET
  if [ $v = helm3 ]; then export GIGAQBX_LIB_PATH=paper_1811_01110_b200/_lib/variants/helm3.so; fi
  if [ $v = onet ]; then export GIGAQBX_ONE_TARGET=1; fi
  for c in "c3 literal" "c3 dense" "c5 literal" "c2 literal"; do
    set -- $c
    echo -n "$v: "; timeout 300 python tools/profile_case.py --case $1 --preset $2 --reps 3 2>&1 | tail -1
  done
done > gpurun_out/helm_ab.log 2>&1
