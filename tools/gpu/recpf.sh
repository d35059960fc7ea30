timeout 900 python -m pytest tests/test_gpu_timed_path.py tests/test_gpu_parity.py -x -q -m gpu > gpurun_out/t_recpf.log 2>&1; echo rc=$? >> gpurun_out/t_recpf.log
for v in default nopfr; do
  unset GIGAQBX_LIB_PATH
  if [ $v != default ]; then export GIGAQBX_LIB_PATH=paper_1811_01110_b200/_lib/variants/$v.so; fi
  for c in "c2 literal" "c4 literal" "c3 literal" "c5 literal" "c2 dense" "c3 dense" "c4 dense" "c5 dense"; do
    set -- $c
    echo -n "$v: "; timeout 300 python tools/profile_case.py --case $1 --preset $2 --reps 3 2>&1 | tail -1
  done
done > gpurun_out/recpf.log 2>&1
