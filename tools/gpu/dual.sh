# dual-source Helmholtz (NT = 1, long rows): parity then timing
timeout 900 python -m pytest tests/test_gpu_timed_path.py tests/test_gpu_parity.py -x -q -k "c5 or helm or Helm" > gpurun_out/t_dual.log 2>&1; echo rc=$? >> gpurun_out/t_dual.log
for c in "c5 dense" "c5 literal"; do
  set -- $c
  timeout 300 python tools/profile_case.py --case $1 --preset $2 --reps 5 2>&1 | tail -1
done > gpurun_out/dual_time.log 2>&1
