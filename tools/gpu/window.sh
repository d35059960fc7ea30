timeout 600 python -m pytest tests/test_gpu_window.py -x -q -m gpu -s > gpurun_out/t_win.log 2>&1; echo rc=$? >> gpurun_out/t_win.log
for f in 1 0; do
  for c in "c2 literal" "c4 literal" "c1 literal"; do
    set -- $c
    echo -n "win=$f "; GIGAQBX_WINDOW=$f timeout 300 python tools/profile_case.py --case $1 --preset $2 --reps 3 2>&1 | tail -1
  done
done > gpurun_out/win_cases.log 2>&1
