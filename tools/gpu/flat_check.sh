timeout 600 python -m pytest tests/test_gpu_flat.py -x -q -m gpu -s > gpurun_out/t_flat.log 2>&1; echo rc=$? >> gpurun_out/t_flat.log
timeout 600 python -m pytest tests/test_gpu_timed_path.py -x -q -m gpu -k "literal" > gpurun_out/t_timed_lit.log 2>&1; echo rc=$? >> gpurun_out/t_timed_lit.log
for f in 1 0; do
  for c in "c1 literal" "c2 literal" "c4 literal" "c2 dense"; do
    set -- $c
    echo -n "flat=$f "; GIGAQBX_FLAT=$f timeout 300 python tools/profile_case.py --case $1 --preset $2 --reps 3 2>&1 | tail -1
  done
done > gpurun_out/flat_cases.log
