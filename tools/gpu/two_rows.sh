timeout 600 python -m pytest tests/test_gpu_two_rows.py -x -q -m gpu -s > gpurun_out/t_two.log 2>&1; echo rc=$? >> gpurun_out/t_two.log
for f in 1 0; do
  for c in "c2 literal" "c4 literal" "c1 literal" "c2 dense"; do
    set -- $c
    echo -n "two=$f "; GIGAQBX_TWO_ROWS=$f timeout 300 python tools/profile_case.py --case $1 --preset $2 --reps 3 2>&1 | tail -1
  done
done > gpurun_out/two_cases.log 2>&1
