# A/B of Helmholtz variants on C5 dense / C3 dense / C5 literal (kernel time, no flush)
for v in default fwd cl_minb2 cl_minb4; do
  if [ $v = default ]; then unset GIGAQBX_LIB_PATH; else export GIGAQBX_LIB_PATH=paper_1811_01110_b200/_lib/variants/$v.so; fi
  for c in "c5 dense" "c3 dense" "c5 literal" "c3 literal"; do
    set -- $c
    echo -n "$v: "; python tools/profile_case.py --case $1 --preset $2 --reps 3 2>&1 | tail -1
  done
done
unset GIGAQBX_LIB_PATH
python -m pytest tests/test_gpu_timed_path.py tests/test_gpu_parity.py -q -x -m gpu -k "helmholtz or c3 or c5 or variants or order_sweep" 2>&1 | tail -3
