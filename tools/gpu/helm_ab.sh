# Helmholtz S SELL kernels: parity, then timings of the Helmholtz presets for the in-tree
# library and every variant under _lib/variants/ (tools/build_variant.sh)
timeout 900 python -m pytest tests/test_gpu_timed_path.py tests/test_gpu_parity.py tests/test_gpu_fused.py -x -q -k "c5 or c3 or helm or Helm or fused" > gpurun_out/t_helm.log 2>&1; echo rc=$? >> gpurun_out/t_helm.log
for v in default $(ls paper_1811_01110_b200/_lib/variants/*.so 2>/dev/null); do
  unset GIGAQBX_LIB_PATH
  [ $v != default ] && export GIGAQBX_LIB_PATH=$PWD/$v
  for c in "c5 dense" "c5 literal" "c3 dense" "c3 literal"; do
    set -- $c
    echo -n "$v "; timeout 300 python tools/profile_case.py --case $1 --preset $2 --reps 5 2>&1 | tail -1
  done
done > gpurun_out/helm_time.log 2>&1
