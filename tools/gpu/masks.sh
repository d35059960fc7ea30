# exact route with member masks: parity tests, then C5 build time with and without
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fused.py -x -q -k "near_list or fused" > gpurun_out/t_masks.log 2>&1; echo rc=$? >> gpurun_out/t_masks.log
for m in 1 0; do
  echo "GIGAQBX_EXACT_MASKS=$m"
  GIGAQBX_EXACT_MASKS=$m timeout 600 python tools/time_build.py c5/dense,c5/literal,c2/dense,c2/literal,c4/dense,c4/literal 2>&1 | grep "sell=True"
done > gpurun_out/masks_time.log 2>&1
