timeout 900 python -m pytest tests/test_gpu_fused.py -x -q -m gpu -s > gpurun_out/t_fused.log 2>&1; echo rc=$? >> gpurun_out/t_fused.log
timeout 900 python tools/e2e_fused.py c2/dense c2/literal c3/dense c4/literal c5/literal c5/dense > gpurun_out/e2e_fused.log 2>&1
