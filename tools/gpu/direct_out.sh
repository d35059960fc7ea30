timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_timed_path.py -x -q -m gpu -k "not near" > gpurun_out/t_do.log 2>&1; echo rc=$? >> gpurun_out/t_do.log
timeout 600 python tools/e2e_fused.py c5/dense c5/literal c2/dense c3/dense c4/dense > gpurun_out/do.log 2>&1
