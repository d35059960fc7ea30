timeout 600 python -m pytest tests/test_gpu_p2p.py -x -q -m gpu > gpurun_out/t_p2p.log 2>&1; echo rc=$? >> gpurun_out/t_p2p.log
timeout 300 python tools/p2p_bench.py > gpurun_out/p2p_default.log 2>&1
GIGAQBX_LIB_PATH=paper_1811_01110_b200/_lib/variants/p2plib.so timeout 300 python tools/p2p_bench.py > gpurun_out/p2p_lib.log 2>&1
