NCCL_DEBUG=WARN timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --force-dist --steps 10 --warmup 3 > gpurun_out/bd.json 2> gpurun_out/bd.err; echo rc=$? >> gpurun_out/bd.err
timeout 900 python bench.py --impl reference --steps 5 --warmup 2 > gpurun_out/bref.json 2> gpurun_out/bref.err; echo rc=$? >> gpurun_out/bref.err
timeout 600 python -m pytest tests/test_gpu_distributed.py -x -q -m gpu > gpurun_out/t_dist.log 2>&1; echo rc=$? >> gpurun_out/t_dist.log
