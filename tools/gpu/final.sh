# end-of-session check: full GPU suite, bench (both arms), launch list, one ncu --set full capture of the headline kernel
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/t_all.log 2>&1; echo rc=$? >> gpurun_out/t_all.log
timeout 1200 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo rc=$? >> gpurun_out/bench.err
timeout 900 python bench.py --impl reference > gpurun_out/bref.json 2> gpurun_out/bref.err; echo rc=$? >> gpurun_out/bref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 2 --warmup 3 --no-secondary --no-cpu-baseline --no-e2e > gpurun_out/ncu_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:helmholtz_sell -s 3 -c 1 -o gpurun_out/ncu_c5dense_s4b python tools/profile_case.py --case c5 --preset dense --reps 3 > gpurun_out/ncu_c5.log 2>&1
NCCL_DEBUG=WARN timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --force-dist --steps 10 --warmup 3 > gpurun_out/bd.json 2> gpurun_out/bd.err; echo rc=$? >> gpurun_out/bd.err
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo rc=$? >> gpurun_out/smoke.log
