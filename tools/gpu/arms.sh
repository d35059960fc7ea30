# both bench arms the way the driver runs them, with wall times; then smoke()
( time timeout 1200 python bench.py --impl reference > gpurun_out/bref.json 2> gpurun_out/bref.err ) 2> gpurun_out/bref.time
( time timeout 1200 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err ) 2> gpurun_out/bench.time
( time python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1 ) 2> gpurun_out/smoke.time
