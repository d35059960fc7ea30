# Round state: full GPU suite, default bench (with secondary), kernel timings per case,
# near-list build times, launch list of the bench.
set -x
python -m pytest tests -x -q -m gpu > gpurun_out/t_all.log 2>&1; echo rc=$? >> gpurun_out/t_all.log
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo rc=$? >> gpurun_out/bench.err
for c in "c2 dense" "c2 literal" "c3 dense" "c3 literal" "c4 dense" "c4 literal" "c5 dense" "c5 literal"; do
  set -- $c
  python tools/profile_case.py --case $1 --preset $2 --reps 3 2>&1 | tail -1
done > gpurun_out/cases.log
python tools/time_build.py c2/dense,c2/literal,c4/literal,c5/literal,c5/dense > gpurun_out/build_times.log 2>&1
