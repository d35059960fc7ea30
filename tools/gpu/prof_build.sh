# near-list build: wall time per case, then ncu launch lists (per-kernel durations)
python tools/time_build.py c2/dense,c2/literal,c5/literal,c5/dense > gpurun_out/build_times.log 2>&1
for c in "c5 dense" "c2 dense" "c5 literal"; do
  set -- $c
  ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/build_launch_$1_$2.csv python tools/prof_build.py $1 $2 > /dev/null 2>&1
done
