# near-list builder: GPU suite, build wall times, launch lists (per-kernel durations)
python -m pytest tests -x -q -m gpu > gpurun_out/t_all.log 2>&1; echo rc=$? >> gpurun_out/t_all.log
python tools/time_build.py ${CASES:-c2/dense,c2/literal,c4/literal,c4/dense,c5/literal,c5/dense} > gpurun_out/build_times.log 2>&1
for c in ${LAUNCH_CASES:-"c5 dense" "c2 dense" "c5 literal"}; do
  set -- $(echo $c | tr / ' ')
  ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/build_launch_$1_$2.csv python tools/prof_build.py $1 $2 > /dev/null 2>&1
done
