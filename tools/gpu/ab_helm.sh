# A/B of Helmholtz variants on C5 / C3 (kernel time, no flush) + Helmholtz parity
for v in default vote; do
  if [ $v = default ]; then unset GIGAQBX_LIB_PATH; else export GIGAQBX_LIB_PATH=paper_1811_01110_b200/_lib/variants/$v.so; fi
  for c in "c5 dense" "c3 dense" "c5 literal" "c3 literal"; do
    set -- $c
    echo -n "$v: "; python tools/profile_case.py --case $1 --preset $2 --reps 3 2>&1 | tail -1
  done
done
unset GIGAQBX_LIB_PATH
python -m pytest tests/test_gpu_timed_path.py tests/test_gpu_parity.py -q -x -m gpu 2>&1 | tail -3
# near-list build: wall time per case, then ncu launch lists (per-kernel durations)
python tools/time_build.py c2/dense,c2/literal,c5/literal,c5/dense > gpurun_out/build_times.log 2>&1
for c in "c5 dense" "c2 dense" "c5 literal"; do
  set -- $c
  ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/build_launch_$1_$2.csv python tools/prof_build.py $1 $2 > /dev/null 2>&1
done
