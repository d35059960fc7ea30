# near-list build launch lists (per-kernel durations) + one full capture of the C5 dense kernel
for c in "c5 dense" "c2 dense" "c5 literal" "c2 literal"; do
  set -- $c
  ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/build_launch_$1_$2.csv python tools/prof_build.py $1 $2 > /dev/null 2>&1
done
ncu --set full --clock-control none --import-source on -k regex:helmholtz_sell -s 3 -c 1 \
    -o gpurun_out/ncu_c5dense_s3 python tools/profile_case.py --case c5 --preset dense --reps 3 \
    > gpurun_out/ncu_c5.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:laplace_sell -s 3 -c 1 \
    -o gpurun_out/ncu_c2lit_s3 python tools/profile_case.py --case c2 --preset literal --reps 3 \
    > gpurun_out/ncu_c2lit.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:sweep_cell -s 2 -c 3 \
    -o gpurun_out/ncu_build_c2dense_s3 python tools/prof_build.py c2 dense \
    > gpurun_out/ncu_build.log 2>&1
