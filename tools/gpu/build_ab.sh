# near-list builder A/B (default vs variants in $VARIANTS) + near-list GPU tests
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "near" > gpurun_out/t_near.log 2>&1; echo rc=$? >> gpurun_out/t_near.log
timeout 300 python tools/time_build.py ${CASES:-c2/dense,c2/literal,c4/literal,c4/dense,c5/literal,c5/dense} > gpurun_out/bt_default.log 2>&1
for v in $VARIANTS; do
  GIGAQBX_LIB_PATH=paper_1811_01110_b200/_lib/variants/$v.so timeout 300 python tools/time_build.py ${CASES:-c2/dense,c2/literal,c4/literal,c4/dense,c5/literal,c5/dense} > gpurun_out/bt_$v.log 2>&1
  GIGAQBX_LIB_PATH=paper_1811_01110_b200/_lib/variants/$v.so timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "near" > gpurun_out/t_near_$v.log 2>&1; echo rc=$? >> gpurun_out/t_near_$v.log
done
for c in ${LAUNCH_CASES:-c5/dense c2/dense c5/literal c2/literal}; do
  set -- $(echo $c | tr / ' ')
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/build_launch_$1_$2.csv python tools/prof_build.py $1 $2 > /dev/null 2>&1
done
