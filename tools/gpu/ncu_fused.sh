timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/fused_launch_c5_dense.csv python tools/prof_fused.py c5 dense > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fused_kernel -s 1 -c 1 -o gpurun_out/ncu_fused_c5dense python tools/prof_fused.py c5 dense > /dev/null 2>&1
