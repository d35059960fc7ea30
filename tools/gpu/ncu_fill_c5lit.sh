ncu --set full --clock-control none --import-source on -k regex:sweep_cell_kernel -s 2 -c 2 -o gpurun_out/ncu_fill_c5lit python tools/prof_build.py c5 literal > /dev/null 2>&1
