ncu --set full --clock-control none --import-source on -k regex:sweep_cell_kernel -s 3 -c 3 -o gpurun_out/ncu_masks_c5dense python tools/prof_build.py c5 dense > gpurun_out/ncu_masks.log 2>&1
