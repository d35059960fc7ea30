# C5 dense Helmholtz kernel: timing, then one ncu --set full capture
python tools/profile_case.py --case c5 --preset dense --reps 3 > gpurun_out/pc5.log 2>&1
python tools/profile_case.py --case c3 --preset dense --reps 3 >> gpurun_out/pc5.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:helmholtz_sell -s 3 -c 1 \
    -o gpurun_out/ncu_c5dense_r02a python tools/profile_case.py --case c5 --preset dense --reps 3 \
    > gpurun_out/ncu_c5.log 2>&1
