python tools/time_build.py c5/literal,c5/dense > gpurun_out/bt_default.log 2>&1
GIGAQBX_LIB_PATH=paper_1811_01110_b200/_lib/variants/ml16.so python tools/time_build.py c5/literal,c5/dense > gpurun_out/bt_ml16.log 2>&1
GIGAQBX_LIB_PATH=paper_1811_01110_b200/_lib/variants/ml16.so ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/bl_ml16_c5_dense.csv python tools/prof_build.py c5 dense > /dev/null 2>&1
GIGAQBX_LIB_PATH=paper_1811_01110_b200/_lib/variants/ml16.so ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/bl_ml16_c5_literal.csv python tools/prof_build.py c5 literal > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:sweep_cell_kernel -s 2 -c 3 -o gpurun_out/ncu_build_c2dense_s3b python tools/prof_build.py c2 dense > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:sweep_cell_kernel -s 2 -c 3 -o gpurun_out/ncu_build_c5lit_s3b python tools/prof_build.py c5 literal > /dev/null 2>&1
