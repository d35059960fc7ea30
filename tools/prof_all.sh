#!/bin/bash
# ncu captures of the top kernels (run under gpurun; one GPU).
#   tools/prof_all.sh TAG "name|ENV=..|case|preset|kernel-regex" ...
TAG=$1; shift
O=gpurun_out
for spec in "$@"; do
  IFS='|' read -r name envs case preset rx <<< "$spec"
  env $envs python tools/profile_case.py --case $case --preset $preset > $O/plain_$name.log 2>&1 &&
  env $envs ncu --set full --clock-control none --import-source on -k regex:$rx -s 2 -c 1 \
      -o $O/${TAG}_$name python tools/profile_case.py --case $case --preset $preset \
      > $O/ncu_$name.log 2>&1
done
