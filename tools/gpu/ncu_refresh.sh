# fresh ncu --set full captures of the secondary presets' kernels, summarised on the box
# (only the JSON summaries come back: the reports together exceed the 64 MiB pull limit)
mkdir -p /tmp/ncu_s4
for c in "c3 dense helmholtz_sell" "c3 literal helmholtz_sell" "c2 dense laplace_sell" "c2 literal laplace_sell" "c4 dense laplace_sell" "c5 literal helmholtz_sell"; do
  set -- $c
  timeout 600 ncu --set full --clock-control none -k regex:$3 -s 3 -c 1 -o /tmp/ncu_s4/ncu_$1_$2_s4 python tools/profile_case.py --case $1 --preset $2 --reps 3 > /dev/null 2>&1
  python tools/ncu_summary.py /tmp/ncu_s4/ncu_$1_$2_s4.ncu-rep --json gpurun_out/ncu_summary_$1_$2_s4.json > /dev/null 2>&1
done
