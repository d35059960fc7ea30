"""Per-kernel time of an ncu launch list (second half of the launches: the
warm repetition), aggregated by kernel name.

    python tools/launch_summary.py gpurun_out/build_launch_c2_dense.csv [...]
"""
import collections
import csv
import sys

for f in sys.argv[1:]:
    rows = list(csv.reader(open(f)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    data = rows[hi + 1:]
    tot, agg = 0.0, collections.OrderedDict()
    for r in data[len(data) // 2:]:
        v = float(r[vi].replace(",", ""))
        agg[r[ki][:70]] = agg.get(r[ki][:70], 0.0) + v
        tot += v
    print(f"{f}: total {tot / 1e3:.1f} us")
    for k, v in agg.items():
        print(f"   {v / 1e3:9.1f} us  {k}")
