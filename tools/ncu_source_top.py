"""Top source lines of one kernel in an ncu report (instructions executed and
warp-stall samples per CUDA source line; needs -lineinfo).

    python tools/ncu_source_top.py report.ncu-rep 'sweep_cell_kernel<(int)1>' [N]
"""
import csv
import io
import subprocess
import sys

rep, pat = sys.argv[1], sys.argv[2]
n_top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
sections, cur = [], None
for r in rows:
    if len(r) >= 2 and r[0] == "Function Name":
        cur = {"name": r[1], "lines": []}
        sections.append(cur)
    elif cur is not None and len(r) > 8 and r[0].isdigit() and r[2] == "-":
        cur["lines"].append(r)
    elif cur is not None and len(r) > 8 and r[0] == "Line No":
        cur["hdr"] = r
# a kernel has one section per source file it inlines code from: merge them
merged = {}
for sec in sections:
    if pat not in sec["name"] or not sec["lines"]:
        continue
    m = merged.setdefault(sec["name"], {"name": sec["name"], "lines": [], "hdr": sec["hdr"]})
    m["lines"] += sec["lines"]
for sec in merged.values():
    h = sec["hdr"]
    ie, sm = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
    tot_i = sum(float(r[ie] or 0) for r in sec["lines"])
    tot_s = sum(float(r[sm] or 0) for r in sec["lines"])
    print(f"{sec['name'][:90]}\n  instructions {tot_i:.3e}, samples {tot_s:.0f}")
    for key, col in (("instructions", ie), ("stall samples", sm)):
        print(f"  top lines by {key}:")
        for r in sorted(sec["lines"], key=lambda r: -float(r[col] or 0))[:n_top]:
            print(f"   {r[0]:>5} {100 * float(r[ie] or 0) / tot_i:5.1f}% inst {100 * float(r[sm] or 0) / max(tot_s, 1):5.1f}% smp  {r[1].strip()[:90]}")
    break
