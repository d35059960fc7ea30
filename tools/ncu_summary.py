"""Summarise ncu reports (run here, on the CPU box): key throughput, stall and
traffic metrics per profiled kernel, as text or JSON.

    python tools/ncu_summary.py gpurun_out/prof_x.ncu-rep [...] [--json out.json]
"""
import csv
import io
import json
import subprocess
import sys

KEYS = [
    ("kernel", "Kernel Name"),
    ("duration_us", "gpu__time_duration.sum"),
    ("registers", "launch__registers_per_thread"),
    ("block", "launch__block_size"),
    ("grid", "launch__grid_size"),
    ("warps_active_pct", "sm__warps_active.avg.pct_of_peak_sustained_active"),
    ("fp64_pipe_pct", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
    ("issue_active_pct", "sm__inst_issued.avg.pct_of_peak_sustained_active"),
    ("inst_executed", "smsp__inst_executed.sum"),
    ("dram_read_bytes", "dram__bytes_read.sum"),
    ("dram_write_bytes", "dram__bytes_write.sum"),
    ("l1_hit_pct", "l1tex__t_sector_hit_rate.pct"),
    ("l2_hit_pct", "lts__t_sector_hit_rate.pct"),
    ("l1_wavefronts", "l1tex__data_pipe_lsu_wavefronts.sum"),
    ("lsu_ld_requests", "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum"),
    ("lsu_ld_sectors", "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum"),
    ("dfma_thread_inst", "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum"),
    ("dmul_thread_inst", "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum"),
    ("dadd_thread_inst", "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum"),
]
STALL = "smsp__average_warps_issue_stalled_"


def load(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        rec = {}
        for k, m in KEYS:
            v = d.get(m)
            if v is None:
                continue
            try:
                f = float(v.replace(",", ""))
                unit = u.get(m, "")
                if m.startswith("dram__bytes") and unit == "Mbyte":
                    f *= 1e6
                elif m.startswith("dram__bytes") and unit == "Gbyte":
                    f *= 1e9
                elif m.startswith("dram__bytes") and unit == "Kbyte":
                    f *= 1e3
                if m == "gpu__time_duration.sum" and unit in ("msecond", "ms"):
                    f *= 1e3
                elif m == "gpu__time_duration.sum" and unit in ("nsecond", "ns"):
                    f *= 1e-3
                rec[k] = f
            except ValueError:
                rec[k] = v
        stalls = {}
        for m, v in d.items():
            if m.startswith(STALL) and m.endswith("_per_issue_active.ratio"):
                try:
                    fv = float(v)
                except ValueError:
                    continue
                if fv >= 0.05:
                    stalls[m[len(STALL):-len("_per_issue_active.ratio")]] = round(fv, 3)
        rec["stalls_per_issue"] = dict(sorted(stalls.items(), key=lambda kv: -kv[1]))
        res.append(rec)
    return res


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    out_json = None
    if "--json" in sys.argv:
        out_json = sys.argv[sys.argv.index("--json") + 1]
        args = [a for a in args if a != out_json]
    allr = {}
    for p in args:
        recs = load(p)
        allr[p] = recs
        for r in recs:
            print(f"== {p}: {str(r.get('kernel'))[:90]}")
            for k, v in r.items():
                if k != "kernel":
                    print(f"   {k:18s} {v}")
    if out_json:
        with open(out_json, "w") as f:
            json.dump(allr, f, indent=1)


if __name__ == "__main__":
    main()
