"""Run one BASELINE case's evaluation a few times (for ncu / launch lists).

    python tools/profile_case.py --case c2 --preset dense --reps 3
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1811_01110_b200 import TsqbxProblem, build_near_lists, configs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--case", default="c2")
ap.add_argument("--preset", default="dense")
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--group-lanes", type=int, default=0)
ap.add_argument("--generic", action="store_true")
a = ap.parse_args()
case = configs.make_case(a.case, a.preset)
near = build_near_lists(case.centers, case.sources, case.near_radii)
prob = TsqbxProblem(case.cfg, case.sources, case.weights, case.centers, case.targets, near,
                    tgt_ptr=case.tgt_ptr, group_lanes=a.group_lanes or None)
for _ in range(a.reps):
    prob.evaluate(generic=a.generic)
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
ev[0].record()
for _ in range(10):
    prob.evaluate(generic=a.generic)
ev[1].record()
torch.cuda.synchronize()
ms = ev[0].elapsed_time(ev[1]) / 10
print(f"{a.case}/{a.preset}: G={prob.group_lanes} pairs={prob.pair_count()} {ms:.4f} ms "
      f"{prob.pair_count() / ms / 1e6:.2f} Gpairs/s")
