"""Time the evaluation of BASELINE cases over group sizes (device-resident, events).

    python tools/sweep.py --cases c2/dense,c2/literal --lanes 4,8,16,32
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1811_01110_b200 import TsqbxProblem, build_near_lists, configs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--cases", default="c2/dense,c2/literal,c3/dense,c3/literal")
ap.add_argument("--lanes", default="0")
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--peak", type=float, default=35.77)
ap.add_argument("--flush", default="write", choices=("write", "write+read", "none"))
ap.add_argument("--validate", action="store_true", help="time the screened (validating) launch")
a = ap.parse_args()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
flush2 = torch.ones(256 << 20, dtype=torch.uint8, device="cuda")


def do_flush():
    if a.flush == "none":
        return
    flush.zero_()
    if a.flush == "write+read":
        flush2.max()      # clean lines displace the dirty ones (write-back outside timing)
from paper_1811_01110_b200 import KernelSpec, TsConfig  # noqa: E402
from paper_1811_01110_b200.kernels import Variant  # noqa: E402

VAR = {"s": Variant.SINGLE_LAYER, "sp": Variant.TARGET_NORMAL_DERIV, "d": Variant.SOURCE_NORMAL_DERIV}
for cs in a.cases.split(","):
    parts = cs.split("/")
    name, preset = parts[0], parts[1]
    case = configs.make_case(name, preset)
    if len(parts) > 2:
        sp = case.cfg.spec
        case.cfg = TsConfig(KernelSpec(equation=sp.equation, variant=VAR[parts[2]],
                                       helmholtz_k=sp.helmholtz_k), case.cfg.p_qbx)
    import numpy as np  # noqa: E402
    tnrm = np.repeat(case.normals, np.diff(case.tgt_ptr), axis=0)
    near = build_near_lists(case.centers, case.sources, case.near_radii)
    fpp = configs.algorithmic_flops_per_pair(case.cfg.spec, case.cfg.p_qbx)
    for G in [int(x) for x in a.lanes.split(",")]:
        prob = TsqbxProblem(case.cfg, case.sources, case.weights, case.centers, case.targets,
                            near, tgt_ptr=case.tgt_ptr, group_lanes=G or None,
                            source_normals=case.normals, target_normals=tnrm)
        pairs = prob.pair_count()
        if a.validate:
            def run(prob=prob):
                prob.prep.launch(torch.view_as_real(prob.out), True)
        else:
            run = prob.evaluate
        for _ in range(3):
            run()
        ts = []
        for _ in range(a.reps):
            do_flush()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            run()
            e1.record()
            ts.append((e0, e1))
        torch.cuda.synchronize()
        ms = sorted(x.elapsed_time(y) for x, y in ts)[len(ts) // 2]
        tf = pairs * fpp / (ms * 1e-3) / 1e12
        print(f"{cs:12s} G={prob.group_lanes:2d} {ms:8.4f} ms  {pairs / ms / 1e6:8.2f} Gpairs/s "
              f"{tf:6.2f} TF  {100 * tf / a.peak:5.1f}% of fp64 peak", flush=True)
        del prob
