"""Row f2 at scale: the driver's direct stage (DirectStage.run) on a synthetic
box structure -- leaf boxes = cells of a uniform grid over the C2 sphere
(262144 sources / centers) plus 65536 conventional targets, List 1 = the 27
neighbour cells -- timed on the device.  Reports TSQBX pairs/s and p2p pairs/s
for the whole stage (box-list expansion included)."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1811_01110_b200 import KernelSpec, configs  # noqa: E402
from paper_1811_01110_b200.direct_stage import DirectStage  # noqa: E402


if __name__ == "__main__":
    case = configs.make_case("c2", "literal")
    rng = np.random.default_rng(1)
    conv = rng.normal(size=(65536, 3))
    conv = 1.02 * conv / np.linalg.norm(conv, axis=1)[:, None]
    cell = float(sys.argv[1]) if len(sys.argv) > 1 else 16 * float(case.expansion_radii.mean())
    tree, lst, sp, cp, tboxes = configs.synthetic_box_tree(case, conv, cell)
    w = case.weights[sp]
    qt = case.targets[case.tgt_ptr[:-1]][cp]        # the on-surface target of each center
    ds = DirectStage(KernelSpec(), 8, tree, tboxes, w, qtargets=qt)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    ds.run(lst)                                   # builds and caches the plan
    e1.record()
    torch.cuda.synchronize()
    first_ms = e0.elapsed_time(e1)
    for _ in range(3):
        conv_add, qbx_add, nts = ds.run(lst)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 10
    e0.record()
    for _ in range(reps):
        conv_add, qbx_add, nts = ds.run(lst)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    ns = tree.owned_end[:, 0] - tree.owned_start[:, 0]
    nt = tree.owned_end[:, 1] - tree.owned_start[:, 1]
    per_box = np.add.reduceat(ns[lst.flat], lst.starts[:-1]) * (np.diff(lst.starts) > 0)
    n_p2p = int((nt * per_box).sum())
    print(json.dumps({"boxes": int(len(lst.starts) - 1), "cell": cell, "ts_pairs": nts,
                      "p2p_pairs": n_p2p, "first_run_ms": round(first_ms, 3), "ms_per_stage": round(ms, 4),
                      "ts_plus_p2p_pairs_per_s": (nts + n_p2p) / (ms * 1e-3)}))
