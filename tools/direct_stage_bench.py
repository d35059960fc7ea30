"""Row f2 at scale: the driver's direct stage (DirectStage.run) on a synthetic
box structure -- leaf boxes = cells of a uniform grid over the C2 sphere
(262144 sources / centers) plus 65536 conventional targets, List 1 = the 27
neighbour cells -- timed on the device.  Reports TSQBX pairs/s and p2p pairs/s
for the whole stage (box-list expansion included)."""
import json
import sys
from types import SimpleNamespace

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1811_01110_b200 import KernelSpec, configs  # noqa: E402
from paper_1811_01110_b200.direct_stage import DirectStage  # noqa: E402


def synthetic_tree(case, conv, cell):
    lo = np.minimum(case.sources.min(0), conv.min(0)) - 1e-9
    def cell_of(x):
        return np.floor((x - lo) / cell).astype(np.int64)
    dims = cell_of(np.maximum(case.sources.max(0), conv.max(0))) + 1
    def key(c):
        return (c[:, 0] * dims[1] + c[:, 1]) * dims[2] + c[:, 2]
    ks, kc, kt = key(cell_of(case.sources)), key(cell_of(case.centers)), key(cell_of(conv))
    boxes = np.unique(np.concatenate([ks, kc, kt]))
    nb = boxes.shape[0]

    def order(keys):
        perm = np.argsort(keys, kind="stable")
        ids = np.searchsorted(boxes, keys[perm])
        return perm, np.searchsorted(ids, np.arange(nb), "left"), \
            np.searchsorted(ids, np.arange(nb), "right")
    sp, s0, s1 = order(ks)
    tp, t0, t1 = order(kt)
    cp, c0, c1 = order(kc)
    owned_start = np.stack([s0, t0, c0], 1)
    owned_end = np.stack([s1, t1, c1], 1)
    # List 1: the existing neighbour cells, in (dx, dy, dz) order
    bx = np.stack([boxes // (dims[1] * dims[2]), (boxes // dims[2]) % dims[1], boxes % dims[2]], 1)
    nbr = np.full((nb, 27), -1, np.int64)
    for q, d in enumerate(np.ndindex(3, 3, 3)):
        c = bx + np.array(d) - 1
        ok = np.all((c >= 0) & (c < dims), axis=1)
        kk = (c[:, 0] * dims[1] + c[:, 1]) * dims[2] + c[:, 2]
        j = np.searchsorted(boxes, kk)
        j = np.minimum(j, nb - 1)
        hit = ok & (boxes[j] == kk)
        nbr[hit, q] = j[hit]
    cnt = (nbr >= 0).sum(1)
    starts = np.concatenate([[0], np.cumsum(cnt)])
    flat = nbr[nbr >= 0]
    tree = SimpleNamespace(points=[case.sources[sp], conv[tp], case.centers[cp]],
                           owned_start=owned_start, owned_end=owned_end)
    lst = SimpleNamespace(starts=starts.astype(np.int64), flat=flat.astype(np.int64))
    return tree, lst, sp, cp, np.arange(nb)


if __name__ == "__main__":
    case = configs.make_case("c2", "literal")
    rng = np.random.default_rng(1)
    conv = rng.normal(size=(65536, 3))
    conv = 1.02 * conv / np.linalg.norm(conv, axis=1)[:, None]
    cell = float(sys.argv[1]) if len(sys.argv) > 1 else 16 * float(case.expansion_radii.mean())
    tree, lst, sp, cp, tboxes = synthetic_tree(case, conv, cell)
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
