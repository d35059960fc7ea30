"""Phase timing of the end-to-end path (host arrays -> potentials) for one case."""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1811_01110_b200 import configs  # noqa: E402
from paper_1811_01110_b200 import _device as dv  # noqa: E402
from paper_1811_01110_b200.nearlist import build_near_lists  # noqa: E402
from paper_1811_01110_b200.tsqbx import _Prepared, near_field_potentials  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--case", default="c2")
ap.add_argument("--preset", default="dense")
a = ap.parse_args()
case = configs.make_case(a.case, a.preset)
pin = lambda x: torch.from_numpy(np.ascontiguousarray(x)).pin_memory()  # noqa: E731
src, w, ctr, rad, tgt, tptr = (pin(x) for x in (case.sources, case.weights, case.centers,
                                               case.near_radii, case.targets, case.tgt_ptr))
dev = torch.device("cuda")
ho = torch.empty(case.n_targets, dtype=torch.complex128).pin_memory()
for _ in range(3):
    near_field_potentials(case.cfg, src, w, ctr, rad, tgt, tgt_ptr=tptr)
torch.cuda.synchronize()
T = {}


def mark(name, t0):
    torch.cuda.synchronize()
    T[name] = T.get(name, 0) + (time.perf_counter() - t0) * 1e3
    return time.perf_counter()


for rep in range(5):
    t = time.perf_counter()
    s_d = src.to(dev, non_blocking=True)
    w_d = torch.view_as_real(w.to(dev, non_blocking=True))
    c_d = ctr.to(dev, non_blocking=True)
    r_d = rad.to(dev, non_blocking=True)
    t_d = tgt.to(dev, non_blocking=True)
    p_d = tptr.to(dev, non_blocking=True)
    t = mark("h2d", t)
    near = build_near_lists(c_d, s_d, r_d, dev)
    t = mark("near_lists", t)
    prep = _Prepared(case.cfg, dev, s_d, w_d, None, c_d, near, t_d, None, p_d)
    t = mark("prepare(pack+order+sell)", t)
    out = torch.empty(prep.n_tgt, dtype=torch.complex128, device=dev)
    prep.launch(torch.view_as_real(out), True)
    t = mark("eval", t)
    prep.check_errors(True)
    t = mark("validate check", t)
    ho.copy_(out)
    t = mark("d2h", t)
tot = sum(T.values())
print("-- full pipeline phases")
for k, v in T.items():
    print(f"{k:28s} {v / 5:8.3f} ms  {100 * v / tot:5.1f}%")
t0 = time.perf_counter()
for _ in range(5):
    near_field_potentials(case.cfg, src, w, ctr, rad, tgt, tgt_ptr=tptr, out=ho)
torch.cuda.synchronize()
print(f"near_field_potentials end-to-end: {(time.perf_counter() - t0) / 5 * 1e3:.3f} ms")

# batch API with prebuilt device near lists (the bench's `e2e`)
from paper_1811_01110_b200.tsqbx import ts_accumulate_batch  # noqa: E402
near0 = build_near_lists(case.centers, case.sources, case.near_radii, dev)
T.clear()
for rep in range(6):
    t = time.perf_counter()
    s_d = src.to(dev, non_blocking=True)
    w_d = torch.view_as_real(w.to(dev, non_blocking=True))
    c_d = ctr.to(dev, non_blocking=True)
    t_d = tgt.to(dev, non_blocking=True)
    p_d = tptr.to(dev, non_blocking=True)
    t = mark("h2d", t)
    prep = _Prepared(case.cfg, dev, s_d, w_d, None, c_d, near0, t_d, None, p_d)
    t = mark("prepare(pack+order)", t)
    out = torch.empty(prep.n_tgt, dtype=torch.complex128, device=dev)
    prep.launch(torch.view_as_real(out), True)
    t = mark("eval", t)
    prep.check_errors(True)
    t = mark("validate check", t)
    ho.copy_(out)
    t = mark("d2h", t)
    if rep == 0:
        T.clear()
tot = sum(T.values())
print("-- batch API phases (prebuilt near lists)")
for k, v in T.items():
    print(f"{k:28s} {v / 5:8.3f} ms  {100 * v / tot:5.1f}%")
t0 = time.perf_counter()
for _ in range(5):
    ts_accumulate_batch(case.cfg, src, w, ctr, tgt, near0, tgt_ptr=tptr, out=ho)
torch.cuda.synchronize()
print(f"ts_accumulate_batch end-to-end: {(time.perf_counter() - t0) / 5 * 1e3:.3f} ms")
