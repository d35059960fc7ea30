"""Wall time of near_field_potentials (pinned host geometry -> potentials in a
pinned host buffer), fused one-shot kernel vs the two-step path, per case.

    python tools/e2e_fused.py c5/dense c2/dense ...
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1811_01110_b200 import configs, near_field_potentials  # noqa: E402

for cs in sys.argv[1:] or ["c2/dense"]:
    name, preset = cs.split("/")
    case = configs.make_case(name, preset)
    pin = lambda x: torch.from_numpy(np.ascontiguousarray(x)).pin_memory()  # noqa: E731
    src, w, ctr, rad, tgt, tptr = (pin(x) for x in (case.sources, case.weights, case.centers,
                                                   case.near_radii, case.targets, case.tgt_ptr))
    ho = torch.empty(case.n_targets, dtype=torch.complex128).pin_memory()
    res = {}
    for fused in ((True, False) if os.environ.get("E2E_FUSED", "0") == "1" else (False,)):
        for _ in range(2):
            near_field_potentials(case.cfg, src, w, ctr, rad, tgt, tgt_ptr=tptr, out=ho,
                                  fused=fused)
        torch.cuda.synchronize()
        ts = []
        for _ in range(5):
            t0 = time.perf_counter()
            near_field_potentials(case.cfg, src, w, ctr, rad, tgt, tgt_ptr=tptr, out=ho,
                                  fused=fused)
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t0)
        res[fused] = (1e3 * float(np.median(ts)), ho.numpy().copy())
    if True in res:
        err = float(np.max(np.abs(res[True][1] - res[False][1])) / np.max(np.abs(res[False][1])))
        print(f"{cs}: fused {res[True][0]:.3f} ms, two-step {res[False][0]:.3f} ms, "
              f"speed-up {res[False][0] / res[True][0]:.2f}x, max rel diff {err:.1e}", flush=True)
    else:
        print(f"{cs}: two-step {res[False][0]:.3f} ms", flush=True)
