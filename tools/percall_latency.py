"""Per-call latency of the reference-shaped entry points (one center, one target):
ts_accumulate (public, validated) and the `cuda` backend's ts_accum_laplace."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_1811_01110_b200 import KernelSpec, TsConfig, get_backend, ts_accumulate  # noqa: E402

rng = np.random.default_rng(0)
cfg = TsConfig(KernelSpec(), 8)
be = get_backend("cuda")
for n in (12, 200):
    src = rng.normal(size=(n, 3)) + np.array([0, 0, 3.0])
    w = rng.normal(size=n) + 0j
    c, t = np.zeros(3), np.array([0.1, 0.0, 0.0])
    for name, fn in (("ts_accumulate", lambda: ts_accumulate(cfg, src, w, c, t)),
                     ("backend.ts_accum_laplace",
                      lambda: be.ts_accum_laplace(0, 8, src, w, None, c, t, None))):
        for _ in range(20):
            fn()
        t0 = time.perf_counter()
        for _ in range(200):
            fn()
        dt = (time.perf_counter() - t0) / 200
        print(f"{name:26s} n={n:4d}: {dt * 1e6:8.1f} us/call")
