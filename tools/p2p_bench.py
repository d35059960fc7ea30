"""Time the P2P direct-sum kernels (dense and rows) on the GPU: pairs/s and
the FP64 roofline fraction with the algorithmic flops per pair of DESIGN.md."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1811_01110_b200 import KernelSpec, P2PProblem  # noqa: E402
from paper_1811_01110_b200.kernels import Equation, Variant  # noqa: E402

FLOPS = {("laplace", 0): 13, ("laplace", 1): 21, ("laplace", 2): 21,
         ("helmholtz", 0): 23, ("helmholtz", 1): 35, ("helmholtz", 2): 35}
PEAK = 35.7e12


def run(eq, v, ns, nt, reps=10):
    rng = np.random.default_rng(0)
    dev = torch.device("cuda")
    src = torch.as_tensor(rng.normal(size=(ns, 3)), device=dev)
    tgt = torch.as_tensor(rng.normal(size=(nt, 3)) + 0.01, device=dev)
    w = torch.as_tensor(rng.normal(size=ns) + 1j * rng.normal(size=ns), device=dev)
    nrm = torch.nn.functional.normalize(torch.as_tensor(rng.normal(size=(max(ns, nt), 3)),
                                                        device=dev), dim=1)
    var = [Variant.SINGLE_LAYER, Variant.TARGET_NORMAL_DERIV, Variant.SOURCE_NORMAL_DERIV][v]
    spec = KernelSpec(equation=Equation(eq), variant=var,
                      helmholtz_k=10.0 if eq == "helmholtz" else None)
    prob = P2PProblem(spec, src, w, nrm[:ns])
    out = torch.empty(nt, dtype=torch.complex128, device=dev)
    tn = nrm[:nt]
    for _ in range(2):
        prob.evaluate(tgt, tn, validate=False, out=out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        prob.evaluate(tgt, tn, validate=False, out=out)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    pairs = ns * nt
    rate = pairs / (ms * 1e-3)
    return dict(eq=eq, variant=v, n_src=ns, n_tgt=nt, ms=round(ms, 4),
                gpairs_s=round(rate / 1e9, 2),
                frac=round(rate * FLOPS[(eq, v)] / PEAK, 3))


if __name__ == "__main__":
    for eq in ("laplace", "helmholtz"):
        for v in (0, 1, 2):
            print(json.dumps(run(eq, v, 65536, 65536)))
    print(json.dumps(run("laplace", 0, 1 << 20, 64)))
    print(json.dumps(run("laplace", 0, 4096, 1 << 20)))
