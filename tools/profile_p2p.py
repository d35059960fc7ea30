"""One dense P2P direct sum (for ncu): python tools/profile_p2p.py [laplace|helmholtz] [n]"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1811_01110_b200 import KernelSpec, P2PProblem  # noqa: E402
from paper_1811_01110_b200.kernels import Equation  # noqa: E402

eq = sys.argv[1] if len(sys.argv) > 1 else "laplace"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 65536
rng = np.random.default_rng(0)
dev = torch.device("cuda")
src = torch.as_tensor(rng.normal(size=(n, 3)), device=dev)
tgt = torch.as_tensor(rng.normal(size=(n, 3)) + 0.01, device=dev)
w = torch.as_tensor(rng.normal(size=n) + 1j * rng.normal(size=n), device=dev)
spec = KernelSpec(equation=Equation(eq), helmholtz_k=10.0 if eq == "helmholtz" else None)
prob = P2PProblem(spec, src, w)
for _ in range(3):
    out = prob.evaluate(tgt, validate=False)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    prob.evaluate(tgt, validate=False, out=out)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 5
print(f"p2p {eq} {n}x{n}: {ms:.3f} ms, {n * n / ms / 1e6:.1f} Gpairs/s")
