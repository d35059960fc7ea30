"""The ``cuda`` backend module: the reference backend functions on the GPU.

Same signatures and conventions as ``_core.ts_accum_laplace`` /
``_core.ts_accum_helmholtz`` (_core.pyx:205-207, :310-312; _ref.py:177, :278):
one (center, target) over a source batch, no validation (backends never
validate; tsqbx._prep does), empty batch -> 0j, Laplace with real weights has
an exactly-zero imaginary part.  Each call is a batch-of-one launch of the
same kernels ``ts_accumulate_batch`` uses.
"""

from __future__ import annotations

import numpy as np
import torch

from .. import _device as dv
from ..kernels import Equation, KernelSpec, Variant
from ..nearlist import NearLists

BACKEND_NAME = "cuda"

_VARIANTS = {0: Variant.SINGLE_LAYER, 1: Variant.TARGET_NORMAL_DERIV,
             2: Variant.SOURCE_NORMAL_DERIV}


def _one(spec: KernelSpec, p, sources, weights, snormals, center, target, tnormal) -> complex:
    from ..tsqbx import TsConfig, _Prepared, _inputs

    sources = np.ascontiguousarray(sources, dtype=np.float64).reshape(-1, 3)
    n = sources.shape[0]
    if n == 0:
        return 0.0 + 0.0j
    cfg = TsConfig(spec, int(p))
    dev = dv.require_cuda()
    tn = None if tnormal is None else np.asarray(tnormal, dtype=np.float64).reshape(1, 3)
    src, w, ctr, tgt, sn, tnd = _inputs(cfg, sources, weights,
                                        np.asarray(center, dtype=np.float64).reshape(1, 3),
                                        np.asarray(target, dtype=np.float64).reshape(1, 3),
                                        snormals, tn, dev)
    near = NearLists(n_ctr=1, n_src=n, n_pairs=n,
                     ptr=torch.tensor([0, n], dtype=torch.int64, device=dev),
                     csr_idx=torch.arange(n, dtype=torch.int32, device=dev))
    prep = _Prepared(cfg, dev, src, w, sn, ctr, near, tgt, tnd,
                     torch.tensor([0, 1], dtype=torch.int64, device=dev))
    out = torch.empty(1, dtype=torch.complex128, device=dev)
    prep.launch(torch.view_as_real(out), validate=False)
    return complex(out.cpu().numpy()[0])


def ts_accum_laplace(variant, p, sources, weights, snormals, center, target, tnormal):
    spec = KernelSpec(equation=Equation.LAPLACE, variant=_VARIANTS[int(variant)])
    return _one(spec, p, sources, weights, snormals, center, target, tnormal)


def ts_accum_helmholtz(variant, k, p, sources, weights, snormals, center, target, tnormal):
    spec = KernelSpec(equation=Equation.HELMHOLTZ, variant=_VARIANTS[int(variant)],
                      helmholtz_k=float(k))
    return _one(spec, p, sources, weights, snormals, center, target, tnormal)


def _p2p(spec, sources, weights, snormals, targets, tnormals):
    from ..p2p import P2PProblem

    targets = np.ascontiguousarray(targets, dtype=np.float64).reshape(-1, 3)
    out = np.zeros(targets.shape[0], dtype=np.complex128)
    if np.asarray(sources).size == 0 or targets.shape[0] == 0:
        return out
    prob = P2PProblem(spec, sources, weights, snormals)
    return prob.evaluate(targets, tnormals).cpu().numpy()


def laplace_p2p(variant, sources, weights, snormals, targets, tnormals):
    """_core.laplace_p2p (_core.pyx:94-125) on the GPU (same ValueError on r = 0)."""
    spec = KernelSpec(equation=Equation.LAPLACE, variant=_VARIANTS[int(variant)])
    return _p2p(spec, sources, weights, snormals, targets, tnormals)


def helmholtz_p2p(variant, k, sources, weights, snormals, targets, tnormals):
    """_core.helmholtz_p2p (_core.pyx:128-165) on the GPU."""
    spec = KernelSpec(equation=Equation.HELMHOLTZ, variant=_VARIANTS[int(variant)],
                      helmholtz_k=float(k))
    return _p2p(spec, sources, weights, snormals, targets, tnormals)
