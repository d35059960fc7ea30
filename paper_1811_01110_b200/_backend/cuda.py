"""The ``cuda`` backend module: the reference backend functions on the GPU.

Same signatures and conventions as ``_core.ts_accum_laplace`` /
``_core.ts_accum_helmholtz`` (_core.pyx:205-207, :310-312; _ref.py:177, :278):
one (center, target) over a source batch, no validation (backends never
validate; tsqbx._prep does), empty batch -> 0j, Laplace with real weights has
an exactly-zero imaginary part.  Each call is one H2D copy, one launch of the
single-call kernel and one D2H copy (``_single.py``); batches belong in
``ts_accumulate_batch``.
"""

from __future__ import annotations

import numpy as np

from ..kernels import Equation, KernelSpec, Variant

BACKEND_NAME = "cuda"

_VARIANTS = {0: Variant.SINGLE_LAYER, 1: Variant.TARGET_NORMAL_DERIV,
             2: Variant.SOURCE_NORMAL_DERIV}


def _one(spec: KernelSpec, p, sources, weights, snormals, center, target, tnormal) -> complex:
    from .._single import one_call
    from ..tsqbx import _equation_code

    sources = np.ascontiguousarray(sources, dtype=np.float64).reshape(-1, 3)
    if sources.shape[0] == 0:
        return 0.0 + 0.0j
    weights = np.ascontiguousarray(weights, dtype=np.complex128).reshape(-1)
    sn = (np.ascontiguousarray(snormals, dtype=np.float64).reshape(-1, 3)
          if spec.needs_source_normals else None)
    tn = (np.asarray(tnormal, dtype=np.float64).reshape(3)
          if spec.needs_target_normals else None)
    value, _ = one_call(_equation_code(spec), spec.variant_code, float(spec.helmholtz_k or 0.0),
                        int(p), sources, weights, sn, np.asarray(center, np.float64).reshape(3),
                        np.asarray(target, np.float64).reshape(3), tn, validate=False)
    return value


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
