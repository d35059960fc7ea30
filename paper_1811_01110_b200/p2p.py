"""Point-to-point direct interactions on the device.

Replaces the reference backends' ``laplace_p2p`` / ``helmholtz_p2p``
(``_core.pyx:94-165``) and mirrors their two callers:

* ``direct_sum`` -- ``kernels.direct_sum`` (kernels.py:114-136): every target
  sees every source; same argument checks and ValueError texts;
* ``p2p_rows`` -- the driver's per-target-box p2p (driver.py:187-210) batched:
  row ``r``'s targets ``[row_tgt[r], row_tgt[r+1])`` see the sources
  ``row_idx[row_ptr[r]:row_ptr[r+1]]``.

Both run ``tsqbx_p2p_packed`` (csrc/p2p.cu).  A singular pair (target ==
source) raises the reference's ``ValueError("singular source/target pair:
target i, source j")`` for the first pair in target-major order.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _device as dv
from . import _lib
from .kernels import KernelSpec


@dataclass
class P2PRows:
    """Device row structure for ``P2PProblem.evaluate`` (checked once)."""

    row_tgt: torch.Tensor
    row_ptr: torch.Tensor
    row_idx: torch.Tensor
    n_rows: int
    n_tgt: int


class P2PProblem:
    """Sources packed once in HBM; evaluate dense or row-restricted sums against
    any set of targets (repeated evaluations reuse the packed sources)."""

    @dv.on_device
    def __init__(self, spec: KernelSpec, sources, weights, source_normals=None, device=None):
        spec = self.spec = KernelSpec.coerce(spec)
        self.dev = dv.require_cuda(device)
        L = _lib.load()
        src = dv.to_device(sources, torch.float64, self.dev, (-1, 3))
        if isinstance(weights, torch.Tensor) and not weights.is_complex():
            weights = weights.to(torch.complex128)
        w = dv.complex_as_f64(dv.to_device(weights, torch.complex128, self.dev, (-1,)))
        if w.shape[0] != src.shape[0]:
            raise ValueError("weights must have one entry per source")
        sn = None
        if spec.needs_source_normals:
            if source_normals is None:
                raise ValueError("kernel variant requires source normals")
            sn = dv.to_device(source_normals, torch.float64, self.dev, (-1, 3))
        self.n_src = int(src.shape[0])
        self.with_normals = sn is not None
        self.src, self.sn = src, sn
        nd = int(L.tsqbx_packed_doubles(self.n_src, int(self.with_normals)))
        self.packed = torch.empty(nd, dtype=torch.float64, device=self.dev)
        self._pack(w)
        self.err = torch.empty(1, dtype=torch.int64, device=self.dev)

    def _pack(self, w: torch.Tensor) -> None:
        L = _lib.load()
        _lib.check(L.tsqbx_pack_sources(self.n_src, self.src.data_ptr(), w.data_ptr(),
                                        dv.ptr(self.sn), None, self.packed.data_ptr(),
                                        dv.stream_handle(self.dev)), "tsqbx_pack_sources")

    @dv.on_own_device
    def set_weights(self, weights) -> None:
        """New source weights (same sources): one pack kernel, no reallocation."""
        if isinstance(weights, torch.Tensor) and not weights.is_complex():
            weights = weights.to(torch.complex128)
        w = dv.complex_as_f64(dv.to_device(weights, torch.complex128, self.dev, (-1,)))
        if w.shape[0] != self.n_src:
            raise ValueError("weights must have one entry per source")
        self._pack(w)

    @dv.on_own_device
    def rows(self, row_tgt, row_ptr, row_idx, n_tgt: int) -> "P2PRows":
        """Checked device copy of a row structure for repeated ``evaluate``."""
        rt = dv.to_device(row_tgt, torch.int64, self.dev, (-1,))
        rp = dv.to_device(row_ptr, torch.int64, self.dev, (-1,))
        ri = dv.to_device(row_idx, torch.int32, self.dev, (-1,))
        n_rows = int(rt.shape[0]) - 1
        if n_rows < 0 or rp.shape[0] != n_rows + 1:
            raise ValueError("row_tgt and row_ptr must both have n_rows + 1 entries")
        if n_rows > 0:
            ends = torch.stack([rt[0], rt[-1], rp[0], rp[-1]]).cpu().tolist()
            if ends[0] != 0 or ends[1] != n_tgt or ends[2] != 0 or ends[3] > ri.shape[0]:
                raise ValueError("rows must partition the targets and index row_idx")
        elif n_tgt:
            raise ValueError("rows must partition the targets")
        return P2PRows(rt, rp, ri, n_rows, n_tgt)

    def _targets(self, targets, target_normals):
        tgt = dv.to_device(targets, torch.float64, self.dev, (-1, 3))
        tn = None
        if self.spec.needs_target_normals:
            if target_normals is None:
                raise ValueError("kernel variant requires target normals")
            tn = dv.to_device(target_normals, torch.float64, self.dev, (-1, 3))
            if tn.shape[0] != tgt.shape[0]:
                raise ValueError("target normals must have one entry per target")
        return tgt, tn

    @dv.on_own_device
    def evaluate(self, targets, target_normals=None, rows=None, validate: bool = True,
                 out: torch.Tensor | None = None) -> torch.Tensor:
        """complex128 (n_tgt,) CUDA tensor.  ``rows = (row_tgt, row_ptr, row_idx)``
        restricts each target row to its source list; None = dense."""
        L = _lib.load()
        tgt, tn = self._targets(targets, target_normals)
        n_tgt = int(tgt.shape[0])
        rt = rp = ri = None
        n_rows = 0
        if rows is not None:
            if not isinstance(rows, P2PRows):
                rows = self.rows(rows[0], rows[1], rows[2], n_tgt)
            elif rows.n_tgt != n_tgt:
                raise ValueError("rows were prepared for a different number of targets")
            rt, rp, ri, n_rows = rows.row_tgt, rows.row_ptr, rows.row_idx, rows.n_rows
        if out is None:
            out = torch.empty(n_tgt, dtype=torch.complex128, device=self.dev)
        o = torch.view_as_real(out)
        wsb = int(L.tsqbx_p2p_workspace_bytes(self.n_src, n_tgt, n_rows, int(rows is None)))
        ws = torch.empty(max(wsb, 1), dtype=torch.uint8, device=self.dev)
        st = dv.stream_handle(self.dev)
        eq = _lib.EQ_LAPLACE if self.spec.is_laplace else _lib.EQ_HELMHOLTZ
        k = float(self.spec.helmholtz_k or 0.0)

        def launch(flags):
            _lib.check(L.tsqbx_p2p_packed(eq, self.spec.variant_code, k, self.packed.data_ptr(),
                                          self.n_src, int(self.with_normals), n_rows,
                                          dv.ptr(rt), dv.ptr(rp), dv.ptr(ri), tgt.data_ptr(),
                                          dv.ptr(tn), n_tgt, flags, ws.data_ptr(), wsb,
                                          o.data_ptr(), self.err.data_ptr(), st),
                       "tsqbx_p2p_packed")

        launch(_lib.FLAG_VALIDATE if validate else 0)
        if validate and n_tgt and int(self.err.item()) != _lib.ERR_KEY_NONE:
            _lib.check(L.tsqbx_p2p_find_singular(self.packed.data_ptr(), self.n_src, n_rows,
                                                 dv.ptr(rt), dv.ptr(rp), dv.ptr(ri),
                                                 tgt.data_ptr(), n_tgt, self.err.data_ptr(), st),
                       "tsqbx_p2p_find_singular")
            key = int(self.err.item())
            if key != _lib.ERR_KEY_NONE:
                raise ValueError(f"singular source/target pair: target {key >> 32}, "
                                 f"source {key & 0xFFFFFFFF}")
            launch(_lib.FLAG_PRECISE)     # non-finite without a singular pair: IEEE path
        return out


def _host_out(sources) -> bool:
    return not (isinstance(sources, torch.Tensor) and sources.is_cuda)


@dv.on_device
def direct_sum(spec: KernelSpec, sources, weights, targets, source_normals=None,
               target_normals=None, device=None):
    """sum_j w_j K(x_i, y_j) for every target (kernels.py:114-136) on the GPU.
    numpy in -> numpy out; CUDA tensors in -> CUDA tensor out."""
    prob = P2PProblem(spec, sources, weights, source_normals, device)
    out = prob.evaluate(targets, target_normals)
    return out.cpu().numpy() if _host_out(sources) else out


_NORMAL_TOL = 1e-12     # kernels.py:23


def _check_normal(normal, name):
    """kernels.py:74-80: present and unit length (same ValueError texts)."""
    if normal is None:
        raise ValueError(f"kernel variant requires a {name} normal")
    normal = np.asarray(normal, dtype=np.float64).reshape(3)
    if abs(float(np.linalg.norm(normal)) - 1.0) > _NORMAL_TOL:
        raise ValueError(f"{name} normal must be unit length")
    return normal


def kernel_value(spec: KernelSpec, target, source, target_normal=None,
                 source_normal=None, device=None) -> complex:
    """K(t, s), nu(t).grad_t K or nu(s).grad_s K at one pair (kernels.py:83-111),
    evaluated by the GPU p2p kernel as a 1 x 1 direct sum; the reference's checks
    and ValueError texts come first (a coincident pair is an error here, not a
    non-finite value)."""
    t = np.asarray(target, dtype=np.float64).reshape(3)
    s = np.asarray(source, dtype=np.float64).reshape(3)
    if float(np.linalg.norm(t - s)) == 0.0:
        raise ValueError("singular point: target coincides with source")
    tn = sn = None
    if spec.needs_target_normals:
        tn = _check_normal(target_normal, "target").reshape(1, 3)
    if spec.needs_source_normals:
        sn = _check_normal(source_normal, "source").reshape(1, 3)
    out = direct_sum(spec, s.reshape(1, 3), np.ones(1, np.complex128), t.reshape(1, 3),
                     source_normals=sn, target_normals=tn, device=device)
    return complex(out[0])


@dv.on_device
def p2p_rows(spec: KernelSpec, sources, weights, targets, row_tgt, row_ptr, row_idx,
             source_normals=None, target_normals=None, device=None):
    """Batched per-box p2p (driver.py:187-210): row r's targets see only the
    sources row_idx[row_ptr[r]:row_ptr[r+1]] (user source indices)."""
    prob = P2PProblem(spec, sources, weights, source_normals, device)
    out = prob.evaluate(targets, target_normals, rows=(row_tgt, row_ptr, row_idx))
    return out.cpu().numpy() if _host_out(sources) else out
