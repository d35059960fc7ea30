"""Target-specific QBX (TSQBX) evaluation on B200.

Drop-in for the reference's public TSQBX API
(/root/reference/pkg/src/gigaqbx/tsqbx.py:28-92):

* ``TsConfig``, ``ts_accumulate`` and ``ts_eval`` keep the reference's names,
  argument meaning, return type and error behaviour (``ValueError`` texts of
  ``_prep``, tsqbx.py:38-65), but evaluate on the GPU through the C ABI.
* ``ts_accumulate_batch`` is the batched form the hardware needs: every center
  with its CSR row of near sources and its run of targets in ONE launch,
  returning per-target potentials.
* ``TsqbxProblem`` keeps a whole problem resident in HBM for repeated
  evaluation (the bench's device-resident measurement).

Validation (``validate=True``) runs on the device: the kernel screens every
pair (``rho^2 > (1+1e-12)^2`` or a non-finite result), and only a flagged
launch runs the exact reference predicate (``tsqbx_validate``) to name the
offending source.  The driver-style path (``driver._ts_accum``,
driver.py:383-389) does no validation; ``validate=False`` matches it.
"""

from __future__ import annotations

import math
import os
from dataclasses import dataclass

import numpy as np
import torch

from . import _device as dv
from . import _lib
from .kernels import Equation, KernelSpec
from .nearlist import NearLists

_SEP_SLACK = 1e-12


@dataclass(frozen=True)
class TsConfig:
    """Same as tsqbx.py:28-35."""

    spec: KernelSpec
    p_qbx: int

    def __post_init__(self):
        object.__setattr__(self, "spec", KernelSpec.coerce(self.spec))
        if self.p_qbx < 0:
            raise ValueError("p_qbx must be nonnegative")


def pick_group_lanes(mean_len: float) -> int:
    """Lanes that share one center in the CSR (group) kernels: ~64 list entries
    per lane, power of two in [1, 32].  Measured on B200 (profiles/): fewer
    lanes amortise the per-center prologue and reduction better."""
    env = os.environ.get("GIGAQBX_GROUP_LANES")
    if env:
        return int(env)
    g = 1 << max(0, int(round(math.log2(max(1.0, mean_len / 64.0)))))
    return max(1, min(32, g))


def pick_split(mean_len: float, n_rows: int, one_target: bool, sms: int = 148,
               uniform: bool = False) -> int:
    """Threads per row on the SELL layout (Laplace S): long rows are split over
    2 threads of a warp (shorter work units: C2 dense +3.5 %, C4 dense +4 %),
    over 4 when the rows fill less than ~1.5 waves of the GPU (C1 dense 2.7x); short
    rows (literal presets) are not split.  A wave is 4 CTAs of 256 threads per
    SM for one target per center or uniform target runs, else 3.
    GIGAQBX_SPLIT overrides."""
    env = os.environ.get("GIGAQBX_SPLIT")
    if env:
        return int(env)
    if mean_len < 48:
        return 1
    waves = n_rows / (sms * (1024 if (one_target or uniform) else 768))
    # 4 threads per row until ~1.5 waves (C2 geometry, 4-CTA kernel: 196 k rows =
    # 1.3 waves 0.213 vs 0.223 ms; 262 k rows = 1.7 waves equal)
    return 4 if waves < 1.5 else 2


# Mean near-list length below which Laplace S would take the short-list kernel
# (laplace_flat_kernel: a warp's 32 rows' CSR entries split evenly over its
# lanes).  0 = never: measured slower than the SELL thread-per-row kernel on
# every literal preset (C2 literal 34.0 vs 27.3 us, C4 literal 74.7 vs 50.0 us;
# ncu: the same FP64 work, 35 % more instructions, 24 instead of 32 warps per
# SM at NT = 2) -- the literal presets are not limited by lane divergence.
FLAT_BELOW = 0.0


def pick_flat(mean_len: float) -> bool:
    """Whether Laplace S takes the short-list kernel; GIGAQBX_FLAT=0/1 overrides."""
    env = os.environ.get("GIGAQBX_FLAT")
    if env is not None:
        return env == "1"
    return mean_len < FLAT_BELOW


# Mean near-list length below which Laplace S would take two rows per thread
# (laplace_sell2_kernel).  0 = never: measured slower on the literal presets
# (C2 literal 31.4 vs 27.1 us, C4 literal 58.2 vs 49.6 us): a thread's row-B
# chain is hidden, but its entries' source gathers now queue behind row A's
# -- the literal kernels wait on per-entry gathers, not on the row heads.
TWO_ROWS_BELOW = 0.0

# Mean near-list length below which Laplace S would use the windowed SELL.
# 0 = never: measured slower on the literal presets (C2 literal 37.8 vs
# 27.4 us, C4 literal 76 vs 50 us): the 40 KB window per CTA costs a quarter
# of the resident warps and the staging adds a dependent step per warp, while
# the per-entry gathers it removes were mostly L1 hits already.
WINDOW_BELOW = 0.0


def pick_window(mean_len: float) -> bool:
    """Short lists: every warp stages its 32 rows' distinct sources in shared
    memory once (tsqbx_sell_window + laplace_sellw_kernel) instead of one
    global gather per entry.  GIGAQBX_WINDOW=0/1 overrides."""
    env = os.environ.get("GIGAQBX_WINDOW")
    if env is not None:
        return env == "1"
    return mean_len < WINDOW_BELOW


def pick_two_rows(mean_len: float) -> bool:
    """Short lists (the literal presets): laplace_sell2_kernel, two rows per
    thread with the second row's loads in flight during the first row's
    arithmetic.  GIGAQBX_TWO_ROWS=0/1 overrides."""
    env = os.environ.get("GIGAQBX_TWO_ROWS")
    if env is not None:
        return env == "1"
    return mean_len < TWO_ROWS_BELOW


def pick_layout() -> str:
    """'sell' (thread per center on the sliced-ELL copy, the default) or 'csr'
    (groups of lanes per center on the CSR rows); GIGAQBX_LAYOUT overrides."""
    return os.environ.get("GIGAQBX_LAYOUT", "sell")


def _equation_code(spec: KernelSpec) -> int:
    return _lib.EQ_LAPLACE if spec.equation is Equation.LAPLACE else _lib.EQ_HELMHOLTZ


class _Prepared:
    """Device-side inputs of one evaluation, in processing order.

    Sources are packed (and Morton-permuted when the near lists come from
    ``build_near_lists``); centers, target runs and targets are reordered to
    the CSR's row order so that row g, its targets and its near sources are
    all addressed by g (what lets a rank evaluate a contiguous row range).
    """

    def __init__(self, cfg: TsConfig, dev, src, w, sn, ctr, near: NearLists, tgt, tn, tptr,
                 group_lanes=None, user_tptr: bool = True):
        L = _lib.load()
        self.cfg, self.dev, self.near = cfg, dev, near
        self.src, self.w, self.sn = src, w, sn
        self.user_ctr, self.user_tgt = ctr, tgt
        self.n_src = int(src.shape[0])
        self.n_ctr = int(ctr.shape[0])
        self.n_tgt = int(tgt.shape[0])
        if near.n_ctr != self.n_ctr:
            raise ValueError(f"near lists have {near.n_ctr} rows for {self.n_ctr} centers")
        if int(tptr.shape[0]) != self.n_ctr + 1:
            raise ValueError("tgt_ptr must have n_centers + 1 entries")
        # err[0]: the evaluation's validation key; err[1]: 1 when a caller's
        # tgt_ptr is malformed (checked on the device by tsqbx_order_targets,
        # reported with the result: no extra synchronisation)
        self.err = torch.zeros(2, dtype=torch.int64, device=dev)
        self.check_tptr = False
        if user_tptr and near.ctr_order is None:
            # rows in the caller's order (a user CSR, already checked with one
            # read-back): check the target offsets the same way
            from .nearlist import check_offsets
            check_offsets(tptr, self.n_tgt, "tgt_ptr")
        spec = cfg.spec
        self.eq = _equation_code(spec)
        self.variant = spec.variant_code
        self.k = float(spec.helmholtz_k or 0.0)
        self.with_normals = 1 if spec.needs_source_normals else 0
        st = dv.stream_handle(dev)
        nd = int(L.tsqbx_packed_doubles(self.n_src, self.with_normals))
        self.packed = torch.empty(max(nd, 4), dtype=torch.float64, device=dev)
        self.pack(w)
        tn = tn if self.variant == 1 else None
        if near.ctr_order is None:
            self.ctr, self.tptr, self.tgt, self.tn, self.tidx = ctr, tptr, tgt, tn, None
        else:
            self.ctr = torch.empty_like(ctr)
            self.tptr = torch.empty_like(tptr)
            self.tgt = torch.empty_like(tgt)
            self.tn = None if tn is None else torch.empty_like(tn)
            self.tidx = torch.empty(max(self.n_tgt, 1), dtype=torch.int64, device=dev)
            wsb = int(L.tsqbx_order_workspace_bytes(self.n_ctr))
            ws = torch.empty(max(wsb, 1), dtype=torch.uint8, device=dev)
            _lib.check(L.tsqbx_order_targets(self.n_ctr, near.ctr_order.data_ptr(),
                                             ctr.data_ptr(), tptr.data_ptr(), tgt.data_ptr(),
                                             dv.ptr(tn), self.n_tgt, ws.data_ptr(), wsb,
                                             self.ctr.data_ptr(), self.tptr.data_ptr(),
                                             self.tgt.data_ptr(), dv.ptr(self.tn),
                                             self.tidx.data_ptr(),
                                             self.err[1:].data_ptr() if user_tptr else None, st),
                       "tsqbx_order_targets")
            self.check_tptr = user_tptr
        self.ws_bytes = int(L.tsqbx_eval_workspace_bytes(self.eq, self.variant, cfg.p_qbx,
                                                         self.n_tgt))
        self.ws = torch.empty(max(self.ws_bytes, 1), dtype=torch.uint8, device=dev)
        self.layout = "csr" if group_lanes else pick_layout()
        if group_lanes:
            self.G = int(group_lanes)
        elif self.layout == "sell":
            # on the SELL layout the ABI's group_lanes is the row split (Laplace S;
            # splitting the Helmholtz rows measured 2 % slower: the per-target
            # Bessel coefficients would be computed S times)
            sms = dv.sm_count(dev.index if dev.index is not None else torch.cuda.current_device())
            self.G = (pick_split(near.mean_len, self.n_ctr, self.n_tgt < 2 * self.n_ctr, sms)
                      if spec.is_laplace and self.variant == 0 else 1)
        else:
            self.G = pick_group_lanes(near.mean_len)
        if self.layout == "sell" and self.n_ctr:
            near.build_sell()
        # real Laplace densities: the pack kernel flags any Im w != 0 on the device
        # and the kernel picks its real-weight path itself (no host round trip)
        self.real_w = False
        self.one_target = os.environ.get("GIGAQBX_ONE_TARGET", "0") == "1"
        self.tuni = 0         # k > 0: every row owns k consecutive targets (set_uniform_targets)
        self.flat = False     # Laplace S, uniform runs of 1-2 targets, short lists: flat kernel
        self.two_rows = False  # Laplace S, uniform runs, unsplit rows: two rows per thread
        self.window = False    # Laplace S, uniform runs, unsplit short rows: windowed SELL
        self._auto_split = (not group_lanes and self.layout == "sell" and spec.is_laplace
                            and self.variant == 0 and "GIGAQBX_SPLIT" not in os.environ)
        # Helmholtz: every near source lies within the largest near radius, so
        # k R is bounded and the kernels can take one sin/cos series without a
        # per-warp vote (the bound is exact: the lists test |s-c|^2 <= rad^2)
        self.kr_flag = 0
        if not spec.is_laplace and near.max_radius is not None:
            kr = self.k * near.max_radius * (1.0 + 1e-12)
            self.kr_flag = (_lib.FLAG_KR_NARROW if kr <= math.pi / 4 else
                            _lib.FLAG_KR_WIDE if kr <= math.pi / 2 else 0)

    def set_uniform_targets(self, known: bool = False) -> None:
        """Let the SELL kernels address row g's targets as [k g, k g + k) instead of
        loading tgt_ptr (one dependent load fewer per row).  ``known``: the caller
        built tgt_ptr as arange * k; otherwise it is checked once on the device."""
        k = self.n_tgt // self.n_ctr if self.n_ctr else 0
        if not (1 <= k <= 255 and k * self.n_ctr == self.n_tgt):
            return
        if known or bool(torch.equal(self.tptr, torch.arange(
                self.n_ctr + 1, dtype=torch.int64, device=self.dev) * k)):
            self.tuni = k
            self.flat = (k <= 2 and self.layout == "sell" and self.cfg.spec.is_laplace
                         and self.variant == 0 and self.cfg.p_qbx <= 16
                         and pick_flat(self.near.mean_len))
            self.two_rows = (k <= 2 and self.layout == "sell" and self.cfg.spec.is_laplace
                             and self.variant == 0 and pick_two_rows(self.near.mean_len))
            if self._auto_split:          # the uniform kernel fits one more CTA per SM
                self.G = pick_split(self.near.mean_len, self.n_ctr, k == 1,
                                    dv.sm_count(self.dev.index if self.dev.index is not None
                                                else torch.cuda.current_device()),
                                    uniform=True)
            self.window = (k <= 2 and self.layout == "sell" and self.cfg.spec.is_laplace
                           and self.variant == 0 and self.cfg.p_qbx <= 16 and self.G == 1
                           and pick_window(self.near.mean_len) and self.near.build_window())

    def pack(self, w: torch.Tensor) -> None:
        """(Re)pack the sources with weights ``w`` (interleaved float64 view)."""
        L = _lib.load()
        if w.shape[0] != self.n_src:
            raise ValueError("weights must have one entry per source")
        self.w = w
        _lib.check(L.tsqbx_pack_sources(self.n_src, dv.ptr(self.src), dv.ptr(w),
                                        dv.ptr(self.sn) if self.with_normals else None,
                                        dv.ptr(self.near.src_perm), self.packed.data_ptr(),
                                        dv.stream_handle(self.dev)), "tsqbx_pack_sources")

    def launch(self, out: torch.Tensor, validate: bool, generic: bool = False,
               rows: tuple[int, int] | None = None, out_offset: int = 0,
               user_order: bool = True) -> None:
        """One evaluation launch.  ``rows=(g0, g1)`` restricts it to a row range
        (a multi-GPU shard or one chunk of it).  The potential of processing-order
        target t goes to ``out[tidx[t] - out_offset]`` (user order) or, with
        ``user_order=False``, to ``out[t - out_offset]``."""
        L = _lib.load()
        flags = ((_lib.FLAG_VALIDATE if validate else 0) | (_lib.FLAG_GENERIC if generic else 0)
                 | (_lib.FLAG_REAL_WEIGHTS if self.real_w else 0)
                 | (_lib.FLAG_ONE_TARGET if self.one_target else 0) | self.kr_flag
                 | (_lib.FLAG_LONG_ROWS if self.near.mean_len >= 48 else 0))
        near = self.near
        g0, g1 = rows if rows is not None else (0, self.n_ctr)
        G = self.G
        if self.tuni:
            # uniform runs: row g of the range owns targets tuni * (g0 + g) ...
            flags |= _lib.FLAG_UNIFORM_TARGETS | (self.tuni << 8)
        if self._auto_split and (g0, g1) != (0, self.n_ctr):
            # a row range (multi-GPU shard) fills fewer waves than the whole problem
            G = pick_split(self.near.mean_len, g1 - g0, self.n_tgt < 2 * self.n_ctr,
                           dv.sm_count(self.dev.index if self.dev.index is not None
                                       else torch.cuda.current_device()),
                           uniform=bool(self.tuni))
        sell = self.layout == "sell" and near.sell_ptr is not None
        if sell and g0 % 32:
            raise ValueError("row ranges on the SELL layout must start at a multiple of 32")
        # the fast S kernels read only the SELL copy; the others need the CSR entries
        fast = self.cfg.p_qbx <= 16 and not generic
        flat = self.flat and fast
        if flat:
            flags |= _lib.FLAG_FLAT
        if self.two_rows and G == 1:
            flags |= _lib.FLAG_TWO_ROWS
        csr = None if (sell and fast and not flat) else near.idx
        if (self.window and sell and fast and not flat and G == 1 and self.tuni
                and near.win_src is not None):
            _lib.check(L.tsqbx_eval_packed_win(
                self.eq, self.variant, self.k, self.cfg.p_qbx, self.packed.data_ptr(),
                self.n_src, self.with_normals, self.ctr.data_ptr() + 24 * g0, g1 - g0,
                near.ptr.data_ptr() + 8 * g0, None,
                near.sell_ptr.data_ptr() + 8 * (g0 // 32), near.sell_loc.data_ptr(),
                near.win_src.data_ptr() + 4 * _lib.WINDOW * (g0 // 32),
                near.win_len.data_ptr() + 4 * (g0 // 32), self.tgt.data_ptr(),
                dv.ptr(self.tn), self.tptr.data_ptr() + 8 * g0, self.n_tgt,
                dv.ptr(self.tidx) if user_order else None, out_offset, self.tuni * g0, flags, G,
                self.ws.data_ptr(), self.ws_bytes, out.data_ptr(), self.err.data_ptr(),
                dv.stream_handle(self.dev)), "tsqbx_eval_packed_win")
            return
        _lib.check(L.tsqbx_eval_packed(
            self.eq, self.variant, self.k, self.cfg.p_qbx, self.packed.data_ptr(), self.n_src,
            self.with_normals, self.ctr.data_ptr() + 24 * g0, g1 - g0,
            near.ptr.data_ptr() + 8 * g0, dv.ptr(csr),
            near.sell_ptr.data_ptr() + 8 * (g0 // 32) if sell else None,
            near.sell_idx.data_ptr() if sell else None, self.tgt.data_ptr(),
            dv.ptr(self.tn), self.tptr.data_ptr() + 8 * g0, self.n_tgt,
            dv.ptr(self.tidx) if user_order else None, out_offset, self.tuni * g0, flags, G,
            self.ws.data_ptr(), self.ws_bytes, out.data_ptr(), self.err.data_ptr(),
            dv.stream_handle(self.dev)), "tsqbx_eval_packed")

    # --- validation -----------------------------------------------------------
    def raise_bad_tptr(self) -> None:
        raise ValueError(f"tgt_ptr must start at 0, be non-decreasing and end at {self.n_tgt}")

    def check_inputs(self) -> None:
        """Raise if the device check of the caller's tgt_ptr failed (one read-back)."""
        if self.check_tptr and int(self.err[1].item()):
            self.raise_bad_tptr()

    def check_errors(self, batch_context: bool) -> None:
        """Raise the reference's ValueError if the screened launch flagged a pair."""
        self.check_inputs()
        if int(self.err[0].item()) == _lib.ERR_KEY_NONE:
            return
        L = _lib.load()
        near = self.near
        _lib.check(L.tsqbx_validate(self.packed.data_ptr(), self.n_src, self.ctr.data_ptr(),
                                    self.n_ctr, near.ptr.data_ptr(), near.idx.data_ptr(),
                                    self.tgt.data_ptr(), self.tptr.data_ptr(), self.n_tgt,
                                    self.err.data_ptr(), dv.stream_handle(self.dev)),
                   "tsqbx_validate")
        key = int(self.err[0].item())
        if key == _lib.ERR_KEY_NONE:
            return            # screen tripped on non-finite weights, not on geometry
        tp, kind, pos = key >> 32, (key >> 31) & 1, key & 0x7FFFFFFF
        g = int(np.searchsorted(self.tptr.cpu().numpy(), tp, side="right") - 1)
        ic = g if near.ctr_order is None else int(near.ctr_order[g].item())
        it = tp if self.tidx is None else int(self.tidx[tp].item())
        s_packed = int(near.idx[int(near.ptr[g].item()) + pos].item())
        s_user = s_packed if near.src_perm is None else int(near.src_perm[s_packed].item())
        where = (f" (target {it}, center {ic}, source index {s_user})" if batch_context else "")
        if kind == 0:
            raise ValueError(f"source {pos} coincides with the expansion center{where}")
        c = self.user_ctr[ic].cpu().numpy()
        s = self.src[s_user].cpu().numpy()
        t = self.user_tgt[it].cpu().numpy()
        R = float(np.linalg.norm(s - c))
        r = float(np.linalg.norm(t - c))
        raise ValueError(f"separation violation for source {pos}: |t-c| = {r} exceeds "
                         f"|s-c| = {R}{where}")


def _inputs(cfg, sources, weights, centers, targets, source_normals, target_normals, dev):
    src = dv.to_device(sources, torch.float64, dev, (-1, 3))
    if isinstance(weights, torch.Tensor) and not weights.is_complex():
        weights = weights.to(torch.complex128)
    w = dv.complex_as_f64(dv.to_device(weights, torch.complex128, dev, (-1,)))
    if w.shape[0] != src.shape[0]:
        raise ValueError("weights must have one entry per source")
    ctr = dv.to_device(centers, torch.float64, dev, (-1, 3))
    tgt = dv.to_device(targets, torch.float64, dev, (-1, 3))
    sn = tn = None
    if cfg.spec.needs_source_normals:
        if source_normals is None:
            raise ValueError("double-layer variant requires source normals")
        sn = dv.to_device(source_normals, torch.float64, dev, (-1, 3))
    if cfg.spec.needs_target_normals:
        if target_normals is None:
            raise ValueError("S' variant requires a target normal")
        tn = dv.to_device(target_normals, torch.float64, dev, (-1, 3))
    return src, w, ctr, tgt, sn, tn


class PendingPotentials:
    """A ``ts_accumulate_batch(..., sync=False)`` evaluation in flight.

    Everything -- the host-to-device copies, the kernels, the copy of the
    potentials into a pinned host buffer and (with validation) of the error key
    -- was enqueued on the stream that was current at the call, so evaluations
    issued on two streams overlap one's PCIe transfers with the other's
    arithmetic.  ``result()`` waits for this one, raises the reference's
    ``ValueError`` if the screen flagged a pair, and returns the potentials."""

    def __init__(self, prep, res: torch.Tensor, out, host_out: bool, validate: bool):
        self._prep, self._res = prep, res
        self._err = None
        self._validate = validate
        if (validate and prep.n_tgt) or prep.check_tptr:
            self._err = torch.empty(2, dtype=torch.int64, pin_memory=True)
            self._err.copy_(prep.err, non_blocking=True)
        self._numpy = out is None and host_out
        if self._numpy:
            out = torch.empty(res.shape, dtype=res.dtype, pin_memory=True)
        if out is not None:
            if not (isinstance(out, torch.Tensor) and out.device.type == "cpu"
                    and out.is_pinned()):
                raise ValueError("sync=False needs `out` to be a pinned host tensor (or None)")
            out.copy_(res, non_blocking=True)
        self._out = out
        self._event = torch.cuda.Event()
        self._event.record()

    def done(self) -> bool:
        return self._event.query()

    def result(self):
        self._event.synchronize()
        if self._err is not None:
            if self._prep.check_tptr and int(self._err[1]):
                self._prep.raise_bad_tptr()
            if self._validate and int(self._err[0]) != _lib.ERR_KEY_NONE:
                self._prep.check_errors(batch_context=True)
        if self._out is None:
            return self._res
        return self._out.numpy() if self._numpy else self._out


@dv.on_device
def ts_accumulate_batch(cfg: TsConfig, sources, weights, centers, targets, near,
                        tgt_ptr=None, source_normals=None, target_normals=None,
                        validate: bool = True, group_lanes: int | None = None, device=None,
                        out=None, sync: bool = True):
    """Per-target TSQBX potentials for many centers in one launch.

    sources (n_src, 3), weights (n_src,) complex, centers (n_ctr, 3),
    targets (n_tgt, 3) grouped by center: targets ``tgt_ptr[c]:tgt_ptr[c+1]``
    belong to center c (default: one target per center).  ``near`` is a
    :class:`NearLists` from :func:`build_near_lists` or a user CSR
    ``(ptr, idx)`` with rows by center and indices into ``sources``.

    Each target's value equals the reference's
    ``ts_accumulate(cfg, sources[near(c)], weights[near(c)], centers[c], t)``
    (tsqbx.py:68-80).  Returns complex128: numpy for host inputs, a CUDA
    tensor when ``sources`` is a CUDA tensor.

    ``sync=False`` returns a :class:`PendingPotentials` instead: the whole call
    is enqueued on the current stream (inputs should be pinned tensors, ``out``
    a pinned tensor or None) and nothing waits for the GPU until ``result()``.
    """
    host_out = not (isinstance(sources, torch.Tensor) and sources.is_cuda)
    dev = dv.require_cuda(device)
    src, w, ctr, tgt, sn, tn = _inputs(cfg, sources, weights, centers, targets,
                                       source_normals, target_normals, dev)
    n_ctr = int(ctr.shape[0])
    if tgt_ptr is None:
        if tgt.shape[0] != n_ctr:
            raise ValueError("tgt_ptr is required unless there is one target per center")
        tptr = torch.arange(n_ctr + 1, dtype=torch.int64, device=dev)
    else:
        tptr = dv.to_device(tgt_ptr, torch.int64, dev)
    if not isinstance(near, NearLists):
        nptr, nidx = near
        near = NearLists.from_user_csr(nptr, nidx, int(src.shape[0]), dev)
    prep = _Prepared(cfg, dev, src, w, sn, ctr, near, tgt, tn, tptr, group_lanes,
                     user_tptr=tgt_ptr is not None)
    if tgt_ptr is None:
        prep.set_uniform_targets(known=True)
    res = torch.empty(prep.n_tgt, dtype=torch.complex128, device=dev)
    if prep.n_tgt:
        prep.launch(torch.view_as_real(res), validate)
    pinned_out = isinstance(out, torch.Tensor) and out.device.type == "cpu" and out.is_pinned()
    if not sync or (prep.n_tgt and (pinned_out or (out is None and host_out))):
        # the potentials and the error key come back in one stream-ordered pass
        # (one synchronisation instead of one for the key and one for the copy)
        pend = PendingPotentials(prep, res, out, host_out, validate)
        return pend if not sync else pend.result()
    if prep.n_tgt and validate:
        prep.check_errors(batch_context=True)
    else:
        prep.check_inputs()
    return _deliver(res, out, host_out)


def _deliver(out_dev: torch.Tensor, out, host_out: bool):
    """Result hand-off: into a caller buffer (a pinned host tensor makes the D2H a
    direct DMA), else numpy for host inputs / the CUDA tensor for device inputs."""
    if out is not None:
        if isinstance(out, np.ndarray):
            out[...] = out_dev.cpu().numpy()
        else:
            out.copy_(out_dev)
        return out
    return out_dev.cpu().numpy() if host_out else out_dev


FUSED_ROW_CAP = 1024     # near sources per row the fused kernel's scratch slice holds


def _uniform_run(tgt_ptr, n_ctr: int, n_tgt: int, dev) -> int:
    """k when every center owns k consecutive targets (tgt_ptr = k * arange), else 0."""
    if tgt_ptr is None:
        return 1 if n_tgt == n_ctr else 0
    k = n_tgt // n_ctr if n_ctr else 0
    if not (1 <= k <= 2 and k * n_ctr == n_tgt):
        return 0
    if isinstance(tgt_ptr, torch.Tensor):
        ok = bool(torch.equal(tgt_ptr.to(device=dev, dtype=torch.int64),
                              torch.arange(n_ctr + 1, dtype=torch.int64, device=dev) * k))
    else:
        ok = bool(np.array_equal(np.asarray(tgt_ptr), np.arange(n_ctr + 1) * k))
    return k if ok else 0


def _fused_potentials(cfg: TsConfig, dev, src, w, ctr, rad, tgt, k_run: int, validate: bool,
                      row_cap: int):
    """One-shot near field through tsqbx_eval_fused (csrc/fused.cu): Morton sorts
    and cell hash (tsqbx_near_index), then one kernel that sweeps every warp's 32
    rows into a scratch slice and evaluates them -- no CSR in HBM.  Returns the
    potentials (CUDA, user order) or None when a row overflowed the scratch slice
    or the validation screen fired (the caller takes the two-step path, which
    names the offending source exactly)."""
    L = _lib.load()
    st = dv.stream_handle(dev)
    spec = cfg.spec
    n_src, n_ctr, n_tgt = int(src.shape[0]), int(ctr.shape[0]), int(tgt.shape[0])
    eq = _equation_code(spec)
    sb = int(L.tsqbx_fused_scratch_bytes(eq, cfg.p_qbx, k_run, int(validate), row_cap))
    if sb < 0:
        return None
    wsb = int(L.tsqbx_near_workspace_bytes(n_ctr, n_src))
    ws = torch.empty(max(wsb, 1), dtype=torch.uint8, device=dev)
    src_perm = torch.empty(max(n_src, 1), dtype=torch.int32, device=dev)
    ctr_order = torch.empty(max(n_ctr, 1), dtype=torch.int32, device=dev)
    _lib.check(L.tsqbx_near_index(ctr.data_ptr(), rad.data_ptr(), n_ctr, src.data_ptr(), n_src,
                                  ws.data_ptr(), wsb, src_perm.data_ptr(), ctr_order.data_ptr(),
                                  st), "tsqbx_near_index")
    nd = int(L.tsqbx_packed_doubles(n_src, 0))
    packed = torch.empty(max(nd, 4), dtype=torch.float64, device=dev)
    _lib.check(L.tsqbx_pack_sources(n_src, src.data_ptr(), w.data_ptr(), None,
                                    src_perm.data_ptr(), packed.data_ptr(), st),
               "tsqbx_pack_sources")
    tptr = torch.arange(n_ctr + 1, dtype=torch.int64, device=dev) * k_run
    ctr_p, tptr_p, tgt_p = torch.empty_like(ctr), torch.empty_like(tptr), torch.empty_like(tgt)
    tidx = torch.empty(max(n_tgt, 1), dtype=torch.int64, device=dev)
    owb = int(L.tsqbx_order_workspace_bytes(n_ctr))
    ows = torch.empty(max(owb, 1), dtype=torch.uint8, device=dev)
    _lib.check(L.tsqbx_order_targets(n_ctr, ctr_order.data_ptr(), ctr.data_ptr(), tptr.data_ptr(),
                                     tgt.data_ptr(), None, n_tgt, ows.data_ptr(), owb,
                                     ctr_p.data_ptr(), tptr_p.data_ptr(), tgt_p.data_ptr(), None,
                                     tidx.data_ptr(), None, st), "tsqbx_order_targets")
    flags = (_lib.FLAG_UNIFORM_TARGETS | (k_run << 8)
             | (_lib.FLAG_VALIDATE if validate else 0))
    if not spec.is_laplace:
        # every member lies within the largest radius: one sin/cos series, no vote
        kr = float(spec.helmholtz_k) * float(rad.max().item()) * (1.0 + 1e-12)
        flags |= (_lib.FLAG_KR_NARROW if kr <= math.pi / 4 else
                  _lib.FLAG_KR_WIDE if kr <= math.pi / 2 else 0)
    scratch = torch.empty(sb, dtype=torch.uint8, device=dev)
    err = torch.empty(2, dtype=torch.int64, device=dev)
    res = torch.empty(n_tgt, dtype=torch.complex128, device=dev)
    _lib.check(L.tsqbx_eval_fused(eq, float(spec.helmholtz_k or 0.0), cfg.p_qbx,
                                  packed.data_ptr(), n_src, ctr.data_ptr(), rad.data_ptr(),
                                  ctr_order.data_ptr(), ws.data_ptr(), wsb, ctr_p.data_ptr(),
                                  n_ctr, tgt_p.data_ptr(), n_tgt, tidx.data_ptr(), flags,
                                  row_cap, scratch.data_ptr(), sb,
                                  torch.view_as_real(res).data_ptr(), err.data_ptr(), st),
               "tsqbx_eval_fused")
    key, overflow = err.tolist()
    if overflow or (validate and key != _lib.ERR_KEY_NONE):
        return None
    return res


@dv.on_device
def near_field_potentials(cfg: TsConfig, sources, weights, centers, near_radii, targets,
                          tgt_ptr=None, source_normals=None, target_normals=None,
                          validate: bool = True, group_lanes: int | None = None, device=None,
                          out=None, fused: bool | None = None):
    """The whole near-field path in one call: geometry -> device radius-ball near
    lists -> TSQBX evaluation -> per-target potentials.

    Host inputs are copied to the device once (asynchronously when they are
    pinned tensors); the result comes back as numpy, into ``out`` (e.g. a
    pinned complex128 tensor) when given, or stays a CUDA tensor when
    ``sources`` is one.

    ``fused=True`` (or GIGAQBX_FUSED=1; S, p <= 16, one or two targets per
    center in runs, no ``group_lanes``): the near lists are swept and evaluated
    in one kernel without a CSR in HBM (``tsqbx_eval_fused``); a row with more
    than FUSED_ROW_CAP sources or a flagged validation screen re-runs through
    ``build_near_lists`` + the evaluation kernels, which also raise the
    reference's ValueError.  Off by default: measured slower than the two-step
    path (C5 dense 48.7 vs 41.5 ms end to end -- the fused kernel's sweep and
    evaluation phases do not overlap on an SM, 26.5 ms against 27 ms for the
    count, fill and evaluation kernels)."""
    from .nearlist import build_near_lists

    host_out = not (isinstance(sources, torch.Tensor) and sources.is_cuda)
    dev = dv.require_cuda(device)
    # the geometry the near lists need goes first, on the current stream; the
    # rest of the payload (weights, targets, offsets, normals) is copied on a
    # side stream while the lists are built
    src = dv.to_device(sources, torch.float64, dev, (-1, 3))
    ctr = dv.to_device(centers, torch.float64, dev, (-1, 3))
    n_ctr = int(ctr.shape[0])
    rad = (near_radii.to(device=dev, dtype=torch.float64) if isinstance(near_radii, torch.Tensor)
           else dv.to_device(np.broadcast_to(np.asarray(near_radii, np.float64), (n_ctr,)),
                             torch.float64, dev))
    main = torch.cuda.current_stream(dev)
    side = dv.side_stream(dev)
    side.wait_stream(main)
    with torch.cuda.stream(side):
        _, w, _, tgt, sn, tn = _inputs(cfg, src, weights, ctr, targets, source_normals,
                                       target_normals, dev)
        tptr = (torch.arange(n_ctr + 1, dtype=torch.int64, device=dev) if tgt_ptr is None
                else dv.to_device(tgt_ptr, torch.int64, dev))
    if fused is None:
        fused = os.environ.get("GIGAQBX_FUSED", "0") == "1"
    fused = (fused and cfg.spec.variant_code == 0 and cfg.p_qbx <= 16 and not group_lanes
             and n_ctr > 0)
    if fused:
        main.wait_stream(side)
        for t in (w, tgt, tptr):
            if t is not None:
                t.record_stream(main)
        if tgt_ptr is None and int(tgt.shape[0]) != n_ctr:
            raise ValueError("tgt_ptr is required unless there is one target per center")
        k_run = _uniform_run(tgt_ptr, n_ctr, int(tgt.shape[0]), dev)
        if k_run:
            row_cap = int(os.environ.get("GIGAQBX_FUSED_ROW_CAP", FUSED_ROW_CAP))
            radc = (rad.reshape(-1).expand(n_ctr) if rad.numel() == 1 else rad.reshape(-1))
            res = _fused_potentials(cfg, dev, src, w, ctr, radc.contiguous(), tgt, k_run,
                                    validate, row_cap)
            if res is not None:
                return _deliver(res, out, host_out)
    near = build_near_lists(ctr, src, rad, dev)
    main.wait_stream(side)
    for t in (w, tgt, sn, tn, tptr):
        if t is not None:
            t.record_stream(main)
    if tgt_ptr is None and int(tgt.shape[0]) != n_ctr:
        raise ValueError("tgt_ptr is required unless there is one target per center")
    prep = _Prepared(cfg, dev, src, w, sn, ctr, near, tgt, tn, tptr, group_lanes,
                     user_tptr=tgt_ptr is not None)
    if tgt_ptr is None:
        prep.set_uniform_targets(known=True)
    if _direct_out(out, prep):
        # the kernel writes the potentials straight into the caller's pinned
        # host buffer (mapped through unified addressing): the device-to-host
        # copy overlaps the evaluation instead of following it
        prep.launch(torch.view_as_real(out), validate)
        if prep.n_tgt and validate:
            prep.check_errors(batch_context=True)
        else:
            prep.check_inputs()
        torch.cuda.current_stream(dev).synchronize()
        return out
    res = torch.empty(prep.n_tgt, dtype=torch.complex128, device=dev)
    if prep.n_tgt:
        prep.launch(torch.view_as_real(res), validate)
    if prep.n_tgt and validate:
        prep.check_errors(batch_context=True)
    else:
        prep.check_inputs()
    return _deliver(res, out, host_out)


# Writing the potentials straight into pinned host memory moves the D2H copy
# under the evaluation, but each scattered 16-byte store crosses PCIe: it pays
# when the evaluation lasts longer than those stores take (~12 GB/s measured
# for scattered complex128 stores): C5 dense 42.1 -> 39.6 ms end to end, C2
# dense 2.18 -> 2.68 ms (a 0.3 ms kernel cannot hide 8 MB of stores).
_DIRECT_OUT_GBS = 12.0
_KERNEL_TFLOPS = 0.65 * 35.7       # the dense kernels' typical rate


def _direct_out(out, prep) -> bool:
    """Whether the kernels write into ``out`` (a pinned complex128 host tensor
    of n_tgt entries) directly; GIGAQBX_DIRECT_OUT=0/1 overrides the estimate."""
    n_tgt = prep.n_tgt
    if not (isinstance(out, torch.Tensor) and out.device.type == "cpu" and out.is_pinned()
            and out.dtype == torch.complex128 and out.is_contiguous()
            and int(out.numel()) == n_tgt and n_tgt > 0):
        return False
    env = os.environ.get("GIGAQBX_DIRECT_OUT")
    if env is not None:
        return env == "1"
    from .configs import algorithmic_flops_per_pair
    pairs = prep.near.n_pairs * n_tgt / max(1, prep.n_ctr)
    kernel_s = pairs * algorithmic_flops_per_pair(prep.cfg.spec, prep.cfg.p_qbx) / (
        _KERNEL_TFLOPS * 1e12)
    return kernel_s >= 16.0 * n_tgt / (_DIRECT_OUT_GBS * 1e9)


class TsqbxProblem:
    """A TSQBX problem resident in HBM: packed sources, CSR, targets, workspace.

    ``evaluate()`` is one launch of the hot path over every (center, target);
    nothing is copied between host and device.
    """

    @dv.on_device
    def __init__(self, cfg: TsConfig, sources, weights, centers, targets, near: NearLists,
                 tgt_ptr=None, source_normals=None, target_normals=None,
                 group_lanes: int | None = None, device=None):
        dev = dv.require_cuda(device)
        src, w, ctr, tgt, sn, tn = _inputs(cfg, sources, weights, centers, targets,
                                           source_normals, target_normals, dev)
        n_ctr = int(ctr.shape[0])
        if tgt_ptr is None and int(tgt.shape[0]) != n_ctr:
            raise ValueError("tgt_ptr is required unless there is one target per center")
        tptr = (torch.arange(n_ctr + 1, dtype=torch.int64, device=dev) if tgt_ptr is None
                else dv.to_device(tgt_ptr, torch.int64, dev))
        self.prep = _Prepared(cfg, dev, src, w, sn, ctr, near, tgt, tn, tptr, group_lanes,
                              user_tptr=tgt_ptr is not None)
        self.prep.check_inputs()        # once per problem (evaluate() never re-checks)
        self.prep.set_uniform_targets(known=tgt_ptr is None)
        self.out = torch.empty(self.prep.n_tgt, dtype=torch.complex128, device=dev)
        self.n_pairs_per_target = None

    @property
    def dev(self) -> torch.device:
        return self.prep.dev

    @dv.on_own_device
    def set_weights(self, weights) -> None:
        """New densities for the same geometry (GMRES matvecs): one pack kernel."""
        if isinstance(weights, torch.Tensor) and not weights.is_complex():
            weights = weights.to(torch.complex128)
        self.prep.pack(dv.complex_as_f64(dv.to_device(weights, torch.complex128,
                                                      self.prep.dev, (-1,))))

    @property
    def group_lanes(self) -> int:
        return self.prep.G

    @property
    def layout(self) -> str:
        return self.prep.layout

    @dv.on_own_device
    def evaluate(self, validate: bool = False, generic: bool = False) -> torch.Tensor:
        if self.prep.n_tgt:
            self.prep.launch(torch.view_as_real(self.out), validate, generic)
            if validate:
                self.prep.check_errors(batch_context=True)
        return self.out

    def pair_count(self) -> int:
        """Number of (target, near source) pairs one evaluate() processes."""
        near, prep = self.prep.near, self.prep
        lens = near.ptr[1:] - near.ptr[:-1]
        tpc = prep.tptr[1:] - prep.tptr[:-1]
        return int((lens * tpc).sum().item())


def ts_accumulate(cfg: TsConfig, sources, weights, center, target,
                  source_normals=None, target_normal=None) -> complex:
    """sum_j w_j * (p-th order target-specific expansion of source j)  (tsqbx.py:68-80).

    Same checks, in the same order, as the reference's ``_prep``
    (tsqbx.py:38-65): coincident source, separation, then the normals.  The
    geometric checks run exactly inside the single-call kernel; the value comes
    from the same launch (one H2D copy, one kernel, one D2H copy)."""
    from ._single import one_call

    sources = np.ascontiguousarray(sources, dtype=np.float64).reshape(-1, 3)
    weights = np.ascontiguousarray(weights, dtype=np.complex128).reshape(-1)
    center = np.asarray(center, dtype=np.float64).reshape(3)
    target = np.asarray(target, dtype=np.float64).reshape(3)
    spec = cfg.spec
    need_sn = spec.needs_source_normals and source_normals is None
    need_tn = spec.needs_target_normals and target_normal is None
    r = float(np.linalg.norm(target - center))
    n = sources.shape[0]
    if need_sn or need_tn or n == 0:
        _prep_geometry(sources, center, r)          # geometry errors come first
        if need_sn:
            raise ValueError("double-layer variant requires source normals")
        if need_tn:
            raise ValueError("S' variant requires a target normal")
        return 0.0 + 0.0j
    sn = (np.ascontiguousarray(source_normals, dtype=np.float64).reshape(-1, 3)
          if spec.needs_source_normals else None)
    tn = (np.asarray(target_normal, dtype=np.float64).reshape(3)
          if spec.needs_target_normals else None)
    value, key = one_call(_equation_code(spec), spec.variant_code, float(spec.helmholtz_k or 0.0),
                          cfg.p_qbx, sources, weights, sn, center, target, tn, validate=True,
                          r_ref=r)
    if key != _lib.ERR_KEY_NONE:
        _prep_geometry(sources, center, r)          # names the source like the reference
        raise RuntimeError(f"device validation key {key:#x} not reproduced on the host")
    return value


def _prep_geometry(sources, center, r):
    """The reference's geometric checks and messages (tsqbx.py:42-51)."""
    R = np.linalg.norm(sources - center, axis=1)
    if np.any(R == 0.0):
        raise ValueError(f"source {int(np.argmin(R))} coincides with the expansion center")
    viol = R * (1.0 + _SEP_SLACK) < r
    if np.any(viol):
        bad = int(np.argmax(viol))
        raise ValueError(
            f"separation violation for source {bad}: |t-c| = {r} exceeds |s-c| = {R[bad]}")


def ts_eval(cfg: TsConfig, source, center, target, source_normal=None,
            target_normal=None) -> complex:
    """Target-specific expansion value for a single unit-weight source (tsqbx.py:83-92)."""
    sn = None if source_normal is None else np.asarray(source_normal).reshape(1, 3)
    return ts_accumulate(cfg, np.asarray(source, dtype=np.float64).reshape(1, 3),
                         np.ones(1, dtype=np.complex128), center, target,
                         source_normals=sn, target_normal=target_normal)
