"""Near-list construction on the device.

BASELINE.json defines a QBX center's near field as every source within a
radius of it (self included).  The reference has no such builder -- its driver
gathers tree lists per target box (driver.py:197-228, ilists.py:93-218) and
uses ``cKDTree.query_ball_point`` elsewhere (costmodel.py:361-365) -- so
``build_near_lists`` is the device replacement for that step:

* sources and centers are Morton-sorted ("tree leaf" order) so that the
  centers one CTA evaluates share a source neighbourhood,
* the CSR rows are stored in that processing order and index the sorted
  sources, ascending within a row,
* membership is ``((dx*dx + dy*dy) + dz*dz) <= rad*rad`` without FMA
  contraction, bit-identical to the oracle (``oracle.near_csr``).

A user-supplied CSR (user center rows, user source indices) is accepted too
(``NearLists.from_user_csr``); it is evaluated in place without reordering.
"""

from __future__ import annotations

import os
from dataclasses import dataclass

import numpy as np
import torch

from . import _device as dv
from . import _lib


@dataclass
class NearLists:
    """Device CSR from centers to near sources.

    ptr[g]..ptr[g+1] is the row of center ``ctr_order[g]`` (identity when
    ``ctr_order`` is None); idx entries index the sources in *packed* order,
    i.e. user source ``src_perm[idx]`` (identity when ``src_perm`` is None).
    """

    n_ctr: int
    n_src: int
    n_pairs: int
    ptr: torch.Tensor
    csr_idx: torch.Tensor | None          # CSR entries; None until first needed
    src_perm: torch.Tensor | None = None
    ctr_order: torch.Tensor | None = None
    sell_ptr: torch.Tensor | None = None
    sell_idx: torch.Tensor | None = None
    max_radius: float | None = None      # every entry has |s - c| <= max_radius (None: unknown)
    # windowed SELL (short lists, build_window): window-local entries + windows
    sell_loc: torch.Tensor | None = None
    win_src: torch.Tensor | None = None
    win_len: torch.Tensor | None = None

    @property
    def dev(self) -> torch.device:
        return self.ptr.device

    @property
    @dv.on_own_device
    def idx(self) -> torch.Tensor:
        """CSR entries (materialised from the SELL copy on first use: the fast
        kernels read only the SELL layout)."""
        if self.csr_idx is None:
            L = _lib.load()
            dev = self.ptr.device
            out = torch.empty(max(self.n_pairs, 1), dtype=torch.int32, device=dev)
            _lib.check(L.tsqbx_sell_to_csr(self.n_ctr, self.ptr.data_ptr(),
                                           self.sell_ptr.data_ptr(), self.sell_idx.data_ptr(),
                                           out.data_ptr(), dv.stream_handle(dev)),
                       "tsqbx_sell_to_csr")
            self.csr_idx = out[:self.n_pairs]
        return self.csr_idx

    @property
    def mean_len(self) -> float:
        return self.n_pairs / max(1, self.n_ctr)

    @dv.on_own_device
    def build_sell(self) -> "NearLists":
        """Add the sliced-ELL (SELL-32) copy the thread-per-center kernels read:
        slices of 32 rows, entries column-major (coalesced index loads)."""
        if self.sell_ptr is not None:
            return self
        L = _lib.load()
        dev = self.ptr.device
        st = dv.stream_handle(dev)
        n_sl = (self.n_ctr + 31) // 32
        wsb = int(L.tsqbx_sell_workspace_bytes(self.n_ctr))
        ws = torch.empty(max(wsb, 1), dtype=torch.uint8, device=dev)
        sptr = torch.empty(n_sl + 1, dtype=torch.int64, device=dev)
        n_ent = torch.zeros(1, dtype=torch.int64, device=dev)
        _lib.check(L.tsqbx_sell_size(self.n_ctr, self.ptr.data_ptr(), ws.data_ptr(), wsb,
                                     sptr.data_ptr(), n_ent.data_ptr(), st), "tsqbx_sell_size")
        sidx = torch.empty(max(int(n_ent.item()), 1), dtype=torch.int32, device=dev)
        _lib.check(L.tsqbx_sell_fill(self.n_ctr, self.ptr.data_ptr(), self.idx.data_ptr(),
                                     sptr.data_ptr(), sidx.data_ptr(), st), "tsqbx_sell_fill")
        self.sell_ptr, self.sell_idx = sptr, sidx
        return self

    @dv.on_own_device
    def build_window(self) -> bool:
        """The windowed SELL copy for short lists (``tsqbx_sell_window``): per
        32-row slice its distinct sources (<= _lib.WINDOW) and the entries as
        indices into them; a slice with more distinct sources than the window
        keeps global indices (counted in ``win_overflow``)."""
        if self.win_src is not None:
            return True
        if self.sell_ptr is None:
            return False
        L = _lib.load()
        dev = self.ptr.device
        n_sl = (self.n_ctr + 31) // 32
        loc = torch.empty_like(self.sell_idx)
        win = torch.empty(max(n_sl * _lib.WINDOW, 1), dtype=torch.int32, device=dev)
        wlen = torch.zeros(max(n_sl, 1), dtype=torch.int32, device=dev)
        flag = torch.zeros(1, dtype=torch.int32, device=dev)
        _lib.check(L.tsqbx_sell_window(self.n_ctr, self.ptr.data_ptr(), self.sell_ptr.data_ptr(),
                                       self.sell_idx.data_ptr(), loc.data_ptr(), win.data_ptr(),
                                       wlen.data_ptr(), flag.data_ptr(), dv.stream_handle(dev)),
                   "tsqbx_sell_window")
        self.win_overflow = int(flag.item())      # slices that keep global indices
        self.sell_loc, self.win_src, self.win_len = loc, win, wlen
        return True

    @property
    def sell_fill(self) -> float:
        """Fraction of SELL slots holding a real entry (1 - padding)."""
        if self.sell_idx is None:
            return float("nan")
        return self.n_pairs / max(1, int(self.sell_ptr[-1].item()))

    @classmethod
    @dv.on_device
    def from_user_csr(cls, ptr, idx, n_src: int, device=None) -> "NearLists":
        """A caller's CSR (rows by center, entries index ``sources``), checked the
        way the reference's indexing would fail: ``ptr[0] == 0``, non-decreasing,
        ``ptr[-1] == len(idx)``, ``0 <= idx < n_src`` (ValueError otherwise)."""
        dev = device
        p = dv.to_device(ptr, torch.int64, dev)
        i = dv.to_device(idx, torch.int32, dev)
        n_ctr = int(p.shape[0]) - 1
        n_pairs = int(i.shape[0])
        if n_ctr < 0:
            raise ValueError("near-list ptr must have n_centers + 1 entries")
        check_offsets(p, n_pairs, "near-list ptr")
        if n_pairs and bool(((i < 0) | (i >= n_src)).any()):
            raise ValueError(f"near-list indices must lie in [0, {n_src})")
        return cls(n_ctr=n_ctr, n_src=n_src, n_pairs=n_pairs, ptr=p, csr_idx=i)

    def to_user_csr(self) -> tuple[np.ndarray, np.ndarray]:
        """(ptr, idx) on the host with rows by user center and user source indices."""
        ptr = self.ptr.cpu().numpy()
        idx = self.idx.cpu().numpy()
        if self.src_perm is not None:
            idx = self.src_perm.cpu().numpy()[idx]
        if self.ctr_order is None:
            return ptr, idx.astype(np.int32)
        order = self.ctr_order.cpu().numpy()
        lens = np.diff(ptr)
        user_lens = np.empty_like(lens)
        user_lens[order] = lens
        uptr = np.zeros(self.n_ctr + 1, dtype=np.int64)
        np.cumsum(user_lens, out=uptr[1:])
        uidx = np.empty_like(idx)
        dest = np.repeat(uptr[order] - ptr[:-1], lens) + np.arange(idx.shape[0])
        uidx[dest] = idx
        return uptr, uidx.astype(np.int32)


def check_offsets(ptr: torch.Tensor, total: int, name: str) -> None:
    """CSR offsets: ptr[0] == 0, non-decreasing, ptr[-1] == total (one read-back);
    malformed offsets would otherwise index outside the device arrays."""
    if ptr.numel() == 0:
        raise ValueError(f"{name} must not be empty")
    ends = torch.stack([ptr[0], ptr[-1], (ptr[1:] < ptr[:-1]).any().to(torch.int64)]).tolist()
    if ends[0] != 0 or ends[1] != total or ends[2]:
        raise ValueError(f"{name} must start at 0, be non-decreasing and end at {total} "
                         f"(got first {ends[0]}, last {ends[1]})")


_BOUND_BYTES_MAX = 16 << 30     # bound-sized SELL buffer above this: count exactly
_COMPACT_ABOVE = 1.5            # bound slots / exact slots above this: compact the slices
# exact route: keep the count's member masks for the fill (GIGAQBX_EXACT_MASKS=0: test twice)
_EXACT_MASKS = os.environ.get("GIGAQBX_EXACT_MASKS", "1") != "0"


@dv.on_device
def build_near_lists(centers, sources, radii, device=None, sell: bool = True) -> NearLists:
    """Radius-ball near lists {s : |s - c|^2 <= rad_c^2} on the device.

    centers (n_ctr, 3), sources (n_src, 3), radii scalar or (n_ctr,) -- numpy
    arrays or torch tensors.  Returns a device :class:`NearLists` in Morton
    processing order, with the SELL-32x4 copy the fast kernels read (``sell``).
    One host read-back (the two totals) sizes the index arrays.
    """
    dev = dv.require_cuda(device)
    L = _lib.load()
    ctr = dv.to_device(centers, torch.float64, dev, (-1, 3))
    src = dv.to_device(sources, torch.float64, dev, (-1, 3))
    n_ctr, n_src = int(ctr.shape[0]), int(src.shape[0])
    if isinstance(radii, torch.Tensor):
        rad = radii.to(device=dev, dtype=torch.float64).reshape(-1).contiguous()
        if rad.numel() == 1:
            rad = rad.expand(n_ctr).contiguous()
    else:
        rad = dv.to_device(np.broadcast_to(np.asarray(radii, dtype=np.float64), (n_ctr,)),
                           torch.float64, dev)
    st = dv.stream_handle(dev)
    ws_bytes = int(L.tsqbx_near_workspace_bytes(n_ctr, n_src))
    ws = torch.empty(max(ws_bytes, 1), dtype=torch.uint8, device=dev)
    src_perm = torch.empty(max(n_src, 1), dtype=torch.int32, device=dev)
    ctr_order = torch.empty(max(n_ctr, 1), dtype=torch.int32, device=dev)
    nptr = torch.empty(n_ctr + 1, dtype=torch.int64, device=dev)
    sptr = torch.empty((n_ctr + 31) // 32 + 1, dtype=torch.int64, device=dev) if sell else None
    totals = torch.zeros(2, dtype=torch.int64, device=dev)
    _lib.check(L.tsqbx_near_count(dv.ptr(ctr), dv.ptr(rad), n_ctr, dv.ptr(src), n_src,
                                  ws.data_ptr(), ws_bytes, src_perm.data_ptr(),
                                  ctr_order.data_ptr(), nptr.data_ptr(), dv.ptr(sptr),
                                  totals.data_ptr(), st), "tsqbx_near_count")
    if sell:
        # slice widths bounded by candidate counts: one read-back sizes the SELL
        # slots, the fill then produces the exact row lengths
        n_sell = int(totals[1].item())
        exact = n_sell * 4 > _BOUND_BYTES_MAX
        mws = None
        if exact:
            # a loose bound (union candidates far above the members, e.g. C5)
            # would need too much memory: count exactly (reusing the sorts and
            # the cell hash), size the slices from the exact lengths, fill them.
            # The count keeps its member masks (one bit per candidate and
            # center, ~1/30 of the bound-sized buffer) so the fill does not
            # test the candidates a second time.
            if _EXACT_MASKS:
                mbytes = int(L.tsqbx_near_mask_bytes(n_ctr, n_sell))
                mws = torch.empty(mbytes, dtype=torch.uint8, device=dev)
                _lib.check(L.tsqbx_near_recount_masks(
                    dv.ptr(ctr), dv.ptr(rad), n_ctr, n_src, ws.data_ptr(), ws_bytes,
                    ctr_order.data_ptr(), nptr.data_ptr(), totals.data_ptr(), mws.data_ptr(),
                    mbytes, st), "tsqbx_near_recount_masks")
            else:
                _lib.check(L.tsqbx_near_recount(dv.ptr(ctr), dv.ptr(rad), n_ctr, n_src,
                                                ws.data_ptr(), ws_bytes, ctr_order.data_ptr(),
                                                nptr.data_ptr(), totals.data_ptr(), st),
                           "tsqbx_near_recount")
            wsb = int(L.tsqbx_sell_workspace_bytes(n_ctr))
            sws = torch.empty(max(wsb, 1), dtype=torch.uint8, device=dev)
            _lib.check(L.tsqbx_sell_size(n_ctr, nptr.data_ptr(), sws.data_ptr(), wsb,
                                         sptr.data_ptr(), totals[1:].data_ptr(), st),
                       "tsqbx_sell_size")
            n_sell = int(totals[1].item())
        idx = None
        sidx = torch.empty(max(n_sell, 4), dtype=torch.int32, device=dev)
    else:
        n_pairs = int(totals[0].item())
        idx = torch.empty(max(n_pairs, 1), dtype=torch.int32, device=dev)
        sidx = None
    if sell and mws is not None:
        _lib.check(L.tsqbx_near_fill_masks(dv.ptr(ctr), dv.ptr(rad), n_ctr, n_src, ws.data_ptr(),
                                           ws_bytes, ctr_order.data_ptr(), nptr.data_ptr(),
                                           sptr.data_ptr(), sidx.data_ptr(), totals.data_ptr(),
                                           mws.data_ptr(), mbytes, st), "tsqbx_near_fill_masks")
    else:
        _lib.check(L.tsqbx_near_fill(dv.ptr(ctr), dv.ptr(rad), n_ctr, dv.ptr(src), n_src,
                                     ws.data_ptr(), ws_bytes, ctr_order.data_ptr(),
                                     nptr.data_ptr(), dv.ptr(idx), dv.ptr(sptr), dv.ptr(sidx),
                                     totals.data_ptr(), st), "tsqbx_near_fill")
    if sell and exact:
        n_pairs = int(totals[0].item())
    elif sell:
        # exact slice widths (the layout a counting build produces), then drop the
        # bound-sized buffer; one read-back gives the pair count and the slot count
        n_sl = (n_ctr + 31) // 32
        wsb = int(L.tsqbx_sell_workspace_bytes(n_ctr))
        sws = torch.empty(max(wsb, 1), dtype=torch.uint8, device=dev)
        xptr = torch.empty(n_sl + 1, dtype=torch.int64, device=dev)
        _lib.check(L.tsqbx_sell_size(n_ctr, nptr.data_ptr(), sws.data_ptr(), wsb, xptr.data_ptr(),
                                     totals[1:].data_ptr(), st), "tsqbx_sell_size")
        n_pairs, n_exact = (int(v) for v in totals.tolist())
        if n_sell > _COMPACT_ABOVE * n_exact:
            xidx = torch.empty(max(n_exact, 4), dtype=torch.int32, device=dev)
            _lib.check(L.tsqbx_sell_compact(n_ctr, sptr.data_ptr(), sidx.data_ptr(),
                                            xptr.data_ptr(), xidx.data_ptr(), st),
                       "tsqbx_sell_compact")
            sptr, sidx = xptr, xidx
        # else: the bound-sized slices are kept as they are -- every index was
        # written once, the kernels never read a slot past a row's length, and
        # the DRAM index stream is the same (a row's blocks stay contiguous)
    return NearLists(n_ctr=n_ctr, n_src=n_src, n_pairs=n_pairs, ptr=nptr,
                     csr_idx=None if idx is None else idx[:n_pairs],
                     src_perm=src_perm[:n_src], ctr_order=ctr_order[:n_ctr],
                     sell_ptr=sptr, sell_idx=sidx,
                     max_radius=float(rad.max().item()) if n_ctr else 0.0)


class NearRowBuilder:
    """Near lists built one processing-row range at a time (multi-GPU shards).

    ``tsqbx_near_count`` runs once over ALL centers (Morton sort of sources and
    centers, source grid/hash, exact row lengths): every rank knows the global
    processing order and every row's length, so it can cut the rows into
    ranges of equal pair count; ``rows(g0, g1)`` then fills only that range's
    lists (``tsqbx_near_fill_rows``, SELL-32x4) -- a rank never stores the
    other ranks' indices.
    """

    @dv.on_device
    def __init__(self, centers, sources, radii, device=None):
        self.dev = dev = device
        L = _lib.load()
        self.ctr = dv.to_device(centers, torch.float64, dev, (-1, 3))
        self.src = dv.to_device(sources, torch.float64, dev, (-1, 3))
        self.n_ctr, self.n_src = int(self.ctr.shape[0]), int(self.src.shape[0])
        if isinstance(radii, torch.Tensor):
            rad = radii.to(device=dev, dtype=torch.float64).reshape(-1).contiguous()
            self.rad = rad.expand(self.n_ctr).contiguous() if rad.numel() == 1 else rad
        else:
            self.rad = dv.to_device(np.broadcast_to(np.asarray(radii, dtype=np.float64),
                                                    (self.n_ctr,)), torch.float64, dev)
        st = dv.stream_handle(dev)
        self.ws_bytes = int(L.tsqbx_near_workspace_bytes(self.n_ctr, self.n_src))
        self.ws = torch.empty(max(self.ws_bytes, 1), dtype=torch.uint8, device=dev)
        self.src_perm = torch.empty(max(self.n_src, 1), dtype=torch.int32, device=dev)
        self.ctr_order = torch.empty(max(self.n_ctr, 1), dtype=torch.int32, device=dev)
        self.ptr = torch.empty(self.n_ctr + 1, dtype=torch.int64, device=dev)
        self.totals = torch.zeros(2, dtype=torch.int64, device=dev)
        _lib.check(L.tsqbx_near_count(self.ctr.data_ptr(), self.rad.data_ptr(), self.n_ctr,
                                      self.src.data_ptr(), self.n_src, self.ws.data_ptr(),
                                      self.ws_bytes, self.src_perm.data_ptr(),
                                      self.ctr_order.data_ptr(), self.ptr.data_ptr(), None,
                                      self.totals.data_ptr(), st), "tsqbx_near_count")
        self.n_pairs = int(self.totals[0].item())
        self.max_radius = float(self.rad.max().item()) if self.n_ctr else 0.0

    @property
    def row_lengths(self) -> torch.Tensor:
        """Exact near-list length of every processing row (device int64)."""
        return self.ptr[1:self.n_ctr + 1] - self.ptr[:self.n_ctr]

    @dv.on_own_device
    def rows(self, g0: int, g1: int) -> NearLists:
        """The lists of processing rows [g0, g1) (g0 a multiple of 32) as a
        NearLists in that range's order (row i = processing row g0 + i; its user
        center is ``ctr_order[g0 + i]``), indices into the packed (Morton)
        source order shared by all ranges."""
        if g0 % 32 or not 0 <= g0 <= g1 <= self.n_ctr:
            raise ValueError("row range must satisfy 0 <= g0 <= g1 <= n_ctr, g0 % 32 == 0")
        L = _lib.load()
        dev = self.dev
        st = dv.stream_handle(dev)
        n = g1 - g0
        lptr = self.ptr[g0:g1 + 1] - self.ptr[g0]
        n_sl = (n + 31) // 32
        wsb = int(L.tsqbx_sell_workspace_bytes(n))
        sws = torch.empty(max(wsb, 1), dtype=torch.uint8, device=dev)
        sptr = torch.empty(n_sl + 1, dtype=torch.int64, device=dev)
        tot = torch.zeros(2, dtype=torch.int64, device=dev)
        _lib.check(L.tsqbx_sell_size(n, lptr.data_ptr(), sws.data_ptr(), wsb, sptr.data_ptr(),
                                     tot[1:].data_ptr(), st), "tsqbx_sell_size")
        sidx = torch.empty(max(int(tot[1].item()), 4), dtype=torch.int32, device=dev)
        nptr = torch.empty(n + 1, dtype=torch.int64, device=dev)
        _lib.check(L.tsqbx_near_fill_rows(self.ctr.data_ptr(), self.rad.data_ptr(), self.n_ctr,
                                          self.src.data_ptr(), self.n_src, self.ws.data_ptr(),
                                          self.ws_bytes, self.ctr_order.data_ptr(), g0, g1,
                                          nptr.data_ptr(), sptr.data_ptr(), sidx.data_ptr(),
                                          tot.data_ptr(), st), "tsqbx_near_fill_rows")
        return NearLists(n_ctr=n, n_src=self.n_src, n_pairs=int(lptr[-1].item()), ptr=nptr,
                         csr_idx=None, src_perm=self.src_perm[:self.n_src], ctr_order=None,
                         sell_ptr=sptr, sell_idx=sidx, max_radius=self.max_radius)
