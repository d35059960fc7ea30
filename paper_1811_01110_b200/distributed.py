"""Multi-GPU TSQBX: centers sharded across ranks, sources replicated, potentials
all-gathered (the reference's unit of independence is the
per-center loop of the driver, driver.py:218-228).

Every (center, target) sum is independent, so the path shards without a halo:

* every rank holds all sources (C5: 8.4 M x 40 B packed = 336 MB) and runs the
  near-list count over all centers (``NearRowBuilder``: Morton order + exact
  row lengths), so all ranks agree on the processing order and the split;
* rows are cut into contiguous ranges of equal (target, source) pair count --
  not equal center count, which would leave the clustered torus imbalanced --
  with inner boundaries on 32-row SELL slices;
* each rank fills the near lists of its own rows only and evaluates them
  (uniform-target kernels kept: the launch passes the range's target base);
* its rows are evaluated in ``chunks`` pieces; the all-gather of chunk c
  (NCCL over NVLink/NVSwitch, ``async_op``) overlaps the evaluation of chunk
  c + 1, and one scatter kernel puts every potential in user order.

The host-side layout (row split, chunking, padding, scatter map) is plain
NumPy (``make_layout``) and is exercised with the gloo backend on CPU at world
sizes 2 and 4 (tests/test_distributed.py).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist


def balanced_rows(row_pairs: np.ndarray, world: int, align: int = 32) -> np.ndarray:
    """Row boundaries b[0..world] splitting rows into `world` contiguous ranges of
    (nearly) equal total pairs.  row_pairs[g] = len(row g) * targets(row g).
    Inner boundaries are multiples of `align` (SELL slices are 32 rows)."""
    row_pairs = np.asarray(row_pairs, dtype=np.int64)
    n = row_pairs.shape[0]
    cum = np.concatenate([[0], np.cumsum(row_pairs)])
    total = cum[-1]
    bounds = np.zeros(world + 1, dtype=np.int64)
    for r in range(1, world):
        b = int(np.searchsorted(cum, total * r / world, side="left"))
        bounds[r] = min(n, int(round(b / align)) * align)
    bounds[world] = n
    return np.maximum.accumulate(bounds)


@dataclass
class ShardLayout:
    """Who evaluates what, and where every potential lands.

    Rank r owns processing rows ``row_bounds[r]:row_bounds[r+1]``, evaluated in
    ``chunks`` row chunks ``chunk_rows[r, c]:chunk_rows[r, c+1]`` whose targets
    are ``chunk_tgts[r, c]:chunk_tgts[r, c+1]`` (processing order).  Chunk c is
    padded to ``pad[c]`` targets on every rank; a rank's send buffer is its
    chunks back to back (chunk c at ``send_off[c]``), and chunk c's all-gather
    fills ``recv[world*send_off[c] : world*send_off[c+1]]`` rank-major.
    ``dest`` maps every receive slot to its user target (padding -> n_tgt).
    """

    world: int
    chunks: int
    row_bounds: np.ndarray      # (world + 1,)
    chunk_rows: np.ndarray      # (world, chunks + 1) absolute processing rows
    chunk_tgts: np.ndarray      # (world, chunks + 1) absolute processing targets
    pad: np.ndarray             # (chunks,)
    send_off: np.ndarray        # (chunks + 1,)
    dest: np.ndarray            # (world * send_off[-1],)
    n_tgt: int

    def rows(self, rank: int) -> tuple[int, int]:
        return int(self.row_bounds[rank]), int(self.row_bounds[rank + 1])

    @property
    def send_len(self) -> int:
        return int(self.send_off[-1])


def make_layout(row_pairs: np.ndarray, tptr_proc: np.ndarray, tidx: np.ndarray | None,
                world: int, chunks: int = 1, align: int = 32) -> ShardLayout:
    """row_pairs: pairs per processing row (length x targets); tptr_proc:
    processing-order target offsets (n_rows + 1); tidx: processing target ->
    user target (None = identity)."""
    row_pairs = np.asarray(row_pairs, dtype=np.int64)
    tptr_proc = np.asarray(tptr_proc, dtype=np.int64)
    n_tgt = int(tptr_proc[-1])
    chunks = max(1, int(chunks))
    rb = balanced_rows(row_pairs, world, align)
    crow = np.zeros((world, chunks + 1), dtype=np.int64)
    for r in range(world):
        g0, g1 = int(rb[r]), int(rb[r + 1])
        # chunk boundaries relative to the rank's first row keep 32-row slices
        # whole (g0 is a multiple of 32)
        crow[r] = g0 + balanced_rows(row_pairs[g0:g1], chunks, align)
    ctgt = tptr_proc[crow]
    pad = np.maximum(1, np.max(np.diff(ctgt, axis=1), axis=0)) if world else np.ones(chunks,
                                                                                     np.int64)
    send_off = np.concatenate([[0], np.cumsum(pad)]).astype(np.int64)
    user = np.arange(n_tgt, dtype=np.int64) if tidx is None else np.asarray(tidx, np.int64)
    dest = np.full(world * int(send_off[-1]), n_tgt, dtype=np.int64)
    for c in range(chunks):
        base = world * int(send_off[c])
        for r in range(world):
            t0, t1 = int(ctgt[r, c]), int(ctgt[r, c + 1])
            at = base + r * int(pad[c])
            dest[at:at + (t1 - t0)] = user[t0:t1]
    return ShardLayout(world=world, chunks=chunks, row_bounds=rb, chunk_rows=crow,
                       chunk_tgts=ctgt, pad=pad.astype(np.int64), send_off=send_off, dest=dest,
                       n_tgt=n_tgt)


def gather_chunks(send: torch.Tensor, recv: torch.Tensor, layout: ShardLayout, group=None,
                  launch_chunk=None) -> None:
    """For each chunk: ``launch_chunk(c)`` (fills this rank's part of ``send``,
    stream-ordered), then an asynchronous all-gather of that chunk -- the next
    chunk's evaluation runs while it travels.  Waits for all gathers at the end
    (the current stream then orders after them)."""
    works = []
    W = layout.world
    for c in range(layout.chunks):
        if launch_chunk is not None:
            launch_chunk(c)
        a, b = int(layout.send_off[c]), int(layout.send_off[c + 1])
        if W == 1:
            continue            # one rank: send is already the receive buffer
        works.append(dist.all_gather_into_tensor(recv[W * a:W * b], send[a:b], group=group,
                                                 async_op=True))
    for w in works:
        w.wait()


def assemble_numpy(gathered: np.ndarray, layout: ShardLayout) -> np.ndarray:
    """Host twin of the device scatter (tests only): received slots -> user order."""
    out = np.zeros(layout.n_tgt + 1, dtype=gathered.dtype)
    out[layout.dest] = gathered
    return out[:layout.n_tgt]


class ShardedProblem:
    """One TSQBX problem split over the ranks of ``group`` (one GPU each).

    Same inputs as ``near_field_potentials``: every rank passes the whole
    geometry (sources replicated); ``evaluate()`` returns every target's
    potential in user order on every rank (a complex128 CUDA tensor).
    """

    def __init__(self, cfg, sources, weights, centers, targets, near_radii, tgt_ptr=None,
                 source_normals=None, target_normals=None, rank: int = 0, world: int = 1,
                 group=None, chunks: int = 0, device=None):
        from . import _device as dv
        from .nearlist import NearRowBuilder
        from .tsqbx import _inputs, _Prepared

        dev = dv.require_cuda(device)
        self.dev, self.rank, self.world, self.group = dev, rank, world, group
        with torch.cuda.device(dev):
            src, w, ctr, tgt, sn, tn = _inputs(cfg, sources, weights, centers, targets,
                                               source_normals, target_normals, dev)
            n_ctr, n_tgt = int(ctr.shape[0]), int(tgt.shape[0])
            if tgt_ptr is None:
                if n_tgt != n_ctr:
                    raise ValueError("tgt_ptr is required unless there is one target per center")
                tptr = torch.arange(n_ctr + 1, dtype=torch.int64, device=dev)
            else:
                tptr = dv.to_device(tgt_ptr, torch.int64, dev)
                from .nearlist import check_offsets
                check_offsets(tptr, n_tgt, "tgt_ptr")
            builder = NearRowBuilder(ctr, src, near_radii, device=dev)
            order = builder.ctr_order[:n_ctr].long()
            # processing-order target runs and the processing -> user target map
            tl = tptr[order + 1] - tptr[order]
            tptr_p = torch.zeros(n_ctr + 1, dtype=torch.int64, device=dev)
            torch.cumsum(tl, 0, out=tptr_p[1:])
            first = torch.repeat_interleave(tptr[order], tl, output_size=n_tgt)
            tidx = first + torch.arange(n_tgt, device=dev) - torch.repeat_interleave(
                tptr_p[:-1], tl, output_size=n_tgt)
            row_pairs = (builder.row_lengths * tl).cpu().numpy()
            if chunks <= 0:
                chunks = 1 if world == 1 else 4
            self.layout = L = make_layout(row_pairs, tptr_p.cpu().numpy(), tidx.cpu().numpy(),
                                          world, chunks)
            g0, g1 = L.rows(rank)
            self.rows = (g0, g1)
            near = builder.rows(g0, g1)
            t0, t1 = int(L.chunk_tgts[rank, 0]), int(L.chunk_tgts[rank, -1])
            tsel = tidx[t0:t1]
            lctr = ctr[order[g0:g1]]
            ltgt = tgt[tsel]
            ltn = None if tn is None else tn[tsel]
            ltptr = tptr_p[g0:g1 + 1] - tptr_p[g0]
            del builder          # the other ranks' rows are never filled
            self.prep = _Prepared(cfg, dev, src, w, sn, lctr, near, ltgt, ltn, ltptr,
                                  user_tptr=False)
            self.prep.set_uniform_targets()
            self.n_tgt = n_tgt
            self.n_pairs_rank = int(row_pairs[g0:g1].sum())
            self.n_pairs = int(row_pairs.sum())
            self.send = torch.zeros(L.send_len, dtype=torch.complex128, device=dev)
            self.recv = (self.send if world == 1 else
                         torch.zeros(world * L.send_len, dtype=torch.complex128, device=dev))
            self.dest = torch.from_numpy(L.dest).to(dev)
            self.out = torch.zeros(n_tgt + 1, dtype=torch.complex128, device=dev)

    def set_weights(self, weights) -> None:
        """A new density for the same geometry: one pack kernel (replicated)."""
        from . import _device as dv
        with torch.cuda.device(self.dev):
            if isinstance(weights, torch.Tensor) and not weights.is_complex():
                weights = weights.to(torch.complex128)
            self.prep.pack(dv.complex_as_f64(dv.to_device(weights, torch.complex128, self.dev,
                                                          (-1,))))

    def _launch_chunk(self, c: int) -> None:
        L, r = self.layout, self.rank
        g0 = self.rows[0]
        c0, c1 = int(L.chunk_rows[r, c]) - g0, int(L.chunk_rows[r, c + 1]) - g0
        if c1 <= c0:
            return
        t_first = int(L.chunk_tgts[r, c]) - int(L.chunk_tgts[r, 0])   # local processing target
        # local target t of this chunk -> send[send_off[c] + t - t_first]
        self.prep.launch(torch.view_as_real(self.send), validate=False, rows=(c0, c1),
                         out_offset=t_first - int(L.send_off[c]), user_order=False)

    def evaluate(self) -> torch.Tensor:
        from . import _lib
        with torch.cuda.device(self.dev):
            gather_chunks(self.send, self.recv, self.layout, self.group, self._launch_chunk)
            Lb = _lib.load()
            _lib.check(Lb.tsqbx_scatter_c128(self.recv.numel(), self.dest.data_ptr(),
                                             torch.view_as_real(self.recv).data_ptr(),
                                             torch.view_as_real(self.out).data_ptr(),
                                             torch.cuda.current_stream(self.dev).cuda_stream),
                       "tsqbx_scatter_c128")
        return self.out[:self.n_tgt]
