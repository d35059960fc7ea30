"""Multi-GPU TSQBX: centers sharded across ranks, sources replicated, one all-gather.

Every (center, target) pair sum is independent, so the path shards without a
halo: each rank holds all sources (C5: 8.4 M x 40 B = 336 MB), evaluates a
contiguous range of CSR rows (Morton processing order) chosen so every rank
gets the same number of (target, source) pairs -- not the same number of
centers, which would leave the clustered-torus case imbalanced -- and then ONE
NCCL all-gather (padded equal shards, over NVLink/NVSwitch) gives every rank
every target's potential, followed by one scatter kernel into user order.

The host logic (row split, padding layout, scatter map) is plain NumPy and is
exercised on CPU with the gloo backend (tests/test_distributed.py).
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
class ShardPlan:
    world: int
    row_bounds: np.ndarray      # (world + 1,) processing rows
    tgt_bounds: np.ndarray      # (world + 1,) processing targets
    shard: int                  # padded shard length (targets)
    dest: np.ndarray            # (world * shard,) user slot of each gathered entry (pad -> n_tgt)
    n_tgt: int

    def rows(self, rank: int) -> tuple[int, int]:
        return int(self.row_bounds[rank]), int(self.row_bounds[rank + 1])

    def targets(self, rank: int) -> tuple[int, int]:
        return int(self.tgt_bounds[rank]), int(self.tgt_bounds[rank + 1])


def make_plan(row_len: np.ndarray, tptr_proc: np.ndarray, tidx: np.ndarray | None,
              world: int) -> ShardPlan:
    """row_len: near-list length per processing row; tptr_proc: processing-order
    target offsets (n_rows + 1); tidx: processing target -> user target (None = identity)."""
    tptr_proc = np.asarray(tptr_proc, dtype=np.int64)
    n_tgt = int(tptr_proc[-1])
    row_pairs = np.asarray(row_len, dtype=np.int64) * np.diff(tptr_proc)
    rb = balanced_rows(row_pairs, world)
    tb = tptr_proc[rb]
    shard = int(max(1, np.max(np.diff(tb)))) if world > 0 else 1
    dest = np.full(world * shard, n_tgt, dtype=np.int64)
    user = np.arange(n_tgt, dtype=np.int64) if tidx is None else np.asarray(tidx, np.int64)
    for r in range(world):
        t0, t1 = int(tb[r]), int(tb[r + 1])
        dest[r * shard: r * shard + (t1 - t0)] = user[t0:t1]
    return ShardPlan(world=world, row_bounds=rb, tgt_bounds=tb, shard=shard, dest=dest,
                     n_tgt=n_tgt)


def assemble_numpy(gathered: np.ndarray, plan: ShardPlan) -> np.ndarray:
    """Host twin of the device scatter (tests only): gathered (world*shard,) -> user order."""
    out = np.zeros(plan.n_tgt + 1, dtype=gathered.dtype)
    out[plan.dest] = gathered
    return out[:plan.n_tgt]


class ShardedEvaluator:
    """Evaluate a TsqbxProblem's rows for this rank, all-gather, scatter to user order."""

    def __init__(self, problem, rank: int, world: int, group=None):
        from . import _lib

        self.problem, self.rank, self.world, self.group = problem, rank, world, group
        prep = problem.prep
        near = prep.near
        row_len = (near.ptr[1:] - near.ptr[:-1]).cpu().numpy()
        tidx = None if prep.tidx is None else prep.tidx[:prep.n_tgt].cpu().numpy()
        self.plan = make_plan(row_len, prep.tptr.cpu().numpy(), tidx, world)
        dev = prep.dev
        S = self.plan.shard
        self.send = torch.zeros(S, dtype=torch.complex128, device=dev)
        self.recv = torch.zeros(world * S, dtype=torch.complex128, device=dev)
        self.dest = torch.from_numpy(self.plan.dest).to(dev)
        self.out = torch.zeros(prep.n_tgt + 1, dtype=torch.complex128, device=dev)
        self._lib = _lib

    def pairs_on_rank(self) -> int:
        prep = self.problem.prep
        g0, g1 = self.plan.rows(self.rank)
        lens = prep.near.ptr[g0 + 1:g1 + 1] - prep.near.ptr[g0:g1]
        tpc = prep.tptr[g0 + 1:g1 + 1] - prep.tptr[g0:g1]
        return int((lens * tpc).sum().item())

    def evaluate(self) -> torch.Tensor:
        prep = self.problem.prep
        g0, g1 = self.plan.rows(self.rank)
        t0, _ = self.plan.targets(self.rank)
        if g1 > g0:
            prep.launch(torch.view_as_real(self.send), validate=False, rows=(g0, g1),
                        out_offset=t0, user_order=False)
        dist.all_gather_into_tensor(self.recv, self.send, group=self.group)
        L = self._lib.load()
        self._lib.check(L.tsqbx_scatter_c128(self.recv.numel(), self.dest.data_ptr(),
                                             self.recv.data_ptr(), self.out.data_ptr(),
                                             torch.cuda.current_stream(prep.dev).cuda_stream),
                        "tsqbx_scatter_c128")
        return self.out[:prep.n_tgt]
