"""Multi-rank host logic on CPU (gloo, world_size 2): row sharding by pair
count, padded all-gather layout, scatter back to user order.  The per-rank
compute is the oracle here (the GPU kernel is covered by the gpu tests); the
assembled result must be bit-identical to the single-process result."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_1811_01110_b200 import configs
from paper_1811_01110_b200.distributed import assemble_numpy, balanced_rows, make_plan


def test_balanced_rows_balances_pairs_and_aligns():
    rng = np.random.default_rng(0)
    pairs = rng.integers(1, 800, size=10000)          # torus-like imbalance
    for world in (1, 2, 3, 4, 8):
        b = balanced_rows(pairs, world)
        assert b[0] == 0 and b[-1] == len(pairs) and np.all(np.diff(b) >= 0)
        assert np.all(b[1:-1] % 32 == 0)
        loads = np.array([pairs[b[r]:b[r + 1]].sum() for r in range(world)])
        assert loads.max() - loads.min() <= 2 * 32 * 800
    b = balanced_rows(np.ones(10), 4)                  # fewer rows than alignment
    assert b[0] == 0 and b[-1] == 10


def test_plan_dest_covers_every_target_once():
    row_len = np.array([3, 0, 5, 2, 7, 1] * 20)
    tptr = np.concatenate([[0], np.cumsum(np.tile([2, 1, 0, 3, 1, 2], 20))])
    tidx = np.random.default_rng(1).permutation(tptr[-1])
    plan = make_plan(row_len, tptr, tidx, 3)
    d = plan.dest[plan.dest < plan.n_tgt]
    assert np.array_equal(np.sort(d), np.arange(plan.n_tgt))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    case = configs.make_case("c2", "literal", n=512)
    ptr, idx = oracle.near_csr(case.centers, case.near_radii, case.sources)
    plan = make_plan(np.diff(ptr), case.tgt_ptr, None, world)
    g0, g1 = plan.rows(rank)
    t0, t1 = plan.targets(rank)
    sub = oracle.ts_batch("laplace", 0, 0.0, 8, case.sources, case.weights,
                          case.centers[g0:g1], ptr[g0:g1 + 1] - ptr[g0], idx[ptr[g0]:ptr[g1]],
                          case.targets[t0:t1], case.tgt_ptr[g0:g1 + 1] - case.tgt_ptr[g0])
    send = torch.zeros(plan.shard, dtype=torch.complex128)
    send[:t1 - t0] = torch.from_numpy(sub)
    recv = torch.zeros(world * plan.shard, dtype=torch.complex128)
    dist.all_gather_into_tensor(recv, send)
    out = assemble_numpy(recv.numpy(), plan)
    if rank == 0:
        full = oracle.ts_batch("laplace", 0, 0.0, 8, case.sources, case.weights, case.centers,
                               ptr, idx, case.targets, case.tgt_ptr)
        q.put(bool(np.array_equal(out, full)))
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_two_rank_allgather_matches_single_process():
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(240)
        assert p.exitcode == 0
    assert q.get() is True
