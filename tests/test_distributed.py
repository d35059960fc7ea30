"""Multi-rank host logic on CPU (gloo, world sizes 2 and 4): row sharding by pair
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
from paper_1811_01110_b200.distributed import (assemble_numpy, balanced_rows, gather_chunks,
                                                   make_layout)


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


@pytest.mark.parametrize("world,chunks", [(1, 1), (2, 1), (3, 4), (8, 3)])
def test_layout_dest_covers_every_target_once(world, chunks):
    rng = np.random.default_rng(1)
    tpc = np.tile([2, 1, 0, 3, 1, 2], 200)
    row_len = rng.integers(0, 9, size=tpc.size)
    tptr = np.concatenate([[0], np.cumsum(tpc)])
    tidx = rng.permutation(tptr[-1])
    L = make_layout(row_len * tpc, tptr, tidx, world, chunks)
    d = L.dest[L.dest < L.n_tgt]
    assert np.array_equal(np.sort(d), np.arange(L.n_tgt))
    assert L.dest.size == world * L.send_len
    assert np.all(L.chunk_rows[:, 1:-1] % 32 == 0) and np.all(L.row_bounds[1:-1] % 32 == 0)
    assert np.array_equal(L.chunk_rows[:, 0], L.row_bounds[:-1])
    assert np.array_equal(L.chunk_rows[:, -1], L.row_bounds[1:])
    assert np.all(np.diff(L.chunk_tgts, axis=1) <= L.pad[None, :])


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, chunks, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    case = configs.make_case("c2", "literal", n=2048)
    ptr, idx = oracle.near_csr(case.centers, case.near_radii, case.sources)
    # a processing order that is not the identity (as the device Morton order)
    order = np.random.default_rng(5).permutation(case.n_centers)
    lens = np.diff(ptr)[order]
    tl = np.diff(case.tgt_ptr)[order]
    tptr_p = np.concatenate([[0], np.cumsum(tl)])
    tidx = np.concatenate([np.arange(case.tgt_ptr[c], case.tgt_ptr[c + 1]) for c in order])
    L = make_layout(lens * tl, tptr_p, tidx, world, chunks)
    send = torch.zeros(L.send_len, dtype=torch.complex128)
    recv = torch.zeros(world * L.send_len, dtype=torch.complex128)

    def launch_chunk(c):
        # this rank's chunk c, evaluated by the oracle (the GPU kernel stands here)
        g0, g1 = int(L.chunk_rows[rank, c]), int(L.chunk_rows[rank, c + 1])
        if g1 <= g0:
            return
        ctr = order[g0:g1]
        sptr = np.concatenate([[0], np.cumsum(np.diff(ptr)[ctr])])
        sidx = np.concatenate([idx[ptr[c_]:ptr[c_ + 1]] for c_ in ctr])
        t0, t1 = int(L.chunk_tgts[rank, c]), int(L.chunk_tgts[rank, c + 1])
        sub = oracle.ts_batch("laplace", 0, 0.0, 8, case.sources, case.weights,
                              case.centers[ctr], sptr, sidx, case.targets[tidx[t0:t1]],
                              tptr_p[g0:g1 + 1] - tptr_p[g0])
        a = int(L.send_off[c])
        send[a:a + (t1 - t0)] = torch.from_numpy(sub)

    if world > 1:
        gather_chunks(send, recv, L, launch_chunk=launch_chunk)
    else:
        for c in range(L.chunks):
            launch_chunk(c)
        recv = send
    out = assemble_numpy(recv.numpy(), L)
    if rank == 0:
        full = oracle.ts_batch("laplace", 0, 0.0, 8, case.sources, case.weights, case.centers,
                               ptr, idx, case.targets, case.tgt_ptr)
        q.put(bool(np.array_equal(out, full)))
    dist.destroy_process_group()


@pytest.mark.timeout(300)
@pytest.mark.parametrize("world,chunks", [(2, 1), (2, 3), (4, 4)])
def test_multi_rank_chunked_allgather_matches_single_process(world, chunks):
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, chunks, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(240)
        assert p.exitcode == 0
    assert q.get() is True
