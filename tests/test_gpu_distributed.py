"""ShardedProblem on the GPU: per-rank near lists (tsqbx_near_fill_rows),
row chunks with the uniform-target kernels (tgt_base), the padded gather
layout and the scatter into user order, against the oracle.

This pool gives one GPU per process, so ranks r > 0 are built in the same
process and their send buffers are assembled by hand (the NCCL all-gather
itself is the library's; its host-side layout is covered with gloo in
tests/test_distributed.py)."""

import numpy as np
import pytest
import torch

import oracle
from paper_1811_01110_b200 import TsqbxProblem, build_near_lists, configs
from paper_1811_01110_b200.distributed import ShardedProblem, assemble_numpy

pytestmark = pytest.mark.gpu


def normwise(a, b):
    return float(np.max(np.abs(a - b)) / np.max(np.abs(b)))


def _oracle(case):
    ptr, idx = oracle.near_csr(case.centers, case.near_radii, case.sources)
    spec = case.cfg.spec
    return oracle.ts_batch("laplace" if spec.is_laplace else "helmholtz", 0,
                           spec.helmholtz_k or 0.0, case.cfg.p_qbx, case.sources, case.weights,
                           case.centers, ptr, idx, case.targets, case.tgt_ptr)


CASES = [("c2", "literal", dict(n=65536)), ("c2", "dense", dict(n=65536)),
         ("c4", "literal", dict(n=65536)), ("c5", "literal", dict(n=16384, spheres=4))]


@pytest.mark.parametrize("name,preset,kw", CASES)
@pytest.mark.parametrize("chunks", [1, 3])
def test_world_one_matches_single_problem(name, preset, kw, chunks):
    case = configs.make_case(name, preset, **kw)
    sp = ShardedProblem(case.cfg, case.sources, case.weights, case.centers, case.targets,
                        case.near_radii, tgt_ptr=case.tgt_ptr, chunks=chunks)
    got = sp.evaluate().cpu().numpy()
    near = build_near_lists(case.centers, case.sources, case.near_radii)
    prob = TsqbxProblem(case.cfg, case.sources, case.weights, case.centers, case.targets, near,
                        tgt_ptr=case.tgt_ptr)
    one = prob.evaluate().cpu().numpy()
    ref = _oracle(case)
    tol = 1e-12 if case.cfg.spec.is_laplace else 1e-10
    assert sp.prep.tuni == case.n_targets // case.n_centers
    assert normwise(got, ref) <= tol
    assert normwise(got, one) <= tol
    assert sp.n_pairs == prob.pair_count()


@pytest.mark.parametrize("name,preset,kw", CASES)
@pytest.mark.parametrize("world,chunks", [(2, 1), (3, 2), (4, 4)])
def test_ranks_assemble_to_oracle(name, preset, kw, world, chunks):
    case = configs.make_case(name, preset, **kw)
    sends, layout, pairs = [], None, 0
    for r in range(world):
        sp = ShardedProblem(case.cfg, case.sources, case.weights, case.centers, case.targets,
                            case.near_radii, tgt_ptr=case.tgt_ptr, rank=r, world=world,
                            chunks=chunks)
        for c in range(sp.layout.chunks):
            sp._launch_chunk(c)
        sends.append(sp.send.cpu().numpy())
        layout = sp.layout
        pairs += sp.n_pairs_rank
        assert sp.prep.near.n_ctr == sp.rows[1] - sp.rows[0]
        del sp
    # the rank-major receive layout of every chunk's all-gather
    recv = np.concatenate([np.concatenate([s[layout.send_off[c]:layout.send_off[c + 1]]
                                           for s in sends]) for c in range(layout.chunks)])
    got = assemble_numpy(recv, layout)
    ref = _oracle(case)
    tol = 1e-12 if case.cfg.spec.is_laplace else 1e-10
    assert normwise(got, ref) <= tol
    loads = [int(np.diff(layout.chunk_tgts[r, [0, -1]])[0]) for r in range(world)]
    assert sum(loads) == case.n_targets
    assert pairs == int(np.diff(oracle.near_csr(case.centers, case.near_radii,
                                                case.sources)[0]) @ np.diff(case.tgt_ptr))
