"""Laplace S with two rows per thread (``laplace_sell2_kernel``: row A = thread
g, row B = g + the grid's threads; both rows' index rings start filling before
row A computes, and row A's first blocks are waited for with row B's cp.async
groups committed behind them).  Compared with the one-row kernel and the
oracle (``_core.pyx:205-259``) on the literal presets, ragged lists (empty rows,
rows of hundreds of sources, odd row counts so the last thread has no row B),
complex weights and the validation screen."""

import numpy as np
import pytest
import torch

import oracle
from paper_1811_01110_b200 import KernelSpec, TsConfig, TsqbxProblem, build_near_lists, configs

pytestmark = pytest.mark.gpu
TOL = 1e-12


def normwise(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.max(np.abs(a - b)) / max(1e-300, np.max(np.abs(b))))


def _prob(monkeypatch, two, cfg, src, w, ctr, tgt, tptr, near):
    monkeypatch.setenv("GIGAQBX_TWO_ROWS", "1" if two else "0")
    prob = TsqbxProblem(cfg, src, w, ctr, tgt, near, tgt_ptr=tptr)
    assert prob.prep.two_rows == two and prob.group_lanes == 1
    return prob


@pytest.mark.parametrize("name,n", [("c1", 4096), ("c2", 65536), ("c4", 65536), ("c2", 12345)])
@pytest.mark.parametrize("validate", [False, True])
def test_two_rows_literal(monkeypatch, name, n, validate):
    case = configs.make_case(name, "literal", n=n)
    near = build_near_lists(case.centers, case.sources, case.near_radii)
    args = (case.cfg, case.sources, case.weights, case.centers, case.targets, case.tgt_ptr, near)
    got = _prob(monkeypatch, True, *args).evaluate(validate=validate).cpu().numpy()
    one = _prob(monkeypatch, False, *args).evaluate(validate=validate).cpu().numpy()
    uptr, uidx = near.to_user_csr()
    ref = oracle.ts_batch("laplace", 0, 0.0, case.cfg.p_qbx, case.sources, case.weights,
                          case.centers, uptr, uidx, case.targets, case.tgt_ptr)
    print(f"{name} n={n}: two rows vs oracle {normwise(got, ref):.2e}, vs one row "
          f"{normwise(got, one):.2e}")
    assert normwise(got, ref) <= TOL and normwise(got, one) <= TOL


@pytest.mark.parametrize("tpc", [1, 2])
@pytest.mark.parametrize("real", [True, False])
def test_two_rows_ragged(monkeypatch, tpc, real):
    rng = np.random.default_rng(11 + tpc)
    n_ctr, n_src = 3001, 12000
    src = rng.normal(size=(n_src, 3))
    src /= np.linalg.norm(src, axis=1)[:, None]
    ctr = rng.normal(size=(n_ctr, 3))
    ctr *= (0.9 / np.linalg.norm(ctr, axis=1))[:, None]
    rad = rng.choice([0.01, 0.12, 0.2, 0.45], n_ctr) * rng.uniform(0.8, 1.2, n_ctr)
    w = rng.uniform(0.5, 1.5, n_src) + (0j if real else 1j * rng.uniform(-1, 1, n_src))
    u = rng.normal(size=(n_ctr * tpc, 3))
    tgt = np.repeat(ctr, tpc, axis=0) + 0.02 * u / np.linalg.norm(u, axis=1)[:, None]
    tptr = np.arange(n_ctr + 1, dtype=np.int64) * tpc
    near = build_near_lists(ctr, src, rad)
    lens = np.diff(near.ptr.cpu().numpy())
    assert (lens == 0).any() and lens.max() > 100
    cfg = TsConfig(KernelSpec(), 7)
    monkeypatch.setenv("GIGAQBX_SPLIT", "1")        # unsplit rows despite the long ones
    got = _prob(monkeypatch, True, cfg, src, w, ctr, tgt, tptr, near).evaluate().cpu().numpy()
    uptr, uidx = near.to_user_csr()
    ref = oracle.ts_batch("laplace", 0, 0.0, 7, src, w, ctr, uptr, uidx, tgt, tptr)
    assert normwise(got, ref) <= TOL


def test_two_rows_validation_error(monkeypatch):
    case = configs.make_case("c2", "literal", n=20000)
    tgt = case.targets.copy()
    c = 19999                                       # a row-B thread's row
    tgt[2 * c] = case.centers[c] + 5.0
    near = build_near_lists(case.centers, case.sources, case.near_radii)
    prob = _prob(monkeypatch, True, case.cfg, case.sources, case.weights, case.centers, tgt,
                 case.tgt_ptr, near)
    with pytest.raises(ValueError, match="separation violation"):
        prob.evaluate(validate=True)


def test_two_rows_row_ranges(monkeypatch):
    """Row-range launches (multi-GPU shards) reproduce the whole evaluation."""
    case = configs.make_case("c2", "literal", n=30000)
    near = build_near_lists(case.centers, case.sources, case.near_radii)
    prob = _prob(monkeypatch, True, case.cfg, case.sources, case.weights, case.centers,
                 case.targets, case.tgt_ptr, near)
    whole = prob.evaluate().clone()
    out = torch.zeros_like(whole)
    cuts = [0, 4096, 9600, 20000, case.n_centers]
    for g0, g1 in zip(cuts[:-1], cuts[1:]):
        prob.prep.launch(torch.view_as_real(out), False, rows=(g0, g1))
    torch.cuda.synchronize()
    assert torch.equal(out, whole)
