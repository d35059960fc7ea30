"""The short-list Laplace S kernel (``laplace_flat_kernel``, csrc/eval_flat.cu).

A warp takes 32 consecutive rows and splits their CSR entries evenly over its
lanes, so rows are cut by lane boundaries and finished by a segmented sum over
the lanes that hold their pieces.  These tests force the kernel
(``GIGAQBX_FLAT=1``) on the literal presets and on ragged synthetic lists --
empty rows, rows of one entry, rows far longer than a lane's share (spanning
many lanes), a last partial slice -- and compare with the oracle
(``_core.pyx:205-307`` restated) and with the SELL kernel.
"""

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


def _problem(monkeypatch, flat, cfg, src, w, ctr, tgt, tptr, near):
    monkeypatch.setenv("GIGAQBX_FLAT", "1" if flat else "0")
    prob = TsqbxProblem(cfg, src, w, ctr, tgt, near, tgt_ptr=tptr)
    assert prob.prep.flat == flat
    return prob


@pytest.mark.parametrize("name,n", [("c1", 4096), ("c2", 65536), ("c4", 65536)])
def test_flat_literal_presets(monkeypatch, name, n):
    case = configs.make_case(name, "literal", n=n)
    near = build_near_lists(case.centers, case.sources, case.near_radii)
    args = (case.cfg, case.sources, case.weights, case.centers, case.targets, case.tgt_ptr, near)
    got = _problem(monkeypatch, True, *args).evaluate().cpu().numpy()
    sell = _problem(monkeypatch, False, *args).evaluate().cpu().numpy()
    uptr, uidx = near.to_user_csr()
    ref = oracle.ts_batch("laplace", 0, 0.0, case.cfg.p_qbx, case.sources, case.weights,
                          case.centers, uptr, uidx, case.targets, case.tgt_ptr)
    err, err_sell = normwise(got, ref), normwise(got, sell)
    print(f"{name} literal n={n}: flat vs oracle {err:.2e}, vs SELL {err_sell:.2e}")
    assert err <= TOL and err_sell <= TOL


def _ragged(seed, n_ctr, tpc, real):
    """Centers on a sphere shell with radii from 0 to far above the spacing:
    empty rows, single-entry rows and rows of hundreds of entries side by side."""
    rng = np.random.default_rng(seed)
    n_src = 4 * n_ctr
    src = rng.normal(size=(n_src, 3))
    src /= np.linalg.norm(src, axis=1)[:, None]
    ctr = rng.normal(size=(n_ctr, 3))
    ctr *= (0.9 / np.linalg.norm(ctr, axis=1))[:, None]
    kind = rng.integers(0, 4, n_ctr)
    rad = np.where(kind == 0, 0.01, np.where(kind == 1, 0.12, np.where(kind == 2, 0.2, 0.45)))
    rad = rad * rng.uniform(0.8, 1.2, n_ctr)
    w = rng.uniform(0.5, 1.5, n_src) + (0j if real else 1j * rng.uniform(-1, 1, n_src))
    # targets inside every ball's separation radius: |t - c| < 0.1 * (distance to the shell)
    u = rng.normal(size=(n_ctr * tpc, 3))
    u /= np.linalg.norm(u, axis=1)[:, None]
    tgt = np.repeat(ctr, tpc, axis=0) + 0.02 * u
    tptr = np.arange(n_ctr + 1, dtype=np.int64) * tpc
    return src, w, ctr, rad, tgt, tptr


@pytest.mark.parametrize("tpc", [1, 2])
@pytest.mark.parametrize("real", [True, False])
@pytest.mark.parametrize("n_ctr", [1000, 4099])
def test_flat_ragged_rows(monkeypatch, tpc, real, n_ctr):
    src, w, ctr, rad, tgt, tptr = _ragged(7 + n_ctr + tpc, n_ctr, tpc, real)
    near = build_near_lists(ctr, src, rad)
    lens = np.diff(near.ptr.cpu().numpy())
    assert (lens == 0).any() and lens.max() > 64      # empty rows and rows over many lanes
    cfg = TsConfig(KernelSpec(), 6)
    args = (cfg, src, w, ctr, tgt, tptr, near)
    got = _problem(monkeypatch, True, *args).evaluate().cpu().numpy()
    uptr, uidx = near.to_user_csr()
    ref = oracle.ts_batch("laplace", 0, 0.0, 6, src, w, ctr, uptr, uidx, tgt, tptr)
    err = normwise(got, ref)
    print(f"ragged n_ctr={n_ctr} tpc={tpc} real={real}: max len {lens.max()}, err {err:.2e}")
    assert err <= TOL
    # rows with no sources get exactly 0
    empty_users = near.ctr_order.cpu().numpy()[lens == 0]
    tsel = (empty_users[:, None] * tpc + np.arange(tpc)[None, :]).ravel()
    assert np.all(got[tsel] == 0)


def test_flat_validation_raises(monkeypatch):
    """A target outside its center's separation radius is reported with the
    reference's message through the flat kernel's screen."""
    src, w, ctr, rad, tgt, tptr = _ragged(3, 2000, 2, True)
    tgt[2 * 777 + 1] = ctr[777] + np.array([0.0, 0.0, 5.0])   # far outside every ball
    near = build_near_lists(ctr, src, rad)
    prob = _problem(monkeypatch, True, TsConfig(KernelSpec(), 6), src, w, ctr, tgt, tptr, near)
    if int(np.diff(near.ptr.cpu().numpy())[np.argsort(near.ctr_order.cpu().numpy())][777]) == 0:
        pytest.skip("center 777 has no near sources")
    with pytest.raises(ValueError, match="separation violation"):
        prob.evaluate(validate=True)
    prob.evaluate(validate=False)      # the driver path does not validate


def test_flat_row_ranges(monkeypatch):
    """Row-range launches (the multi-GPU shards) through the flat kernel
    reproduce the whole-problem evaluation."""
    case = configs.make_case("c2", "literal", n=20000)
    near = build_near_lists(case.centers, case.sources, case.near_radii)
    prob = _problem(monkeypatch, True, case.cfg, case.sources, case.weights, case.centers,
                    case.targets, case.tgt_ptr, near)
    whole = prob.evaluate().clone()
    out = torch.zeros_like(whole)
    cuts = [0, 4096, 5120, 13344, case.n_centers]   # SELL row ranges start at multiples of 32
    for g0, g1 in zip(cuts[:-1], cuts[1:]):
        prob.prep.launch(torch.view_as_real(out), False, rows=(g0, g1))
    torch.cuda.synchronize()
    assert torch.equal(out, whole)
