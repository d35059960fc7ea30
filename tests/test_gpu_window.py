"""Windowed SELL for short lists (``tsqbx_sell_window`` + ``laplace_sellw_kernel``):
per 32-row slice the distinct sources are staged in shared memory once and the
rows read them by window index.  Checked against the plain SELL kernel and the
oracle (``_core.pyx:205-259``) on the literal presets, with complex weights,
ragged rows, validation, row-range launches, and the overflow fallback (a slice
with more distinct sources than the window keeps the plain layout)."""

import numpy as np
import pytest
import torch

import oracle
from paper_1811_01110_b200 import KernelSpec, TsConfig, TsqbxProblem, _lib, build_near_lists, configs

pytestmark = pytest.mark.gpu
TOL = 1e-12


def normwise(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.max(np.abs(a - b)) / max(1e-300, np.max(np.abs(b))))


def _prob(monkeypatch, win, cfg, src, w, ctr, tgt, tptr, near):
    monkeypatch.setenv("GIGAQBX_WINDOW", "1" if win else "0")
    return TsqbxProblem(cfg, src, w, ctr, tgt, near, tgt_ptr=tptr)


def test_window_layout_holds_the_rows():
    case = configs.make_case("c2", "literal", n=20000)
    near = build_near_lists(case.centers, case.sources, case.near_radii)
    assert near.build_window()
    p = near.ptr.cpu().numpy()
    sp = near.sell_ptr.cpu().numpy()
    loc = near.sell_loc.cpu().numpy()
    win = near.win_src.cpu().numpy()
    wl = near.win_len.cpu().numpy()
    d = near.idx.cpu().numpy()
    assert wl.max() <= _lib.WINDOW
    for g in range(0, near.n_ctr, 97):
        s = g // 32
        i = np.arange(p[g + 1] - p[g])
        cells = sp[s] + (i // 4) * 128 + (g % 32) * 4 + i % 4
        li = loc[cells]
        if wl[s] < 0:                          # overflowed slice: global indices kept
            assert np.array_equal(li, d[p[g]:p[g + 1]])
            continue
        assert np.all(li < wl[s])
        assert np.array_equal(win[s * _lib.WINDOW + li], d[p[g]:p[g + 1]])
        w = win[s * _lib.WINDOW: s * _lib.WINDOW + wl[s]]
        assert len(np.unique(w)) == wl[s]
    print(f"slices over the window: {near.win_overflow} of {len(wl)}")
    assert near.win_overflow == int((wl < 0).sum())


@pytest.mark.parametrize("name,n", [("c1", 4096), ("c2", 65536), ("c4", 65536), ("c2", 12345)])
@pytest.mark.parametrize("validate", [False, True])
def test_window_literal(monkeypatch, name, n, validate):
    case = configs.make_case(name, "literal", n=n)
    near = build_near_lists(case.centers, case.sources, case.near_radii)
    args = (case.cfg, case.sources, case.weights, case.centers, case.targets, case.tgt_ptr, near)
    pw = _prob(monkeypatch, True, *args)
    assert pw.prep.window
    got = pw.evaluate(validate=validate).cpu().numpy()
    plain = _prob(monkeypatch, False, *args).evaluate(validate=validate).cpu().numpy()
    uptr, uidx = near.to_user_csr()
    ref = oracle.ts_batch("laplace", 0, 0.0, case.cfg.p_qbx, case.sources, case.weights,
                          case.centers, uptr, uidx, case.targets, case.tgt_ptr)
    print(f"{name} n={n}: window vs oracle {normwise(got, ref):.2e}, vs plain {normwise(got, plain):.2e}")
    assert normwise(got, ref) <= TOL and normwise(got, plain) <= TOL


@pytest.mark.parametrize("tpc", [1, 2])
def test_window_complex_weights(monkeypatch, tpc):
    case = configs.make_case("c2", "literal", n=30000)
    rng = np.random.default_rng(4)
    w = case.weights * (1 + 0.5j * rng.uniform(-1, 1, case.n_sources))
    if tpc == 1:
        tgt, tptr = case.targets[0::2], np.arange(case.n_centers + 1, dtype=np.int64)
    else:
        tgt, tptr = case.targets, case.tgt_ptr
    near = build_near_lists(case.centers, case.sources, case.near_radii)
    pw = _prob(monkeypatch, True, case.cfg, case.sources, w, case.centers, tgt, tptr, near)
    assert pw.prep.window
    got = pw.evaluate().cpu().numpy()
    uptr, uidx = near.to_user_csr()
    ref = oracle.ts_batch("laplace", 0, 0.0, case.cfg.p_qbx, case.sources, w, case.centers,
                          uptr, uidx, tgt, tptr)
    assert normwise(got, ref) <= TOL


def test_window_overflow_slices_gather_globally(monkeypatch):
    """Dense lists (several hundred distinct sources per slice > the 128-record
    window): every slice keeps global indices and its warp gathers as the plain
    kernel does."""
    case = configs.make_case("c2", "dense", n=8192)
    near = build_near_lists(case.centers, case.sources, case.near_radii)
    monkeypatch.setenv("GIGAQBX_SPLIT", "1")
    p = _prob(monkeypatch, True, case.cfg, case.sources, case.weights, case.centers,
              case.targets, case.tgt_ptr, near)
    assert p.prep.window and near.win_overflow == (case.n_centers + 31) // 32
    uptr, uidx = near.to_user_csr()
    ref = oracle.ts_batch("laplace", 0, 0.0, case.cfg.p_qbx, case.sources, case.weights,
                          case.centers, uptr, uidx, case.targets, case.tgt_ptr)
    assert normwise(p.evaluate().cpu().numpy(), ref) <= TOL


def test_window_validation_and_row_ranges(monkeypatch):
    case = configs.make_case("c2", "literal", n=30000)
    near = build_near_lists(case.centers, case.sources, case.near_radii)
    p = _prob(monkeypatch, True, case.cfg, case.sources, case.weights, case.centers,
              case.targets, case.tgt_ptr, near)
    whole = p.evaluate().clone()
    out = torch.zeros_like(whole)
    cuts = [0, 4096, 9600, 20000, case.n_centers]
    for g0, g1 in zip(cuts[:-1], cuts[1:]):
        p.prep.launch(torch.view_as_real(out), False, rows=(g0, g1))
    torch.cuda.synchronize()
    assert torch.equal(out, whole)
    tgt = case.targets.copy()
    tgt[2 * 777 + 1] = case.centers[777] + 5.0
    pv = _prob(monkeypatch, True, case.cfg, case.sources, case.weights, case.centers, tgt,
               case.tgt_ptr, near)
    with pytest.raises(ValueError, match="separation violation"):
        pv.evaluate(validate=True)
