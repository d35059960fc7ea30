"""The CPU oracle (oracle/tsqbx_oracle.c) pinned against the reference.

Pins: the reference's known-answer tests (pkg/tests/test_tsqbx.py:28-43,88-98),
golden vectors produced by the reference itself (tests/golden/make_golden.py),
and -- when built -- the reference's compiled Cython core (oracle/_ref)."""

import math
import os

import numpy as np
import pytest

import oracle


def normwise(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.max(np.abs(a - b)) / max(1e-300, np.max(np.abs(b))))


def test_collinear_geometric_sum():
    # test_tsqbx.py:28-36: gamma = 0, p = 2, r = 0.5, R = 1
    v = oracle.ts_accum_laplace(0, 2, [[0, 0, 1.0]], [1.0], None, np.zeros(3), [0, 0, 0.5], None)
    assert v == pytest.approx((1 + 0.5 + 0.25) / (4 * math.pi), rel=1e-14)
    assert v == pytest.approx(0.139261, abs=1e-6)


def test_target_at_center():
    # test_tsqbx.py:39-43: only n = 0 survives
    s = np.array([0.3, -0.4, 1.2])
    v = oracle.ts_accum_laplace(0, 8, s[None], [1.0], None, np.zeros(3), np.zeros(3), None)
    assert v == pytest.approx(1.0 / (4 * math.pi * np.linalg.norm(s)), rel=1e-14)


def test_empty_batch():
    assert oracle.ts_accum_laplace(0, 8, np.zeros((0, 3)), [], None, np.zeros(3),
                                   np.zeros(3), None) == 0.0


def test_pairs_golden(golden_dir):
    g = np.load(os.path.join(golden_dir, "pairs_p8.npz"))
    for i in range(g["value"].shape[0]):
        eq, var, k = int(g["equation"][i]), int(g["variant"][i]), float(g["k"][i])
        sn = g["snrm"][i][None] if var == 2 else None
        tn = g["tnrm"][i] if var == 1 else None
        if eq == 0:
            a = oracle.ts_accum_laplace(var, 8, g["src"][i][None], [1.0], sn, g["ctr"][i],
                                        g["tgt"][i], tn)
        else:
            a = oracle.ts_accum_helmholtz(var, k, 8, g["src"][i][None], [1.0], sn, g["ctr"][i],
                                          g["tgt"][i], tn)
        b = g["value"][i]
        assert abs(a - b) <= 1e-13 * max(1.0, abs(b)), (i, eq, var, a, b)


def test_backend_batch_golden(golden_dir):
    g = np.load(os.path.join(golden_dir, "backend_batch.npz"))
    for v in range(3):
        for it, t in enumerate(g["targets"]):
            a = oracle.ts_accum_laplace(v, 8, g["src"], g["w"], g["snrm"], np.zeros(3), t,
                                        g["tnrm"])
            b = oracle.ts_accum_helmholtz(v, 1.7, 8, g["src"], g["w"], g["snrm"], np.zeros(3),
                                          t, g["tnrm"])
            assert normwise(a, g["laplace"][v, it]) <= 5e-13
            assert normwise(b, g["helmholtz"][v, it]) <= 5e-13


@pytest.mark.parametrize("name,tol", [("c1_literal", 1e-13), ("c2_small_literal", 1e-13),
                                      ("c3_small_literal", 1e-12)])
def test_batch_golden(golden_dir, name, tol):
    g = np.load(os.path.join(golden_dir, name + ".npz"))
    k = float(g["k"])
    out = oracle.ts_batch("helmholtz" if k else "laplace", 0, k, int(g["p"]), g["sources"],
                          g["weights"], g["centers"], g["near_ptr"], g["near_idx"],
                          g["targets"], g["tgt_ptr"])
    assert normwise(out, g["value"]) <= tol


def test_near_csr_matches_golden_and_kdtree(golden_dir):
    from scipy.spatial import cKDTree
    g = np.load(os.path.join(golden_dir, "c1_literal.npz"))
    h = math.sqrt(4 * math.pi / 4096)
    ptr, idx = oracle.near_csr(g["centers"], 3 * 0.5 * h, g["sources"])
    assert np.array_equal(ptr, g["near_ptr"]) and np.array_equal(idx, g["near_idx"])
    tree = cKDTree(g["sources"])
    balls = tree.query_ball_point(g["centers"], 3 * 0.5 * h)
    for ic in range(0, 4096, 7):
        assert sorted(balls[ic]) == list(idx[ptr[ic]:ptr[ic + 1]])


def test_reference_core_agrees_with_port():
    core = oracle.ref_core()
    if core is None:
        pytest.skip("oracle/_ref not built (make -C oracle ref)")
    rng = np.random.default_rng(5)
    src = rng.normal(size=(30, 3)) + np.array([0, 0, 2.5])
    w = rng.normal(size=30) + 1j * rng.normal(size=30)
    sn = rng.normal(size=(30, 3))
    sn /= np.linalg.norm(sn, axis=1)[:, None]
    tn = np.array([0.6, 0.0, 0.8])
    for t in (np.zeros(3), np.array([0.1, -0.2, 0.05])):
        for v in range(3):
            for p in (0, 1, 5, 12):
                a = core.ts_accum_laplace(v, p, src, w, sn, np.zeros(3), t, tn)
                b = oracle.ts_accum_laplace(v, p, src, w, sn, np.zeros(3), t, tn)
                assert normwise(b, a) <= 1e-14
                a = core.ts_accum_helmholtz(v, 3.1, p, src, w, sn, np.zeros(3), t, tn)
                b = oracle.ts_accum_helmholtz(v, 3.1, p, src, w, sn, np.zeros(3), t, tn)
                assert normwise(b, a) <= 1e-14


# ---- point-to-point direct sum (_core.pyx:94-165) ------------------------

@pytest.mark.parametrize("tag", ["small", "cloud"])
def test_p2p_golden(golden_dir, tag):
    g = np.load(os.path.join(golden_dir, "p2p.npz"))
    for v in range(3):
        a = oracle.p2p("laplace", v, None, g[f"{tag}_src"], g[f"{tag}_w"], g[f"{tag}_tgt"],
                       g[f"{tag}_snrm"], g[f"{tag}_tnrm"])
        b = oracle.p2p("helmholtz", v, float(g["k"]), g[f"{tag}_src"], g[f"{tag}_w"],
                       g[f"{tag}_tgt"], g[f"{tag}_snrm"], g[f"{tag}_tnrm"])
        assert normwise(a, g[f"{tag}_laplace_{v}"]) <= 1e-15
        assert normwise(b, g[f"{tag}_helmholtz_{v}"]) <= 1e-15


def test_p2p_known_answers():
    # test_kernels.py:18-22 (1/(4 pi) at unit distance), :102-105 (empty sources),
    # :137-141 (Laplace, real weights: imaginary part exactly zero)
    v = oracle.p2p("laplace", 0, None, [[0, 0, 0.0]], [1.0], [[1.0, 0, 0]])
    assert v[0] == pytest.approx(1 / (4 * math.pi), rel=1e-15)
    assert np.all(oracle.p2p("laplace", 0, None, np.zeros((0, 3)), [], np.ones((4, 3))) == 0)
    rng = np.random.default_rng(3)
    out = oracle.p2p("laplace", 0, None, rng.normal(size=(30, 3)), np.ones(30),
                     rng.normal(size=(9, 3)) + 5)
    assert np.all(out.imag == 0)


def test_p2p_singular_pair_message():
    # test_kernels.py:130-134: the first (target-major) coincident pair is named
    src = np.array([[0, 0, 0.0], [1, 0, 0]])
    tgt = np.array([[2, 0, 0.0], [1, 0, 0], [0, 0, 0]])
    with pytest.raises(ValueError, match=r"singular source/target pair: target 1, source 1"):
        oracle.p2p("laplace", 0, None, src, np.ones(2), tgt)


def test_p2p_rows_match_per_row_dense():
    rng = np.random.default_rng(5)
    src = rng.normal(size=(80, 3))
    w = rng.normal(size=80) + 1j * rng.normal(size=80)
    tgt = rng.normal(size=(25, 3)) + 4
    row_tgt = np.array([0, 3, 3, 11, 25])
    row_ptr = np.array([0, 10, 30, 30, 77])
    row_idx = rng.integers(0, 80, size=77).astype(np.int32)
    out = oracle.p2p("helmholtz", 0, 2.5, src, w, tgt, rows=(row_tgt, row_ptr, row_idx))
    for r in range(4):
        sel = row_idx[row_ptr[r]:row_ptr[r + 1]]
        ref = oracle.p2p("helmholtz", 0, 2.5, src[sel], w[sel], tgt[row_tgt[r]:row_tgt[r + 1]])
        assert np.array_equal(out[row_tgt[r]:row_tgt[r + 1]], ref)


def test_p2p_reference_core_agrees():
    core = oracle.ref_core()
    if core is None:
        pytest.skip("oracle/_ref not built")
    rng = np.random.default_rng(9)
    src = rng.normal(size=(120, 3))
    tgt = rng.normal(size=(50, 3))
    w = rng.normal(size=120) + 1j * rng.normal(size=120)
    sn = rng.normal(size=(120, 3))
    tn = rng.normal(size=(50, 3))
    for v in range(3):
        assert np.array_equal(oracle.p2p("laplace", v, None, src, w, tgt, sn, tn),
                              core.laplace_p2p(v, src, w, sn, tgt, tn))
        assert np.array_equal(oracle.p2p("helmholtz", v, 3.0, src, w, tgt, sn, tn),
                              core.helmholtz_p2p(v, 3.0, src, w, sn, tgt, tn))
