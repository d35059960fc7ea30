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
