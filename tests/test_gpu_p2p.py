"""GPU parity of the point-to-point direct interactions (csrc/p2p.cu) against the
oracle (oracle.p2p, pinned bit-for-bit to the reference's _core p2p) and the
reference-generated golden vectors (tests/golden/p2p.npz).

Mirrors pkg/tests/test_kernels.py:18-141 and test_backends.py:38-44.
Tolerances: normwise relative l-inf <= 1e-12 Laplace, <= 1e-10 Helmholtz.
"""

import math
import os

import numpy as np
import pytest
import torch

import oracle
from paper_1811_01110_b200 import KernelSpec, P2PProblem, direct_sum, get_backend, p2p_rows
from paper_1811_01110_b200.kernels import Equation, Variant

pytestmark = pytest.mark.gpu

LAP_TOL = 1e-12
HELM_TOL = 1e-10
VARIANTS = [Variant.SINGLE_LAYER, Variant.TARGET_NORMAL_DERIV, Variant.SOURCE_NORMAL_DERIV]
LAPLACE = KernelSpec()


def normwise(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.max(np.abs(a - b)) / max(1e-300, np.max(np.abs(b))))


def spec_of(eq, v, k=1.7):
    return KernelSpec(equation=eq, variant=v, helmholtz_k=k if eq is Equation.HELMHOLTZ else None)


def cloud(rng, ns, nt, shift=0.0):
    src = rng.normal(size=(ns, 3))
    tgt = rng.normal(size=(nt, 3)) + shift
    w = rng.normal(size=ns) + 1j * rng.normal(size=ns)
    sn = rng.normal(size=(ns, 3))
    sn /= np.linalg.norm(sn, axis=1)[:, None]
    tn = rng.normal(size=(nt, 3))
    tn /= np.linalg.norm(tn, axis=1)[:, None]
    return src, tgt, w, sn, tn


@pytest.mark.parametrize("tag", ["small", "cloud"])
def test_backend_p2p_matches_reference_golden(golden_dir, tag):
    # test_backends.py:38-44 through the `cuda` backend module
    g = np.load(os.path.join(golden_dir, "p2p.npz"))
    be = get_backend("cuda")
    src, w, sn, tgt, tn = (g[f"{tag}_{x}"] for x in ("src", "w", "snrm", "tgt", "tnrm"))
    for v in range(3):
        assert normwise(be.laplace_p2p(v, src, w, sn, tgt, tn),
                        g[f"{tag}_laplace_{v}"]) <= LAP_TOL
        assert normwise(be.helmholtz_p2p(v, float(g["k"]), src, w, sn, tgt, tn),
                        g[f"{tag}_helmholtz_{v}"]) <= HELM_TOL


def test_known_answers():
    # test_kernels.py:18-22: 1/(4 pi) at unit distance
    v = direct_sum(LAPLACE, [[0, 0, 0.0]], [1.0], [[1.0, 0, 0]])
    assert v[0] == pytest.approx(1 / (4 * math.pi), rel=1e-14)
    # :24-30: Helmholtz with small k approaches Laplace
    rng = np.random.default_rng(0)
    s, t = rng.normal(size=(5, 3)), rng.normal(size=(3, 3)) + 4
    h = direct_sum(KernelSpec(equation=Equation.HELMHOLTZ, helmholtz_k=1e-8), s, np.ones(5), t)
    lap = direct_sum(LAPLACE, s, np.ones(5), t)
    assert normwise(h, lap) < 1e-7
    # :102-105: empty sources
    out = direct_sum(LAPLACE, np.zeros((0, 3)), np.zeros(0), rng.normal(size=(4, 3)))
    assert out.shape == (4,) and np.all(out == 0)
    # :137-141: Laplace with real weights has an exactly zero imaginary part
    out = direct_sum(LAPLACE, rng.normal(size=(30, 3)), np.ones(30, dtype=complex),
                     rng.normal(size=(9, 3)) + 5)
    assert np.all(out.imag == 0)


def test_single_pair_matches_kernel_value():
    # test_kernels.py:107-112
    s = np.array([[0.1, 0.2, 0.3]])
    t = np.array([[1.0, -0.5, 2.0]])
    r = np.linalg.norm(t - s)
    out = direct_sum(KernelSpec(equation=Equation.HELMHOLTZ, helmholtz_k=2.0), s, [1.0], t)
    assert out[0] == pytest.approx(np.exp(2j * r) / (4 * math.pi * r), rel=1e-14)


def test_singular_pair_reports_indices():
    # test_kernels.py:130-134
    src = np.array([[0, 0, 0.0], [1, 0, 0]])
    tgt = np.array([[2, 0, 0.0], [1, 0, 0], [0, 0, 0]])
    with pytest.raises(ValueError, match=r"singular source/target pair: target 1, source 1"):
        direct_sum(LAPLACE, src, np.ones(2), tgt)


def test_argument_errors():
    with pytest.raises(ValueError, match="one entry per source"):
        direct_sum(LAPLACE, np.zeros((3, 3)), np.ones(2), np.ones((1, 3)))
    with pytest.raises(ValueError, match="requires source normals"):
        direct_sum(spec_of(Equation.LAPLACE, Variant.SOURCE_NORMAL_DERIV), np.zeros((3, 3)),
                   np.ones(3), np.ones((1, 3)))
    with pytest.raises(ValueError, match="requires target normals"):
        direct_sum(spec_of(Equation.HELMHOLTZ, Variant.TARGET_NORMAL_DERIV), np.zeros((3, 3)),
                   np.ones(3), np.ones((1, 3)))


@pytest.mark.parametrize("eq", [Equation.LAPLACE, Equation.HELMHOLTZ])
@pytest.mark.parametrize("variant", VARIANTS)
@pytest.mark.parametrize("ns,nt", [(1, 1), (129, 3), (3000, 257), (20000, 7), (4099, 4097)])
def test_dense_matches_oracle(eq, variant, ns, nt):
    # covers tiles of 1..128 targets, source lanes, partial tiles and the
    # chunked (blockIdx.y) sums with their ordered reduction
    rng = np.random.default_rng(ns * 7 + nt)
    src, tgt, w, sn, tn = cloud(rng, ns, nt, shift=0.01)
    spec = spec_of(eq, variant)
    got = direct_sum(spec, src, w, tgt, sn, tn)
    ref = oracle.p2p(eq.value, spec.variant_code, spec.helmholtz_k, src, w, tgt, sn, tn)
    assert normwise(got, ref) <= (LAP_TOL if eq is Equation.LAPLACE else HELM_TOL)


@pytest.mark.parametrize("eq", [Equation.LAPLACE, Equation.HELMHOLTZ])
@pytest.mark.parametrize("variant", VARIANTS)
def test_rows_match_oracle(eq, variant):
    # ragged target rows (0, 1, 5, 300 targets) over ragged source lists (incl. empty)
    rng = np.random.default_rng(21)
    src, tgt, w, sn, tn = cloud(rng, 5000, 1 + 5 + 300 + 40 + 2, shift=0.01)
    tcount = np.array([0, 1, 5, 300, 0, 40, 2])
    scount = np.array([10, 0, 700, 1500, 3, 129, 1])
    row_tgt = np.concatenate([[0], np.cumsum(tcount)])
    row_ptr = np.concatenate([[0], np.cumsum(scount)])
    row_idx = rng.integers(0, 5000, size=row_ptr[-1]).astype(np.int32)
    spec = spec_of(eq, variant)
    got = p2p_rows(spec, src, w, tgt, row_tgt, row_ptr, row_idx, sn, tn)
    ref = oracle.p2p(eq.value, spec.variant_code, spec.helmholtz_k, src, w, tgt, sn, tn,
                     rows=(row_tgt, row_ptr, row_idx))
    assert normwise(got, ref) <= (LAP_TOL if eq is Equation.LAPLACE else HELM_TOL)
    assert np.all(got[row_tgt[1]:row_tgt[2]] == 0)      # row with no sources


def test_rows_singular_pair_names_global_indices():
    rng = np.random.default_rng(4)
    src = rng.normal(size=(50, 3))
    tgt = rng.normal(size=(6, 3)) + 3
    tgt[4] = src[17]
    row_tgt = np.array([0, 2, 6])
    row_ptr = np.array([0, 20, 45])
    row_idx = np.concatenate([np.arange(20), np.arange(5, 30)]).astype(np.int32)
    with pytest.raises(ValueError, match=r"target 4, source 17"):
        p2p_rows(LAPLACE, src, np.ones(50), tgt, row_tgt, row_ptr, row_idx)
    # the same target in a row that does not list source 17 is fine
    out = p2p_rows(LAPLACE, src, np.ones(50), tgt, row_tgt, np.array([0, 20, 20]),
                   row_idx[:20])
    assert np.all(np.isfinite(out))


def test_chunked_dense_singular_pair():
    rng = np.random.default_rng(6)
    src = rng.normal(size=(60000, 3))
    tgt = rng.normal(size=(5, 3)) + 0.5
    tgt[3] = src[51234]
    with pytest.raises(ValueError, match=r"target 3, source 51234"):
        direct_sum(LAPLACE, src, np.ones(60000), tgt)


def test_subnormal_distance_takes_precise_path():
    # r^2 is subnormal: the fast rsqrt flushes it, the screen trips, no pair is
    # singular, and the IEEE re-run gives the reference's finite value
    src = np.array([[0.0, 0.0, 0.0], [1.0, 0.0, 0.0]])
    tgt = np.array([[1e-160, 0.0, 0.0], [0.0, 2.0, 0.0]])
    w = np.array([1.0, 2.0])
    got = direct_sum(LAPLACE, src, w, tgt)
    ref = oracle.p2p("laplace", 0, None, src, w, tgt)
    assert np.all(np.isfinite(got))
    assert normwise(got, ref) <= 1e-15


def test_device_tensors_and_problem_reuse():
    rng = np.random.default_rng(8)
    src, tgt, w, _, _ = cloud(rng, 2000, 300, 0.02)
    dev = torch.device("cuda")
    spec = spec_of(Equation.HELMHOLTZ, Variant.SINGLE_LAYER, 10.0)
    prob = P2PProblem(spec, torch.as_tensor(src, device=dev),
                      torch.as_tensor(w, device=dev))
    a = prob.evaluate(torch.as_tensor(tgt, device=dev))
    b = prob.evaluate(tgt[:100])
    assert a.is_cuda and torch.equal(a[:100], b)
    ref = oracle.p2p("helmholtz", 0, 10.0, src, w, tgt)
    assert normwise(a.cpu().numpy(), ref) <= HELM_TOL


def test_derivative_variants_match_finite_differences():
    # test_kernels.py:77-95: S' = grad_t K . nu_t, D = grad_s K . nu_s
    rng = np.random.default_rng(12)
    s = rng.normal(size=(1, 3))
    t = s + np.array([[0.7, -0.4, 0.9]])
    nu = np.array([0.6, 0.0, 0.8])
    h = 1e-5
    for eq in (Equation.LAPLACE, Equation.HELMHOLTZ):
        sv = spec_of(eq, Variant.SINGLE_LAYER, 3.0)
        fd_t = (direct_sum(sv, s, [1.0], t + h * nu) - direct_sum(sv, s, [1.0], t - h * nu)) / (2 * h)
        fd_s = (direct_sum(sv, s + h * nu, [1.0], t) - direct_sum(sv, s - h * nu, [1.0], t)) / (2 * h)
        sp = direct_sum(spec_of(eq, Variant.TARGET_NORMAL_DERIV, 3.0), s, [1.0], t,
                        target_normals=nu[None])
        d = direct_sum(spec_of(eq, Variant.SOURCE_NORMAL_DERIV, 3.0), s, [1.0], t,
                       source_normals=nu[None])
        assert abs(sp[0] - fd_t[0]) <= 1e-8 * abs(sp[0])
        assert abs(d[0] - fd_s[0]) <= 1e-8 * abs(d[0])


# --- kernel_value (kernels.py:83-111) ------------------------------------------------
def _unit(v):
    return v / np.linalg.norm(v)


def test_kernel_value_known_answers_and_symmetry():
    # test_kernels.py:18-48, 98-100
    from paper_1811_01110_b200 import kernel_value
    t, s = np.array([1.0, -0.5, 2.0]), np.array([0.1, 0.2, 0.3])
    r = float(np.linalg.norm(t - s))
    assert kernel_value(LAPLACE, t, s) == pytest.approx(1 / (4 * math.pi * r), rel=1e-14)
    helm = KernelSpec(equation=Equation.HELMHOLTZ, helmholtz_k=2.0)
    assert kernel_value(helm, t, s) == pytest.approx(np.exp(2j * r) / (4 * math.pi * r),
                                                     rel=1e-14)
    rng = np.random.default_rng(4)
    t, s = rng.normal(size=3), rng.normal(size=3)
    assert kernel_value(LAPLACE, t, s) == kernel_value(LAPLACE, s, t)
    assert kernel_value(LAPLACE, t, s).imag == 0.0


def test_kernel_value_source_normal_deriv_on_sphere_vs_finite_differences():
    # test_kernels.py:57-65
    from paper_1811_01110_b200 import kernel_value
    s_hat = _unit(np.array([0.3, 0.5, 0.81]))
    t = 2.0 * s_hat
    val = kernel_value(KernelSpec(variant=Variant.SOURCE_NORMAL_DERIV), t, s_hat,
                       source_normal=s_hat)
    h = 1e-6
    fd = (kernel_value(LAPLACE, t, s_hat + h * s_hat)
          - kernel_value(LAPLACE, t, s_hat - h * s_hat)) / (2 * h)
    assert abs(val - fd) < 1e-7 * abs(fd)


@pytest.mark.parametrize("spec", [
    KernelSpec(variant=Variant.TARGET_NORMAL_DERIV),
    KernelSpec(variant=Variant.SOURCE_NORMAL_DERIV),
    KernelSpec(equation=Equation.HELMHOLTZ, helmholtz_k=1.3, variant=Variant.TARGET_NORMAL_DERIV),
    KernelSpec(equation=Equation.HELMHOLTZ, helmholtz_k=1.3, variant=Variant.SOURCE_NORMAL_DERIV),
])
def test_kernel_value_derivatives_match_finite_differences(spec):
    # test_kernels.py:68-95 (20 random pairs instead of 100)
    from paper_1811_01110_b200 import kernel_value
    rng = np.random.default_rng(8)
    h = 1e-5
    base = KernelSpec(equation=spec.equation, helmholtz_k=spec.helmholtz_k)
    for _ in range(20):
        t, s = rng.normal(size=3), rng.normal(size=3)
        if np.linalg.norm(t - s) < 0.1:
            s = t + _unit(s - t) * 0.1
        nu = _unit(rng.normal(size=3))
        if spec.variant is Variant.TARGET_NORMAL_DERIV:
            val = kernel_value(spec, t, s, target_normal=nu)
            fd = (kernel_value(base, t + h * nu, s) - kernel_value(base, t - h * nu, s)) / (2 * h)
        else:
            val = kernel_value(spec, t, s, source_normal=nu)
            fd = (kernel_value(base, t, s + h * nu) - kernel_value(base, t, s - h * nu)) / (2 * h)
        assert abs(val - fd) <= 1e-6 * max(1e-3, abs(fd))
