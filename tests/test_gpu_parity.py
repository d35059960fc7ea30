"""GPU parity: the sm_100a kernels (through the C ABI) against the oracle.

Mirrors the reference's hot-path tests (pkg/tests/test_tsqbx.py,
test_backends.py) plus config-level parity on the BASELINE geometries.
Tolerances (north_star): normwise relative l-inf <= 1e-12 Laplace,
<= 1e-10 Helmholtz; near-list membership bit-exact.
"""

import math
import os

import numpy as np
import pytest
import torch

import oracle
from paper_1811_01110_b200 import (KernelSpec, TsConfig, TsqbxProblem, build_near_lists,
                                   get_backend, ts_accumulate, ts_accumulate_batch, ts_eval)
from paper_1811_01110_b200 import configs
from paper_1811_01110_b200.kernels import Equation, Variant

pytestmark = pytest.mark.gpu

LAP_TOL = 1e-12
HELM_TOL = 1e-10
VARIANTS = [Variant.SINGLE_LAYER, Variant.TARGET_NORMAL_DERIV, Variant.SOURCE_NORMAL_DERIV]


def normwise(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.max(np.abs(a - b)) / max(1e-300, np.max(np.abs(b))))


def sorted_rows(ptr, idx):
    return [np.sort(idx[ptr[i]:ptr[i + 1]]) for i in range(len(ptr) - 1)]


# --- reference known answers (test_tsqbx.py) --------------------------------------
def test_collinear_geometric_sum():
    v = ts_eval(TsConfig(KernelSpec(), 2), [0, 0, 1.0], np.zeros(3), [0, 0, 0.5])
    assert v == pytest.approx((1 + 0.5 + 0.25) / (4 * math.pi), rel=1e-14)
    assert v == pytest.approx(0.139261, abs=1e-6)


def test_target_at_center():
    s = np.array([0.3, -0.4, 1.2])
    v = ts_eval(TsConfig(KernelSpec(), 8), s, np.zeros(3), np.zeros(3))
    assert v == pytest.approx(1.0 / (4 * math.pi * np.linalg.norm(s)), rel=1e-14)


def test_separation_violation_raises():
    with pytest.raises(ValueError, match="separation violation"):
        ts_eval(TsConfig(KernelSpec(), 8), [0, 0, 1.0], np.zeros(3), [0, 1.1, 0])


def test_singular_center_raises():
    with pytest.raises(ValueError, match="coincides"):
        ts_eval(TsConfig(KernelSpec(), 8), np.zeros(3), np.zeros(3), np.zeros(3))


def test_separation_error_names_source_index():
    src = np.array([[0, 0, 2.0], [0, 0, 0.4]])
    with pytest.raises(ValueError, match="source 1"):
        ts_accumulate(TsConfig(KernelSpec(), 8), src, np.ones(2), np.zeros(3), [0, 0.5, 0])


def test_coincidence_outranks_separation():
    src = np.array([[0, 0, 0.4], [0, 0, 0.0]])
    with pytest.raises(ValueError, match="source 1 coincides"):
        ts_accumulate(TsConfig(KernelSpec(), 8), src, np.ones(2), np.zeros(3), [0, 0.5, 0])


def test_empty_batch_and_single_source():
    cfg = TsConfig(KernelSpec(), 8)
    assert ts_accumulate(cfg, np.zeros((0, 3)), np.zeros(0), np.zeros(3), np.zeros(3)) == 0.0
    s, c, t = np.array([0.2, 0.9, -0.5]), np.array([0.1, 0.0, 0.0]), np.array([0.3, 0.1, 0.2])
    a = ts_accumulate(cfg, s[None], np.array([1.3 - 0.4j]), c, t)
    assert a == pytest.approx((1.3 - 0.4j) * ts_eval(cfg, s, c, t), rel=1e-14)


def test_laplace_outputs_real():
    v = ts_eval(TsConfig(KernelSpec(), 8), [0.2, 0.9, -0.5], [0.1, 0, 0], [0.3, 0.1, 0.2])
    assert v.imag == 0.0


def test_normals_required():
    with pytest.raises(ValueError, match="source normals"):
        ts_eval(TsConfig(KernelSpec(variant=Variant.SOURCE_NORMAL_DERIV), 4), [0, 0, 1.0],
                np.zeros(3), [0, 0, 0.1])
    with pytest.raises(ValueError, match="target normal"):
        ts_eval(TsConfig(KernelSpec(variant=Variant.TARGET_NORMAL_DERIV), 4), [0, 0, 1.0],
                np.zeros(3), [0, 0, 0.1])


# --- golden vectors produced by the reference ---------------------------------------
def test_all_variants_match_reference_pairs(golden_dir):
    """60 random admissible configs x (Laplace, Helmholtz) x (S, S', D), p = 8
    (test_tsqbx.py:71-85), against the reference's own ts_eval values."""
    g = np.load(os.path.join(golden_dir, "pairs_p8.npz"))
    for i in range(g["value"].shape[0]):
        eq, var, k = int(g["equation"][i]), int(g["variant"][i]), float(g["k"][i])
        spec = KernelSpec(equation=Equation.LAPLACE if eq == 0 else Equation.HELMHOLTZ,
                          variant=VARIANTS[var], helmholtz_k=None if eq == 0 else k)
        a = ts_eval(TsConfig(spec, 8), g["src"][i], g["ctr"][i], g["tgt"][i],
                    source_normal=g["snrm"][i] if var == 2 else None,
                    target_normal=g["tnrm"][i] if var == 1 else None)
        b = g["value"][i]
        assert abs(a - b) <= 1e-12 * max(1.0, abs(b)), (i, eq, var, a, b)


def test_cuda_backend_matches_reference_backends(golden_dir):
    """test_backends.py:47-59 on the cuda backend module."""
    g = np.load(os.path.join(golden_dir, "backend_batch.npz"))
    be = get_backend("cuda")
    for v in range(3):
        for it, t in enumerate(g["targets"]):
            a = be.ts_accum_laplace(v, 8, g["src"], g["w"], g["snrm"], np.zeros(3), t, g["tnrm"])
            b = be.ts_accum_helmholtz(v, 1.7, 8, g["src"], g["w"], g["snrm"], np.zeros(3), t,
                                      g["tnrm"])
            assert normwise(a, g["laplace"][v, it]) <= 5e-13
            assert normwise(b, g["helmholtz"][v, it]) <= 5e-13


@pytest.mark.parametrize("name,tol", [("c1_literal", LAP_TOL), ("c2_small_literal", LAP_TOL),
                                      ("c3_small_literal", HELM_TOL)])
def test_batch_matches_reference_golden(golden_dir, name, tol):
    g = np.load(os.path.join(golden_dir, name + ".npz"))
    k = float(g["k"])
    spec = KernelSpec(equation=Equation.HELMHOLTZ, helmholtz_k=k) if k else KernelSpec()
    cfg = TsConfig(spec, int(g["p"]))
    out = ts_accumulate_batch(cfg, g["sources"], g["weights"], g["centers"], g["targets"],
                              (g["near_ptr"], g["near_idx"]), tgt_ptr=g["tgt_ptr"])
    assert normwise(out, g["value"]) <= tol
    # same values through the device-built near lists
    h = math.sqrt(4 * math.pi / g["sources"].shape[0])
    mult = 3.0 if name.startswith("c1") else 4.0
    near = build_near_lists(g["centers"], g["sources"], mult * 0.5 * h)
    uptr, uidx = near.to_user_csr()
    assert np.array_equal(uptr, g["near_ptr"])
    assert all(np.array_equal(a, b) for a, b in zip(sorted_rows(uptr, uidx),
                                                    sorted_rows(g["near_ptr"], g["near_idx"])))
    out2 = ts_accumulate_batch(cfg, g["sources"], g["weights"], g["centers"], g["targets"], near,
                               tgt_ptr=g["tgt_ptr"])
    assert normwise(out2, g["value"]) <= tol


# --- near-list builder vs oracle membership ------------------------------------------
@pytest.mark.parametrize("name,preset", [("c1", "literal"), ("c1", "dense"), ("c2", "literal"),
                                         ("c4", "literal"), ("c5", "literal")])
def test_near_lists_bit_exact(name, preset):
    kw = {"n": 65536, "spheres": 4} if name == "c5" else {}
    case = configs.make_case(name, preset, **kw)
    near = build_near_lists(case.centers, case.sources, case.near_radii)
    uptr, uidx = near.to_user_csr()
    optr, oidx = oracle.near_csr(case.centers, case.near_radii, case.sources)
    assert near.n_pairs == len(oidx)
    assert np.array_equal(uptr, optr)
    srt = np.concatenate([np.sort(uidx[uptr[i]:uptr[i + 1]]) for i in range(case.n_centers)])
    assert np.array_equal(srt, oidx)
    # the SELL-32x4 copy holds exactly the CSR rows
    sp = near.sell_ptr.cpu().numpy()
    si = near.sell_idx.cpu().numpy()
    p = near.ptr.cpu().numpy()
    d = near.idx.cpu().numpy()
    for g in range(0, case.n_centers, max(1, case.n_centers // 257)):
        n_g = p[g + 1] - p[g]
        i = np.arange(n_g)
        cells = sp[g // 32] + (i // 4) * 128 + (g % 32) * 4 + i % 4
        assert np.array_equal(si[cells], d[p[g]:p[g + 1]])


def _assert_sell_holds_csr(near, stride=1):
    sp = near.sell_ptr.cpu().numpy()
    si = near.sell_idx.cpu().numpy()
    p = near.ptr.cpu().numpy()
    d = near.idx.cpu().numpy()
    for g in range(0, near.n_ctr, stride):
        n_g = p[g + 1] - p[g]
        i = np.arange(n_g)
        cells = sp[g // 32] + (i // 4) * 128 + (g % 32) * 4 + i % 4
        assert cells.size == 0 or cells.max() < sp[g // 32 + 1]
        assert np.array_equal(si[cells], d[p[g]:p[g + 1]])


@pytest.mark.parametrize("mode", ["bound", "exact", "exact_nomask", "csr"])
def test_near_list_build_paths_agree(mode, monkeypatch):
    """The bound-sized SELL build (+ compaction), the exact-count fallback it
    takes when the bound would be too large, and the CSR-only build give the
    same rows, the same SELL layout, and the oracle's membership."""
    from paper_1811_01110_b200 import nearlist
    case = configs.make_case("c5", "literal", n=32768, spheres=4)
    if mode.startswith("exact"):
        monkeypatch.setattr(nearlist, "_BOUND_BYTES_MAX", 0)
        monkeypatch.setattr(nearlist, "_EXACT_MASKS", mode == "exact")
    near = build_near_lists(case.centers, case.sources, case.near_radii, sell=mode != "csr")
    if mode == "csr":
        near.build_sell()
    monkeypatch.undo()
    ref = build_near_lists(case.centers, case.sources, case.near_radii)
    assert torch.equal(near.ptr, ref.ptr)
    assert torch.equal(near.idx, ref.idx)
    # slice widths may differ (the bound build keeps its bound-sized slices when
    # they are within 1.5x of exact), the rows they hold may not
    _assert_sell_holds_csr(near)
    uptr, uidx = near.to_user_csr()
    optr, oidx = oracle.near_csr(case.centers, case.near_radii, case.sources)
    assert np.array_equal(uptr, optr)
    srt = np.concatenate([np.sort(uidx[uptr[i]:uptr[i + 1]]) for i in range(case.n_centers)])
    assert np.array_equal(srt, oidx)


@pytest.mark.gpu
@pytest.mark.parametrize("kind", ["c2_dense", "c4_dense", "mixed", "sparse", "ragged"])
def test_near_lists_exact_route_masks(kind, monkeypatch):
    """The exact route with the count's member masks reused by the fill
    (tsqbx_near_recount_masks / tsqbx_near_fill_masks): dense lists (union
    mode, the uniform walk over 32-candidate groups), radii of mixed levels and
    sparse centers (per-cell mode, which tests twice), a center count that is
    not a multiple of 32 -- rows, SELL layout and oracle membership."""
    from paper_1811_01110_b200 import nearlist
    rng = np.random.default_rng(11)
    if kind in ("c2_dense", "c4_dense"):
        case = configs.make_case(kind[:2], "dense", n=16384)
        ctr, src, rad = case.centers, case.sources, case.near_radii
    elif kind == "mixed":
        n = 30000
        src = np.vstack([rng.normal(scale=0.05, size=(n // 2, 3)), rng.uniform(-1, 1, (n // 2, 3))])
        ctr = src[rng.permutation(n)[: n // 2]] + rng.normal(scale=1e-3, size=(n // 2, 3))
        rad = 0.004 * np.exp(rng.uniform(0.0, np.log(7.0), size=n // 2))
    elif kind == "sparse":
        src = rng.uniform(0, 1, (20000, 3))
        ctr = rng.uniform(0, 1, (300, 3))
        rad = np.full(300, 0.03)
    else:
        src = rng.normal(size=(3000, 3))
        ctr = rng.normal(size=(1001, 3))
        rad = rng.uniform(0.0, 0.6, size=1001)
    monkeypatch.setattr(nearlist, "_BOUND_BYTES_MAX", 0)
    monkeypatch.setattr(nearlist, "_EXACT_MASKS", True)
    near = build_near_lists(ctr, src, rad)
    monkeypatch.setattr(nearlist, "_EXACT_MASKS", False)
    twice = build_near_lists(ctr, src, rad)
    assert torch.equal(near.ptr, twice.ptr)
    assert torch.equal(near.sell_ptr, twice.sell_ptr)
    assert torch.equal(near.idx, twice.idx)
    _assert_sell_holds_csr(near, stride=7)
    uptr, uidx = near.to_user_csr()
    optr, oidx = oracle.near_csr(ctr, rad, src)
    assert np.array_equal(uptr, optr)
    order = np.lexsort((uidx, np.repeat(np.arange(np.asarray(ctr).shape[0]), np.diff(uptr))))
    assert np.array_equal(uidx[order], oidx)


def test_near_lists_repeated_builds_are_exact():
    """Alternating builds of different sizes reuse device memory; every build must
    reproduce the oracle membership exactly (guards against stale-memory and
    divergence bugs in the count/fill sweeps)."""
    ref = {}
    for name, preset in [("c2", "literal"), ("c1", "literal"), ("c2", "literal"), ("c1", "dense"),
                         ("c2", "literal"), ("c2", "dense"), ("c2", "literal")]:
        case = configs.make_case(name, preset)
        near = build_near_lists(case.centers, case.sources, case.near_radii)
        uptr, uidx = near.to_user_csr()
        key = (name, preset)
        if key not in ref:
            ref[key] = oracle.near_csr(case.centers, case.near_radii, case.sources)
        optr, oidx = ref[key]
        assert np.array_equal(uptr, optr)
        order = np.lexsort((uidx, np.repeat(np.arange(case.n_centers), np.diff(uptr))))
        assert np.array_equal(uidx[order], oidx)


def test_near_lists_edge_cases():
    rng = np.random.default_rng(3)
    src = rng.normal(size=(500, 3))
    ctr = np.vstack([rng.normal(size=(50, 3)), [[100.0, 100.0, 100.0]]])   # last: no sources
    rad = rng.uniform(0.0, 0.8, size=51)
    rad[0] = 0.0                                                            # zero radius
    near = build_near_lists(ctr, src, rad)
    uptr, uidx = near.to_user_csr()
    optr, oidx = oracle.near_csr(ctr, rad, src)
    assert np.array_equal(uptr, optr) and uptr[-1] - uptr[-2] == 0
    assert all(np.array_equal(a, b) for a, b in zip(sorted_rows(uptr, uidx),
                                                    sorted_rows(optr, oidx)))
    near0 = build_near_lists(ctr, np.zeros((0, 3)), rad)     # no sources at all
    assert near0.n_pairs == 0
    # duplicate points (ties) and a source exactly on the sphere of the radius
    src2 = np.array([[0.0, 0.0, 1.0], [0.0, 0.0, 1.0], [0.0, 0.0, 1.0 + 1e-15], [0.5, 0, 0]])
    near2 = build_near_lists(np.zeros((1, 3)), src2, 1.0)
    u2p, u2i = near2.to_user_csr()
    o2p, o2i = oracle.near_csr(np.zeros((1, 3)), [1.0], src2)
    assert sorted(u2i.tolist()) == o2i.tolist()


@pytest.mark.gpu
@pytest.mark.parametrize("spread", [2.0, 7.0, 40.0])
def test_near_lists_mixed_radii_levels(spread):
    """Radii spanning `spread`x: centers search cells of different levels (up to
    four, the fine grid following the smallest radius; beyond 8x the smallest
    radii share level 0), warps mix levels (per-cell mode, one head per distinct
    (cell, level)), and clustered points make union tiles span many small cells.
    Membership must equal the oracle's exactly."""
    rng = np.random.default_rng(int(spread * 10))
    n = 40000
    # a dense cluster and a sparse background, radii from 0.004 to 0.004 * spread
    src = np.vstack([rng.normal(scale=0.05, size=(n // 2, 3)), rng.uniform(-1, 1, (n // 2, 3))])
    ctr = src[rng.permutation(n)[: n // 2]] + rng.normal(scale=1e-3, size=(n // 2, 3))
    rad = 0.004 * np.exp(rng.uniform(0.0, np.log(spread), size=n // 2))
    near = build_near_lists(ctr, src, rad)
    uptr, uidx = near.to_user_csr()
    optr, oidx = oracle.near_csr(ctr, rad, src)
    assert np.array_equal(uptr, optr)
    assert all(np.array_equal(a, b) for a, b in zip(sorted_rows(uptr, uidx),
                                                    sorted_rows(optr, oidx)))
    # the bound-sized SELL holds every row: CSR derived from it equals the rows
    assert near.n_pairs == len(oidx)


@pytest.mark.gpu
def test_near_lists_wide_extent_full_key_bits():
    """Clusters 1e6 apart with small radii: the fine grid is capped by the
    extent (2^21 cells per axis), the sort uses all 63 key bits, and cells far
    larger than the radii still give the oracle's membership."""
    rng = np.random.default_rng(5)
    offs = np.array([[0.0, 0.0, 0.0], [1e6, -3e5, 2e5], [-7e5, 9e5, -1e6]])
    src = np.vstack([o + rng.normal(scale=0.02, size=(3000, 3)) for o in offs])
    ctr = src[::2] + rng.normal(scale=1e-3, size=src[::2].shape)
    rad = rng.uniform(0.005, 0.03, size=len(ctr))
    near = build_near_lists(ctr, src, rad)
    uptr, uidx = near.to_user_csr()
    optr, oidx = oracle.near_csr(ctr, rad, src)
    assert np.array_equal(uptr, optr)
    assert all(np.array_equal(a, b) for a, b in zip(sorted_rows(uptr, uidx),
                                                    sorted_rows(optr, oidx)))


# --- config-level parity ------------------------------------------------------------
def _case_parity(case, tol, subset=None, generic=False):
    near = build_near_lists(case.centers, case.sources, case.near_radii)
    prob = TsqbxProblem(case.cfg, case.sources, case.weights, case.centers, case.targets, near,
                        tgt_ptr=case.tgt_ptr, source_normals=case.normals,
                        target_normals=case.targets * 0 + case.normals[0])
    out = prob.evaluate(validate=True, generic=generic).cpu().numpy()
    uptr, uidx = near.to_user_csr()
    spec = case.cfg.spec
    eq = "laplace" if spec.is_laplace else "helmholtz"
    if subset is None:
        ref = oracle.ts_batch(eq, spec.variant_code, spec.helmholtz_k or 0.0, case.cfg.p_qbx,
                              case.sources, case.weights, case.centers, uptr, uidx,
                              case.targets, case.tgt_ptr)
        err = normwise(out, ref)
    else:
        rng = np.random.default_rng(11)
        sel = np.sort(rng.choice(case.n_centers, subset, replace=False))
        lens = np.diff(uptr)[sel]
        sptr = np.concatenate([[0], np.cumsum(lens)])
        sidx = np.concatenate([uidx[uptr[c]:uptr[c + 1]] for c in sel])
        tl = np.diff(case.tgt_ptr)[sel]
        tptr = np.concatenate([[0], np.cumsum(tl)])
        tsel = np.concatenate([np.arange(case.tgt_ptr[c], case.tgt_ptr[c + 1]) for c in sel])
        ref = oracle.ts_batch(eq, spec.variant_code, spec.helmholtz_k or 0.0, case.cfg.p_qbx,
                              case.sources, case.weights, case.centers[sel], sptr, sidx,
                              case.targets[tsel], tptr)
        err = normwise(out[tsel], ref)
    assert err <= tol, err
    return out, near


@pytest.mark.parametrize("name,preset", [("c4", "literal"), ("c4", "dense"), ("c5", "literal")])
def test_c4_c5_full_size_one_percent(name, preset):
    # parity on a >= 1% seeded subset at the full C4/C5 sizes
    case = configs.make_case(name, preset)
    _case_parity(case, LAP_TOL if name == "c4" else HELM_TOL,
                 subset=max(4096, case.n_centers // 100))


def test_c5_dense_full_size_one_percent():
    """C5 dense at full size (8.39 M centers, 1.69 G pairs): a seeded 1 % subset
    of the centers against the oracle; the subset's rows are cut out of the
    device lists on the device (the full CSR is 6.7 GB)."""
    case = configs.make_case("c5", "dense")
    near = build_near_lists(case.centers, case.sources, case.near_radii)
    prob = TsqbxProblem(case.cfg, case.sources, case.weights, case.centers, case.targets, near,
                        tgt_ptr=case.tgt_ptr)
    out = prob.evaluate(validate=True).cpu().numpy()
    rng = np.random.default_rng(12)
    sel = np.sort(rng.choice(case.n_centers, case.n_centers // 100, replace=False))
    dev = near.ptr.device
    row_of = torch.empty_like(near.ctr_order)
    row_of[near.ctr_order.long()] = torch.arange(case.n_centers, dtype=row_of.dtype, device=dev)
    rows = row_of[torch.as_tensor(sel, device=dev)].long()
    b, e = near.ptr[rows], near.ptr[rows + 1]
    lens = e - b
    sptr = torch.zeros(len(sel) + 1, dtype=torch.int64, device=dev)
    sptr[1:] = torch.cumsum(lens, 0)
    pos = torch.arange(int(sptr[-1].item()), device=dev) - torch.repeat_interleave(sptr[:-1], lens)
    ent = near.idx[torch.repeat_interleave(b, lens) + pos].long()
    sidx = near.src_perm[ent].cpu().numpy().astype(np.int32)
    sptr = sptr.cpu().numpy()
    tl = np.diff(case.tgt_ptr)[sel]
    tptr = np.concatenate([[0], np.cumsum(tl)])
    tsel = np.concatenate([np.arange(case.tgt_ptr[c], case.tgt_ptr[c + 1]) for c in sel])
    spec = case.cfg.spec
    ref = oracle.ts_batch("helmholtz", 0, spec.helmholtz_k, case.cfg.p_qbx, case.sources,
                          case.weights, case.centers[sel], sptr, sidx, case.targets[tsel], tptr)
    assert sptr[-1] > 10_000_000
    assert normwise(out[tsel], ref) <= HELM_TOL


@pytest.mark.parametrize("name,preset", [("c1", "literal"), ("c1", "dense")])
def test_c1_full(name, preset):
    _case_parity(configs.make_case(name, preset), LAP_TOL)


@pytest.mark.parametrize("preset", ["literal", "dense"])
def test_c2_c3_full_size_subset(preset):
    _case_parity(configs.make_case("c2", preset), LAP_TOL, subset=4096)
    _case_parity(configs.make_case("c3", preset), HELM_TOL, subset=4096)


def test_c4_c5_subset():
    _case_parity(configs.make_case("c4", "literal", n=262144), LAP_TOL, subset=4096)
    _case_parity(configs.make_case("c4", "dense", n=65536), LAP_TOL, subset=2048)
    _case_parity(configs.make_case("c5", "literal", n=65536, spheres=4), HELM_TOL, subset=4096)


@pytest.mark.parametrize("p", list(range(0, 17)) + [20, 33])
def test_order_sweep(p):
    for name in ("c1", "c3"):
        case = configs.make_case(name, "literal", n=2048)
        case.cfg = TsConfig(case.cfg.spec, p)
        _case_parity(case, LAP_TOL if name == "c1" else HELM_TOL)


@pytest.mark.parametrize("eq,variant", [(e, v) for e in ("laplace", "helmholtz")
                                        for v in VARIANTS])
def test_variants_batch(eq, variant):
    case = configs.make_case("c1" if eq == "laplace" else "c3", "literal", n=2048)
    spec = KernelSpec(equation=Equation(eq), variant=variant,
                      helmholtz_k=None if eq == "laplace" else 10.0)
    case.cfg = TsConfig(spec, 8)
    near = build_near_lists(case.centers, case.sources, case.near_radii)
    tn = np.repeat(case.normals, np.diff(case.tgt_ptr), axis=0)
    out = ts_accumulate_batch(case.cfg, case.sources, case.weights, case.centers, case.targets,
                              near, tgt_ptr=case.tgt_ptr, source_normals=case.normals,
                              target_normals=tn)
    uptr, uidx = near.to_user_csr()
    ref = oracle.ts_batch(eq, spec.variant_code, spec.helmholtz_k or 0.0, 8, case.sources,
                          case.weights, case.centers, uptr, uidx, case.targets, case.tgt_ptr,
                          snormals=case.normals, tnormals=tn)
    assert normwise(out, ref) <= (LAP_TOL if eq == "laplace" else HELM_TOL)


def test_fast_and_generic_kernels_agree():
    for name, tol in (("c2", LAP_TOL), ("c3", HELM_TOL)):
        case = configs.make_case(name, "dense", n=16384)
        a, _ = _case_parity(case, tol)
        b, _ = _case_parity(case, tol, generic=True)
        assert normwise(a, b) <= tol


@pytest.mark.parametrize("G", [1, 2, 4, 8, 16, 32])
def test_group_lanes_all_agree(G):
    case = configs.make_case("c2", "dense", n=8192)
    near = build_near_lists(case.centers, case.sources, case.near_radii)
    uptr, uidx = near.to_user_csr()
    ref = oracle.ts_batch("laplace", 0, 0.0, 8, case.sources, case.weights, case.centers, uptr,
                          uidx, case.targets, case.tgt_ptr)
    prob = TsqbxProblem(case.cfg, case.sources, case.weights, case.centers, case.targets, near,
                        tgt_ptr=case.tgt_ptr, group_lanes=G)
    assert normwise(prob.evaluate().cpu().numpy(), ref) <= LAP_TOL


def test_ragged_targets_and_empty_rows():
    rng = np.random.default_rng(7)
    src = rng.normal(size=(300, 3)) * 0.5 + np.array([0, 0, 3.0])
    ctr = rng.normal(size=(40, 3)) * 0.1
    ntg = rng.integers(0, 4, size=40)                      # 0..3 targets per center
    tptr = np.concatenate([[0], np.cumsum(ntg)])
    tgt = np.repeat(ctr, ntg, axis=0) + rng.normal(size=(tptr[-1], 3)) * 0.05
    lens = rng.integers(0, 30, size=40)
    lens[::5] = 0                                          # empty rows
    nptr = np.concatenate([[0], np.cumsum(lens)])
    nidx = rng.integers(0, 300, size=nptr[-1]).astype(np.int32)
    w = rng.normal(size=300) + 1j * rng.normal(size=300)
    for spec, tol in ((KernelSpec(), LAP_TOL),
                      (KernelSpec(equation=Equation.HELMHOLTZ, helmholtz_k=3.0), HELM_TOL)):
        cfg = TsConfig(spec, 8)
        out = ts_accumulate_batch(cfg, src, w, ctr, tgt, (nptr, nidx), tgt_ptr=tptr)
        ref = oracle.ts_batch("laplace" if spec.is_laplace else "helmholtz", 0,
                              spec.helmholtz_k or 0.0, 8, src, w, ctr, nptr, nidx, tgt, tptr)
        assert normwise(out, ref) <= tol
        for ic in np.nonzero(lens == 0)[0]:
            assert np.all(out[tptr[ic]:tptr[ic + 1]] == 0)


@pytest.mark.parametrize("split", ["1", "2", "4"])
def test_row_split_matches_oracle(split, monkeypatch):
    """Rows split over 1, 2 or 4 threads (SELL, Laplace S): ragged rows (0..70
    entries, lengths not multiples of 4, rows shorter than the split), 0..3
    targets per center, real and complex weights, validation on; and a dense
    C2 subset."""
    monkeypatch.setenv("GIGAQBX_SPLIT", split)
    rng = np.random.default_rng(70 + int(split))
    src = rng.normal(size=(500, 3)) * 0.5 + np.array([0, 0, 3.0])
    n_ctr = 150
    ctr = rng.normal(size=(n_ctr, 3)) * 0.1
    ntg = rng.integers(0, 4, size=n_ctr)
    tptr = np.concatenate([[0], np.cumsum(ntg)])
    tgt = np.repeat(ctr, ntg, axis=0) + rng.normal(size=(tptr[-1], 3)) * 0.05
    lens = rng.integers(0, 71, size=n_ctr)
    lens[::7] = 0
    lens[1::7] = 1
    nptr = np.concatenate([[0], np.cumsum(lens)])
    nidx = rng.integers(0, 500, size=nptr[-1]).astype(np.int32)
    for w in (rng.uniform(0.5, 1.5, size=500) + 0j, rng.normal(size=500) + 1j * rng.normal(size=500)):
        for p in (4, 8, 12):
            out = ts_accumulate_batch(TsConfig(KernelSpec(), p), src, w, ctr, tgt, (nptr, nidx),
                                      tgt_ptr=tptr)
            ref = oracle.ts_batch("laplace", 0, 0.0, p, src, w, ctr, nptr, nidx, tgt, tptr)
            assert normwise(out, ref) <= LAP_TOL
    _case_parity(configs.make_case("c2", "dense", n=16384), LAP_TOL)


def test_batch_validation_names_target_and_source():
    case = configs.make_case("c1", "literal", n=1024)
    tg = case.targets.copy()
    tg[37] = case.centers[37] + 10.0 * case.expansion_radii[37]     # far outside: violation
    near = build_near_lists(case.centers, case.sources, case.near_radii)
    with pytest.raises(ValueError, match=r"separation violation for source \d+: .*target 37"):
        ts_accumulate_batch(case.cfg, case.sources, case.weights, case.centers, tg, near)
    out = ts_accumulate_batch(case.cfg, case.sources, case.weights, case.centers, tg, near,
                              validate=False)
    assert out.shape == (1024,)


def test_full_size_properties_c2_dense():
    """At BASELINE size: linearity in the weights and invariance under a
    permutation of the source order (size-independent properties)."""
    case = configs.make_case("c2", "dense")
    near = build_near_lists(case.centers, case.sources, case.near_radii)
    p1 = TsqbxProblem(case.cfg, case.sources, case.weights, case.centers, case.targets, near,
                      tgt_ptr=case.tgt_ptr)
    u1 = p1.evaluate().clone()
    w2 = np.random.default_rng(4).normal(size=case.n_sources) + 0j
    p2 = TsqbxProblem(case.cfg, case.sources, w2, case.centers, case.targets, near,
                      tgt_ptr=case.tgt_ptr)
    u2 = p2.evaluate().clone()
    p3 = TsqbxProblem(case.cfg, case.sources, case.weights + 2.0 * w2, case.centers,
                      case.targets, near, tgt_ptr=case.tgt_ptr)
    u3 = p3.evaluate().clone()
    assert normwise((u1 + 2 * u2).cpu().numpy(), u3.cpu().numpy()) <= 1e-12
    perm = np.random.default_rng(5).permutation(case.n_sources)
    near_p = build_near_lists(case.centers, case.sources[perm], case.near_radii)
    assert near_p.n_pairs == near.n_pairs
    p4 = TsqbxProblem(case.cfg, case.sources[perm], case.weights[perm], case.centers,
                      case.targets, near_p, tgt_ptr=case.tgt_ptr)
    assert normwise(p4.evaluate().cpu().numpy(), u1.cpu().numpy()) <= 1e-13
    assert np.all(np.isfinite(u1.cpu().numpy()))


@pytest.mark.parametrize("p", [0, 1, 2, 5, 8, 12, 16, 20])
@pytest.mark.parametrize("eq", ["laplace", "helmholtz"])
def test_derivative_variants_all_orders(p, eq):
    """S' and D through the compile-time-order SELL kernels (p <= 16) and the
    generic kernel (p = 20), including targets AT their center (r = 0
    conventions, _core.pyx:262-264, 285-288, 357-359, 400-408)."""
    rng = np.random.default_rng(100 + p)
    n_src, n_ctr = 400, 60
    src = rng.normal(size=(n_src, 3)) * 0.4 + np.array([0.0, 0.0, 2.0])
    sn = rng.normal(size=(n_src, 3))
    sn /= np.linalg.norm(sn, axis=1)[:, None]
    w = rng.normal(size=n_src) + 1j * rng.normal(size=n_src)
    ctr = rng.normal(size=(n_ctr, 3)) * 0.05
    tptr = np.arange(0, 2 * n_ctr + 1, 2)
    tgt = np.repeat(ctr, 2, axis=0) + rng.normal(size=(2 * n_ctr, 3)) * 0.05
    tgt[::6] = ctr[::3]                              # every third center: a target at r = 0
    tn = rng.normal(size=(2 * n_ctr, 3))
    tn /= np.linalg.norm(tn, axis=1)[:, None]
    lens = rng.integers(5, 40, size=n_ctr)
    nptr = np.concatenate([[0], np.cumsum(lens)])
    nidx = rng.integers(0, n_src, size=nptr[-1]).astype(np.int32)
    for variant in (Variant.TARGET_NORMAL_DERIV, Variant.SOURCE_NORMAL_DERIV):
        spec = KernelSpec(equation=Equation(eq), variant=variant,
                          helmholtz_k=None if eq == "laplace" else 2.3)
        cfg = TsConfig(spec, p)
        out = ts_accumulate_batch(cfg, src, w, ctr, tgt, (nptr, nidx), tgt_ptr=tptr,
                                  source_normals=sn, target_normals=tn)
        ref = oracle.ts_batch(eq, spec.variant_code, spec.helmholtz_k or 0.0, p, src, w, ctr,
                              nptr, nidx, tgt, tptr, snormals=sn, tnormals=tn)
        assert normwise(out, ref) <= (LAP_TOL if eq == "laplace" else HELM_TOL), (variant, p)


@pytest.mark.parametrize("variant", VARIANTS)
@pytest.mark.parametrize("band", [(0.05, 0.7), (0.5, 1.5), (1.2, 1.6), (0.5, 6.0)])
def test_helmholtz_sin_cos_ranges(variant, band):
    """kR inside pi/4 (narrow series), straddling it (wide series), near pi/2,
    and beyond (library sincos) -- mixed within warps -- against the oracle."""
    rng = np.random.default_rng(int(band[1] * 10))
    k = 20.0
    n_ctr, per = 96, 24
    ctr = rng.normal(size=(n_ctr, 3))
    dirs = rng.normal(size=(n_ctr * per, 3))
    dirs /= np.linalg.norm(dirs, axis=1)[:, None]
    R = rng.uniform(band[0], band[1], size=n_ctr * per) / k
    src = np.repeat(ctr, per, axis=0) + dirs * R[:, None]
    sn = rng.normal(size=src.shape)
    sn /= np.linalg.norm(sn, axis=1)[:, None]
    w = rng.normal(size=src.shape[0]) + 1j * rng.normal(size=src.shape[0])
    nptr = np.arange(0, n_ctr * per + 1, per)
    nidx = np.arange(n_ctr * per, dtype=np.int32)
    tdir = rng.normal(size=(n_ctr, 3))
    tdir /= np.linalg.norm(tdir, axis=1)[:, None]
    tgt = ctr + tdir * (0.4 * band[0] / k)
    tn = rng.normal(size=(n_ctr, 3))
    tn /= np.linalg.norm(tn, axis=1)[:, None]
    spec = KernelSpec(equation=Equation.HELMHOLTZ, variant=variant, helmholtz_k=k)
    cfg = TsConfig(spec, 10)
    out = ts_accumulate_batch(cfg, src, w, ctr, tgt, (nptr, nidx), source_normals=sn,
                              target_normals=tn)
    ref = oracle.ts_batch("helmholtz", spec.variant_code, k, 10, src, w, ctr, nptr, nidx, tgt,
                          np.arange(n_ctr + 1, dtype=np.int64), snormals=sn, tnormals=tn)
    assert normwise(out, ref) <= HELM_TOL


# --- convergence to the free-space kernel (test_tsqbx.py:93-99, 131-157) -------------
def test_accumulate_single_equals_eval_times_weight():
    rng = np.random.default_rng(4)
    c = rng.normal(size=3)
    s = c + 1.3 * rng.normal(size=3) / np.linalg.norm(rng.normal(size=3))
    s = c + (s - c) / np.linalg.norm(s - c) * 1.1
    t = c + 0.4 * (rng.normal(size=3) / np.linalg.norm(rng.normal(size=3)))
    w = 1.3 - 0.4j
    a = ts_accumulate(TsConfig(KernelSpec(), 8), s[None, :], np.array([w]), c, t)
    b = w * ts_eval(TsConfig(KernelSpec(), 8), s, c, t)
    assert a == pytest.approx(b, rel=1e-14)


def test_laplace_convergence_order():
    # fixed rho = r/R = 0.5: the truncation error decays like rho^{p+1}
    from paper_1811_01110_b200 import direct_sum
    c = np.zeros(3)
    s = np.array([0.0, 0.8, 0.6])
    t = 0.5 * np.array([0.6, -0.64, 0.48])
    exact = direct_sum(KernelSpec(), s[None], [1.0], t[None])[0]
    orders = np.arange(2, 16)
    errs = [abs(ts_eval(TsConfig(KernelSpec(), int(p)), s, c, t) - exact) / abs(exact)
            for p in orders]
    slope = np.polyfit(orders + 1, np.log(errs), 1)[0]
    assert abs(slope - math.log(0.5)) < 0.15 * abs(math.log(0.5))


def test_helmholtz_convergence_trend():
    # kR = 4: the error decreases monotonically with p towards the kernel value
    from paper_1811_01110_b200 import direct_sum
    spec = KernelSpec(equation=Equation.HELMHOLTZ, helmholtz_k=2.5)
    c = np.zeros(3)
    s = np.array([0.0, 0.0, 1.6])
    t = np.array([0.4, 0.3, 0.0])
    exact = direct_sum(spec, s[None], [1.0], t[None])[0]
    errs = [abs(ts_eval(TsConfig(spec, p), s, c, t) - exact) / abs(exact)
            for p in range(2, 20, 3)]
    assert all(b < a for a, b in zip(errs, errs[1:]))
    assert errs[-1] < 1e-8


def test_helmholtz_small_k_matches_oracle():
    # k -> 0: h_n(kR) and j_n(kr) at tiny arguments (Miller start p + 16 + ceil(kr))
    case = configs.make_case("c3", "literal", n=4096)
    spec = KernelSpec(equation=Equation.HELMHOLTZ, helmholtz_k=1e-6)
    case.cfg = TsConfig(spec, 8)
    near = build_near_lists(case.centers, case.sources, case.near_radii)
    out = ts_accumulate_batch(case.cfg, case.sources, case.weights, case.centers, case.targets,
                              near, tgt_ptr=case.tgt_ptr)
    uptr, uidx = near.to_user_csr()
    ref = oracle.ts_batch("helmholtz", 0, 1e-6, 8, case.sources, case.weights, case.centers,
                          uptr, uidx, case.targets, case.tgt_ptr)
    assert normwise(out, ref) <= HELM_TOL


def test_set_weights_reuses_the_problem():
    case = configs.make_case("c2", "literal", n=8192)
    near = build_near_lists(case.centers, case.sources, case.near_radii)
    prob = TsqbxProblem(case.cfg, case.sources, case.weights, case.centers, case.targets, near,
                        tgt_ptr=case.tgt_ptr)
    a = prob.evaluate().cpu().numpy().copy()
    prob.set_weights(2.5 * case.weights)
    b = prob.evaluate().cpu().numpy()
    assert normwise(b, 2.5 * a) <= 1e-15


@pytest.mark.gpu
def test_uniform_target_runs_flag():
    """TSQBX_FLAG_UNIFORM_TARGETS (row g owns targets [k g, k g + k), no tgt_ptr
    load) gives the same potentials as the tgt_ptr path; a ragged tgt_ptr is
    detected and keeps the tgt_ptr path."""
    case = configs.make_case("c2", "literal", n=4096)
    near = build_near_lists(case.centers, case.sources, case.near_radii)
    prob = TsqbxProblem(case.cfg, case.sources, case.weights, case.centers, case.targets,
                        near, tgt_ptr=case.tgt_ptr)
    assert prob.prep.tuni == 2
    fast = prob.evaluate(validate=True).cpu().numpy().copy()
    prob.prep.tuni = 0
    slow = prob.evaluate(validate=True).cpu().numpy()
    assert np.array_equal(fast, slow)
    ragged = case.tgt_ptr.copy()
    ragged[1] -= 1                      # center 0 one target, center 1 three
    rp = TsqbxProblem(case.cfg, case.sources, case.weights, case.centers, case.targets, near,
                      tgt_ptr=ragged)
    assert rp.prep.tuni == 0
    one = TsqbxProblem(case.cfg, case.sources, case.weights, case.centers, case.sources, near)
    assert one.prep.tuni == 1
    # three targets per center: uniform runs, but wider than a kernel pass (NT = 2),
    # so the kernels keep the tgt_ptr path; all equations and variants stay exact
    rng = np.random.default_rng(2)
    tg3 = np.repeat(case.centers, 3, axis=0) + rng.normal(scale=1e-4, size=(3 * case.n_centers, 3))
    tp3 = np.arange(case.n_centers + 1) * 3
    uptr, uidx = near.to_user_csr()
    for spec, tol in ((KernelSpec(), LAP_TOL),
                      (KernelSpec(equation=Equation.HELMHOLTZ, helmholtz_k=10.0), HELM_TOL)):
        cfg = TsConfig(spec, 8)
        p3 = TsqbxProblem(cfg, case.sources, case.weights, case.centers, tg3, near, tgt_ptr=tp3)
        assert p3.prep.tuni == 3
        got = p3.evaluate(validate=True).cpu().numpy()
        ref = oracle.ts_batch("laplace" if spec.is_laplace else "helmholtz", 0,
                              spec.helmholtz_k or 0.0, 8, case.sources, case.weights,
                              case.centers, uptr, uidx, tg3, tp3)
        assert normwise(got, ref) <= tol


@pytest.mark.gpu
def test_async_batches_on_two_streams():
    """ts_accumulate_batch(sync=False) on two streams (the overlapped e2e path):
    same potentials as the synchronous call; the screen's ValueError surfaces at
    result()."""
    case = configs.make_case("c2", "literal", n=4096)
    near = build_near_lists(case.centers, case.sources, case.near_radii)
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()  # noqa: E731
    args = (pin(case.sources), pin(case.weights), pin(case.centers), pin(case.targets), near)
    ref = ts_accumulate_batch(case.cfg, *args, tgt_ptr=pin(case.tgt_ptr))
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    outs = [torch.empty(case.n_targets, dtype=torch.complex128).pin_memory() for _ in range(2)]
    pend = []
    for i in range(4):
        with torch.cuda.stream(streams[i % 2]):
            if len(pend) >= 2:
                got = pend.pop(0).result()
                assert np.array_equal(got.numpy(), ref)
            pend.append(ts_accumulate_batch(case.cfg, *args, tgt_ptr=pin(case.tgt_ptr),
                                            out=outs[i % 2], sync=False))
    for p in pend:
        assert np.array_equal(p.result().numpy(), ref)
    # numpy result when no `out` is given
    p = ts_accumulate_batch(case.cfg, *args, tgt_ptr=pin(case.tgt_ptr), sync=False)
    assert np.array_equal(p.result(), ref)
    # a separation violation is reported by result()
    src = np.array([[0.0, 0.0, 1.0], [0.0, 0.0, 0.2]])
    w = np.ones(2, complex)
    p = ts_accumulate_batch(case.cfg, src, w, np.zeros((1, 3)), np.array([[0.0, 0.0, 0.5]]),
                            (np.array([0, 2]), np.array([0, 1], np.int32)), sync=False)
    with pytest.raises(ValueError, match="separation violation for source 1"):
        p.result()


@pytest.mark.gpu
@pytest.mark.parametrize("pinned", [False, True])
def test_near_field_potentials_matches_oracle(pinned):
    """geometry -> device near lists -> potentials in one call (payload copied on a
    side stream while the lists are built) equals the oracle on the oracle's lists."""
    from paper_1811_01110_b200.tsqbx import near_field_potentials
    case = configs.make_case("c3", "literal", n=4096)
    conv = ((lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()) if pinned
            else (lambda a: a))
    got = near_field_potentials(case.cfg, conv(case.sources), conv(case.weights),
                                conv(case.centers), conv(case.near_radii), conv(case.targets),
                                tgt_ptr=conv(case.tgt_ptr))
    got = got.numpy() if isinstance(got, torch.Tensor) else got
    ptr, idx = oracle.near_csr(case.centers, case.near_radii, case.sources)
    ref = oracle.ts_batch("helmholtz", 0, case.cfg.spec.helmholtz_k, case.cfg.p_qbx,
                          case.sources, case.weights, case.centers, ptr, idx, case.targets,
                          case.tgt_ptr)
    assert normwise(got, ref) <= HELM_TOL


@pytest.mark.gpu
@pytest.mark.parametrize("name,variant", [("c2", Variant.SINGLE_LAYER), ("c3", Variant.SINGLE_LAYER),
                                          ("c2", Variant.TARGET_NORMAL_DERIV),
                                          ("c3", Variant.SOURCE_NORMAL_DERIV)])
def test_row_range_launches_match_full(name, variant):
    """The multi-GPU shard path: launches over row ranges (multiples of 32, each
    with its own row split and the tgt_ptr kernels), in user order and in
    processing order with an output offset, reproduce the whole-problem
    evaluation (which takes the uniform-target kernels)."""
    case = configs.make_case(name, "literal", n=8192)
    sp = case.cfg.spec
    cfg = TsConfig(KernelSpec(equation=sp.equation, variant=variant, helmholtz_k=sp.helmholtz_k),
                   case.cfg.p_qbx)
    tnrm = np.repeat(case.normals, np.diff(case.tgt_ptr), axis=0)
    near = build_near_lists(case.centers, case.sources, case.near_radii)
    prob = TsqbxProblem(cfg, case.sources, case.weights, case.centers, case.targets, near,
                        tgt_ptr=case.tgt_ptr, source_normals=case.normals, target_normals=tnrm)
    prep = prob.prep
    assert prep.tuni == 2
    full = prob.evaluate().clone()
    tol = LAP_TOL if sp.is_laplace else HELM_TOL
    bounds = [0, 2048, 5120, prep.n_ctr]
    out = torch.zeros_like(full)
    for g0, g1 in zip(bounds[:-1], bounds[1:]):
        prep.launch(torch.view_as_real(out), False, rows=(g0, g1))
    assert normwise(out.cpu().numpy(), full.cpu().numpy()) <= tol
    # processing order, each range into its own buffer at offset tptr[g0]
    tptr = prep.tptr.cpu().numpy()
    proc = torch.zeros_like(full)
    for g0, g1 in zip(bounds[:-1], bounds[1:]):
        t0, t1 = int(tptr[g0]), int(tptr[g1])
        part = torch.zeros(t1 - t0, dtype=full.dtype, device=full.device)
        prep.launch(torch.view_as_real(part), False, rows=(g0, g1), out_offset=t0,
                    user_order=False)
        proc[t0:t1] = part
    user = torch.empty_like(proc)
    user[prep.tidx] = proc
    assert normwise(user.cpu().numpy(), full.cpu().numpy()) <= tol
