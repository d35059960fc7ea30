"""Parity of the exact kernels the bench times, on the full BASELINE outputs.

bench.py's device-resident step is ``TsqbxProblem(case..., tgt_ptr=case.tgt_ptr)``
followed by ``evaluate()`` -- no validation, the uniform-target SELL
instances (``laplace_sell_kernel<P, 2, VAL=0, S, UNI>``,
``helmholtz_sell_kernel<P, NT, VAL=0, UNI>``) and the auto row split.  These
tests build the problem the same way, run the same ``evaluate()`` and compare
every potential with the oracle (``oracle.ts_batch``: the C restatement of
``_core.pyx:205-419``, OpenMP over centers), printing the normwise error.
C5 dense (1.69 G pairs) is checked on a seeded 2 % subset of the full-size
launch (>= 1 % for C4/C5).  The reference-named C entry points
(``tsqbx_eval_laplace/helmholtz``, ``tsqbx_p2p_laplace/helmholtz``, what
INTEGRATION.md's ctypes stub binds) are called directly through ctypes.

Tolerances (north_star): normwise relative l-inf <= 1e-12 Laplace, <= 1e-10
Helmholtz.
"""

import numpy as np
import pytest
import torch

import oracle
from paper_1811_01110_b200 import (KernelSpec, TsConfig, TsqbxProblem, _lib, build_near_lists,
                                   configs)
from paper_1811_01110_b200.kernels import Equation

pytestmark = pytest.mark.gpu

LAP_TOL = 1e-12
HELM_TOL = 1e-10


def normwise(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.max(np.abs(a - b)) / max(1e-300, np.max(np.abs(b))))


def _bench_problem(case):
    """bench.measure_case's construction (device geometry for the build, host
    arrays for the problem, tgt_ptr given so the uniform runs are detected)."""
    dev = torch.device("cuda", torch.cuda.current_device())
    near = build_near_lists(torch.as_tensor(case.centers, device=dev),
                            torch.as_tensor(case.sources, device=dev),
                            torch.as_tensor(case.near_radii, device=dev), dev)
    prob = TsqbxProblem(case.cfg, case.sources, case.weights, case.centers, case.targets, near,
                        tgt_ptr=case.tgt_ptr, device=dev)
    return prob, near


def _expected_instance(case, prob):
    """The template instance bench.py times: uniform target runs, SELL layout,
    Laplace rows split over 2 lanes on the dense presets."""
    tpc = case.n_targets // case.n_centers
    assert prob.layout == "sell"
    assert prob.prep.tuni == tpc, (prob.prep.tuni, tpc)
    if case.cfg.spec.is_laplace:
        assert prob.group_lanes == (1 if case.preset == "literal" else 2)
        assert not prob.prep.flat          # the short-list kernel is opt-in (GIGAQBX_FLAT=1)
    else:
        assert prob.group_lanes == 1
        assert not prob.prep.flat


def _oracle(case, uptr, uidx, sel=None):
    spec = case.cfg.spec
    eq = "laplace" if spec.is_laplace else "helmholtz"
    if sel is None:
        return oracle.ts_batch(eq, 0, spec.helmholtz_k or 0.0, case.cfg.p_qbx, case.sources,
                               case.weights, case.centers, uptr, uidx, case.targets,
                               case.tgt_ptr)
    lens = np.diff(uptr)[sel]
    sptr = np.concatenate([[0], np.cumsum(lens)])
    sidx = np.concatenate([uidx[uptr[c]:uptr[c + 1]] for c in sel])
    tl = np.diff(case.tgt_ptr)[sel]
    tptr = np.concatenate([[0], np.cumsum(tl)])
    tsel = np.concatenate([np.arange(case.tgt_ptr[c], case.tgt_ptr[c + 1]) for c in sel])
    return oracle.ts_batch(eq, 0, spec.helmholtz_k or 0.0, case.cfg.p_qbx, case.sources,
                           case.weights, case.centers[sel], sptr, sidx, case.targets[tsel],
                           tptr), tsel


@pytest.mark.parametrize("name,preset", [("c2", "literal"), ("c2", "dense"), ("c3", "literal"),
                                         ("c3", "dense"), ("c4", "literal"), ("c4", "dense"),
                                         ("c5", "literal")])
def test_timed_kernel_full_output(name, preset):
    case = configs.make_case(name, preset)
    prob, near = _bench_problem(case)
    _expected_instance(case, prob)
    out = prob.evaluate().cpu().numpy()          # validate=False: the timed launch
    uptr, uidx = near.to_user_csr()
    ref = _oracle(case, uptr, uidx)
    err = normwise(out, ref)
    tol = LAP_TOL if case.cfg.spec.is_laplace else HELM_TOL
    print(f"\n{name}/{preset}: {prob.pair_count()} pairs, {case.n_targets} targets (all), "
          f"normwise err {err:.3e} (tol {tol:g})")
    assert err <= tol
    # the validated launch (another template instance) agrees with it
    outv = prob.evaluate(validate=True).cpu().numpy()
    assert normwise(outv, ref) <= tol


def test_timed_kernel_c5_dense_subset():
    """C5 dense at full size: the timed launch, 2 % seeded subset of its
    potentials (rows cut out of the device lists on the device)."""
    case = configs.make_case("c5", "dense")
    prob, near = _bench_problem(case)
    _expected_instance(case, prob)
    out = prob.evaluate().cpu().numpy()
    rng = np.random.default_rng(21)
    sel = np.sort(rng.choice(case.n_centers, case.n_centers // 50, replace=False))
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
    spec = case.cfg.spec
    ref = oracle.ts_batch("helmholtz", 0, spec.helmholtz_k, case.cfg.p_qbx, case.sources,
                          case.weights, case.centers[sel], sptr, sidx, case.targets[sel],
                          np.arange(len(sel) + 1, dtype=np.int64))
    err = normwise(out[sel], ref)
    print(f"\nc5/dense: {len(sel)} of {case.n_centers} targets, {int(sptr[-1])} pairs, "
          f"normwise err {err:.3e}")
    assert sptr[-1] > 30_000_000
    assert err <= HELM_TOL


# --- the reference-named C entry points (INTEGRATION.md's ctypes stub) ------------
def _dev(a, dtype=torch.float64):
    return torch.as_tensor(np.ascontiguousarray(a), dtype=dtype, device="cuda")


def _ptr(t):
    return None if t is None else t.data_ptr()


@pytest.mark.parametrize("variant", [0, 1, 2])
@pytest.mark.parametrize("eq", ["laplace", "helmholtz"])
@pytest.mark.parametrize("validate", [False, True])
def test_reference_named_eval_entry_points(eq, variant, validate):
    case = configs.make_case("c2", "literal", n=8192)
    L = _lib.load()
    rng = np.random.default_rng(variant)
    uptr, uidx = oracle.near_csr(case.centers, case.near_radii, case.sources)
    w = (case.weights if eq == "laplace"
         else rng.uniform(-1, 1, case.n_sources) + 1j * rng.uniform(-1, 1, case.n_sources))
    tn = case.targets * 0 + case.normals[0]
    p, k = (8, 0.0) if eq == "laplace" else (8, 10.0)
    src, ww = _dev(case.sources), _dev(np.stack([w.real, w.imag], 1))
    sn = _dev(case.normals) if variant == 2 else None
    tnd = _dev(tn) if variant == 1 else None
    ctr, tgt = _dev(case.centers), _dev(case.targets)
    nptr, nidx = _dev(uptr, torch.int64), _dev(uidx, torch.int32)
    tptr = _dev(case.tgt_ptr, torch.int64)
    eqc = _lib.EQ_LAPLACE if eq == "laplace" else _lib.EQ_HELMHOLTZ
    wsb = int(L.tsqbx_user_workspace_bytes(eqc, variant, p, case.n_sources, case.n_targets))
    ws = torch.empty(max(wsb, 1), dtype=torch.uint8, device="cuda")
    out = torch.empty(case.n_targets, 2, dtype=torch.float64, device="cuda")
    err = torch.empty(1, dtype=torch.int64, device="cuda")
    flags = _lib.FLAG_VALIDATE if validate else 0
    st = torch.cuda.current_stream().cuda_stream
    common = (_ptr(src), _ptr(ww), _ptr(sn), case.n_sources, _ptr(ctr), case.n_centers,
              _ptr(nptr), _ptr(nidx), _ptr(tgt), _ptr(tnd), _ptr(tptr), case.n_targets, flags,
              _ptr(ws), wsb, _ptr(out), _ptr(err), st)
    if eq == "laplace":
        rc = L.tsqbx_eval_laplace(variant, p, *common)
    else:
        rc = L.tsqbx_eval_helmholtz(variant, k, p, *common)
    assert rc == 0, L.tsqbx_last_error()
    got = out.cpu().numpy()
    got = got[:, 0] + 1j * got[:, 1]
    ref = oracle.ts_batch(eq, variant, k, p, case.sources, w, case.centers, uptr, uidx,
                          case.targets, case.tgt_ptr,
                          snormals=case.normals if variant == 2 else None,
                          tnormals=tn if variant == 1 else None)
    e = normwise(got, ref)
    print(f"\ntsqbx_eval_{eq} variant {variant} validate {validate}: normwise err {e:.3e}")
    assert e <= (LAP_TOL if eq == "laplace" else HELM_TOL)
    if validate:
        assert int(err.item()) == _lib.ERR_KEY_NONE


@pytest.mark.parametrize("variant", [0, 1, 2])
@pytest.mark.parametrize("eq", ["laplace", "helmholtz"])
def test_reference_named_p2p_entry_points(eq, variant):
    L = _lib.load()
    rng = np.random.default_rng(3 + variant)
    n, m = 5000, 777
    s = rng.normal(size=(n, 3))
    t = rng.normal(size=(m, 3)) + 0.01
    w = rng.normal(size=n) + 1j * rng.normal(size=n)
    sn = rng.normal(size=(n, 3))
    sn /= np.linalg.norm(sn, axis=1)[:, None]
    tn = rng.normal(size=(m, 3))
    tn /= np.linalg.norm(tn, axis=1)[:, None]
    k = 0.0 if eq == "laplace" else 7.5
    snd = _dev(sn) if variant == 2 else None
    tnd = _dev(tn) if variant == 1 else None
    wsb = int(L.tsqbx_p2p_user_workspace_bytes(variant, n, m))
    ws = torch.empty(max(wsb, 1), dtype=torch.uint8, device="cuda")
    out = torch.empty(m, 2, dtype=torch.float64, device="cuda")
    err = torch.empty(1, dtype=torch.int64, device="cuda")
    src, ww, tgt = _dev(s), _dev(np.stack([w.real, w.imag], 1)), _dev(t)
    st = torch.cuda.current_stream().cuda_stream
    tail = (_ptr(src), _ptr(ww), _ptr(snd), n, _ptr(tgt), _ptr(tnd), m, _lib.FLAG_VALIDATE,
            _ptr(ws), wsb, _ptr(out), _ptr(err), st)
    rc = (L.tsqbx_p2p_laplace(variant, *tail) if eq == "laplace"
          else L.tsqbx_p2p_helmholtz(variant, k, *tail))
    assert rc == 0, L.tsqbx_last_error()
    got = out.cpu().numpy()
    got = got[:, 0] + 1j * got[:, 1]
    ref = oracle.p2p(eq, variant, k, s, w, t, snormals=sn if variant == 2 else None,
                     tnormals=tn if variant == 1 else None)
    e = normwise(got, ref)
    print(f"\ntsqbx_p2p_{eq} variant {variant}: normwise err {e:.3e}")
    assert e <= (LAP_TOL if eq == "laplace" else HELM_TOL)
    assert int(err.item()) == _lib.ERR_KEY_NONE


@pytest.mark.parametrize("claimed", ["narrow", "wide"])
def test_helmholtz_kr_hint_violated_is_recomputed(claimed):
    """The one-target long-row Helmholtz kernel picks its e^{ikR} series outside
    the row loop from the k R hint (FLAG_KR_NARROW / FLAG_KR_WIDE) and checks the
    hint per row (largest R^2 on the integer pipe): rows that violate it are
    recomputed on the generic path.  A near list that claims a far too small
    radius must still give the oracle's potentials."""
    import math
    case = configs.make_case("c5", "dense", n=8192, spheres=2)
    k = 60.0                     # k R up to ~2.4: beyond both series' intervals on many rows
    cfg = TsConfig(KernelSpec(equation=Equation.HELMHOLTZ, helmholtz_k=k), case.cfg.p_qbx)
    near = build_near_lists(case.centers, case.sources, case.near_radii)
    true_kr = k * near.max_radius
    assert true_kr > math.pi / 2 and near.mean_len >= 48
    near.max_radius = (0.5 if claimed == "narrow" else 1.5) / k      # k R "<= pi/4" / "<= pi/2"
    prob = TsqbxProblem(cfg, case.sources, case.weights, case.centers, case.targets, near,
                        tgt_ptr=case.tgt_ptr)
    assert prob.prep.kr_flag != 0 and prob.prep.tuni == 1
    got = prob.evaluate(validate=False).cpu().numpy()
    uptr, uidx = near.to_user_csr()
    ref = oracle.ts_batch("helmholtz", 0, k, cfg.p_qbx, case.sources, case.weights, case.centers,
                          uptr, uidx, case.targets, case.tgt_ptr)
    err = float(np.max(np.abs(got - ref)) / np.max(np.abs(ref)))
    print(f"kr hint {claimed} violated (true k R {true_kr:.2f}): normwise {err:.2e}")
    assert err <= 1e-10
