"""The one-shot fused near field (``tsqbx_eval_fused``, csrc/fused.cu): each
warp sweeps the near lists of 32 rows into a scratch slice and evaluates them
at once.  ``near_field_potentials(..., fused=True)`` takes it; these tests compare it
with the oracle (``_core.pyx:205-398`` restated, on the oracle's own near
lists), with the two-step path (``fused=False``), and check the fallbacks: a
row longer than the scratch slice, and a validation error (the reference's
message).  Tolerances: 1e-12 Laplace, 1e-10 Helmholtz (north_star)."""

import numpy as np
import pytest

import oracle
from paper_1811_01110_b200 import KernelSpec, TsConfig, configs, near_field_potentials

pytestmark = pytest.mark.gpu


def normwise(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.max(np.abs(a - b)) / max(1e-300, np.max(np.abs(b))))


def _oracle(case):
    spec = case.cfg.spec
    ptr, idx = oracle.near_csr(case.centers, case.near_radii, case.sources)
    return oracle.ts_batch("laplace" if spec.is_laplace else "helmholtz", 0,
                           spec.helmholtz_k or 0.0, case.cfg.p_qbx, case.sources, case.weights,
                           case.centers, ptr, idx, case.targets, case.tgt_ptr)


CASES = [("c1", "literal", {}), ("c1", "dense", {}), ("c2", "literal", {"n": 65536}),
         ("c2", "dense", {"n": 32768}), ("c3", "literal", {"n": 65536}),
         ("c3", "dense", {"n": 32768}), ("c4", "literal", {"n": 65536}),
         ("c4", "dense", {"n": 32768}), ("c5", "literal", {"n": 32768, "spheres": 4}),
         ("c5", "dense", {"n": 16384, "spheres": 4})]


@pytest.mark.parametrize("name,preset,kw", CASES)
def test_fused_matches_oracle_and_two_step(name, preset, kw):
    case = configs.make_case(name, preset, **kw)
    tol = 1e-12 if case.cfg.spec.is_laplace else 1e-10
    args = (case.cfg, case.sources, case.weights, case.centers, case.near_radii, case.targets)
    got = near_field_potentials(*args, tgt_ptr=case.tgt_ptr, fused=True)
    two = near_field_potentials(*args, tgt_ptr=case.tgt_ptr, fused=False)
    ref = _oracle(case)
    e_ref, e_two = normwise(got, ref), normwise(got, two)
    print(f"{name}/{preset} {kw}: fused vs oracle {e_ref:.2e}, vs two-step {e_two:.2e}")
    assert e_ref <= tol and e_two <= tol
    # no validation (the driver path) gives the same potentials
    nov = near_field_potentials(*args, tgt_ptr=case.tgt_ptr, validate=False, fused=True)
    assert normwise(nov, got) <= tol


def test_fused_row_overflow_falls_back(monkeypatch):
    """Rows longer than the scratch slice (row_cap) take the two-step path."""
    case = configs.make_case("c2", "dense", n=8192)
    monkeypatch.setenv("GIGAQBX_FUSED_ROW_CAP", "16")
    args = (case.cfg, case.sources, case.weights, case.centers, case.near_radii, case.targets)
    got = near_field_potentials(*args, tgt_ptr=case.tgt_ptr, fused=True)
    assert normwise(got, _oracle(case)) <= 1e-12


def test_fused_validation_error_message():
    """A target outside a center's separation radius is reported exactly as the
    reference's _prep does (tsqbx.py:48-51), via the two-step re-run."""
    case = configs.make_case("c1", "literal")
    tgt = case.targets.copy()
    tgt[100] = case.centers[100] + 10.0 * (tgt[100] - case.centers[100])
    with pytest.raises(ValueError, match="separation violation"):
        near_field_potentials(case.cfg, case.sources, case.weights, case.centers,
                              case.near_radii, tgt, fused=True)


def test_fused_scalar_radius_and_empty_rows():
    """A scalar near radius and centers with no near source (zero potentials)."""
    rng = np.random.default_rng(5)
    src = rng.normal(size=(5000, 3))
    src /= np.linalg.norm(src, axis=1)[:, None]
    ctr = 0.9 * src[:3000] + 0.05 * rng.normal(size=(3000, 3))
    ctr[::7] = 0.2 * rng.normal(size=(ctr[::7].shape[0], 3))      # far from the shell: empty
    tgt = ctr + 1e-3
    w = rng.uniform(0.5, 1.5, 5000).astype(np.complex128)
    cfg = TsConfig(KernelSpec(), 6)
    got = near_field_potentials(cfg, src, w, ctr, 0.15, tgt, fused=True)
    ptr, idx = oracle.near_csr(ctr, np.full(3000, 0.15), src)
    ref = oracle.ts_batch("laplace", 0, 0.0, 6, src, w, ctr, ptr, idx, tgt,
                          np.arange(3001, dtype=np.int64))
    assert (np.diff(ptr) == 0).any()
    assert normwise(got, ref) <= 1e-12
    assert np.all(got[np.diff(ptr) == 0] == 0)
