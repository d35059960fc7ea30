"""Malformed caller inputs raise ValueError instead of reading or writing
outside the device arrays, and ``device=`` selects the GPU a call runs on."""

import numpy as np
import pytest
import torch

from paper_1811_01110_b200 import TsqbxProblem, build_near_lists, configs, ts_accumulate_batch
from paper_1811_01110_b200.nearlist import NearLists

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def case():
    return configs.make_case("c2", "literal", n=4096)


def _bad_tptrs(case):
    good = np.asarray(case.tgt_ptr, dtype=np.int64)
    a = good.copy(); a[0] = 1                                       # noqa: E702
    b = good.copy(); b[-1] = case.n_targets + 7                     # noqa: E702
    c = good.copy(); c[10] = c[12] + 1                              # noqa: E702  decreasing
    d = good.copy(); d[5] = 10 * case.n_targets                     # noqa: E702  past the end
    e = good.copy(); e[-1] = case.n_targets - 1                     # noqa: E702
    return [a, b, c, d, e]


@pytest.mark.parametrize("which", range(5))
def test_malformed_tgt_ptr_morton_path(case, which):
    near = build_near_lists(case.centers, case.sources, case.near_radii)
    bad = _bad_tptrs(case)[which]
    with pytest.raises(ValueError, match="tgt_ptr"):
        ts_accumulate_batch(case.cfg, case.sources, case.weights, case.centers, case.targets,
                            near, tgt_ptr=bad)
    with pytest.raises(ValueError, match="tgt_ptr"):
        ts_accumulate_batch(case.cfg, case.sources, case.weights, case.centers, case.targets,
                            near, tgt_ptr=bad, validate=False)
    with pytest.raises(ValueError, match="tgt_ptr"):
        TsqbxProblem(case.cfg, case.sources, case.weights, case.centers, case.targets, near,
                     tgt_ptr=bad)
    # the device is still usable and a good call still agrees
    torch.cuda.synchronize()
    ok = ts_accumulate_batch(case.cfg, case.sources, case.weights, case.centers, case.targets,
                             near, tgt_ptr=case.tgt_ptr)
    assert np.all(np.isfinite(ok))


@pytest.mark.parametrize("which", range(5))
def test_malformed_tgt_ptr_user_csr_path(case, which):
    import oracle
    uptr, uidx = oracle.near_csr(case.centers, case.near_radii, case.sources)
    bad = _bad_tptrs(case)[which]
    with pytest.raises(ValueError, match="tgt_ptr"):
        ts_accumulate_batch(case.cfg, case.sources, case.weights, case.centers, case.targets,
                            (uptr, uidx), tgt_ptr=bad)


def test_malformed_user_csr(case):
    import oracle
    uptr, uidx = oracle.near_csr(case.centers, case.near_radii, case.sources)
    args = (case.cfg, case.sources, case.weights, case.centers, case.targets)
    p = uptr.copy(); p[-1] += 3                                      # noqa: E702
    with pytest.raises(ValueError, match="near-list ptr"):
        ts_accumulate_batch(*args, (p, uidx), tgt_ptr=case.tgt_ptr)
    p = uptr.copy(); p[3] = p[5] + 1                                 # noqa: E702
    with pytest.raises(ValueError, match="near-list ptr"):
        ts_accumulate_batch(*args, (p, uidx), tgt_ptr=case.tgt_ptr)
    i = uidx.copy(); i[17] = case.n_sources                          # noqa: E702
    with pytest.raises(ValueError, match="near-list indices"):
        ts_accumulate_batch(*args, (uptr, i), tgt_ptr=case.tgt_ptr)
    i = uidx.copy(); i[0] = -1                                       # noqa: E702
    with pytest.raises(ValueError, match="near-list indices"):
        NearLists.from_user_csr(uptr, i, case.n_sources)


def test_missing_tgt_ptr_needs_one_target_per_center(case):
    near = build_near_lists(case.centers, case.sources, case.near_radii)
    # case has two targets per center: without tgt_ptr that is an error everywhere
    with pytest.raises(ValueError, match="tgt_ptr is required"):
        TsqbxProblem(case.cfg, case.sources, case.weights, case.centers, case.targets, near)
    with pytest.raises(ValueError, match="tgt_ptr is required"):
        ts_accumulate_batch(case.cfg, case.sources, case.weights, case.centers, case.targets,
                            near)


def test_explicit_device_argument(case):
    dev = torch.device("cuda", torch.cuda.device_count() - 1)
    near = build_near_lists(case.centers, case.sources, case.near_radii, device=dev)
    assert near.ptr.device == dev
    out = ts_accumulate_batch(case.cfg, torch.as_tensor(case.sources, device=dev),
                              torch.as_tensor(case.weights, device=dev),
                              torch.as_tensor(case.centers, device=dev),
                              torch.as_tensor(case.targets, device=dev), near,
                              tgt_ptr=case.tgt_ptr, device=dev)
    assert out.device == dev
    ref = ts_accumulate_batch(case.cfg, case.sources, case.weights, case.centers, case.targets,
                              build_near_lists(case.centers, case.sources, case.near_radii),
                              tgt_ptr=case.tgt_ptr)
    assert np.allclose(out.cpu().numpy(), ref, rtol=0, atol=1e-13 * np.abs(ref).max())


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs two GPUs")
def test_non_current_device(case):
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 1)
    near = build_near_lists(case.centers, case.sources, case.near_radii, device=dev)
    prob = TsqbxProblem(case.cfg, case.sources, case.weights, case.centers, case.targets, near,
                        tgt_ptr=case.tgt_ptr, device=dev)
    out = prob.evaluate().cpu().numpy()
    assert torch.cuda.current_device() == 0
    ref = ts_accumulate_batch(case.cfg, case.sources, case.weights, case.centers, case.targets,
                              build_near_lists(case.centers, case.sources, case.near_radii),
                              tgt_ptr=case.tgt_ptr)
    assert np.allclose(out, ref, rtol=0, atol=1e-13 * np.abs(ref).max())
