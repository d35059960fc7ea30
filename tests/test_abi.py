"""CPU-side checks of the C ABI library and the host logic (no GPU needed)."""

import ctypes
import os
import re

import numpy as np
import pytest
import torch

from paper_1811_01110_b200 import _lib, configs, geometry, tsqbx
from paper_1811_01110_b200.kernels import Equation, KernelSpec, Variant
from paper_1811_01110_b200.nearlist import NearLists

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include",
                      "tsqbx.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^[A-Za-z_][\w\s\*]*?\b(tsqbx_\w+)\s*\(", text, re.M)))


def test_library_exports_every_declared_symbol():
    L = _lib.load()
    syms = declared_symbols()
    assert len(syms) >= 14
    for s in syms:
        assert hasattr(L, s), s
    assert set(syms) == set(_lib.SIGNATURES), "ctypes table out of sync with include/tsqbx.h"


def test_abi_queries_without_gpu():
    L = _lib.load()
    ver = int(re.search(r"#define TSQBX_ABI_VERSION (\d+)", open(HEADER).read()).group(1))
    assert L.tsqbx_abi_version() == ver
    assert L.tsqbx_packed_doubles(10, 0) == 56 and L.tsqbx_packed_doubles(10, 1) == 96
    assert L.tsqbx_eval_workspace_bytes(_lib.EQ_LAPLACE, 0, 8, 100) == 0
    assert L.tsqbx_eval_workspace_bytes(_lib.EQ_HELMHOLTZ, 0, 8, 100) >= 100 * 9 * 8
    assert L.tsqbx_near_workspace_bytes(1000, 2000) > 2000 * 32
    assert L.tsqbx_near_workspace_bytes(-1, 0) == -1


def test_abi_rejects_bad_arguments_without_launching():
    L = _lib.load()
    rc = L.tsqbx_eval_packed(7, 0, 0.0, 4, None, 0, 0, None, 0, None, None, None, None, None,
                             None, None, 0, None, 0, 0, 0, 8, None, 0, None, None, None)
    assert rc == _lib.ERR_ARGUMENT and "equation" in _lib.last_error()
    rc = L.tsqbx_eval_packed(1, 0, -1.0, 4, None, 0, 0, None, 0, None, None, None, None, None,
                             None, None, 0, None, 0, 0, 0, 8, None, 0, None, None, None)
    assert rc == _lib.ERR_ARGUMENT and "k > 0" in _lib.last_error()
    rc = L.tsqbx_eval_packed(0, 0, 0.0, 65, None, 0, 0, None, 0, None, None, None, None, None,
                             None, None, 0, None, 0, 0, 0, 8, None, 0, None, None, None)
    assert rc == _lib.ERR_ARGUMENT
    rc = L.tsqbx_eval_packed(0, 2, 0.0, 4, None, 0, 0, None, 0, None, None, None, None, None,
                             None, None, 0, None, 0, 0, 0, 8, None, 0, None, None, None)
    assert rc == _lib.ERR_ARGUMENT and "normals" in _lib.last_error()


def test_product_fails_loudly_without_gpu():
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    cfg = tsqbx.TsConfig(KernelSpec(), 4)
    with pytest.raises(RuntimeError, match="CUDA device"):
        tsqbx.ts_eval(cfg, [0, 0, 1.0], np.zeros(3), [0, 0, 0.5])


def test_config_validation_mirrors_reference():
    with pytest.raises(ValueError):
        tsqbx.TsConfig(KernelSpec(), -1)
    with pytest.raises(ValueError):
        KernelSpec(equation=Equation.HELMHOLTZ)
    with pytest.raises(ValueError):
        KernelSpec(helmholtz_k=1.0)
    s = KernelSpec(variant=Variant.SOURCE_NORMAL_DERIV)
    assert s.variant_code == 2 and s.needs_source_normals and not s.needs_target_normals


def test_group_lanes_heuristic(monkeypatch):
    monkeypatch.delenv("GIGAQBX_GROUP_LANES", raising=False)
    assert tsqbx.pick_group_lanes(200) == 4
    assert tsqbx.pick_group_lanes(12) == 1
    assert tsqbx.pick_group_lanes(4096) == 32
    monkeypatch.setenv("GIGAQBX_GROUP_LANES", "16")
    assert tsqbx.pick_group_lanes(200) == 16


def test_near_lists_user_export_roundtrip():
    # processing order g -> user center order[g]; sorted source s -> user perm[s]
    ptr = torch.tensor([0, 2, 3, 3, 6])
    idx = torch.tensor([0, 1, 2, 0, 1, 2], dtype=torch.int32)
    perm = torch.tensor([2, 0, 1], dtype=torch.int32)
    order = torch.tensor([3, 1, 0, 2], dtype=torch.int32)
    nl = NearLists(n_ctr=4, n_src=3, n_pairs=6, ptr=ptr, csr_idx=idx, src_perm=perm,
                   ctr_order=order)
    uptr, uidx = nl.to_user_csr()
    assert uptr.tolist() == [0, 0, 1, 4, 6]
    rows = [uidx[uptr[c]:uptr[c + 1]].tolist() for c in range(4)]
    assert rows == [[], [1], [2, 0, 1], [2, 0]]


def test_place_qbx_centers_matches_reference_semantics():
    y, n = geometry.fibonacci_sphere(64)
    disc = geometry.point_cloud_discretization(y, n, np.ones(64), 0.2)
    cs = geometry.place_qbx_centers(disc, -1, 0.5)
    assert np.allclose(cs.centers, y - 0.1 * n) and np.all(cs.radii == 0.1)
    with pytest.raises(ValueError):
        geometry.place_qbx_centers(disc, 0, 0.5)
    with pytest.raises(ValueError):
        geometry.place_qbx_centers(disc, 1, 1.5)


def test_configs_shapes_and_rng_order():
    c2 = configs.make_case("c2", "literal", n=512)
    c3 = configs.make_case("c3", "literal", n=512)
    assert c2.n_targets == 1024 and np.array_equal(c2.targets, c3.targets)
    assert np.all(c2.weights.imag == 0) and np.any(c3.weights.imag != 0)
    r_off = np.linalg.norm(c2.targets[1::2] - c2.centers, axis=1)
    assert np.allclose(r_off, 0.5 * c2.expansion_radii)
    c5 = configs.make_case("c5", "literal", n=256, spheres=3)
    assert c5.n_sources == 768 and c5.cfg.p_qbx == 10 and c5.cfg.spec.helmholtz_k == 20.0
    c4 = configs.make_case("c4", "literal", n=4096)
    assert c4.cfg.p_qbx == 12 and c4.n_targets == 4096
    assert configs.algorithmic_flops_per_pair(c2.cfg.spec, 8) == 73
    assert configs.algorithmic_flops_per_pair(c3.cfg.spec, 8) == 142
