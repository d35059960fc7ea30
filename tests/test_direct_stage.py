"""The driver's direct stages (driver.py:197-228) batched: host logic and the
oracle against the reference-generated fixture (tests/golden/direct_stage.npz,
the reference's own tree + interaction lists + compiled core), and the GPU
path (DirectStage) against the same fixture."""

import os

import numpy as np
import pytest

import oracle
from paper_1811_01110_b200.direct_stage import CENTERS, SOURCES, TARGETS, _owner_rows

LISTS = ("list1", "list3close", "list4close")
KERNELS = {"lap_s": ("laplace", 0, None, 4), "lap_d": ("laplace", 2, None, 6),
           "helm_sp": ("helmholtz", 1, 1.3, 5)}


def normwise(a, b):
    return float(np.max(np.abs(a - b)) / max(1e-300, np.max(np.abs(b))))


@pytest.fixture(scope="module")
def g(golden_dir):
    return dict(np.load(os.path.join(golden_dir, "direct_stage.npz")))


def expand(g, lname, row_box):
    """Host restatement of tsqbx_box_rows (_gather_sources, driver.py:109-113)."""
    st, fl = g[f"{lname}_starts"], g[f"{lname}_flat"]
    s0, s1 = g["owned_start"][:, SOURCES], g["owned_end"][:, SOURCES]
    ptr, idx = [0], []
    for b in row_box:
        if b >= 0:
            for d in fl[st[b]:st[b + 1]]:
                idx.extend(range(s0[d], s1[d]))
        ptr.append(len(idx))
    return np.array(ptr, np.int64), np.array(idx, np.int32)


def rows_of(g):
    tb = np.zeros(g["owned_start"].shape[0], bool)
    tb[g["target_boxes"]] = True
    c_start, c_box = _owner_rows(g["owned_start"], g["owned_end"], CENTERS,
                                 g["qcenters"].shape[0], tb)
    t_start, t_box = _owner_rows(g["owned_start"], g["owned_end"], TARGETS,
                                 g["conv"].shape[0], tb)
    return np.repeat(c_box, np.diff(c_start)), t_start, t_box


def test_owner_rows_partition(g):
    center_box, t_start, t_box = rows_of(g)
    assert center_box.shape[0] == g["qcenters"].shape[0]
    assert t_start[0] == 0 and t_start[-1] == g["conv"].shape[0]
    assert np.all(np.diff(t_start) > 0)
    with pytest.raises(ValueError, match="partition"):
        bad_end = g["owned_end"].copy()
        bad_end[np.argmax(bad_end[:, TARGETS] > g["owned_start"][:, TARGETS]), TARGETS] -= 1
        _owner_rows(g["owned_start"], bad_end, TARGETS, g["conv"].shape[0],
                    np.ones(bad_end.shape[0], bool))


@pytest.mark.parametrize("lname", LISTS)
def test_oracle_replays_reference_direct_stage(g, lname):
    center_box, t_start, t_box = rows_of(g)
    ptr, idx = expand(g, lname, center_box)
    tptr, tidx = expand(g, lname, t_box)
    for kname, (eq, var, k, p) in KERNELS.items():
        assert idx.shape[0] == int(g[f"{lname}_{kname}_nts"])
        q = oracle.ts_batch(eq, var, k, p, g["sources"], g["weights"], g["qcenters"], ptr, idx,
                            g["qtargets"], np.arange(ptr.shape[0], dtype=np.int64),
                            snormals=g["snormals"], tnormals=g["qnormals"])
        assert normwise(q, g[f"{lname}_{kname}_qbx"]) <= 1e-14
        c = oracle.p2p(eq, var, k, g["sources"], g["weights"], g["conv"], g["snormals"],
                       g["conv_normals"], rows=(t_start, tptr, tidx))
        assert normwise(c, g[f"{lname}_{kname}_conv"]) <= 1e-14


@pytest.mark.gpu
@pytest.mark.parametrize("kname", list(KERNELS))
def test_gpu_direct_stage_matches_reference(g, kname):
    from types import SimpleNamespace

    from paper_1811_01110_b200 import KernelSpec
    from paper_1811_01110_b200.direct_stage import DirectStage
    from paper_1811_01110_b200.kernels import Equation, Variant

    eq, var, k, p = KERNELS[kname]
    spec = KernelSpec(equation=Equation(eq), helmholtz_k=k,
                      variant=[Variant.SINGLE_LAYER, Variant.TARGET_NORMAL_DERIV,
                               Variant.SOURCE_NORMAL_DERIV][var])
    tree = SimpleNamespace(points=[g["sources"], g["conv"], g["qcenters"]],
                           owned_start=g["owned_start"], owned_end=g["owned_end"])
    ds = DirectStage(spec, p, tree, g["target_boxes"], g["weights"],
                     source_normals=g["snormals"] if var == 2 else None,
                     qtargets=g["qtargets"], qnormals=g["qnormals"] if var == 1 else None,
                     conv_normals=g["conv_normals"] if var == 1 else None)
    tol = 1e-12 if eq == "laplace" else 1e-10
    for lname in LISTS:
        conv, qbx, nts = ds.run(SimpleNamespace(starts=g[f"{lname}_starts"],
                                                flat=g[f"{lname}_flat"]))
        assert nts == int(g[f"{lname}_{kname}_nts"])
        assert normwise(qbx.cpu().numpy(), g[f"{lname}_{kname}_qbx"]) <= tol
        assert normwise(conv.cpu().numpy(), g[f"{lname}_{kname}_conv"]) <= tol
    # GMRES-style reuse: a new density on the cached plans (linear in the weights)
    ds.set_weights((2.0 - 0.5j) * g["weights"])
    for lname in LISTS:
        conv, qbx, _ = ds.run(SimpleNamespace(starts=g[f"{lname}_starts"],
                                              flat=g[f"{lname}_flat"]))
        assert normwise(qbx.cpu().numpy(), (2.0 - 0.5j) * g[f"{lname}_{kname}_qbx"]) <= tol
        assert normwise(conv.cpu().numpy(), (2.0 - 0.5j) * g[f"{lname}_{kname}_conv"]) <= tol
