"""Geometry files (reference format, geometry.py:432-498) and center placement
against files written / read by the reference itself (tests/golden)."""

import os

import numpy as np

from paper_1811_01110_b200 import geometry as geo


def test_load_reference_file(golden_dir):
    disc, centers = geo.load_geometry(os.path.join(golden_dir, "geom_sphere.json"))
    g = np.load(os.path.join(golden_dir, "geometry.npz"))
    assert np.array_equal(disc.nodes, g["nodes"])
    assert centers is not None and centers.side == -1
    assert np.array_equal(centers.centers, g["centers"])
    assert np.array_equal(centers.radii, g["radii"])
    # center placement reproduces the reference's bit for bit
    again = geo.place_qbx_centers(disc, -1, 0.5)
    assert np.array_equal(again.centers, centers.centers)
    assert np.array_equal(again.radii, centers.radii)


def test_minimal_file_recovers_targets_like_reference(golden_dir):
    disc, centers = geo.load_geometry(os.path.join(golden_dir, "geom_sphere_min.json"))
    g = np.load(os.path.join(golden_dir, "geometry.npz"))
    assert centers is None
    assert np.array_equal(disc.target_element_id, g["target_element_id"])
    assert np.array_equal(disc.target_normals, g["target_normals"])


def test_round_trip(tmp_path, golden_dir):
    disc, centers = geo.load_geometry(os.path.join(golden_dir, "geom_sphere.json"))
    path = tmp_path / "g.json"
    geo.save_geometry(path, disc, centers)
    d2, c2 = geo.load_geometry(path)
    for a in ("nodes", "weights", "normals", "element_id", "element_size", "target_nodes",
              "target_normals", "target_element_id"):
        assert np.array_equal(getattr(disc, a), getattr(d2, a))
    assert np.array_equal(centers.centers, c2.centers) and c2.side == centers.side
    # byte-identical to the reference writer's output
    with open(os.path.join(golden_dir, "geom_sphere.json")) as f:
        assert f.read() == path.read_text()


import pytest  # noqa: E402


@pytest.mark.gpu
def test_device_geometry_near_field_matches_oracle(golden_dir):
    import oracle
    from paper_1811_01110_b200 import KernelSpec, TsConfig

    disc, centers = geo.load_geometry(os.path.join(golden_dir, "geom_sphere.json"))
    dg = geo.DeviceGeometry.from_host(disc, centers)
    dens = np.random.default_rng(3).normal(size=disc.n_nodes)
    cfg = TsConfig(KernelSpec(), 6)
    got = dg.near_field(cfg, dens, near_mult=3.0).cpu().numpy()
    ptr, idx = oracle.near_csr(centers.centers, 3.0 * centers.radii, disc.nodes)
    ref = oracle.ts_batch("laplace", 0, None, 6, disc.nodes, disc.weights * dens,
                          centers.centers, ptr, idx, disc.target_nodes[centers.target_index],
                          np.arange(centers.n_centers + 1, dtype=np.int64))
    assert np.max(np.abs(got - ref)) <= 1e-12 * np.max(np.abs(ref))
