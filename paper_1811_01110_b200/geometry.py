"""Geometry / center / target setup for the TSQBX path (host side).

Keeps the reference's container types and center placement
(/root/reference/pkg/src/gigaqbx/geometry.py:29-66, 413-427) and adds the
synthetic point clouds the BASELINE.json configurations are defined on
(Fibonacci spheres, a clustered torus, packed spheres).  This is setup, not
the hot path: plain NumPy, run once per problem.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np


@dataclass
class Discretization:
    """Same fields and checks as geometry.py:29-54."""

    nodes: np.ndarray            # (N, 3) source quadrature nodes
    weights: np.ndarray          # (N,)  quadrature weight x surface Jacobian
    normals: np.ndarray          # (N, 3) unit normals
    element_id: np.ndarray       # (N,)  owning element per node
    element_size: np.ndarray     # (K,)  diameter proxy h per element
    target_nodes: np.ndarray     # (T, 3) on-surface targets
    target_normals: np.ndarray   # (T, 3)
    target_element_id: np.ndarray  # (T,)

    def __post_init__(self):
        n = self.nodes.shape[0]
        if not (self.weights.shape[0] == self.normals.shape[0] == self.element_id.shape[0] == n):
            raise ValueError("inconsistent discretization array lengths")
        if np.any(self.weights <= 0):
            raise ValueError("quadrature weights must be positive")

    @property
    def n_nodes(self) -> int:
        return self.nodes.shape[0]

    @property
    def n_targets(self) -> int:
        return self.target_nodes.shape[0]


@dataclass
class QbxCenterSet:
    """Same fields as geometry.py:57-66."""

    centers: np.ndarray       # (T, 3)
    radii: np.ndarray         # (T,) expansion radius r_c
    target_index: np.ndarray  # (T,) target driven by each center
    side: int                 # +1 exterior, -1 interior

    @property
    def n_centers(self) -> int:
        return self.centers.shape[0]


def place_qbx_centers(disc: Discretization, side: int, alpha: float) -> QbxCenterSet:
    """One center per on-surface target at ``t + side * r_c * n`` with
    ``r_c = alpha * element_size`` (geometry.py:413-427)."""
    if not 0.0 < alpha <= 1.0:
        raise ValueError("alpha must be in (0, 1]")
    if side not in (+1, -1):
        raise ValueError("side must be +1 (exterior) or -1 (interior)")
    radii = alpha * disc.element_size[disc.target_element_id]
    centers = disc.target_nodes + side * radii[:, None] * disc.target_normals
    return QbxCenterSet(centers=centers, radii=radii,
                        target_index=np.arange(disc.n_targets, dtype=np.int64), side=side)


def point_cloud_discretization(nodes, normals, weights, spacing) -> Discretization:
    """Discretization of a point cloud: every node is its own element of size
    ``spacing`` (scalar or per node) and its own on-surface target."""
    nodes = np.ascontiguousarray(nodes, dtype=np.float64)
    n = nodes.shape[0]
    h = np.broadcast_to(np.asarray(spacing, dtype=np.float64), (n,)).copy()
    ids = np.arange(n, dtype=np.int64)
    return Discretization(nodes=nodes, weights=np.asarray(weights, dtype=np.float64),
                          normals=np.ascontiguousarray(normals, dtype=np.float64),
                          element_id=ids, element_size=h, target_nodes=nodes.copy(),
                          target_normals=np.ascontiguousarray(normals, dtype=np.float64),
                          target_element_id=ids.copy())


# ---------------------------------------------------------------------------
# synthetic point clouds used by the BASELINE.json configurations
# ---------------------------------------------------------------------------
def fibonacci_sphere(n: int, radius: float = 1.0, origin=(0.0, 0.0, 0.0)):
    """Fibonacci lattice: z_i = 1 - (2i+1)/n, phi_i = i*pi*(3 - sqrt 5).
    Returns (points, outward unit normals)."""
    i = np.arange(n, dtype=np.float64)
    z = 1.0 - (2.0 * i + 1.0) / n
    phi = i * math.pi * (3.0 - math.sqrt(5.0))
    rho = np.sqrt(np.maximum(0.0, 1.0 - z * z))
    nrm = np.stack([rho * np.cos(phi), rho * np.sin(phi), z], axis=1)
    pts = np.asarray(origin, dtype=np.float64)[None, :] + radius * nrm
    return pts, nrm


def _inverse_cdf(pdf, lo, hi, u, m=1 << 16):
    """Invert the CDF of an unnormalised density on [lo, hi] at u in (0, 1)."""
    x = np.linspace(lo, hi, m + 1)
    f = pdf(x)
    cdf = np.concatenate([[0.0], np.cumsum(0.5 * (f[1:] + f[:-1]) * np.diff(x))])
    cdf /= cdf[-1]
    return np.interp(u, cdf, x)


def clustered_torus(n: int, rng: np.random.Generator, major: float = 1.0, minor: float = 0.35,
                    amp: float = 4.0, width: float = 0.05, jitter: float = 0.1):
    """Torus points with area density proportional to 1 + amp*exp(-phi^2/width)
    (clustered near phi = 0), Kronecker-lattice placed, with a tangential jitter
    of ``jitter`` times the local spacing.  Returns (points, normals, h_loc) with
    h_loc = (n * rho_A)^(-1/2) the analytic local spacing."""
    i = np.arange(n, dtype=np.float64)
    u = (i + 0.5) / n
    v = np.mod(i * (math.sqrt(5.0) - 1.0) / 2.0, 1.0)
    fphi = lambda x: 1.0 + amp * np.exp(-x * x / width)  # noqa: E731
    phi = _inverse_cdf(fphi, -math.pi, math.pi, u)
    theta = _inverse_cdf(lambda x: 1.0 + (minor / major) * np.cos(x), -math.pi, math.pi, v)
    # points per unit area: n * f(phi)/Z / (2 pi minor)   (the theta factor cancels the metric)
    xs = np.linspace(-math.pi, math.pi, 1 << 16)
    zf = np.trapezoid(fphi(xs), xs)
    rho_a = n * fphi(phi) / zf / (2.0 * math.pi * minor * major)
    h_loc = 1.0 / np.sqrt(rho_a)
    xi = rng.uniform(-1.0, 1.0, size=(n, 2))
    ring = major + minor * np.cos(theta)
    phi = phi + jitter * h_loc * xi[:, 0] / ring
    theta = theta + jitter * h_loc * xi[:, 1] / minor
    ring = major + minor * np.cos(theta)
    pts = np.stack([ring * np.cos(phi), ring * np.sin(phi), minor * np.sin(theta)], axis=1)
    nrm = np.stack([np.cos(theta) * np.cos(phi), np.cos(theta) * np.sin(phi), np.sin(theta)],
                   axis=1)
    return pts, nrm, h_loc


def pack_spheres(count: int, rng: np.random.Generator, box: float = 10.0, rmin: float = 0.5,
                 rmax: float = 1.5, gap: float = 0.1, max_tries: int = 100000):
    """Non-overlapping spheres (radii U(rmin, rmax)) in [-box, box]^3 by seeded
    rejection sampling with a surface gap >= ``gap``.  Returns (origins, radii)."""
    origins, radii = [], []
    tries = 0
    while len(radii) < count:
        tries += 1
        if tries > max_tries:
            raise RuntimeError("could not place spheres")
        R = rng.uniform(rmin, rmax)
        o = rng.uniform(-box + R, box - R, size=3)
        if all(np.linalg.norm(o - q) >= R + Rq + gap for q, Rq in zip(origins, radii)):
            origins.append(o)
            radii.append(R)
    return np.array(origins), np.array(radii)


# ---------------------------------------------------------------------------
# geometry files: the reference's JSON format
# (geometry.py:432-498): arrays of numbers written as strings with 17
# significant digits, optional centers block.
# ---------------------------------------------------------------------------
def _num_rows(a):
    return [[format(float(x), ".17g") for x in row] for row in np.atleast_2d(a)]


def _nums(a):
    return [format(float(x), ".17g") for x in np.asarray(a).reshape(-1)]


def save_geometry(path, disc: Discretization, centers: QbxCenterSet | None = None) -> None:
    """Write ``disc`` (and ``centers``) in the reference's file format."""
    import json

    doc = {"nodes": _num_rows(disc.nodes), "weights": _nums(disc.weights),
           "normals": _num_rows(disc.normals), "element_id": disc.element_id.tolist(),
           "element_size": _nums(disc.element_size), "targets": _num_rows(disc.target_nodes),
           "target_normals": _num_rows(disc.target_normals),
           "target_element_id": disc.target_element_id.tolist()}
    if centers is not None:
        doc.update(centers=_num_rows(centers.centers), radii=_nums(centers.radii),
                   target_index=centers.target_index.tolist(),
                   side="exterior" if centers.side > 0 else "interior")
    with open(path, "w") as f:
        json.dump(doc, f)
        f.write("\n")


def load_geometry(path):
    """(Discretization, QbxCenterSet | None) from a reference geometry file.
    Missing target element ids / normals come from each target's nearest
    quadrature node, as in the reference."""
    import json

    with open(path) as f:
        doc = json.load(f)
    f64 = lambda key: np.asarray(doc[key], dtype=np.float64)  # noqa: E731
    nodes = f64("nodes").reshape(-1, 3)
    targets = f64("targets").reshape(-1, 3)
    element_id = np.asarray(doc["element_id"], dtype=np.int64)
    normals = f64("normals").reshape(-1, 3)
    nearest = None
    if "target_element_id" not in doc or "target_normals" not in doc:
        from scipy.spatial import cKDTree

        nearest = cKDTree(nodes).query(targets)[1]
    if "target_element_id" in doc:
        teid = np.asarray(doc["target_element_id"], dtype=np.int64)
    else:
        teid = element_id[nearest]
    if "target_normals" in doc:
        tnrm = f64("target_normals").reshape(-1, 3)
    else:
        tnrm = normals[nearest]
        tnrm = tnrm / np.linalg.norm(tnrm, axis=1)[:, None]
    disc = Discretization(nodes=nodes, weights=f64("weights"), normals=normals,
                          element_id=element_id, element_size=f64("element_size"),
                          target_nodes=targets, target_normals=tnrm, target_element_id=teid)
    centers = None
    if "centers" in doc:
        centers = QbxCenterSet(centers=f64("centers").reshape(-1, 3), radii=f64("radii"),
                               target_index=np.asarray(doc["target_index"], dtype=np.int64),
                               side=+1 if doc.get("side", "exterior") == "exterior" else -1)
    return disc, centers


@dataclass
class DeviceGeometry:
    """A geometry resident in HBM, laid out for the TSQBX path: sources with
    their quadrature weights and normals, centers with radii, and each center's
    on-surface target (and its normal) -- one target per center."""

    nodes: "object"
    weights: "object"
    normals: "object"
    centers: "object"
    radii: "object"
    targets: "object"
    target_normals: "object"

    @classmethod
    def from_host(cls, disc: Discretization, centers: QbxCenterSet, device=None):
        import torch

        from . import _device as dv

        dev = dv.require_cuda(device)
        with torch.cuda.device(dev):
            return cls._from_host(disc, centers, dev)

    @classmethod
    def _from_host(cls, disc, centers, dev):
        import torch

        from . import _device as dv

        put = lambda a: dv.to_device(a, torch.float64, dev)  # noqa: E731
        return cls(nodes=put(disc.nodes), weights=put(disc.weights), normals=put(disc.normals),
                   centers=put(centers.centers), radii=put(centers.radii),
                   targets=put(disc.target_nodes[centers.target_index]),
                   target_normals=put(disc.target_normals[centers.target_index]))

    def near_field(self, cfg, density, near_mult: float = 3.0, validate: bool = True):
        """Per-center near-field TSQBX potentials of ``density`` (one value per
        node; source weights = quadrature weight x density): near lists are
        the radius balls |s - c| <= near_mult * r_c (BASELINE's definition),
        built and evaluated on the device.  Returns a complex128 CUDA tensor
        (the center's target order)."""
        import torch

        from . import _device as dv
        from .tsqbx import near_field_potentials

        dev = self.nodes.device
        dens = dv.to_device(density, torch.complex128, dev, (-1,))
        if dens.shape[0] != self.nodes.shape[0]:
            raise ValueError("density must have one value per source node")
        w = self.weights.to(torch.complex128) * dens
        nrm = self.normals if cfg.spec.needs_source_normals else None
        tn = self.target_normals if cfg.spec.needs_target_normals else None
        return near_field_potentials(cfg, self.nodes, w, self.centers, self.radii * near_mult,
                                     self.targets, source_normals=nrm, target_normals=tn,
                                     validate=validate, device=dev)
