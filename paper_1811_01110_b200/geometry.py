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
