"""The five BASELINE.json workloads as seeded synthetic problems.

Every case is a cloud of sources y_j with outward normals n_j, one QBX
center per source at c_j = y_j - r_j n_j (``place_qbx_centers`` with side -1),
the on-surface target t = y_j (C2/C3 add one off-surface target per center)
and a radius-ball near list of radius m * r_j.

BASELINE.json is inconsistent about the near radius:
the literal radii (3r / 4r) give ~7-12 sources per center while the text
states a mean of ~200, which the same geometry reaches at 16r.  Both are
available: ``preset="literal"`` (3r for C1/C4/C5, 4r for C2/C3) and
``preset="dense"`` (16r; for C4 a global r = 0.5*sqrt(area/N), the only
variant giving the stated ~30..~800 spread).  The choices SURVEY.md
Appendix B leaves open are recorded in DESIGN.md.

RNG (``np.random.default_rng(seed)``) draw order, fixed:
  C1-C3:  w_lap = U(0.5, 1.5)^N, u_off = normal(N, 3), w_re = U(-1, 1)^N, w_im = U(-1, 1)^N
  C4:     jitter (N, 2), w_lap
  C5:     sphere placement, then per sphere w_re, w_im
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from . import geometry as geo
from .kernels import Equation, KernelSpec
from .tsqbx import TsConfig

PRESETS = ("literal", "dense")


@dataclass
class TsqbxCase:
    name: str
    preset: str
    seed: int
    cfg: TsConfig
    sources: np.ndarray        # (N, 3)
    weights: np.ndarray        # (N,) complex128
    normals: np.ndarray        # (N, 3)
    centers: np.ndarray        # (C, 3)
    expansion_radii: np.ndarray  # (C,) r_j
    near_radii: np.ndarray     # (C,) m * r_j
    targets: np.ndarray        # (T, 3) grouped by center
    tgt_ptr: np.ndarray        # (C + 1,)
    notes: dict = field(default_factory=dict)

    @property
    def n_sources(self) -> int:
        return self.sources.shape[0]

    @property
    def n_centers(self) -> int:
        return self.centers.shape[0]

    @property
    def n_targets(self) -> int:
        return self.targets.shape[0]

    def describe(self) -> dict:
        spec = self.cfg.spec
        return {"case": self.name, "preset": self.preset, "seed": self.seed,
                "equation": spec.equation.value, "variant": spec.variant.value,
                "k": spec.helmholtz_k, "p": self.cfg.p_qbx, "n_sources": self.n_sources,
                "n_centers": self.n_centers, "n_targets": self.n_targets, **self.notes}


def _sphere_case(name, n, p, spec, preset, seed, off_surface, helmholtz_weights, mult_literal):
    rng = np.random.default_rng(seed)
    y, nrm = geo.fibonacci_sphere(n)
    h = math.sqrt(4.0 * math.pi / n)
    r = 0.5 * h
    w_lap = (4.0 * math.pi / n) * rng.uniform(0.5, 1.5, n)
    u_off = rng.normal(size=(n, 3))
    w_re = rng.uniform(-1.0, 1.0, n)
    w_im = rng.uniform(-1.0, 1.0, n)
    weights = ((4.0 * math.pi / n) * (w_re + 1j * w_im) if helmholtz_weights
               else w_lap.astype(np.complex128))
    disc = geo.point_cloud_discretization(y, nrm, np.full(n, 4.0 * math.pi / n), h)
    cs = geo.place_qbx_centers(disc, -1, 0.5)
    m = mult_literal if preset == "literal" else 16.0
    if off_surface:
        u = u_off / np.linalg.norm(u_off, axis=1)[:, None]
        toff = cs.centers + 0.5 * r * u
        targets = np.empty((2 * n, 3))
        targets[0::2] = y
        targets[1::2] = toff
        tptr = np.arange(0, 2 * n + 1, 2, dtype=np.int64)
    else:
        targets = y.copy()
        tptr = np.arange(n + 1, dtype=np.int64)
    return TsqbxCase(name=name, preset=preset, seed=seed, cfg=TsConfig(spec, p), sources=y,
                     weights=weights, normals=nrm, centers=cs.centers,
                     expansion_radii=cs.radii, near_radii=m * cs.radii, targets=targets,
                     tgt_ptr=tptr, notes={"near_mult": m, "h": h})


def make_case(name: str, preset: str = "dense", seed: int = 0, n: int | None = None,
              spheres: int | None = None) -> TsqbxCase:
    """Build configuration ``name`` in {c1..c5}.  ``n`` (points per sphere / torus)
    and ``spheres`` (C5) shrink a case for tests; defaults are BASELINE sizes."""
    if preset not in PRESETS:
        raise ValueError(f"preset must be one of {PRESETS}")
    name = name.lower()
    lap = KernelSpec()
    if name == "c1":
        return _sphere_case("c1", n or 4096, 4, lap, preset, seed, False, False, 3.0)
    if name == "c2":
        return _sphere_case("c2", n or 262144, 8, lap, preset, seed, True, False, 4.0)
    if name == "c3":
        spec = KernelSpec(equation=Equation.HELMHOLTZ, helmholtz_k=10.0)
        return _sphere_case("c3", n or 262144, 8, spec, preset, seed, True, True, 4.0)
    if name == "c4":
        return _torus_case(n or 1048576, preset, seed)
    if name == "c5":
        return _spheres_case(n or 524288, spheres or 16, preset, seed)
    raise ValueError(f"unknown case {name!r}")


def _torus_case(n, preset, seed):
    rng = np.random.default_rng(seed)
    y, nrm, h_loc = geo.clustered_torus(n, rng)
    area = 4.0 * math.pi ** 2 * 1.0 * 0.35
    w = (area / n) * rng.uniform(0.5, 1.5, n)
    if preset == "literal":
        r, m = 0.5 * h_loc, 3.0                     # per-source r = half the local spacing
    else:
        r, m = np.full(n, 0.5 * math.sqrt(area / n)), 16.0   # global r: ~30..~800 per list
    disc = geo.point_cloud_discretization(y, nrm, np.full(n, area / n), 2.0 * r)
    cs = geo.place_qbx_centers(disc, -1, 0.5)
    return TsqbxCase(name="c4", preset=preset, seed=seed, cfg=TsConfig(KernelSpec(), 12),
                     sources=y, weights=w.astype(np.complex128), normals=nrm,
                     centers=cs.centers, expansion_radii=cs.radii, near_radii=m * cs.radii,
                     targets=y.copy(), tgt_ptr=np.arange(n + 1, dtype=np.int64),
                     notes={"near_mult": m})


def _spheres_case(n_per, count, preset, seed):
    rng = np.random.default_rng(seed)
    origins, radii = geo.pack_spheres(count, rng)
    ys, ns, ws, rs = [], [], [], []
    for o, R in zip(origins, radii):
        y, nrm = geo.fibonacci_sphere(n_per, R, o)
        a = 4.0 * math.pi * R * R / n_per
        w = a * (rng.uniform(-1.0, 1.0, n_per) + 1j * rng.uniform(-1.0, 1.0, n_per))
        ys.append(y)
        ns.append(nrm)
        ws.append(w)
        rs.append(np.full(n_per, 0.5 * R * math.sqrt(4.0 * math.pi / n_per)))
    y, nrm, w, r = (np.concatenate(v) for v in (ys, ns, ws, rs))
    m = 3.0 if preset == "literal" else 16.0
    centers = y - r[:, None] * nrm
    spec = KernelSpec(equation=Equation.HELMHOLTZ, helmholtz_k=20.0)
    N = y.shape[0]
    return TsqbxCase(name="c5", preset=preset, seed=seed, cfg=TsConfig(spec, 10), sources=y,
                     weights=w, normals=nrm, centers=centers, expansion_radii=r,
                     near_radii=m * r, targets=y.copy(), tgt_ptr=np.arange(N + 1, dtype=np.int64),
                     notes={"near_mult": m, "spheres": count})


def algorithmic_flops_per_pair(spec: KernelSpec, p: int) -> int:
    """Algorithmic flops per (target, near source) pair, SURVEY.md 8(d)'s
    convention (add/sub/mul 1, FMA 2, sqrt/rsqrt/div/sin/cos 1; per-target work
    -- t - c, r, t-hat, n_t . t-hat, j_n(kr) and its scaled tables, the 1/(4 pi)
    or ik/(4 pi) factor -- excluded):

    * Laplace S   7p + 17 (_core.pyx:229-259).
    * Laplace S'  12p + 22 (_core.pyx:260-282): the S geometry (s - c 3, R^2 5,
      1/R 1, cos g 6, rho 1 = 16); n_t . s-hat 6; (n_t.s-hat - n_t.t-hat cos g) 2;
      1/R^2 1; per order n = 1..p the term radial (n n_t.t-hat P_n + X P'_n),
      s += : 5p; for n < p Legendre 4, P' ladder 2, radial *= rho 1: 7(p - 1);
      complex-weight accumulate 4.
    * Laplace D   13p + 29 (_core.pyx:283-304): geometry 16; n_s . s-hat 6;
      n_s . t-hat 5; (n_s.t-hat - n_s.s-hat cos g) 2; 1/R^2 1; n = 0 term 1;
      per order radial *= rho and -(n+1) n_s.s-hat P_n + Y P'_n, s += : 7p;
      Legendre + P' ladder for n < p: 6(p - 1); accumulate 4.
    * Helmholtz S 14p + 30 (_core.pyx:363-398).
    * Helmholtz S' 19p + 37 (_core.pyx:399-407): the S terms with the
      derivative ladder 2(p - 1), n_t . s-hat 6, (n_t.s-hat - n_t.t-hat cos g) 2,
      and 8 instead of 5 flops per order for h_n (a_n P_n + X b_n P'_n).
    * Helmholtz D 27p + 50 (_core.pyx:408-416): the S terms with the derivative
      ladder 2(p - 1), h'_n = h_{n-1} - (n+1)/x h_n 4p, n_s . s-hat 6,
      n_s . t-hat 5, Y 2, k n_s.s-hat 1, Y/R 1, and 12 instead of 5 flops per
      order for c_n (k n_s.s-hat h'_n P_n + (Y/R) h_n P'_n).
    """
    v = spec.variant_code
    if spec.is_laplace:
        return (7 * p + 17, 12 * p + 22, 13 * p + 29)[v]
    return (14 * p + 30, 19 * p + 37, 27 * p + 50)[v]


def synthetic_box_tree(case, conv, cell):
    """A box structure for the driver's direct stages at BASELINE scale (row f2
    measurements): leaf boxes = the occupied cells of a uniform grid of size
    ``cell`` over the case's sources / centers and the conventional targets
    ``conv``; List 1 of a box = its existing 27 neighbour cells.  Returns
    (tree, list1, source order, center order, target boxes) duck-typed like the
    reference's Octree / _Csr (points in tree order, owned ranges per box).
    Not the reference's adaptive octree -- a stand-in of the same shape."""
    from types import SimpleNamespace

    lo = np.minimum(case.sources.min(0), conv.min(0)) - 1e-9
    def cell_of(x):
        return np.floor((x - lo) / cell).astype(np.int64)
    dims = cell_of(np.maximum(case.sources.max(0), conv.max(0))) + 1
    def key(c):
        return (c[:, 0] * dims[1] + c[:, 1]) * dims[2] + c[:, 2]
    ks, kc, kt = key(cell_of(case.sources)), key(cell_of(case.centers)), key(cell_of(conv))
    boxes = np.unique(np.concatenate([ks, kc, kt]))
    nb = boxes.shape[0]

    def order(keys):
        perm = np.argsort(keys, kind="stable")
        ids = np.searchsorted(boxes, keys[perm])
        return perm, np.searchsorted(ids, np.arange(nb), "left"), \
            np.searchsorted(ids, np.arange(nb), "right")
    sp, s0, s1 = order(ks)
    tp, t0, t1 = order(kt)
    cp, c0, c1 = order(kc)
    owned_start = np.stack([s0, t0, c0], 1)
    owned_end = np.stack([s1, t1, c1], 1)
    # List 1: the existing neighbour cells, in (dx, dy, dz) order
    bx = np.stack([boxes // (dims[1] * dims[2]), (boxes // dims[2]) % dims[1], boxes % dims[2]], 1)
    nbr = np.full((nb, 27), -1, np.int64)
    for q, d in enumerate(np.ndindex(3, 3, 3)):
        c = bx + np.array(d) - 1
        ok = np.all((c >= 0) & (c < dims), axis=1)
        kk = (c[:, 0] * dims[1] + c[:, 1]) * dims[2] + c[:, 2]
        j = np.searchsorted(boxes, kk)
        j = np.minimum(j, nb - 1)
        hit = ok & (boxes[j] == kk)
        nbr[hit, q] = j[hit]
    cnt = (nbr >= 0).sum(1)
    starts = np.concatenate([[0], np.cumsum(cnt)])
    flat = nbr[nbr >= 0]
    tree = SimpleNamespace(points=[case.sources[sp], conv[tp], case.centers[cp]],
                           owned_start=owned_start, owned_end=owned_end)
    lst = SimpleNamespace(starts=starts.astype(np.int64), flat=flat.astype(np.int64))
    return tree, lst, sp, cp, np.arange(nb)
