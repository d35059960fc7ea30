"""Generate the golden vectors in tests/golden/ from the REFERENCE itself.

Run in the build container (needs /root/reference; never at test time):

    python tests/golden/make_golden.py [name ...]     # default: all

The reference package is imported read-only from /root/reference/pkg/src.
Its backend selection falls back to the NumPy twin there (the compiled
`_core` is not built in the read-only tree); the compiled Cython core built by
`make -C oracle ref` (oracle/_ref/_core*.so) is called directly as well, so
every vector is produced by both reference backends and they are checked to
agree before saving.
"""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, REPO)

import gigaqbx.tsqbx as rts  # noqa: E402
from gigaqbx._backend import _ref as ref_numpy  # noqa: E402
from gigaqbx.kernels import Equation, KernelSpec, Variant  # noqa: E402

import oracle  # noqa: E402

core = oracle.ref_core()
assert core is not None, "build oracle/_ref first: make -C oracle ref"

VARIANTS = [Variant.SINGLE_LAYER, Variant.TARGET_NORMAL_DERIV, Variant.SOURCE_NORMAL_DERIV]


def unit(v):
    return v / np.linalg.norm(v)


def pair_cases():
    """60 random admissible (s, c, t) per (equation, variant), p = 8, k = 2.2,
    drawn like pkg/tests/test_tsqbx.py:19-25 (rho <= 0.9)."""
    rng = np.random.default_rng(99)
    rows = []
    for eq, k in ((Equation.LAPLACE, None), (Equation.HELMHOLTZ, 2.2)):
        for var in VARIANTS:
            spec = KernelSpec(equation=eq, helmholtz_k=k, variant=var)
            cfg = rts.TsConfig(spec, 8)
            for _ in range(60):
                c = rng.normal(size=3)
                R = rng.uniform(0.5, 2.0)
                s = c + R * unit(rng.normal(size=3))
                r = rng.uniform(0.0, 0.9) * R
                t = c + r * unit(rng.normal(size=3))
                sn = unit(rng.normal(size=3))
                tn = unit(rng.normal(size=3))
                v = rts.ts_eval(cfg, s, c, t, source_normal=sn if spec.needs_source_normals
                                else None, target_normal=tn if spec.needs_target_normals
                                else None)
                rows.append((0 if eq is Equation.LAPLACE else 1, spec.variant_code,
                             k or 0.0, s, c, t, sn, tn, v))
    return dict(equation=np.array([r[0] for r in rows]), variant=np.array([r[1] for r in rows]),
                k=np.array([r[2] for r in rows]), p=np.array(8),
                src=np.array([r[3] for r in rows]), ctr=np.array([r[4] for r in rows]),
                tgt=np.array([r[5] for r in rows]), snrm=np.array([r[6] for r in rows]),
                tnrm=np.array([r[7] for r in rows]), value=np.array([r[8] for r in rows]))


def backend_batch():
    """pkg/tests/test_backends.py:17-27,47-59 data: 40 sources at z~3, complex
    weights, variants 0/1/2, target at / off center, p = 8, k = 1.7; values
    from the compiled reference core (checked against the NumPy twin)."""
    rng = np.random.default_rng(8)
    src = rng.normal(size=(40, 3)) + np.array([0, 0, 3.0])
    w = (rng.normal(size=40) + 1j * rng.normal(size=40)).astype(np.complex128)
    sn = rng.normal(size=(40, 3))
    sn /= np.linalg.norm(sn, axis=1)[:, None]
    tn = np.array([0.0, 0.6, 0.8])
    targets = np.array([[0.0, 0.0, 0.0], [0.05, 0.02, -0.03]])
    lap = np.zeros((3, 2), complex)
    hel = np.zeros((3, 2), complex)
    c = np.zeros(3)
    for v in range(3):
        for it, t in enumerate(targets):
            lap[v, it] = core.ts_accum_laplace(v, 8, src, w, sn, c, t, tn)
            hel[v, it] = core.ts_accum_helmholtz(v, 1.7, 8, src, w, sn, c, t, tn)
            a = ref_numpy.ts_accum_laplace(v, 8, src, w, sn, c, t, tn)
            b = ref_numpy.ts_accum_helmholtz(v, 1.7, 8, src, w, sn, c, t, tn)
            assert abs(a - lap[v, it]) <= 5e-13 * abs(a) and abs(b - hel[v, it]) <= 5e-13 * abs(b)
    return dict(src=src, w=w, snrm=sn, tnrm=tn, targets=targets, p=np.array(8), k=np.array(1.7),
                laplace=lap, helmholtz=hel)


def sphere_case(n, p, k, mult, off_surface, seed):
    """Fibonacci-sphere batch (BASELINE config geometry at size n) through the
    reference's PUBLIC ts_accumulate, one call per (center, target)."""
    from paper_1811_01110_b200 import configs
    name = "c3" if k else ("c2" if off_surface else "c1")
    case = configs.make_case(name, "literal", seed=seed, n=n)
    ptr, idx = oracle.near_csr(case.centers, mult * case.expansion_radii, case.sources)
    spec = case.cfg.spec
    cfg = rts.TsConfig(rts.KernelSpec(equation=Equation(spec.equation.value),
                                      variant=Variant(spec.variant.value),
                                      helmholtz_k=spec.helmholtz_k), p)
    out = np.zeros(case.n_targets, complex)
    out_core = np.zeros(case.n_targets, complex)
    for ic in range(case.n_centers):
        sel = idx[ptr[ic]:ptr[ic + 1]]
        for it in range(case.tgt_ptr[ic], case.tgt_ptr[ic + 1]):
            out[it] = rts.ts_accumulate(cfg, case.sources[sel], case.weights[sel],
                                        case.centers[ic], case.targets[it])
            if k:
                out_core[it] = core.ts_accum_helmholtz(0, k, p, np.ascontiguousarray(
                    case.sources[sel]), np.ascontiguousarray(case.weights[sel]), None,
                    case.centers[ic], case.targets[it], None)
            else:
                out_core[it] = core.ts_accum_laplace(0, p, np.ascontiguousarray(
                    case.sources[sel]), np.ascontiguousarray(case.weights[sel]), None,
                    case.centers[ic], case.targets[it], None)
    err = np.max(np.abs(out - out_core)) / np.max(np.abs(out_core))
    assert err < 1e-14, err
    return dict(sources=case.sources, weights=case.weights, centers=case.centers,
                targets=case.targets, tgt_ptr=case.tgt_ptr, near_ptr=ptr, near_idx=idx,
                p=np.array(p), k=np.array(k or 0.0), value=out)


def p2p_cases():
    """Direct sums through the reference's p2p backends (_core.pyx:94-165; the
    compiled core and the NumPy twin must agree): test_backends.py:17-45 style
    data (40 sources, 7 targets, k = 1.7) and a 300 x 200 random cloud, every
    (equation, variant)."""
    out = {}
    rng = np.random.default_rng(11)
    for tag, ns, nt in (("small", 40, 7), ("cloud", 300, 200)):
        src = rng.normal(size=(ns, 3)) + np.array([0, 0, 3.0])
        tgt = rng.normal(size=(nt, 3))
        w = (rng.normal(size=ns) + 1j * rng.normal(size=ns)).astype(np.complex128)
        sn = rng.normal(size=(ns, 3))
        sn /= np.linalg.norm(sn, axis=1)[:, None]
        tn = rng.normal(size=(nt, 3))
        tn /= np.linalg.norm(tn, axis=1)[:, None]
        out.update({f"{tag}_src": src, f"{tag}_tgt": tgt, f"{tag}_w": w, f"{tag}_snrm": sn,
                    f"{tag}_tnrm": tn})
        for v in range(3):
            a = core.laplace_p2p(v, src, w, sn, tgt, tn)
            b = core.helmholtz_p2p(v, 1.7, src, w, sn, tgt, tn)
            a2 = ref_numpy.laplace_p2p(v, src, w, sn, tgt, tn)
            b2 = ref_numpy.helmholtz_p2p(v, 1.7, src, w, sn, tgt, tn)
            assert np.max(abs(a - a2)) <= 1e-13 * np.max(abs(a))
            assert np.max(abs(b - b2)) <= 1e-13 * np.max(abs(b))
            out[f"{tag}_laplace_{v}"] = a
            out[f"{tag}_helmholtz_{v}"] = b
    out["k"] = np.array(1.7)
    return out


def direct_stage_case():
    """The driver's direct stages (driver.py:197-228) on the reference's own tree
    and interaction lists (build_tree / compute_lists, the test_driver.py sphere
    with TREE = TreeParams(nmax=40, t_f=0.9), plus 200 conventional targets):
    the per-box loop is replayed with the compiled reference core, for three
    kernels (Laplace S p=4, Laplace D p=6, Helmholtz S' k=1.3 p=5)."""
    from gigaqbx import geometry as geo
    from gigaqbx.ilists import compute_lists
    from gigaqbx.tree import CENTERS, SOURCES, TARGETS, TreeParams, build_tree

    disc = geo.make_sphere(1.0, 1, 6)
    centers = geo.place_qbx_centers(disc, +1, 0.5)
    rng = np.random.default_rng(17)
    extra = rng.normal(size=(200, 3)) * 1.5
    extra_n = rng.normal(size=(200, 3))
    extra_n /= np.linalg.norm(extra_n, axis=1)[:, None]
    tree = build_tree(disc.nodes, extra, centers.centers, centers.radii,
                      TreeParams(nmax=40, t_f=0.9))
    lists = compute_lists(tree, 20.0)
    dens = rng.normal(size=disc.n_nodes) + 1j * rng.normal(size=disc.n_nodes)
    w_src = disc.weights * dens
    sperm = tree.perms[SOURCES]
    w = np.empty_like(w_src)
    w[...] = w_src[sperm]
    sn = disc.normals[sperm]
    tgt_of_center = centers.target_index[tree.perms[CENTERS]]
    qtargets = disc.target_nodes[tgt_of_center]
    qnormals = disc.target_normals[tgt_of_center]
    conv = tree.points[TARGETS]
    conv_n = extra_n[tree.perms[TARGETS]]
    src = tree.points[SOURCES]
    qc = tree.points[CENTERS]
    out = dict(sources=src, weights=w, snormals=sn, conv=conv, conv_normals=conv_n,
               qcenters=qc, qtargets=qtargets, qnormals=qnormals,
               owned_start=tree.owned_start, owned_end=tree.owned_end,
               target_boxes=lists.target_boxes)
    kernels = [("lap_s", 0, 0, None, 4), ("lap_d", 0, 2, None, 6), ("helm_sp", 1, 1, 1.3, 5)]
    for lname in ("list1", "list3close", "list4close"):
        lst = getattr(lists, lname)
        out[f"{lname}_starts"] = lst.starts
        out[f"{lname}_flat"] = lst.flat
        for kname, eq, var, k, p in kernels:
            conv_near = np.zeros(conv.shape[0], complex)
            qbx = np.zeros(qc.shape[0], complex)
            n_ts = 0
            for b in lists.target_boxes:                     # driver.py:199-227
                b = int(b)
                boxes = lst.get(b)
                if boxes.shape[0] == 0:
                    continue
                sl = [tree.owned_slice(int(d), SOURCES) for d in boxes]
                idx = np.concatenate([np.arange(x.start, x.stop) for x in sl])
                if idx.shape[0] == 0:
                    continue
                ct = tree.owned_slice(b, TARGETS)
                sn_b = np.ascontiguousarray(sn[idx]) if var == 2 else None
                if ct.stop > ct.start:
                    tn = np.ascontiguousarray(conv_n[ct]) if var == 1 else None
                    if eq == 0:
                        conv_near[ct] += core.laplace_p2p(var, src[idx], w[idx], sn_b,
                                                          conv[ct], tn)
                    else:
                        conv_near[ct] += core.helmholtz_p2p(var, k, src[idx], w[idx], sn_b,
                                                            conv[ct], tn)
                cs = tree.owned_slice(b, CENTERS)
                s_b = np.ascontiguousarray(src[idx])
                w_b = np.ascontiguousarray(w[idx])
                for ic in range(cs.start, cs.stop):
                    tn_i = qnormals[ic] if var == 1 else None
                    if eq == 0:
                        qbx[ic] += core.ts_accum_laplace(var, p, s_b, w_b, sn_b, qc[ic],
                                                         qtargets[ic], tn_i)
                    else:
                        qbx[ic] += core.ts_accum_helmholtz(var, k, p, s_b, w_b, sn_b, qc[ic],
                                                           qtargets[ic], tn_i)
                    n_ts += idx.shape[0]
            out[f"{lname}_{kname}_conv"] = conv_near
            out[f"{lname}_{kname}_qbx"] = qbx
            out[f"{lname}_{kname}_nts"] = np.array(n_ts)
    return out


def geometry_case():
    """Geometry files written by the reference (geometry.save_geometry,
    geometry.py:436-455): a sphere with centers, and the same file without the
    optional target_element_id / target_normals / centers keys (load_geometry
    then recovers them by nearest node, :464-476).  The npz holds what the
    reference's load_geometry returns for the minimal file."""
    import json

    from gigaqbx import geometry as geo

    disc = geo.make_sphere(1.0, 0, 3)
    centers = geo.place_qbx_centers(disc, -1, 0.5)
    full = os.path.join(HERE, "geom_sphere.json")
    geo.save_geometry(full, disc, centers)
    with open(full) as f:
        doc = json.load(f)
    for key in ("target_element_id", "target_normals", "centers", "radii", "target_index",
                "side"):
        doc.pop(key)
    minimal = os.path.join(HERE, "geom_sphere_min.json")
    with open(minimal, "w") as f:
        json.dump(doc, f)
        f.write("\n")
    d2, c2 = geo.load_geometry(minimal)
    assert c2 is None
    return dict(target_element_id=d2.target_element_id, target_normals=d2.target_normals,
                nodes=disc.nodes, centers=centers.centers, radii=centers.radii)


GOLDEN = {
    "geometry": geometry_case,
    "direct_stage": direct_stage_case,
    "pairs_p8": pair_cases,
    "backend_batch": backend_batch,
    "c1_literal": lambda: sphere_case(4096, 4, None, 3.0, False, 0),
    "c2_small_literal": lambda: sphere_case(2048, 8, None, 4.0, True, 1),
    "c3_small_literal": lambda: sphere_case(2048, 8, 10.0, 4.0, True, 2),
    "p2p": p2p_cases,
}


def main(names):
    for name in names or GOLDEN:
        np.savez_compressed(os.path.join(HERE, name + ".npz"), **GOLDEN[name]())
    for f in sorted(os.listdir(HERE)):
        print(f, os.path.getsize(os.path.join(HERE, f)))


if __name__ == "__main__":
    main(sys.argv[1:])
