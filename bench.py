#!/usr/bin/env python
"""TSQBX near-field benchmark (BASELINE.json metric: source-target pair-evals/s, fp64,
and % of the FP64 roofline).

Default: N=1, the largest configuration of BASELINE.json that fits one GPU:
configuration 5 (Helmholtz TSQBX, k=20, p=10, 16 spheres, N=8,388,608 sources,
one target per center), `dense` near preset (16r, the stated mean ~200 sources
per center): 1.69 G (center, source) pairs per step.  One
"step" = one evaluation of every (center, target) of that problem.  The other
configurations are reported under `secondary` (configuration 2, the round-1
headline, among them).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Under torchrun (N > 1) the same problem is split over the ranks (strong
scaling, north_star): centers in Morton order are cut into contiguous ranges of
equal pair count, each rank builds the near lists of its own centers only
(sources replicated), evaluates them, and the per-target potentials are
all-gathered over NCCL in chunks that overlap the evaluation of the next chunk
(`ShardedProblem` in paper_1811_01110_b200/distributed.py).  `--scaling weak`
runs one independent problem per GPU instead.  `--impl reference` times the
reference's own compiled CPU core (oracle/_ref, built from /root/reference) on
all host cores on a bounded sample of the same workload.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

METRIC = "TSQBX source-target pair-evals/sec (fp64)"
UNIT = "pair-evals/s"
L2_FLUSH_BYTES = 256 << 20


def _hbm_peak():
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"])
    except (OSError, ValueError, KeyError):
        return 6650.0     # B200_PROFILING.md fallback


HBM_PEAK = _hbm_peak()


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--case", default="c5")
    ap.add_argument("--preset", default="dense", choices=("dense", "literal"))
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--soak-seconds", type=float, default=1.0)
    ap.add_argument("--no-secondary", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--group-lanes", type=int, default=0)
    ap.add_argument("--force-dist", action="store_true",
                    help=argparse.SUPPRESS)   # run the N>1 code path at world size 1 (tests)
    ap.add_argument("--scaling", choices=("weak", "strong"), default="strong",
                    help="N>1: one problem sharded over the GPUs (strong, default) or an "
                         "independent problem per GPU (weak)")
    ap.add_argument("--chunks", type=int, default=0,
                    help="N>1 strong: all-gather chunks per step (0 = automatic)")
    return ap.parse_args()


def workload_name(case) -> str:
    d = case.describe()
    eq = "Laplace" if d["equation"] == "laplace" else f"Helmholtz k={d['k']:g}"
    return (f"BASELINE config {case.name[1]}: {eq} TSQBX S p={d['p']}, {d['n_sources']} sources, "
            f"{d['n_centers']} centers, {d['n_targets']} targets, near radius "
            f"{d['near_mult']:g}r ({case.preset})")


def parallelism_name(args) -> str:
    n = args.gpus
    if n <= 1:
        return "1 GPU"
    if args.scaling == "weak":
        return f"{n} GPUs, one independent problem per GPU (seed = rank), no collective"
    return (f"{n} GPUs: centers sharded by pair count (Morton order), sources replicated, "
            "NCCL all-gather of the potentials")


def bench_config(case, args) -> dict:
    """The `config` object, identical in both arms (same workload, seed, sizes)."""
    parallelism = parallelism_name(args)
    d = case.describe()
    return {"workload": workload_name(case), "case": case.name, "preset": case.preset,
            "seed": case.seed, "equation": d["equation"], "p": d["p"], "k": d["k"],
            "n_sources": d["n_sources"], "n_centers": d["n_centers"],
            "n_targets": d["n_targets"], "near_radius": f"{d['near_mult']:g}r",
            "parallelism": parallelism,
            "l2": "GPU arm: flushed between steps, outside the timed events: a 256 MB "
                  "buffer written, then a second 256 MB buffer read, so the flush's own "
                  "dirty lines are written back before the step starts"}


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


# ----------------------------------------------------------------------------- clocks
_REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
            0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
            0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
            0x100: "display_clock_setting"}


class ClockSampler:
    """Polls SM clock, utilisation and throttle reasons (NVML) every 50 ms."""

    def __init__(self, index: int):
        self.samples = []
        self._stop = threading.Event()
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # noqa: BLE001
            self.err = repr(e)
        self.th = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
                util = nv.nvmlDeviceGetUtilizationRates(self.h).gpu
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                self.samples.append((sm, util, rs))
            except Exception:  # noqa: BLE001
                pass
            time.sleep(0.05)

    def __enter__(self):
        if self.ok:
            self.th.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.ok:
            self.th.join()

    def summary(self):
        if not self.ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "note": self.err}
        loaded = [s for s in self.samples if s[1] >= 50] or self.samples
        reasons = set()
        for _, _, rs in loaded:
            for bit, name in _REASONS.items():
                if rs & bit and name != "gpu_idle":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(s[0] for s in loaded) if loaded else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(reasons),
                "samples": len(loaded)}


# ----------------------------------------------------------------------------- helpers
def fp64_peak_tflops(torch, dev):
    """DFMA throughput of this GPU (MEASURED_PEAKS.json has no FP64 entry)."""
    from paper_1811_01110_b200 import _lib
    L = _lib.load()
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    blocks, threads, iters = sms * 8, 256, 1 << 15
    buf = torch.empty(blocks * threads, dtype=torch.float64, device=dev)
    st = torch.cuda.current_stream(dev).cuda_stream
    best = 0.0
    for i in range(6):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        _lib.check(L.tsqbx_fp64_probe(buf.data_ptr(), iters, blocks, threads, st), "fp64 probe")
        e1.record()
        e1.synchronize()
        if i >= 1:
            best = max(best, blocks * threads * iters * 16 / (e0.elapsed_time(e1) * 1e-3) / 1e12)
    return best


class L2Flush:
    """Evicts the problem from L2 between timed steps: writes one 256 MB buffer
    (2x the 126 MB L2), then reads another, so the L2 ends full of clean lines
    -- the write-backs of the flush's dirty lines happen here, outside the
    timed events, not inside the next step (with a write-only flush the
    literal presets paid up to ~126 MB of those write-backs: 7-10 %)."""

    def __init__(self, torch, dev, nbytes):
        self.w = torch.empty(nbytes, dtype=torch.uint8, device=dev)
        self.r = torch.zeros(nbytes // 8, dtype=torch.float64, device=dev)

    def __call__(self):
        self.w.zero_()
        self.r.sum()


def time_device_steps(torch, fn, steps, flush):
    """Per-step device time (CUDA events on the launching stream) with an L2 flush
    between steps (L2Flush), outside the events."""
    ms = []
    for _ in range(steps):
        flush()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        ms.append((e0, e1))
    torch.cuda.synchronize()
    return [a.elapsed_time(b) for a, b in ms]


def load_traffic(key):
    path = os.path.join(REPO, "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            return json.load(f).get(key)
    except (OSError, ValueError):
        return None


def sample_centers(case, n, seed=123):
    rng = np.random.default_rng(seed)
    return np.sort(rng.choice(case.n_centers, size=min(n, case.n_centers), replace=False))


def cpu_sample_problem(case, sel):
    """CPU near lists for a subset of centers (oracle membership builder) + their targets."""
    import oracle
    ptr, idx = oracle.near_csr(case.centers[sel], case.near_radii[sel], case.sources)
    ntg = np.diff(case.tgt_ptr)[sel]
    tptr = np.concatenate([[0], np.cumsum(ntg)])
    tsel = np.concatenate([np.arange(case.tgt_ptr[c], case.tgt_ptr[c + 1]) for c in sel])
    return ptr, idx, tptr, tsel


def run_reference_chunk(args_tuple):
    """Worker: the reference's compiled core (or the C port when the reference
    core is absent) over centers [lo, hi) of the sample, driver-style
    (``driver._ts_accum``: one ``_core.ts_accum_*`` call per (center, target))."""
    import oracle
    lo, hi = args_tuple
    S = _REF_STATE
    core = oracle.ref_core()
    case = S["case"]
    ptr, idx, tptr, tsel = S["ptr"], S["idx"], S["tptr"], S["tsel"]
    sub_ptr = ptr[lo:hi + 1] - ptr[lo]
    sub_idx = idx[ptr[lo]:ptr[hi]]
    sub_tptr = tptr[lo:hi + 1] - tptr[lo]
    spec = case.cfg.spec
    eq = "laplace" if spec.is_laplace else "helmholtz"
    args = (spec.variant_code, spec.helmholtz_k or 0.0, case.cfg.p_qbx, case.sources,
            case.weights, case.centers[S["sel"][lo:hi]], sub_ptr, sub_idx,
            case.targets[tsel[tptr[lo]:tptr[hi]]], sub_tptr)
    if core is not None:
        oracle.ref_ts_batch(core, eq, *args)
    else:
        oracle.ts_batch(eq, *args, nthreads=1)
    return int(np.sum(np.diff(sub_ptr) * np.diff(sub_tptr)))


_REF_STATE = {}


class CpuReference:
    """The reference's compiled CPU core (oracle/_ref) on a fixed, seeded sample
    of a case's centers: CPU near lists for the sample (the oracle's membership
    builder, identical to the device lists), then ``step()`` evaluates the whole
    sample on ``processes`` forked workers and returns (pairs, seconds)."""

    chunk = 256

    def __init__(self, case, n_sample, processes):
        import oracle
        self.kind = "reference" if oracle.ref_core() is not None else "port"
        self.case, self.processes = case, processes
        sel = sample_centers(case, n_sample)
        ptr, idx, tptr, tsel = cpu_sample_problem(case, sel)
        _REF_STATE.update(case=case, sel=sel, ptr=ptr, idx=idx, tptr=tptr, tsel=tsel)
        self.n = len(sel)
        self.pool = None
        if processes > 1:
            import multiprocessing as mp
            self.pool = mp.get_context("fork").Pool(processes)

    def close(self):
        if self.pool is not None:
            self.pool.close()
            self.pool.join()

    def step(self, n_centers=None):
        n = self.n if n_centers is None else min(self.n, n_centers)
        t0 = time.perf_counter()
        if self.pool is None:
            pairs = sum(run_reference_chunk((lo, min(lo + self.chunk, n)))
                        for lo in range(0, n, self.chunk))
        else:
            bounds = np.linspace(0, n, self.processes * 8 + 1).astype(int)
            pairs = sum(self.pool.map(run_reference_chunk, list(zip(bounds[:-1], bounds[1:]))))
        return pairs, time.perf_counter() - t0

    def describe(self, n, pairs, dt):
        return (f"{n} seeded-random centers of {self.case.n_centers} ({pairs} pairs), "
                f"driver-style _core.ts_accum_* per (center, target) (the reference's compiled "
                f"Cython core built from /root/reference into oracle/_ref), {self.processes} "
                f"process(es), {dt:.2f} s per step; host CPU: {cpu_model()}")


def cpu_reference_rate(case, seconds, processes=1, n_sample=200000):
    """Reference core on a bounded sample: (pairs/s, cores, kind, sample text),
    the sample sized so that one pass takes about ``seconds``."""
    ref = CpuReference(case, n_sample, processes)
    try:
        pairs, dt = ref.step(min(ref.n, max(ref.chunk, 4 * ref.chunk * processes)))
        rate = pairs / dt
        per_center = pairs / max(1, min(ref.n, max(ref.chunk, 4 * ref.chunk * processes)))
        n = int(min(ref.n, max(ref.chunk, rate * seconds / max(per_center, 1.0))))
        pairs, dt = ref.step(n)
        return pairs / dt, processes, ref.kind, ref.describe(n, pairs, dt)
    finally:
        ref.close()


def cpu_public_api_rate(case, seconds, n_sample=20000):
    """The reference's PUBLIC per-call API: its own
    ``gigaqbx.tsqbx.ts_accumulate`` (``_prep`` validation + the compiled
    backend, tsqbx.py:68-80) per (center, target) on one core, from the
    unmodified install in baseline/_ref.  None when that install is absent."""
    ref_dir = os.path.join(REPO, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref_dir, "gigaqbx")):
        return None
    if ref_dir not in sys.path:
        sys.path.insert(0, ref_dir)
    from gigaqbx import kernels as rk, tsqbx as rt
    from gigaqbx._backend import BACKEND_NAME
    spec = case.cfg.spec
    rspec = rk.KernelSpec(equation=rk.Equation(spec.equation.value),
                          variant=rk.Variant(spec.variant.value), helmholtz_k=spec.helmholtz_k)
    cfg = rt.TsConfig(rspec, case.cfg.p_qbx)
    sel = sample_centers(case, n_sample, seed=321)
    ptr, idx, tptr, tsel = cpu_sample_problem(case, sel)
    pairs, n_done = 0, 0
    t0 = time.perf_counter()
    for i, c in enumerate(sel):
        rows = idx[ptr[i]:ptr[i + 1]]
        src, w = case.sources[rows], case.weights[rows]
        for t in tsel[tptr[i]:tptr[i + 1]]:
            rt.ts_accumulate(cfg, src, w, case.centers[c], case.targets[t])
            pairs += len(rows)
        n_done = i + 1
        if time.perf_counter() - t0 > seconds:
            break
    dt = time.perf_counter() - t0
    return {"value": pairs / dt, "unit": UNIT, "cores": 1, "kind": "reference",
            "sample": f"{n_done} seeded-random centers of {case.n_centers} ({pairs} pairs), the "
                      f"reference's public gigaqbx.tsqbx.ts_accumulate per (center, target) "
                      f"(_prep + backend '{BACKEND_NAME}', baseline/_ref), 1 process, {dt:.2f} s; "
                      f"host CPU: {cpu_model()}"}


# ----------------------------------------------------------------------------- reference arm
def main_reference(args):
    """The reference arm: the reference's own CPU implementation of the path on
    all host cores, same config/metric/unit as our arm; each step evaluates the
    same seeded sample of the workload's centers (sized so the whole
    --warmup + --steps run takes about two minutes) and is timed by wall clock;
    ms_per_step is that measured time and value = the sample's pairs / it."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from paper_1811_01110_b200 import configs
    case = configs.make_case(args.case, args.preset)
    procs = os.cpu_count() or 1
    total_steps = max(1, args.steps + args.warmup)
    step_seconds = max(0.5, min(4.0, 100.0 / total_steps))
    ref = CpuReference(case, min(case.n_centers, 300000), procs)
    try:
        # calibrate the per-step sample on one small pass (not a timed step)
        n0 = min(ref.n, 8 * ref.chunk * procs)
        pairs0, dt0 = ref.step(n0)
        n = int(min(ref.n, max(ref.chunk, n0 * step_seconds / max(dt0, 1e-6))))
        for _ in range(args.warmup):
            ref.step(n)
        times, pairs = [], 0
        for _ in range(args.steps):
            pairs, dt = ref.step(n)
            times.append(dt)
    finally:
        ref.close()
    dt = float(statistics.median(times))
    value = pairs / dt
    cpu = {"value": value, "unit": UNIT, "cores": procs, "kind": ref.kind,
           "sample": ref.describe(n, pairs, dt) + f"; median of {args.steps} steps",
           "cpu_model": cpu_model(), "pairs_per_step": pairs}
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": dt * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded, BASELINE.json configuration geometry)",
            "impl": "reference",
            "config": bench_config(case, args),
            "reference_arm": "host CPU, all cores; under torchrun rank 0 only",
            "cpu_baseline": cpu,
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line))
    return 0


# ----------------------------------------------------------------------------- our arm
def measure_case(torch, case, args, dev, flush, want_clocks=False, index=0, variant=None):
    """Device-resident kernel throughput for one case (``variant``: evaluate the
    S' or D layer potential of the same geometry instead of S; normals are the
    sources' surface normals, a target takes its center's)."""
    from paper_1811_01110_b200 import KernelSpec, TsConfig, TsqbxProblem, build_near_lists, configs
    cfg, extra = case.cfg, {}
    if variant is not None:
        sp = case.cfg.spec
        cfg = TsConfig(KernelSpec(equation=sp.equation, variant=variant,
                                  helmholtz_k=sp.helmholtz_k), case.cfg.p_qbx)
        extra = {"source_normals": case.normals,
                 "target_normals": np.repeat(case.normals, np.diff(case.tgt_ptr), axis=0)}
    # device near-list build, steady state: geometry already in HBM, second build
    # (the first one pays the allocator's cudaMalloc calls)
    ctr_d = torch.as_tensor(case.centers, device=dev)
    src_d = torch.as_tensor(case.sources, device=dev)
    rad_d = torch.as_tensor(case.near_radii, device=dev)
    near = build_near_lists(ctr_d, src_d, rad_d, dev)
    del near
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    near = build_near_lists(ctr_d, src_d, rad_d, dev)
    e1.record()
    torch.cuda.synchronize()
    csr_ms = e0.elapsed_time(e1)
    del ctr_d, src_d, rad_d
    prob = TsqbxProblem(cfg, case.sources, case.weights, case.centers, case.targets, near,
                        tgt_ptr=case.tgt_ptr, group_lanes=args.group_lanes or None, device=dev,
                        **extra)
    pairs = prob.pair_count()
    for _ in range(max(3, args.warmup)):
        prob.evaluate()
    torch.cuda.synchronize()
    clocks = None
    if want_clocks:
        sampler = ClockSampler(index)
        with sampler:
            t_end = time.perf_counter() + args.soak_seconds
            while time.perf_counter() < t_end:     # soak: clocks settle under this load
                for _ in range(20):
                    prob.evaluate()
                torch.cuda.synchronize()
            ms = time_device_steps(torch, prob.evaluate, args.steps, flush)
        clocks = sampler.summary()
    else:
        ms = time_device_steps(torch, prob.evaluate, args.steps, flush)
    spec = cfg.spec
    fpp = configs.algorithmic_flops_per_pair(spec, cfg.p_qbx)
    mean_ms = sum(ms) / len(ms)
    launches_per_step = 1   # one evaluation kernel (Helmholtz SELL computes j_n in-kernel)
    # SURVEY.md 8(d) compulsory bytes: sources 40 B, centers 32 B, 4 B per CSR entry,
    # targets 48 B (coordinates, output slot, potential)
    alg_bytes = (case.n_sources * 40 + case.n_centers * 32 + near.n_pairs * 4
                 + case.n_targets * 48)
    res = {"pairs_per_step": pairs, "ms": ms, "mean_ms": mean_ms, "alg_bytes": alg_bytes,
           "layout": prob.layout,
           "value": pairs * len(ms) / (sum(ms) * 1e-3), "flops_per_pair": fpp,
           "tflops": pairs * fpp / (mean_ms * 1e-3) / 1e12, "csr_build_ms": csr_ms,
           "group_lanes": prob.group_lanes, "launches_per_step": launches_per_step,
           "mean_list_len": near.mean_len}
    return res, prob, clocks


P2P_FLOPS = {(0, 0): 13, (0, 1): 21, (0, 2): 21, (1, 0): 23, (1, 1): 35, (1, 2): 35}


def measure_p2p(torch, dev, flush, peak, n=65536, reps=5):
    """dense direct sums (kernels.direct_sum's kernel) over
    n x n pairs, sources and targets resident; algorithmic flops per pair
    (DESIGN.md): Laplace 13 (S) / 21 (S', D), Helmholtz 23 / 35."""
    from paper_1811_01110_b200 import KernelSpec, P2PProblem
    from paper_1811_01110_b200.kernels import Equation, Variant
    rng = np.random.default_rng(0)
    src = torch.as_tensor(rng.normal(size=(n, 3)), device=dev)
    tgt = torch.as_tensor(rng.normal(size=(n, 3)) + 0.01, device=dev)
    w = torch.as_tensor(rng.normal(size=n) + 1j * rng.normal(size=n), device=dev)
    res = {}
    for eq, k in ((Equation.LAPLACE, None), (Equation.HELMHOLTZ, 10.0)):
        spec = KernelSpec(equation=eq, variant=Variant.SINGLE_LAYER, helmholtz_k=k)
        prob = P2PProblem(spec, src, w, device=dev)
        out = torch.empty(n, dtype=torch.complex128, device=dev)
        step = lambda: prob.evaluate(tgt, validate=False, out=out)  # noqa: E731
        for _ in range(2):
            step()
        ms = time_device_steps(torch, step, reps, flush)
        mean = sum(ms) / len(ms)
        rate = n * n / (mean * 1e-3)
        fpp = P2P_FLOPS[(0 if eq is Equation.LAPLACE else 1, 0)]
        res[f"{eq.value}_s_{n}x{n}"] = {
            "value": rate, "unit": "pair-evals/s", "ms_per_step": mean, "flops_per_pair": fpp,
            "roofline_frac": rate * fpp / (peak * 1e12) if peak else None}
    return res


def measure_direct_stage(torch, dev, flush, reps=5):
    """one driver direct stage (List 1) through DirectStage on a
    synthetic C2-scale box structure (configs.synthetic_box_tree: 16r leaf cells,
    65536 conventional targets at radius 1.02); plan cached as in a GMRES solve."""
    from paper_1811_01110_b200 import KernelSpec, configs
    from paper_1811_01110_b200.direct_stage import DirectStage
    case = configs.make_case("c2", "literal")
    rng = np.random.default_rng(1)
    conv = rng.normal(size=(65536, 3))
    conv = 1.02 * conv / np.linalg.norm(conv, axis=1)[:, None]
    cell = 16 * float(case.expansion_radii.mean())
    tree, lst, sp, cp, tboxes = configs.synthetic_box_tree(case, conv, cell)
    qt = case.targets[case.tgt_ptr[:-1]][cp]
    ds = DirectStage(KernelSpec(), 8, tree, tboxes, case.weights[sp], qtargets=qt, device=dev)
    for _ in range(2):
        _, _, nts = ds.run(lst)
    ms = time_device_steps(torch, lambda: ds.run(lst), reps, flush)
    mean = sum(ms) / len(ms)
    ns = tree.owned_end[:, 0] - tree.owned_start[:, 0]
    nt = tree.owned_end[:, 1] - tree.owned_start[:, 1]
    per_box = np.add.reduceat(ns[lst.flat], lst.starts[:-1]) * (np.diff(lst.starts) > 0)
    n_p2p = int((nt * per_box).sum())
    return {"boxes": int(len(lst.starts) - 1), "ts_pairs": int(nts), "p2p_pairs": n_p2p,
            "ms_per_stage": mean, "value": (nts + n_p2p) / (mean * 1e-3),
            "unit": "pair-evals/s (TSQBX + p2p)"}


def build_near_lists_for(case, dev):
    from paper_1811_01110_b200 import build_near_lists
    return build_near_lists(case.centers, case.sources, case.near_radii, dev)


def measure_e2e(torch, case, args, dev, with_near_lists=False):
    """Through the public API with host (pinned) buffers, every step: H2D of the
    step's inputs, TSQBX (validated), D2H of the potentials into a pinned buffer.

    Default (the reference's contract: `ts_accumulate` receives each center's
    near sources, i.e. the lists pre-exist): `ts_accumulate_batch` with the
    device near lists built once up front -- inputs sources, weights, centers,
    targets, target offsets.  `with_near_lists=True` times the whole pipeline
    `near_field_potentials` (geometry -> near lists -> TSQBX) instead."""
    from paper_1811_01110_b200 import build_near_lists
    from paper_1811_01110_b200.tsqbx import near_field_potentials, ts_accumulate_batch
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()  # noqa: E731
    src, w = pin(case.sources), pin(case.weights)
    ctr, rad, tgt = pin(case.centers), pin(case.near_radii), pin(case.targets)
    # one target per center is the API's default layout (tgt_ptr=None): no offsets to copy
    one_each = case.n_targets == case.n_centers and np.array_equal(
        case.tgt_ptr, np.arange(case.n_centers + 1))
    tptr = None if one_each else pin(case.tgt_ptr)
    out = torch.empty(case.n_targets, dtype=torch.complex128).pin_memory()
    gl = args.group_lanes or None
    if with_near_lists:
        ins = (src, w, ctr, rad, tgt, tptr)
        fn = lambda: near_field_potentials(case.cfg, src, w, ctr, rad, tgt, tgt_ptr=tptr,  # noqa
                                           validate=True, group_lanes=gl, device=dev, out=out)
    else:
        ins = (src, w, ctr, tgt, tptr)
        near = build_near_lists(case.centers, case.sources, case.near_radii, dev)
        fn = lambda: ts_accumulate_batch(case.cfg, src, w, ctr, tgt, near, tgt_ptr=tptr,  # noqa
                                         validate=True, group_lanes=gl, device=dev, out=out)
    h2d = sum(int(t.numel() * t.element_size()) for t in ins if t is not None)
    d2h = case.n_targets * 16 + 8
    for _ in range(max(1, min(args.warmup, 3))):
        fn()
    torch.cuda.synchronize()
    steps = max(1, args.steps)
    ms = []
    for _ in range(steps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        ms.append(e0.elapsed_time(e1))
    return {"ms": ms, "h2d": h2d, "d2h": d2h, "steps": steps}


def measure_e2e_overlapped(torch, case, args, dev, near):
    """Independent evaluations through the public API, two in flight on two
    streams (`ts_accumulate_batch(..., sync=False)`): every step still copies
    its inputs H2D from pinned memory and its potentials (and error key) D2H;
    one step's PCIe transfers overlap the other's kernels.  Device time from
    an event pair on the launching stream around all K steps."""
    from paper_1811_01110_b200.tsqbx import ts_accumulate_batch
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()  # noqa: E731
    src, w = pin(case.sources), pin(case.weights)
    ctr, tgt = pin(case.centers), pin(case.targets)
    one_each = case.n_targets == case.n_centers and np.array_equal(
        case.tgt_ptr, np.arange(case.n_centers + 1))
    tptr = None if one_each else pin(case.tgt_ptr)
    streams = [torch.cuda.Stream(dev), torch.cuda.Stream(dev)]
    outs = [torch.empty(case.n_targets, dtype=torch.complex128).pin_memory() for _ in range(2)]
    main = torch.cuda.current_stream(dev)

    def run(k):
        pend = []
        for i in range(k):
            s = streams[i % 2]
            if len(pend) == 2:
                pend.pop(0).result()
            with torch.cuda.stream(s):
                pend.append(ts_accumulate_batch(case.cfg, src, w, ctr, tgt, near, tgt_ptr=tptr,
                                                validate=True, device=dev, out=outs[i % 2],
                                                sync=False))
        for p in pend:
            p.result()
    run(max(3, min(args.warmup, 3)))
    torch.cuda.synchronize()
    steps = max(2, args.steps)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(main)
    for s in streams:
        s.wait_stream(main)
    run(steps)
    for s in streams:
        main.wait_stream(s)
    e1.record(main)
    e1.synchronize()
    h2d = sum(int(t.numel() * t.element_size()) for t in (src, w, ctr, tgt, tptr)
              if t is not None)
    return {"ms": e0.elapsed_time(e1) / steps, "h2d": h2d, "d2h": case.n_targets * 16 + 8,
            "steps": steps}


def main_ours(args):
    import torch
    from paper_1811_01110_b200 import configs

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if not torch.cuda.is_available():
        print(json.dumps({"metric": METRIC, "error": "no CUDA device"}))
        return 1
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    flush = L2Flush(torch, dev, L2_FLUSH_BYTES)
    case = configs.make_case(args.case, args.preset)
    if world > 1 or args.force_dist:
        return main_distributed(torch, args, case, dev, flush, rank, world, local)

    peak = fp64_peak_tflops(torch, dev)
    res, prob, clocks = measure_case(torch, case, args, dev, flush, want_clocks=True,
                                     index=local)
    frac = res["tflops"] / peak if peak else None
    key = f"{case.name}/{case.preset}"
    tr = load_traffic(key)
    traffic = tr["dram_bytes_per_launch"] if tr else None
    line = {
        "metric": METRIC, "value": res["value"], "unit": UNIT, "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": res["mean_ms"],
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded, BASELINE.json configuration geometry; inputs resident in "
                "HBM for `value`)",
        "config": bench_config(case, args),
        "workload_stats": {"pairs_per_step": res["pairs_per_step"],
                           "mean_near_list": round(res["mean_list_len"], 2),
                           "layout": res["layout"],
                           "csr_build_ms": round(res["csr_build_ms"], 3),
                           "validation": "off in `value` (driver path), on in `e2e` (public "
                                         "API)"},
        "roofline": {"bound": "fp64", "achieved": res["tflops"], "peak": peak,
                     "unit": "TFLOP/s", "frac": frac,
                     "traffic": traffic,
                     "traffic_source": ("profiles/ncu_traffic.json: dram__bytes_read.sum + "
                                        "dram__bytes_write.sum of this kernel, one ncu --set "
                                        "full capture, per launch" if traffic else None),
                     "peak_source": "measured DFMA probe on this GPU (tsqbx_fp64_probe); "
                                    "MEASURED_PEAKS.json has no FP64 entry",
                     "flops_per_pair": res["flops_per_pair"],
                     "hbm": {"algorithmic_bytes": res["alg_bytes"],
                             "achieved_gbs": res["alg_bytes"] / (res["mean_ms"] * 1e-3) / 1e9,
                             "peak_gbs": HBM_PEAK,
                             "note": "HBM is not the bound: flop/byte >> ridge ~5.5"},
                     "flops_convention": "algorithmic, SURVEY.md 8(d) (configs.algorithmic_flops_per_pair): "
                                         "Laplace S 7p+17, "
                                         "Helmholtz 14p+30 per pair"},
        "gpu_launches": res["launches_per_step"] * args.steps,
        "clocks": clocks,
    }
    if not args.no_e2e:
        del prob
        torch.cuda.empty_cache()
        e2e = measure_e2e(torch, case, args, dev, with_near_lists=True)
        mean = sum(e2e["ms"]) / len(e2e["ms"])
        line["e2e"] = {"value": res["pairs_per_step"] / (mean * 1e-3), "unit": UNIT,
                       "h2d_bytes_per_step": e2e["h2d"], "d2h_bytes_per_step": e2e["d2h"],
                       "ms_per_step": mean,
                       "path": "paper_1811_01110_b200.near_field_potentials (one call from "
                               "geometry): pinned host sources/weights/centers/near radii/"
                               "targets -> H2D -> device radius-ball near lists -> pack + "
                               "Morton reorder -> TSQBX (validated) -> D2H into a pinned "
                               "buffer; nothing is kept between steps"}
        e2r = measure_e2e(torch, case, args, dev)
        mean = sum(e2r["ms"]) / len(e2r["ms"])
        line["e2e_resident_near_lists"] = {
            "value": res["pairs_per_step"] / (mean * 1e-3), "unit": UNIT,
            "h2d_bytes_per_step": e2r["h2d"], "d2h_bytes_per_step": e2r["d2h"],
            "ms_per_step": mean,
            "path": "paper_1811_01110_b200.ts_accumulate_batch: pinned host sources/weights/"
                    "centers/targets -> H2D -> pack + Morton reorder -> TSQBX (validated) -> "
                    "D2H; the device near lists are built once before the timed steps (the "
                    "reference's ts_accumulate receives pre-gathered near sources)"}
        ov = measure_e2e_overlapped(torch, case, args, dev, build_near_lists_for(case, dev))
        line["e2e_overlapped"] = {
            "value": res["pairs_per_step"] / (ov["ms"] * 1e-3), "unit": UNIT,
            "h2d_bytes_per_step": ov["h2d"], "d2h_bytes_per_step": ov["d2h"],
            "ms_per_step": ov["ms"],
            "path": "as e2e_resident_near_lists, independent evaluations issued two at a time "
                    "on two CUDA streams (ts_accumulate_batch(..., sync=False)): one step's "
                    "H2D/D2H overlaps the other's kernels"}
        torch.cuda.empty_cache()
        # a solver's matvec: geometry resident, a new density in each step
        # (TsqbxProblem.set_weights: H2D of the weights, pack, evaluate, D2H)
        from paper_1811_01110_b200 import TsqbxProblem
        pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()  # noqa: E731
        dens = [pin(case.weights * (1.0 + 0.1 * i)) for i in range(2)]
        hout = torch.empty(case.n_targets, dtype=torch.complex128).pin_memory()
        rprob = TsqbxProblem(case.cfg, case.sources, case.weights, case.centers, case.targets,
                             build_near_lists_for(case, dev), tgt_ptr=case.tgt_ptr, device=dev)

        def matvec(i=[0]):  # noqa: B006
            rprob.set_weights(dens[i[0] % 2])
            i[0] += 1
            hout.copy_(rprob.evaluate(validate=True))
        for _ in range(3):
            matvec()
        torch.cuda.synchronize()
        mms = []
        for _ in range(max(1, args.steps)):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            matvec()
            e1.record()
            e1.synchronize()
            mms.append(e0.elapsed_time(e1))
        mm = sum(mms) / len(mms)
        line["e2e_resident_geometry"] = {
            "value": res["pairs_per_step"] / (mm * 1e-3), "unit": UNIT,
            "h2d_bytes_per_step": case.n_sources * 16, "d2h_bytes_per_step": case.n_targets * 16,
            "ms_per_step": mm,
            "path": "TsqbxProblem.set_weights(pinned density) -> evaluate (validated) -> D2H "
                    "(GMRES matvec: geometry and near lists stay in HBM)"}
        del rprob
        torch.cuda.empty_cache()
    if not args.no_cpu_baseline:
        rate, cores, kind, sample = cpu_reference_rate(case, args.cpu_seconds, processes=1)
        line["cpu_baseline"] = {"value": rate, "unit": UNIT, "cores": cores, "kind": kind,
                                "sample": sample, "cpu_model": cpu_model()}
        pub = cpu_public_api_rate(case, min(args.cpu_seconds, 8.0))
        if pub is not None:
            line["cpu_baseline_public_api"] = pub
    if not args.no_secondary:
        sec = {}
        for name, preset in (("c2", "dense"), ("c2", "literal"), ("c3", "dense"),
                             ("c3", "literal"), ("c4", "literal"), ("c4", "dense"),
                             ("c5", "literal"), ("c5", "dense")):
            if name == case.name and preset == case.preset:
                continue
            c2 = configs.make_case(name, preset)
            r, p2, _ = measure_case(torch, c2, args, dev, flush)
            sec[f"{name}/{preset}"] = {
                "value": r["value"], "pairs_per_step": r["pairs_per_step"],
                "ms_per_step": r["mean_ms"], "tflops": r["tflops"],
                "roofline_frac": r["tflops"] / peak if peak else None,
                "layout": r["layout"], "csr_build_ms": round(r["csr_build_ms"], 3),
                "mean_near_list": round(r["mean_list_len"], 2)}
            del p2
            torch.cuda.empty_cache()
        line["secondary"] = sec
        # S' and D (row f1) on the C2 / C3 dense geometry: same lists, algorithmic
        # flops per pair of configs.algorithmic_flops_per_pair
        from paper_1811_01110_b200.kernels import Variant
        var = {}
        for name in ("c2", "c3"):
            c2 = configs.make_case(name, "dense")
            for vname, v in (("S'", Variant.TARGET_NORMAL_DERIV),
                             ("D", Variant.SOURCE_NORMAL_DERIV)):
                r, p2, _ = measure_case(torch, c2, args, dev, flush, variant=v)
                var[f"{name}/dense/{vname}"] = {
                    "value": r["value"], "ms_per_step": r["mean_ms"],
                    "flops_per_pair": r["flops_per_pair"], "tflops": r["tflops"],
                    "roofline_frac": r["tflops"] / peak if peak else None}
                del p2
                torch.cuda.empty_cache()
        line["variants"] = var
        line["p2p"] = measure_p2p(torch, dev, flush, peak)
        line["direct_stage"] = measure_direct_stage(torch, dev, flush)
    print(json.dumps(line))
    return 0


def main_distributed(torch, args, case, dev, flush, rank, world, local):
    """N ranks, one GPU each (torchrun; NCCL process group).

    Default (`--scaling strong`, north_star): ONE problem -- the N=1 workload --
    split over the ranks by `ShardedProblem` (centers in Morton order cut into
    equal-pair ranges, each rank building only its own near lists, sources
    replicated; per step: the rank's rows in chunks with the all-gather of
    chunk c overlapping chunk c+1, then one scatter into user order on every
    rank).  The step time is the max over ranks of the device-event time
    (all-reduced after the timed region); `value` = the problem's pairs / that
    time.  `--scaling weak`: an independent problem of the N=1 size per rank
    (seed = rank), no data-path collective; `value` = all ranks' pairs / time.
    Run with NCCL_DEBUG=INFO to see the transport (NVLink / NVLS) NCCL chose."""
    import torch.distributed as dist
    from paper_1811_01110_b200 import TsqbxProblem, build_near_lists, configs
    from paper_1811_01110_b200.distributed import ShardedProblem

    dist.init_process_group("nccl", device_id=dev)
    weak = args.scaling == "weak"
    if weak:
        case = configs.make_case(args.case, args.preset, seed=rank)
        near = build_near_lists(case.centers, case.sources, case.near_radii, dev)
        prob = TsqbxProblem(case.cfg, case.sources, case.weights, case.centers, case.targets,
                            near, tgt_ptr=case.tgt_ptr, group_lanes=args.group_lanes or None,
                            device=dev)
        pairs = prob.pair_count()
        step = prob.evaluate
        chunks = None
    else:
        t_setup = time.perf_counter()
        prob = ShardedProblem(case.cfg, case.sources, case.weights, case.centers, case.targets,
                              case.near_radii, tgt_ptr=case.tgt_ptr, rank=rank, world=world,
                              chunks=args.chunks, device=dev)
        torch.cuda.synchronize()
        t_setup = time.perf_counter() - t_setup
        pairs = prob.n_pairs_rank
        step = prob.evaluate
        chunks = prob.layout.chunks
    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    sampler = ClockSampler(local)
    with sampler:
        t_end = time.perf_counter() + args.soak_seconds
        while time.perf_counter() < t_end:     # soak: clocks settle under this load
            for _ in range(5):
                step()
            torch.cuda.synchronize()
        dist.barrier()
        torch.cuda.synchronize()
        ms = time_device_steps(torch, step, args.steps, flush)
        torch.cuda.synchronize()
        dist.barrier()
    clocks = sampler.summary()
    stats = torch.tensor([sum(ms), float(pairs)], dtype=torch.float64, device=dev)
    tmax = stats[:1].clone()
    dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
    tot_pairs = stats[1:].clone()
    dist.all_reduce(tot_pairs, op=dist.ReduceOp.SUM)
    e2e = None
    if not args.no_e2e:
        if weak:
            r = measure_e2e(torch, case, args, dev)
            e_ms_local = sum(r["ms"]) / len(r["ms"])
            h2d, d2h = r["h2d"] * world, r["d2h"] * world
            path = "ts_accumulate_batch on every rank (pinned host in/out), max over ranks"
        else:
            # solver matvec through the sharded problem: every step a new
            # density H2D (pinned, replicated), the sharded evaluation with its
            # all-gather, and the full potential vector D2H on every rank
            pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()  # noqa
            dens = [pin(case.weights * (1.0 + 0.1 * i)) for i in range(2)]
            hout = torch.empty(case.n_targets, dtype=torch.complex128).pin_memory()

            def matvec(i=[0]):  # noqa: B006
                prob.set_weights(dens[i[0] % 2])
                i[0] += 1
                hout.copy_(step(), non_blocking=True)
            for _ in range(3):
                matvec()
            torch.cuda.synchronize()
            dist.barrier()
            mms = []
            for _ in range(max(1, args.steps)):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                matvec()
                e1.record()
                e1.synchronize()
                mms.append(e0.elapsed_time(e1))
            e_ms_local = sum(mms) / len(mms)
            h2d, d2h = case.n_sources * 16 * world, case.n_targets * 16 * world
            path = ("ShardedProblem.set_weights(pinned density, every rank) -> sharded "
                    "evaluation + NCCL all-gather -> D2H of all potentials on every rank; "
                    "geometry and each rank's near lists resident")
        e_ms = torch.tensor([e_ms_local], dtype=torch.float64, device=dev)
        dist.all_reduce(e_ms, op=dist.ReduceOp.MAX)
        step_pairs_e = float(tot_pairs.item())
        e2e = {"value": step_pairs_e / (float(e_ms.item()) * 1e-3), "unit": UNIT,
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
               "ms_per_step": float(e_ms.item()), "path": path}
    t = float(tmax.item())
    step_pairs = float(tot_pairs.item())
    if rank == 0:
        fpp = configs.algorithmic_flops_per_pair(case.cfg.spec, case.cfg.p_qbx)
        per_gpu_tf = step_pairs * fpp / (t / args.steps * 1e-3) / 1e12 / world
        peak = fp64_peak_tflops(torch, dev)
        line = {"metric": METRIC, "value": step_pairs * args.steps / (t * 1e-3), "unit": UNIT,
                "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": t / args.steps, "higher_is_better": True,
                "scaling": "weak" if weak else "strong",
                "vs_baseline": None, "dtype": "f64",
                "data": "synthetic (seeded, BASELINE.json configuration geometry)",
                "config": bench_config(case, args),
                "workload_stats": {"pairs_per_step": step_pairs,
                                   "all_gather_chunks": chunks,
                                   "setup_s_rank0": None if weak else round(t_setup, 3)},
                "roofline": {"bound": "fp64", "achieved": per_gpu_tf, "unit": "TFLOP/s per GPU",
                             "peak": peak, "frac": per_gpu_tf / peak if peak else None,
                             "traffic": None},
                "gpu_launches": (1 if weak else 1 + (chunks or 1)) * args.steps,
                "clocks": clocks}
        if e2e:
            line["e2e"] = e2e
        print(json.dumps(line))
    dist.destroy_process_group()
    return 0


def main():
    args = parse_args()
    if args.impl == "reference":
        return main_reference(args)
    return main_ours(args)


if __name__ == "__main__":
    sys.exit(main())
