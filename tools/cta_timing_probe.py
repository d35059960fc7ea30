"""Per-CTA start/end times (globaltimer) of the Laplace SELL kernel, from a
debug build of the library with timing stores (row split):

    make -C paper_1811_01110_b200/csrc OUT=$PWD/paper_1811_01110_b200/_lib/dbg_timing.so \
        OBJDIR=/tmp/obj_dbg EXTRA_NVFLAGS=-DTSQBX_CTA_TIMING
    python tools/cta_timing_probe.py [case] [preset]     # GIGAQBX_LIB_PATH -> debug build
"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("GIGAQBX_LIB_PATH", os.path.join(
    os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
    "paper_1811_01110_b200", "_lib", "dbg_timing.so"))
from paper_1811_01110_b200 import TsqbxProblem, build_near_lists, configs, _lib  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
preset = sys.argv[2] if len(sys.argv) > 2 else "dense"
case = configs.make_case(name, preset)
near = build_near_lists(case.centers, case.sources, case.near_radii)
prob = TsqbxProblem(case.cfg, case.sources, case.weights, case.centers, case.targets, near,
                    tgt_ptr=case.tgt_ptr)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
L = _lib.load()
fn = L.tsqbx_debug_cta_times
fn.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]
N = 8192
t = np.zeros(2 * N, np.uint64)
sm = np.zeros(N, np.uint32)
for _ in range(3):
    prob.evaluate()
torch.cuda.synchronize()
fn(t.ctypes.data, sm.ctypes.data, N)
flush.zero_()
torch.cuda.synchronize()
prob.evaluate()
torch.cuda.synchronize()
fn(t.ctypes.data, sm.ctypes.data, N)
st = t[0::2].astype(np.int64)
en = t[1::2].astype(np.int64)
used = en > 0
st, en, sm = st[used], en[used], sm[used]
t0 = st.min()
st -= t0
en -= t0
d = (en - st) / 1e3
order = np.argsort(st)
slots = np.bincount(sm[order[:min(len(order), 4096)]], minlength=148).max() * 148
print(f"{name}/{preset}: split {prob.group_lanes}, {used.sum()} CTAs, ~{slots} slots, "
      f"kernel span {en.max() / 1e3:.1f} us, CTA duration mean {d.mean():.1f} "
      f"min {d.min():.1f} max {d.max():.1f} us, total CTA-us / slots = "
      f"{d.sum() / slots:.1f} us")
for lo in range(0, len(order), max(1, slots)):
    idx = order[lo:lo + slots]
    print(f"  CTAs {lo}-{lo + len(idx)}: start {st[idx].min() / 1e3:.1f}-{st[idx].max() / 1e3:.1f}"
          f" us, end {en[idx].min() / 1e3:.1f}-{en[idx].max() / 1e3:.1f}, dur mean "
          f"{d[idx].mean():.1f}")
