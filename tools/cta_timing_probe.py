import ctypes, os, sys
import numpy as np, torch
sys.path.insert(0, "/root/repo")
os.environ["GIGAQBX_LIB_PATH"] = "/root/repo/paper_1811_01110_b200/_lib/dbg_timing.so"
from paper_1811_01110_b200 import TsqbxProblem, build_near_lists, configs, _lib
case = configs.make_case("c2", "dense")
near = build_near_lists(case.centers, case.sources, case.near_radii)
prob = TsqbxProblem(case.cfg, case.sources, case.weights, case.centers, case.targets, near, tgt_ptr=case.tgt_ptr)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
L = _lib.load()
fn = L.tsqbx_debug_cta_times
fn.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]
for _ in range(3): prob.evaluate()
torch.cuda.synchronize()
t = np.zeros(2 * 1024, np.uint64); sm = np.zeros(1024, np.uint32)
fn(t.ctypes.data, sm.ctypes.data, 1024)
flush.zero_(); torch.cuda.synchronize()
prob.evaluate(); torch.cuda.synchronize()
fn(t.ctypes.data, sm.ctypes.data, 1024)
st = t[0::2].astype(np.int64); en = t[1::2].astype(np.int64)
t0 = st.min(); st -= t0; en -= t0
d = (en - st) / 1e3
lens = (near.ptr[1:] - near.ptr[:-1]).cpu().numpy()
cta_len = np.add.reduceat(lens, np.arange(0, 262144, 256))
print("kernel span us", en.max() / 1e3)
order = np.argsort(st)
for lo, hi in ((0, 444), (444, 888), (888, 1024)):
    idx = order[lo:hi]
    print(f"CTAs {lo}-{hi}: start {st[idx].min()/1e3:.1f}-{st[idx].max()/1e3:.1f} us, end {en[idx].min()/1e3:.1f}-{en[idx].max()/1e3:.1f}, dur mean {d[idx].mean():.1f} min {d[idx].min():.1f} max {d[idx].max():.1f}, pairs/CTA mean {cta_len[idx].mean():.0f}")
print("ctas per sm first wave:", np.bincount(sm[order[:444]]).max(), np.bincount(sm[order[:444]], minlength=148).min())
print("duration vs pairs corr", np.corrcoef(d, cta_len)[0,1])
