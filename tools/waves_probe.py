import sys, torch
sys.path.insert(0, "/root/repo")
from paper_1811_01110_b200 import TsqbxProblem, build_near_lists, configs
case = configs.make_case("c2", "dense")
near = build_near_lists(case.centers, case.sources, case.near_radii)
prob = TsqbxProblem(case.cfg, case.sources, case.weights, case.centers, case.targets, near, tgt_ptr=case.tgt_ptr)
p = prob.prep
out = torch.view_as_real(prob.out)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
lens = (near.ptr[1:] - near.ptr[:-1]).cpu()
for g1 in (444*256, 2*444*256, 2*444*256 + 64*256, 2*444*256 + 136*256, 3*444*256 if 3*444*256 <= p.n_ctr else p.n_ctr, p.n_ctr):
    g1 = min(g1, p.n_ctr)
    for _ in range(3): p.launch(out, False, rows=(0, g1))
    ts = []
    for _ in range(20):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); p.launch(out, False, rows=(0, g1)); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort(); ms = ts[len(ts)//2]
    pairs = int(lens[:g1].sum()) * 2
    print(f"rows {g1:7d} ctas {g1/256:7.1f} waves {g1/256/444:5.2f}  {ms:.4f} ms  {pairs/ms/1e6:.1f} Gpairs/s")
