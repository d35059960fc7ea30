import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1811_01110_b200 import configs, build_near_lists
for name, preset in [("c2", "dense"), ("c2", "literal"), ("c4", "dense"), ("c5", "literal")]:
    case = configs.make_case(name, preset)
    dev = torch.device("cuda")
    c = torch.from_numpy(case.centers).to(dev); s = torch.from_numpy(case.sources).to(dev)
    r = torch.from_numpy(case.near_radii).to(dev)
    for _ in range(2):
        near = build_near_lists(c, s, r)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(5):
        near = build_near_lists(c, s, r)
    torch.cuda.synchronize()
    print(f"{name}/{preset}: build {1e3 * (time.perf_counter() - t) / 5:.3f} ms, pairs {near.n_pairs}, "
          f"SELL fill {near.sell_fill:.3f}", flush=True)
