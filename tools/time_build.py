import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1811_01110_b200 import configs, build_near_lists
cases = sys.argv[1].split(",") if len(sys.argv) > 1 else ["c2/dense", "c2/literal", "c4/dense", "c5/literal"]
for cs in cases:
    name, preset = cs.split("/")
    case = configs.make_case(name, preset)
    dev = torch.device("cuda")
    c = torch.from_numpy(case.centers).to(dev); s = torch.from_numpy(case.sources).to(dev)
    r = torch.from_numpy(case.near_radii).to(dev)
    for sell in (True, False):
        for _ in range(2):
            near = build_near_lists(c, s, r, sell=sell)
        torch.cuda.synchronize()
        t = time.perf_counter()
        for _ in range(5):
            near = build_near_lists(c, s, r, sell=sell)
        torch.cuda.synchronize()
        slots = int(near.sell_ptr[-1].item()) if sell else near.n_pairs
        print(f"{name}/{preset} sell={sell}: build {1e3 * (time.perf_counter() - t) / 5:.3f} ms, "
              f"pairs {near.n_pairs}, index slots {slots} ({slots / max(1, near.n_pairs):.2f}x)",
              flush=True)
