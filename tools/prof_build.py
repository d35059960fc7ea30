import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1811_01110_b200 import configs, build_near_lists
name, preset = sys.argv[1], sys.argv[2]
case = configs.make_case(name, preset, **({"n": int(sys.argv[3])} if len(sys.argv) > 3 else {}))
dev = torch.device("cuda")
c = torch.from_numpy(case.centers).to(dev); s = torch.from_numpy(case.sources).to(dev)
r = torch.from_numpy(case.near_radii).to(dev)
for _ in range(2):
    near = build_near_lists(c, s, r)
torch.cuda.synchronize()
print("ok", near.n_pairs)
