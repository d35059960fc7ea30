import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1811_01110_b200 import configs, near_field_potentials
name, preset = sys.argv[1], sys.argv[2]
case = configs.make_case(name, preset)
dev = torch.device("cuda")
args = [torch.as_tensor(x, device=dev) for x in (case.sources, case.weights, case.centers, case.near_radii, case.targets)]
for _ in range(2):
    near_field_potentials(case.cfg, *args, tgt_ptr=torch.as_tensor(case.tgt_ptr, device=dev), fused=True)
torch.cuda.synchronize()
print("ok")
