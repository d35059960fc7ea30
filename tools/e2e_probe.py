"""Which earlier bench phase slows the e2e measurement?  Runs bench.measure_e2e
before and after each phase of bench.main_ours and prints the mean ms."""
import argparse
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_1811_01110_b200 import configs  # noqa: E402

case = configs.make_case("c2", "dense")
dev = torch.device("cuda", 0)
args = argparse.Namespace(steps=10, warmup=3, group_lanes=0, soak_seconds=1.0)


def e2e(tag):
    r = bench.measure_e2e(torch, case, args, dev)
    print(f"{tag:28s} e2e {sum(r['ms']) / len(r['ms']):.3f} ms", flush=True)


e2e("fresh")
e2e("again")
flush = torch.empty(bench.L2_FLUSH_BYTES, dtype=torch.uint8, device=dev)
e2e("after flush alloc")
bench.fp64_peak_tflops(torch, dev)
e2e("after fp64 probe")
res, prob, clocks = bench.measure_case(torch, case, args, dev, flush, want_clocks=False)
e2e("after measure_case")
del prob
torch.cuda.empty_cache()
e2e("after del prob")
res, prob, clocks = bench.measure_case(torch, case, args, dev, flush, want_clocks=True)
e2e("after measure_case+clocks")
