"""The paper-shaped layer sweep alone (bench.py side_paper_sweep): ms per frame against L."""
import json
import sys
import torch
sys.path.insert(0, ".")
import bench
from paper_2309_16818_b200 import mem as M

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 100
out = bench.side_paper_sweep(torch, M, torch.cuda.current_stream(), iters=iters)
for k in ("exponential_averaging", "bayesian"):
    print(k, out[k]["layers"], [round(x, 4) for x in out[k]["ms_per_frame"]])
print("height only", round(out["height_only_ms"], 4))
