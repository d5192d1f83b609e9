"""C5a probe: one batched point input of N maps (default 512) -- for ncu / timing of the small-map path."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2309_16818_b200 import mem as M
from synth import scenes as S

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
c = S.C5A
bt = [S.c5a_batch(f, 0, n) for f in range(2)]
dev = [torch.from_numpy(b["points"]).cuda() for b in bt]
mp = M.Map(c["res"], c["rows"], c["cols"], [dict(name="feat", rule=0, n_channels=1, w=c["w"])], n_maps=n,
          fuse_sorted=len(sys.argv) > 2 and sys.argv[2] == "sorted")
for i in range(6):
    b = bt[i % 2]
    mp.move_to_batch(b["move"])
    mp.input_pointcloud_batch(dev[i % 2], b["offsets"], [(0, 1, 0)], b["R"], b["t"], c["noise"])
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for i in range(10):
    b = bt[i % 2]
    mp.move_to_batch(b["move"])
    mp.input_pointcloud_batch(dev[i % 2], b["offsets"], [(0, 1, 0)], b["R"], b["t"], c["noise"])
e1.record()
torch.cuda.synchronize()
print(f"{n} maps: {e0.elapsed_time(e1) / 10 * 1e3:.1f} us per step")
