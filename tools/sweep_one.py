"""One point of the paper layer sweep (L channels, rule 0 = averaging / 3 = Bayesian), for ncu."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2309_16818_b200 import mem as M
from synth import scenes as S

L = int(sys.argv[1]) if len(sys.argv) > 1 else 2
rule = int(sys.argv[2]) if len(sys.argv) > 2 else 0
n = int(sys.argv[3]) if len(sys.argv) > 3 else 20
c = S.PAPER
clouds = [S.paper_cloud(L, f) for f in range(2)]
dev = [torch.from_numpy(np.ascontiguousarray(cl["points"][:, :3 + L])).cuda() for cl in clouds]
mp = M.Map(c["res"], c["rows"], c["cols"], [dict(name="sem", rule=rule, n_channels=L, w=0.5, alpha0=1.0)])
for i in range(n):
    cl = clouds[i % 2]
    mp.move_to(*cl["move"])
    mp.input_pointcloud(dev[i % 2], [(0, L, 0)], cl["R"], cl["t"], c["noise"])
torch.cuda.synchronize()
print("stats", mp.stats())
