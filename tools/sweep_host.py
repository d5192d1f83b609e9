import sys, time
import numpy as np, torch
sys.path.insert(0, ".")
from paper_2309_16818_b200 import mem as M
from synth import scenes as S
L = 2
c = S.PAPER
clouds = [S.paper_cloud(L, f) for f in range(2)]
dev = [torch.from_numpy(np.ascontiguousarray(cl["points"][:, :3 + L])).cuda() for cl in clouds]
mp = M.Map(c["res"], c["rows"], c["cols"], [dict(name="sem", rule=0, n_channels=L, w=0.5, alpha0=1.0)])
ts = []
for i in range(60):
    cl = clouds[i % 2]
    t0 = time.perf_counter()
    mp.move_to(*cl["move"])
    mp.input_pointcloud(dev[i % 2], [(0, L, 0)], cl["R"], cl["t"], c["noise"])
    ts.append(time.perf_counter() - t0)
torch.cuda.synchronize()
print("host us per call", [round(x * 1e6) for x in ts[:12]], "median", round(np.median(ts) * 1e6))
evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(40)]
for i in range(40):
    cl = clouds[i % 2]
    mp.move_to(*cl["move"])
    evs[i][0].record()
    mp.input_pointcloud(dev[i % 2], [(0, L, 0)], cl["R"], cl["t"], c["noise"])
    evs[i][1].record()
torch.cuda.synchronize()
print("device us per call", [round(a.elapsed_time(b) * 1e3) for a, b in evs[:20]])
mp.profile(True)
for i in range(4):
    cl = clouds[i % 2]
    mp.move_to(*cl["move"])
    mp.input_pointcloud(dev[i % 2], [(0, L, 0)], cl["R"], cl["t"], c["noise"])
torch.cuda.synchronize()
print("stages", mp.profile_read(reset=True))
