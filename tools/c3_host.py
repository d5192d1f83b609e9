"""C3 frame: host time per call vs device time per stage (events between the calls)."""
import sys
import time
import torch
sys.path.insert(0, ".")
from paper_2309_16818_b200 import mem as M
from synth import scenes as S

c = S.C3
fr = [S.c3_frame(f) for f in range(4)]
groups = [dict(name="sem", rule=3, n_channels=c["n_classes"], alpha0=1.0),
          dict(name="top", rule=4, n_channels=c["n_classes"])]
binds = [(0, c["n_classes"], 0), (0, c["n_classes"], 1)]
mp = M.Map(c["res"], c["rows"], c["cols"], groups)
dev = [dict(clouds=[torch.from_numpy(cl["points"]).cuda() for cl in f["clouds"]],
            img=torch.from_numpy(f["image"]["img"]).cuda()) for f in fr]
N = int(sys.argv[1]) if len(sys.argv) > 1 else 40
host = {k: 0.0 for k in ("move", "c0", "c1", "c2", "img")}
ev = [[torch.cuda.Event(enable_timing=True) for _ in range(6)] for _ in range(N)]
for i in range(N + 5):
    f, d = fr[i % 4], dev[i % 4]
    j = i - 5
    if j >= 0:
        ev[j][0].record()
    t0 = time.perf_counter()
    mp.move_to(*f["move"])
    t1 = time.perf_counter()
    if j >= 0:
        host["move"] += t1 - t0
    for k, (cl, dp) in enumerate(zip(f["clouds"], d["clouds"])):
        t0 = time.perf_counter()
        mp.input_pointcloud(dp, [], cl["R"], cl["t"], c["noise"])
        t1 = time.perf_counter()
        if j >= 0:
            host[f"c{k}"] += t1 - t0
            ev[j][k + 1].record()
    t0 = time.perf_counter()
    mp.input_image(d["img"], binds, f["image"]["K"], f["image"]["R"], f["image"]["t"])
    t1 = time.perf_counter()
    if j >= 0:
        host["img"] += t1 - t0
        ev[j][4].record()
torch.cuda.synchronize()
print("host us per call:", {k: round(v / N * 1e6, 1) for k, v in host.items()})
dt = [[ev[j][k].elapsed_time(ev[j][k + 1]) * 1e3 for k in range(4)] for j in range(N)]
import numpy as np
a = np.array(dt)
print("device us between events (move+c0, c1, c2, img):", np.round(np.median(a, 0), 1), "frame", round(float(np.median([ev[j][0].elapsed_time(ev[j][4]) for j in range(N)]) * 1e3), 1))
