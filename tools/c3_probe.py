"""C3 probe: the RGB-D semantic frame (3 depth clouds + 20-class image) -- per-launch breakdown
under ncu, and live per-frame time / per-cloud time without it."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2309_16818_b200 import mem as M
from synth import scenes as S

c = S.C3
fr = [S.c3_frame(f) for f in range(2)]
groups = [dict(name="sem", rule=3, n_channels=c["n_classes"], alpha0=1.0),
          dict(name="top", rule=4, n_channels=c["n_classes"])]
binds = [(0, c["n_classes"], 0), (0, c["n_classes"], 1)]
mp = M.Map(c["res"], c["rows"], c["cols"], groups, fuse_sorted=len(sys.argv) > 2 and sys.argv[2] == "sorted")
dev = [dict(clouds=[torch.from_numpy(cl["points"]).cuda() for cl in f["clouds"]],
            img=torch.from_numpy(f["image"]["img"]).cuda()) for f in fr]
n = int(sys.argv[1]) if len(sys.argv) > 1 else 50


def step(i, clouds=True, image=True):
    f, d = fr[i % 2], dev[i % 2]
    mp.move_to(*f["move"])
    if clouds:
        for cl, dp in zip(f["clouds"], d["clouds"]):
            mp.input_pointcloud(dp, [], cl["R"], cl["t"], c["noise"])
    if image:
        mp.input_image(d["img"], binds, f["image"]["K"], f["image"]["R"], f["image"]["t"])


for kw in (dict(), dict(image=False), dict(clouds=False)):
    for i in range(5):
        step(i, **kw)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(n):
        step(i, **kw)
    e1.record()
    torch.cuda.synchronize()
    print(kw, f"{e0.elapsed_time(e1) / n * 1e3:.1f} us per frame")
st = mp.stats() if hasattr(mp, "stats") else None
print("stats", st)

# C4: 64-channel feature image, average-fused (as bench.py side_c3_c4)
c4 = S.C4
m4 = M.Map(c4["res"], c4["rows"], c4["cols"], [dict(name="feat", rule=0, n_channels=c4["d"], w=c4["w"])])
m4.move_to(*fr[0]["move"])
for cl, dp in zip(fr[0]["clouds"], dev[0]["clouds"]):
    m4.input_pointcloud(dp, [], cl["R"], cl["t"], c["noise"])
ims = [S.c4_image(f) for f in range(2)]
dims = [torch.from_numpy(im["img"]).cuda() for im in ims]
for i in range(5):
    m4.input_image(dims[i % 2], [(0, c4["d"], 0)], ims[i % 2]["K"], ims[i % 2]["R"], ims[i % 2]["t"])
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for i in range(n):
    m4.input_image(dims[i % 2], [(0, c4["d"], 0)], ims[i % 2]["K"], ims[i % 2]["R"], ims[i % 2]["t"])
e1.record()
torch.cuda.synchronize()
print(f"C4 {e0.elapsed_time(e1) / n * 1e3:.1f} us per image")
