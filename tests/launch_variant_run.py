"""Runs a fixed set of seeded scenarios through libmem and saves every layer of every map
(and the frame counters) to an .npz: tests/test_launch_config_gpu.py runs it once with the
shipped library and once with a copy built with other launch configurations (MEM_LIB) and
compares the two bit for bit.  Covers every point path (certified REDs + refold, the sort
pipeline for fast and generic groups, k_smap), the image pass and the PCA readout."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2309_16818_b200 import mem as M  # noqa: E402
from synth import scenes as S  # noqa: E402

out = {}


def save(tag, mp):
    for nm in mp.layer_names():
        out[f"{tag}/{nm}"] = np.asarray(mp.get_layer(nm))
    out[f"{tag}/stats"] = np.array(list(mp.stats().values()), dtype=np.int64)


# C1 colour (RED path, float4), 6 frames with moves
c = S.C1
groups = [dict(name="rgb", rule=M.MEM_COLOR, n_channels=3, w=0.5)]
for sorted_ in (False, True):
    mp = M.Map(c["res"], c["rows"], c["cols"], groups, fuse_sorted=sorted_)
    rng = np.random.default_rng(5)
    for f in range(6):
        fr = S.c1_frame(f)
        pts = fr["points"].copy()
        pts[:, 3] = S.pack_rgb(rng.integers(0, 256, (len(pts), 3)).astype(np.uint8))
        mp.move_to(*fr["move"])
        mp.input_pointcloud(torch.from_numpy(pts).cuda(), [(0, 1, 0)], fr["R"], fr["t"], c["noise"])
    save(f"c1_colour_sorted{int(sorted_)}", mp)
# C3: three dense depth clouds (stride 3, refolds) + the 20-class image, 2 frames
c = S.C3
groups = [dict(name="sem", rule=M.MEM_CLASS_BAYESIAN, n_channels=c["n_classes"], alpha0=1.0),
          dict(name="top", rule=M.MEM_CLASS_MAX, n_channels=c["n_classes"])]
mp = M.Map(c["res"], c["rows"], c["cols"], groups)
for f in range(2):
    fr = S.c3_frame(f)
    mp.move_to(*fr["move"])
    for cl in fr["clouds"]:
        mp.input_pointcloud(torch.from_numpy(cl["points"]).cuda(), [], cl["R"], cl["t"], c["noise"])
    im = fr["image"]
    mp.input_image(torch.from_numpy(im["img"]).cuda(), [(0, c["n_classes"], 0), (0, c["n_classes"], 1)],
                   im["K"], im["R"], im["t"])
save("c3", mp)
# the paper cloud with an 8-channel average group (sort path, generic), 2 frames
c = S.PAPER
mp = M.Map(c["res"], c["rows"], c["cols"], [dict(name="sem", rule=M.MEM_AVERAGE, n_channels=8, w=0.5)])
for f in range(2):
    cl = S.paper_cloud(8, f)
    mp.move_to(*cl["move"])
    mp.input_pointcloud(torch.from_numpy(np.ascontiguousarray(cl["points"])).cuda(), [(0, 8, 0)], cl["R"], cl["t"],
                        c["noise"])
save("paper8", mp)
# 64 C5a maps (k_smap), 2 frames
c = S.C5A
mp = M.Map(c["res"], c["rows"], c["cols"], [dict(name="feat", rule=M.MEM_AVERAGE, n_channels=1, w=c["w"])], n_maps=64)
for f in range(2):
    bt = S.c5a_batch(f, 0, 64)
    mp.move_to_batch(bt["move"])
    mp.input_pointcloud_batch(torch.from_numpy(bt["points"]).cuda(), bt["offsets"], [(0, 1, 0)], bt["R"], bt["t"],
                              c["noise"])
save("c5a64", mp)
# uncertified cells (refold: sorted lists and the whole-map walk)
for rows, n in ((16, 20000), (4, 100000)):
    rng = np.random.default_rng(11 + rows)
    noise = dict(a=1e-4, b=0.0, r_min=0.0, r_max=100.0, h_min=-10.0, h_max=10.0, tau2=1e30, v_out=0.01)
    mp = M.Map(0.1, rows, rows, [dict(name="feat", rule=M.MEM_AVERAGE, n_channels=1, w=0.5)])
    half = rows * 0.1 / 2 - 0.01
    for f in range(3):
        xy = rng.uniform(-half, half, (n, 2))
        z = rng.choice([1e-12, 1e-9, 1e-6, 1e-3, 1.0], n) * rng.choice([-1.0, 1.0], n) * rng.uniform(1, 2, n)
        feat = rng.choice([1e-20, 1e-10, 1.0, 1e10], n) * rng.uniform(1, 2, n)
        pts = np.stack([xy[:, 0], xy[:, 1], z - 1.0, feat], 1).astype(np.float32)
        mp.input_pointcloud(torch.from_numpy(pts).cuda(), [(0, 1, 0)], np.eye(3), [0.0, 0.0, 1.0], noise)
    save(f"refold{rows}", mp)
# C4: 64-channel image and the PCA readout
c4 = S.C4
mp = M.Map(c4["res"], c4["rows"], c4["cols"], [dict(name="feat", rule=M.MEM_AVERAGE, n_channels=c4["d"], w=c4["w"])])
fr = S.c3_frame(0)
mp.move_to(*fr["move"])
for cl in fr["clouds"]:
    mp.input_pointcloud(torch.from_numpy(cl["points"]).cuda(), [], cl["R"], cl["t"], S.C3["noise"])
im = S.c4_image(0)
mp.input_image(torch.from_numpy(im["img"]).cuda(), [(0, c4["d"], 0)], im["K"], im["R"], im["t"])
save("c4", mp)
out["c4/pca"] = np.asarray(mp.pca_readout("feat", 3))
np.savez(sys.argv[1], **out)
print("saved", len(out), "arrays")
