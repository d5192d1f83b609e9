"""C1 (3 frames) through every point path -- certified atomics + k_refold, the sort-by-cell
pipeline, the small-map kernel -- plus an image input and a readout, for compute-sanitizer
(tests/test_sanitizer_gpu.py).  Exits 0 when the run completes."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2309_16818_b200 import mem as M  # noqa: E402
from synth import scenes as S  # noqa: E402

c = S.C1
groups = [dict(name="feat", rule=M.MEM_AVERAGE, n_channels=1, w=c["w"])]
for sorted_ in (False, True):
    g = M.Map(c["res"], c["rows"], c["cols"], groups, debug_points=True, fuse_sorted=sorted_)
    for f in range(3):
        fr = S.c1_frame(f)
        g.move_to(*fr["move"])
        g.input_pointcloud(torch.from_numpy(fr["points"]).cuda(), [(0, 1, 0)], fr["R"], fr["t"], c["noise"])
    g.debug_codes()
    img = np.random.default_rng(0).uniform(0, 1, (1, 48, 64)).astype(np.float32)
    K = np.array([[50.0, 0, 32], [0, 50.0, 24], [0, 0, 1]])
    g.input_image(torch.from_numpy(img).cuda(), [(0, 1, 0)], K, S.camera_looking_at([-2.0, 0.0, 1.5], [0, 0, 0]),
                  [-2.0, 0.0, 1.5])
    g.get_layer("elevation")
    g.close()
B = 64  # the small-map kernel
gb = M.Map(c["res"], c["rows"], c["cols"], groups, n_maps=B)
fr = S.c1_frame(0)
pts = np.tile(fr["points"], (B, 1))
gb.input_pointcloud_batch(torch.from_numpy(pts).cuda(), np.arange(B + 1, dtype=np.int64) * len(fr["points"]),
                          [(0, 1, 0)], np.tile(fr["R"], (B, 1, 1)), np.tile(fr["t"], (B, 1)), c["noise"])
gb.get_layer("elevation")
torch.cuda.synchronize()
print("sanitize_c1: ok")
