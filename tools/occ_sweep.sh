#!/bin/bash
for b in ${@:-4 8 16}; do
  MEM_NVCC_EXTRA="-DMEM_OCC_BATCH=$b" python paper_2309_16818_b200/build.py --force > gpurun_out/ob.log 2>&1
  echo "batch=$b $(grep -c k_image gpurun_out/ob.log) spill-lines"
  timeout 600 python - <<'PY'
import sys, numpy as np, torch
sys.path.insert(0, ".")
from paper_2309_16818_b200 import mem as M
from synth import scenes as S
c = S.C3
fr = [S.c3_frame(f) for f in range(2)]
groups = [dict(name="sem", rule=3, n_channels=c["n_classes"], alpha0=1.0), dict(name="top", rule=4, n_channels=c["n_classes"])]
binds = [(0, c["n_classes"], 0), (0, c["n_classes"], 1)]
mp = M.Map(c["res"], c["rows"], c["cols"], groups)
for f in fr:
    mp.move_to(*f["move"])
    for cl in f["clouds"]:
        mp.input_pointcloud(torch.from_numpy(cl["points"]).cuda(), [], cl["R"], cl["t"], c["noise"])
mp.set_image_occlusion(True)
img = [torch.from_numpy(f["image"]["img"]).cuda() for f in fr]
for i in range(3):
    im = fr[i % 2]["image"]; mp.input_image(img[i % 2], binds, im["K"], im["R"], im["t"])
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for i in range(50):
    im = fr[i % 2]["image"]; mp.input_image(img[i % 2], binds, im["K"], im["R"], im["t"])
e1.record(); torch.cuda.synchronize()
print("image us", e0.elapsed_time(e1) / 50 * 1e3)
PY
done
