"""C4 PCA readout: device time per readout and per kernel (mem_profile stage 'read')."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2309_16818_b200 import mem as M
from synth import scenes as S
c, c3 = S.C4, S.C3
m4 = M.Map(c["res"], c["rows"], c["cols"], [dict(name="feat", rule=0, n_channels=c["d"], w=c["w"])])
fr = S.c3_frame(0)
m4.move_to(*fr["move"])
for cl in fr["clouds"]:
    m4.input_pointcloud(torch.from_numpy(cl["points"]).cuda(), [], cl["R"], cl["t"], c3["noise"])
im = S.c4_image(0)
m4.input_image(torch.from_numpy(im["img"]).cuda(), [(0, c["d"], 0)], im["K"], im["R"], im["t"])
out = torch.empty((3, c["rows"], c["cols"]), device="cuda")
for _ in range(3):
    m4.pca_readout("feat", 3, out)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    m4.pca_readout("feat", 3, out)
e1.record()
torch.cuda.synchronize()
print("pca readout us", e0.elapsed_time(e1) / 20 * 1e3)
