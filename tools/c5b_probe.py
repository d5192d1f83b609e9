"""C5b probe: one 2000x2000 map, 4M uniform points per frame -- RED path vs sort path timing."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2309_16818_b200 import mem as M
from synth import scenes as S

c = S.C5B
fr = [S.c5b_shard(f, 0, 1) for f in range(2)]
dev = [torch.from_numpy(f["points"]).cuda() for f in fr]
for sorted_ in (False, True):
    mp = M.Map(c["res"], c["rows"], c["cols"], [dict(name="feat", rule=0, n_channels=1, w=c["w"])], fuse_sorted=sorted_)
    def step(i):
        f = fr[i % 2]
        mp.move_to(*f["move"])
        mp.input_pointcloud(dev[i % 2], [(0, 1, 0)], f["R"], f["t"], c["noise"])
    for i in range(3):
        step(i)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(10):
        step(i)
    e1.record()
    torch.cuda.synchronize()
    print("sorted" if sorted_ else "RED", f"{e0.elapsed_time(e1) / 10 * 1e3:.1f} us per frame")
    mp.close()
