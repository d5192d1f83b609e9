import sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_2309_16818_b200 import mem as M
from synth import scenes as S
c = S.C2
fr = [S.c2_frame(f) for f in range(4)]
dev = [torch.from_numpy(f["points"]).cuda() for f in fr]
mp = M.Map(c["res"], c["rows"], c["cols"], [dict(name="rgb", rule=5, n_channels=3, w=0.5)])
s = torch.cuda.Stream()
M.mem_set_stream(mp.h, s)
def step(i):
    f = fr[i % 4]
    mp.move_to(*f["move"]); mp.input_pointcloud(dev[i % 4], [(0, 1, 0)], f["R"], f["t"], c["noise"])
with torch.cuda.stream(s):
    for i in range(3): step(i)
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=s):
    print("capturing:", torch.cuda.is_current_stream_capturing(), s.cuda_stream, torch.cuda.current_stream().cuda_stream)
    for i in range(4): step(i)
torch.cuda.synchronize()
a0 = np.asarray(mp.get_layer("variance")).copy()
with torch.cuda.stream(s):
    g.replay()
torch.cuda.synchronize()
a1 = np.asarray(mp.get_layer("variance")).copy()
print("changed by replay:", int((np.nan_to_num(a0) != np.nan_to_num(a1)).sum()))
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
with torch.cuda.stream(s):
    e0.record(s); g.replay(); e1.record(s)
e1.synchronize(); print("replay ms (4 frames)", e0.elapsed_time(e1))
