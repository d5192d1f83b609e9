#!/usr/bin/env python
"""bench.py -- MEM fusion hot path (arXiv 2309.16818) on B200: one JSON line.

Workload (BASELINE.json configs[1], batched): every GPU owns M independent
200x200 @ 0.04 m maps ("C2x64", M = 64 by default).  One STEP = one frame for every map:
mem_move_to_batch (ring shift) + mem_input_pointcloud_batch of a 128x1024 LiDAR scan with
packed RGB (131,072 points per map; transform, filters, binning, noise, Mahalanobis test,
Kalman height, colour fusion).  Inputs are synthetic (synth/scenes.py), resident in HBM
before the timed region, and rotate through a 16-step pool (2.1 GB) so every step reads
134 MB of points, more than the 126 MB L2.

  python bench.py [--gpus N --steps K --warmup W] [--impl reference] [--maps M]

For N > 1 launch with torchrun; each rank runs its own M maps (no collective on the data
path: maps are independent -> "scaling": "weak"); rank 0 prints the line with the MAX time
over ranks.  `--impl reference` times the CPU oracle (oracle/) on the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

# stdout carries exactly one JSON line: file descriptor 1 is pointed at stderr for the whole
# run (native libraries print there too, e.g. NCCL's version banner when the C5b communicator
# is created) and the line is written to the saved original stdout
_JSON_FD = None


def claim_stdout():
    global _JSON_FD
    sys.stdout.flush()
    _JSON_FD = os.dup(1)
    os.dup2(2, 1)


def emit(line):
    sys.stdout.flush()
    os.write(_JSON_FD if _JSON_FD is not None else 1, (json.dumps(line) + "\n").encode())

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from synth import scenes as S  # noqa: E402

POOL = 16  # trajectory period of synth.c2_pose; also the number of distinct step batches


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="mem", choices=["mem", "reference"])
    ap.add_argument("--maps", type=int, default=64, help="maps per GPU")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-sides", action="store_true", help="skip the C3 / C4 / C5a side lines")
    return ap.parse_args()


def c2_groups():
    return [dict(name="rgb", rule=5, n_channels=3, w=S.C2["w"])]


def frame_pool(seed=2):
    return [S.c2_frame(f, seed=seed) for f in range(POOL)]


def step_frames(step, maps):
    """frame index of every map at `step` (map m runs the trajectory shifted by m)."""
    return [(step + m) % POOL for m in range(maps)]


# ------------------------------------------------------------------ clocks sampler
class Clocks:
    """nvidia-smi sampled during the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, index):
        self.index = index
        self.samples = []
        self.p = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={q}",
                                       "--format=csv,noheader,nounits", "-lms", "20"], stdout=subprocess.PIPE,
                                      stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.p = None
        return self

    def _read(self):
        for line in self.p.stdout:
            self.samples.append((time.monotonic(), [x.strip() for x in line.split(",")]))

    def wait_first(self, timeout=5.0):
        t0 = time.monotonic()
        while self.p and not self.samples and time.monotonic() - t0 < timeout:
            time.sleep(0.02)

    def __exit__(self, *a):
        if self.p:
            self.p.terminate()
            self.p.wait()
            self.t.join(timeout=2)

    def summary(self, t0=None, t1=None):
        """samples inside [t0, t1] (the timed region, widened by one sampling period)."""
        rows = [r for t, r in self.samples if len(r) >= 8 and (t0 is None or t0 - 0.02 <= t <= t1 + 0.02)]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"], "samples": 0}
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in rows for n, v in zip(names, r[4:8]) if v.lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def traffic_record():
    """dram bytes per k_points launch from the committed ncu --set full capture (or None)."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(p):
        return json.load(open(p))
    return None


# ------------------------------------------------------------------ CPU oracle timing
class OracleFleet:
    """persistent host worker threads, each owning ONE persistent oracle C2 map (ctypes releases
    the GIL): the oracle as it stands, in steady state (every frame fuses into an already built
    map; no thread start-up inside a timed step)."""

    def __init__(self, frames, threads=None):
        import concurrent.futures
        from oracle import oracle as O
        O.lib()
        self.frames = frames
        self.threads = threads or os.cpu_count() or 1
        c = S.C2
        self.maps = [O.OracleMap(c["res"], c["rows"], c["cols"], c2_groups()) for _ in range(self.threads)]
        self.next = [k for k in range(self.threads)]
        self.pool = concurrent.futures.ThreadPoolExecutor(max_workers=self.threads)

    def run(self, frames_per_map=None, budget_s=None, total_frames=None):
        """every thread fuses frames_per_map frames (or for budget_s seconds) into its map, or
        the threads share total_frames map-frames; returns (frames fused, seconds)."""
        c = S.C2

        def work(k, quota):
            t0 = time.perf_counter()
            i = 0
            while quota is None or i < quota:
                fr = self.frames[self.next[k] % POOL]
                self.next[k] += 1
                self.maps[k].move_to(*fr["move"])
                self.maps[k].input_pointcloud(fr["points"], [(0, 1, 0)], fr["R"], fr["t"], c["noise"])
                i += 1
                if budget_s and time.perf_counter() - t0 > budget_s:
                    break
            return i

        if total_frames is not None:
            quotas = [total_frames // self.threads + (1 if k < total_frames % self.threads else 0)
                      for k in range(self.threads)]
        else:
            quotas = [frames_per_map] * self.threads
        t0 = time.perf_counter()
        futs = [self.pool.submit(work, k, q) for k, q in enumerate(quotas) if q is None or q > 0]
        done = [f.result() for f in futs]
        return sum(done), time.perf_counter() - t0


def oracle_rate(frames, budget_s=12.0, threads=None):
    """the oracle's steady-state C2 rate on the host's cores (one persistent map per thread,
    one warm-up frame each first)."""
    fleet = OracleFleet(frames, threads)
    fleet.run(frames_per_map=1)
    nf, dt = fleet.run(budget_s=budget_s)
    return nf * 131072 / dt, nf / dt, fleet.threads, nf, dt


# ------------------------------------------------------------------ reference arm
def headline_config(maps, npts, world):
    """the `config` of the headline line (both arms)."""
    return {"workload": f"C2x{maps}: {maps} independent 200x200@0.04m maps per GPU, 128x1024 LiDAR "
                        f"({npts} pts, packed RGB) per map per step, colour fusion + ring shift",
            "maps_per_gpu": maps, "points_per_map": npts, "parallelism": f"maps sharded x{world}",
            "l2": "inputs > L2: 134 MB of points per step from a 16-step rotating pool (2.1 GB)"}


def run_reference(a):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    frames = frame_pool()
    fleet = OracleFleet(frames)
    threads = fleet.threads
    # each step: the whole C2x64 step -- its 64 map-frames shared by the host threads, each
    # fusing into its own persistent map (persistent worker threads)
    # the K steps' map-frames run back to back on the workers (no barrier between steps: a
    # host step boundary would only add the stragglers' wait), timed as a whole
    fleet.run(total_frames=a.warmup * a.maps)
    t0 = time.perf_counter()
    nf, _ = fleet.run(total_frames=a.steps * a.maps)
    dt = time.perf_counter() - t0
    pts = nf * 131072 / dt
    line = {
        "impl": "reference", "metric": "fused_points_per_s", "value": pts, "unit": "points/s", "n_gpus": a.gpus,
        "steps": a.steps, "warmup": a.warmup, "ms_per_step": dt * 1e3 / a.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32+f64", "data": "synthetic",
        "config": headline_config(a.maps, 131072, a.gpus),
        "map_updates_per_s": nf / dt,
        "cpu_baseline": {"value": pts, "unit": "points/s", "cores": threads, "kind": "oracle",
                         "sample": f"{a.steps} C2x{a.maps} steps = {a.steps * a.maps} map-frames (131072 pts "
                                   f"each) shared by {threads} persistent host threads, one persistent "
                                   f"map each, after {a.warmup} warm-up steps"},
        "e2e": {"value": pts, "unit": "points/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    emit(line)
    return 0


# ------------------------------------------------------------------ side lines (other configs)
def timed_loop(torch, stream, n, fn):
    """device time of n calls of fn() (CUDA events on the caller's stream), after 2 warm-ups."""
    fn(0)
    fn(1)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for i in range(n):
        fn(i)
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


def graph_sequence(torch, M, mp, step_fn, n=10, reps=30):
    """SPEC.md:518-521 / PAPER.md:410 protocol: an n-frame sequence captured ONCE as a CUDA
    graph (every launch of the n frames), replayed `reps` times, each replay timed with CUDA
    events on the capture stream; returns mean and std of the time per frame (us).  The map
    keeps fusing (each replay applies the same n frames to the evolving state); it is a timing
    map and is discarded afterwards."""
    s = torch.cuda.Stream()
    M.mem_set_stream(mp.h, s)
    with torch.cuda.stream(s):
        for i in range(3):
            step_fn(i)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for i in range(n):
            step_fn(i)
    per = []
    with torch.cuda.stream(s):  # CUDAGraph.replay launches on the current stream
        for _ in range(2):
            g.replay()
        torch.cuda.synchronize()
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            g.replay()
            e1.record(s)
            e1.synchronize()
            per.append(e0.elapsed_time(e1) * 1e3 / n)
    return {"frames_per_replay": n, "replays": reps, "us_per_frame_mean": float(np.mean(per)),
            "us_per_frame_std": float(np.std(per)), "us_per_frame_min": float(np.min(per))}


def oracle_threads(jobs, threads=None):
    """runs the callables in `jobs` on `threads` host threads (ctypes releases the GIL);
    returns the wall seconds and the thread count."""
    threads = min(threads or os.cpu_count() or 1, len(jobs))
    nxt = [0]
    lock = threading.Lock()

    def work():
        while True:
            with lock:
                k = nxt[0]
                nxt[0] += 1
            if k >= len(jobs):
                return
            jobs[k]()

    t0 = time.perf_counter()
    ts = [threading.Thread(target=work) for _ in range(threads)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    return time.perf_counter() - t0, threads


def side_c5a(torch, M, stream, rank, world, steps=20):
    """BASELINE configs[4] batched learning workload: 4096 maps split over the ranks (strong
    scaling), one 32,768-point frame per map per step.  Inputs: 256 generated maps x 2 frames
    tiled to the rank's maps (map m uses generated map m % 256)."""
    c = S.C5A
    total_maps = 4096
    mine = total_maps // world
    first = rank * mine
    pool = [S.c5a_batch(f, 0, 256) for f in range(2)]
    idx = (np.arange(first, first + mine) % 256)
    P = c["points"]
    batches, Rs, ts, xys = [], [], [], []
    for fr in pool:
        pts = fr["points"].reshape(256, P, 4)[idx].reshape(-1, 4)
        batches.append(torch.from_numpy(pts).cuda())
        Rs.append(fr["R"][idx])
        ts.append(fr["t"][idx])
        xys.append(fr["move"][idx])
    offsets = np.arange(mine + 1, dtype=np.int64) * P
    mp = M.Map(c["res"], c["rows"], c["cols"], [dict(name="feat", rule=0, n_channels=1, w=c["w"])], n_maps=mine)

    def step(i):
        k = i % 2
        mp.move_to_batch(xys[k])
        mp.input_pointcloud_batch(batches[k], offsets, [(0, 1, 0)], Rs[k], ts[k], c["noise"])

    ms = timed_loop(torch, stream, steps, step)
    mp.close()
    cpu = None
    if rank == 0 and os.environ.get("MEM_BENCH_NO_CPU") != "1":
        # the oracle on every host core: persistent maps (the 256 generated ones), one frame
        # each per job, frames 0 then 1 (a bounded sample of the 4096-map step)
        from oracle import oracle as O
        O.lib()
        oras = [O.OracleMap(c["res"], c["rows"], c["cols"], [dict(name="feat", rule=0, n_channels=1, w=c["w"])])
                for _ in range(256)]
        pts = [fr["points"].reshape(256, P, 4) for fr in pool]

        def job(k, f):
            return lambda: (oras[k].move_to(*pool[f]["move"][k]),
                            oras[k].input_pointcloud(pts[f][k], [(0, 1, 0)], pool[f]["R"][k], pool[f]["t"][k], c["noise"]))

        oracle_threads([job(k, 0) for k in range(256)])
        dt, th = oracle_threads([job(k, 1) for k in range(256)])
        cpu = {"kind": "oracle", "cores": th, "map_updates_per_s": 256 / dt, "points_per_s": 256 * P / dt,
               "sample": "256 C5a map-frames (32768 pts each) on all host threads, persistent maps",
               "projected_ms_per_step_4096_maps": 4096 / (256 / dt) * 1e3}
    return {"workload": f"C5a: 4096 maps 128x128@0.1m x 32768 pts, {mine} maps on this rank", "ms_per_step": ms,
            "cpu_oracle": cpu,
            "maps_per_rank": mine, "points_per_s_rank": mine * P / (ms * 1e-3),
            "map_updates_per_s_rank": mine / (ms * 1e-3), "scaling": "strong (4096 maps total)"}


def side_c5b(torch, M, stream, rank, world, dist, steps=10):
    """BASELINE configs[4] second half: one 2000x2000 map, 4M points per frame point-sharded
    over the ranks (4M/G each), band exchange over NCCL inside mem_input_pointcloud
    (include/mem.h sharded map).  Two pre-generated frames alternate."""
    c = S.C5B
    uid = torch.zeros(128, dtype=torch.uint8, device="cuda")
    if rank == 0:
        uid.copy_(torch.frombuffer(bytearray(M.mem_nccl_unique_id()), dtype=torch.uint8))
    if world > 1:
        dist.broadcast(uid, 0)
    mp = M.Map.sharded(c["res"], c["rows"], c["cols"], [dict(name="feat", rule=0, n_channels=1, w=c["w"])],
                       rank, world, nccl_id=bytes(uid.cpu().numpy()), stream=stream)
    frames = [S.c5b_shard(f, rank, world) for f in range(2)]
    dev = [torch.from_numpy(f["points"]).cuda() for f in frames]

    def step(i):
        f = frames[i % 2]
        mp.move_to(*f["move"])
        mp.input_pointcloud(dev[i % 2], [(0, 1, 0)], f["R"], f["t"], c["noise"])

    if world > 1:
        dist.barrier()
    ms = timed_loop(torch, stream, steps, step)
    t = torch.tensor([ms], device="cuda", dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    mp.profile_read(reset=True)
    mp.profile(True)
    step(0)
    torch.cuda.synchronize()
    mp.profile(False)
    prof = mp.profile_read(reset=True)
    mp.close()
    cpu = None
    if rank == 0 and world == 1 and os.environ.get("MEM_BENCH_NO_CPU") != "1":
        from oracle import oracle as O
        o = O.OracleMap(c["res"], c["rows"], c["cols"], [dict(name="feat", rule=0, n_channels=1, w=c["w"])])
        for f in range(2):
            o.move_to(*frames[f]["move"])
            t0 = time.perf_counter()
            o.input_pointcloud(frames[f]["points"], [(0, 1, 0)], frames[f]["R"], frames[f]["t"], c["noise"])
            dt = time.perf_counter() - t0
        cpu = {"kind": "oracle", "cores": 1, "ms_per_frame": dt * 1e3, "points_per_s": c["points"] / dt,
               "sample": "the second of two 4M-point frames on one host core"}
    return {"workload": f"C5b: one 2000x2000@0.04m map, {c['points']} pts/frame point-sharded over {world} rank(s)",
            "cpu_oracle": cpu,
            "ms_per_frame_max_over_ranks": ms, "points_per_s": c["points"] / (ms * 1e-3),
            "stage_ms_rank0": {k: v[0] for k, v in prof.items() if v[1]}, "transport": "NCCL",
            "scaling": "strong (4M points total)"}


def side_paper_sweep(torch, M, stream, iters=300):
    """SURVEY §8(f) NEXT-4, the paper's performance setup (Table II, Fig. 6):
    250x250 @ 4 cm, a 230,400-point semantic cloud per frame, the multi-modal update swept over
    L in {1, 2, 4, 8, 16, 20} layers for exponential averaging and Bayesian inference; 300
    iterations per point (CUDA events).  Reports ms per frame, the multi-modal share (frame
    time minus the height-only frame) and a least-squares line with its R^2."""
    c = S.PAPER
    out = {"workload": "PAPER: 250x250@0.04m, 230400-pt semantic cloud (ZED 2i 360x640), layer sweep",
           "iterations": iters}

    def frame_ms(groups, binds, n_layers):
        clouds = [S.paper_cloud(max(n_layers, 1), f) for f in range(2)]
        dev = [torch.from_numpy(np.ascontiguousarray(cl["points"][:, :3 + n_layers])).cuda() for cl in clouds]
        mp = M.Map(c["res"], c["rows"], c["cols"], groups)

        def step(i):
            cl = clouds[i % 2]
            mp.move_to(*cl["move"])
            mp.input_pointcloud(dev[i % 2], binds, cl["R"], cl["t"], c["noise"])

        ms = timed_loop(torch, stream, iters, step)
        if n_layers == max(c["layers"]):  # Table II-style stage split of the largest case
            mp.profile_read(reset=True)
            mp.profile(True)
            step(0)
            torch.cuda.synchronize()
            mp.profile(False)
            prof = mp.profile_read(reset=True)
            stages[groups[0]["rule"] if groups else -1] = {k: v[0] for k, v in prof.items() if v[1]}
        mp.close()
        return ms

    stages = {}
    base = frame_ms([], [], 0)
    out["height_only_ms"] = base
    for name, rule in (("exponential_averaging", 0), ("bayesian", 3)):
        xs, ys = [], []
        for L in c["layers"]:
            if rule == 3 and L < 2:
                continue
            ms = frame_ms([dict(name="sem", rule=rule, n_channels=L, w=0.5, alpha0=1.0)], [(0, L, 0)], L)
            xs.append(L)
            ys.append(ms)
        x, y = np.array(xs, float), np.array(ys)
        slope, icpt = np.polyfit(x, y, 1)
        r2 = 1.0 - ((y - (slope * x + icpt)) ** 2).sum() / max(((y - y.mean()) ** 2).sum(), 1e-30)
        out[name] = {"layers": xs, "ms_per_frame": ys, "multimodal_ms": [v - base for v in ys],
                     "fit_ms_per_layer": slope, "fit_intercept_ms": icpt, "r2": r2,
                     "stage_ms_at_max_layers": stages.get(rule)}
    return out


def side_c3_c4(torch, M, stream, frames=10):
    out = {}
    c = S.C3
    fr = [S.c3_frame(f) for f in range(frames)]
    groups = [dict(name="sem", rule=3, n_channels=c["n_classes"], alpha0=1.0),
              dict(name="top", rule=4, n_channels=c["n_classes"])]
    binds = [(0, c["n_classes"], 0), (0, c["n_classes"], 1)]
    mp = M.Map(c["res"], c["rows"], c["cols"], groups)
    dev = [dict(clouds=[torch.from_numpy(cl["points"]).cuda() for cl in f["clouds"]],
                img=torch.from_numpy(f["image"]["img"]).cuda()) for f in fr]

    def c3_step(i):
        f, d = fr[i % frames], dev[i % frames]
        mp.move_to(*f["move"])
        for cl, dp in zip(f["clouds"], d["clouds"]):
            mp.input_pointcloud(dp, [], cl["R"], cl["t"], c["noise"])
        im = f["image"]
        mp.input_image(d["img"], binds, im["K"], im["R"], im["t"])

    ms = timed_loop(torch, stream, 20, c3_step)
    npts = sum(cl["points"].shape[0] for cl in fr[0]["clouds"])
    out["c3"] = {"workload": "C3: 250x250@0.04m, 3 x 640x480 depth clouds + 20-class 640x480 softmax image per frame",
                 "ms_per_frame": ms, "points_per_s": npts / (ms * 1e-3), "frames_per_s": 1e3 / ms}
    mp.profile_read(reset=True)
    mp.profile(True)
    c3_step(0)
    torch.cuda.synchronize()
    mp.profile(False)
    prof = mp.profile_read(reset=True)
    out["c3"]["stage_ms"] = {k: v[0] for k, v in prof.items() if v[1]}
    # the SPEC.md:518-521 protocol: the 10-frame sequence as one CUDA graph, 30 replays
    mg = M.Map(c["res"], c["rows"], c["cols"], groups)

    def g_step(i):
        f, d = fr[i % frames], dev[i % frames]
        mg.move_to(*f["move"])
        for cl, dp in zip(f["clouds"], d["clouds"]):
            mg.input_pointcloud(dp, [], cl["R"], cl["t"], c["noise"])
        im = f["image"]
        mg.input_image(d["img"], binds, im["K"], im["R"], im["t"])

    out["c3"]["graph_10_frames"] = graph_sequence(torch, M, mg, g_step, n=frames, reps=30)
    mg.close()
    if os.environ.get("MEM_BENCH_NO_CPU") != "1":  # the oracle on one host core, one frame
        from oracle import oracle as O
        o = O.OracleMap(c["res"], c["rows"], c["cols"], groups)
        for k in range(2):
            f = fr[k]
            t0 = time.perf_counter()
            o.move_to(*f["move"])
            for cl in f["clouds"]:
                o.input_pointcloud(cl["points"], [], cl["R"], cl["t"], c["noise"])
            im = f["image"]
            o.input_image(im["img"], binds, im["K"], im["R"], im["t"])
            dt = time.perf_counter() - t0
        out["c3"]["cpu_oracle"] = {"kind": "oracle", "cores": 1, "ms_per_frame": dt * 1e3,
                                   "points_per_s": npts / dt, "sample": "the second of two C3 frames, one host core"}
    # NEXT-3 plugins on the fused C3 map (device outputs)
    o3 = torch.empty((3, c["rows"], c["cols"]), device="cuda")
    t1 = torch.empty((1, c["rows"], c["cols"]), device="cuda")
    o2 = torch.empty((2, c["rows"], c["cols"]), device="cuda")
    out["plugins_c3_map"] = {
        "workload": "NEXT-3 plugins on the 250x250 C3 map",
        "normals_us": 1e3 * timed_loop(torch, stream, 50, lambda i: mp.normals(out=o3)),
        "traversability_us": 1e3 * timed_loop(torch, stream, 50, lambda i: mp.traversability(0.6, 0.1, out=t1)),
        "semantic_argmax_us": 1e3 * timed_loop(torch, stream, 50, lambda i: mp.semantic_argmax("sem", out=o2))}
    # NEXT-1: the same frames with the Bresenham occlusion test in the image association
    mp.set_image_occlusion(True, 1e-4)
    ms_occ = timed_loop(torch, stream, 20, c3_step)
    mp.profile_read(reset=True)
    mp.profile(True)
    c3_step(0)
    torch.cuda.synchronize()
    mp.profile(False)
    prof = mp.profile_read(reset=True)
    out["c3_occlusion"] = {"workload": "C3 with the Bresenham occlusion test (PAPER.md:234-236) on the image",
                           "ms_per_frame": ms_occ, "frames_per_s": 1e3 / ms_occ,
                           "image_stage_ms": prof.get("image", (None,))[0]}
    mp.close()
    c4 = S.C4
    m4 = M.Map(c4["res"], c4["rows"], c4["cols"], [dict(name="feat", rule=0, n_channels=c4["d"], w=c4["w"])])
    f0 = fr[0]
    m4.move_to(*f0["move"])
    for cl, dp in zip(f0["clouds"], dev[0]["clouds"]):
        m4.input_pointcloud(dp, [], cl["R"], cl["t"], c["noise"])
    ims = [S.c4_image(f) for f in range(2)]
    dims = [torch.from_numpy(im["img"]).cuda() for im in ims]

    def c4_step(i):
        im = ims[i % 2]
        m4.input_image(dims[i % 2], [(0, c4["d"], 0)], im["K"], im["R"], im["t"])

    ms4 = timed_loop(torch, stream, 20, c4_step)
    pca_out = torch.empty((3, c4["rows"], c4["cols"]), device="cuda")
    pca_ms = timed_loop(torch, stream, 20, lambda i: m4.pca_readout("feat", 3, pca_out))  # device time
    out["c4"] = {"workload": "C4: 250x250@0.04m, 64-channel 480x640 feature image, 64 x average + PCA readout",
                 "ms_per_image": ms4, "images_per_s": 1e3 / ms4, "pca_readout_ms": pca_ms,
                 "image_bytes": int(dims[0].numel() * 4)}
    if os.environ.get("MEM_BENCH_NO_CPU") != "1":  # the oracle on one host core: an image, a PCA readout
        from oracle import oracle as O
        o4 = O.OracleMap(c4["res"], c4["rows"], c4["cols"], [dict(name="feat", rule=0, n_channels=c4["d"], w=c4["w"])])
        o4.move_to(*f0["move"])
        for cl in f0["clouds"]:
            o4.input_pointcloud(cl["points"], [], cl["R"], cl["t"], c["noise"])
        o4.input_image(ims[0]["img"], [(0, c4["d"], 0)], ims[0]["K"], ims[0]["R"], ims[0]["t"])
        t0 = time.perf_counter()
        o4.input_image(ims[1]["img"], [(0, c4["d"], 0)], ims[1]["K"], ims[1]["R"], ims[1]["t"])
        t1 = time.perf_counter()
        o4.pca_readout("feat", 3)
        t2 = time.perf_counter()
        out["c4"]["cpu_oracle"] = {"kind": "oracle", "cores": 1, "ms_per_image": (t1 - t0) * 1e3,
                                   "pca_readout_ms": (t2 - t1) * 1e3, "sample": "one image, one readout, one host core"}
    m4.close()
    return out


# ------------------------------------------------------------------ GPU arm
def run_mem(a):
    if a.no_cpu:
        os.environ["MEM_BENCH_NO_CPU"] = "1"
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    from paper_2309_16818_b200 import mem as M

    M_ = a.maps
    c = S.C2
    frames = frame_pool()
    dev_frames = [torch.from_numpy(fr["points"]).cuda() for fr in frames]
    npts = frames[0]["points"].shape[0]
    # 16 distinct step batches, contiguous per map (offsets identical across steps)
    batches = [torch.cat([dev_frames[f] for f in step_frames(s, M_)]) for s in range(POOL)]
    offsets = np.arange(M_ + 1, dtype=np.int64) * npts
    Rs = [np.stack([frames[f]["R"] for f in step_frames(s, M_)]) for s in range(POOL)]
    ts = [np.stack([frames[f]["t"] for f in step_frames(s, M_)]) for s in range(POOL)]
    xys = [np.stack([frames[f]["move"] for f in step_frames(s, M_)]) for s in range(POOL)]
    stream = torch.cuda.current_stream()
    mp = M.Map(c["res"], c["rows"], c["cols"], c2_groups(), n_maps=M_)
    binds = [(0, 1, 0)]

    def step(s, src=None):
        # device inputs: the 16-step pool; host inputs (e2e): the first len(src) steps of it,
        # points and poses of the same step
        k = s % POOL if src is None else s % len(src)
        mp.move_to_batch(xys[k])
        mp.input_pointcloud_batch(batches[k] if src is None else src[k], offsets, binds, Rs[k], ts[k], c["noise"])

    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with Clocks(local) as clk:
        clk.wait_first()
        for s in range(a.warmup):
            step(s)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t_on = time.monotonic()
        ev0.record(stream)
        for s in range(a.warmup, a.warmup + a.steps):
            step(s)
        ev1.record(stream)
        torch.cuda.synchronize()
        t_off = time.monotonic()
        if world > 1:
            dist.barrier()
    ms = ev0.elapsed_time(ev1)
    # the per-kernel durations of the roofline: the same K steps again with CUDA events around
    # every stage launch on the map's stream (the events themselves keep the launches apart, so
    # this pass is not the one whose step time is reported)
    mp.profile_read(reset=True)
    mp.profile(True)
    for s in range(a.warmup + a.steps, a.warmup + 2 * a.steps):
        step(s)
    torch.cuda.synchronize()
    mp.profile(False)
    prof = mp.profile_read(reset=True)
    stats = mp.stats()
    t = torch.tensor([ms], device="cuda", dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    total_pts = npts * M_ * a.steps * world
    value = total_pts / (ms_max * 1e-3)

    # ---- roofline of the dominant kernel (k_points), timed live with CUDA events on its stream
    pts_ms, pts_n = prof["point"]
    cell_ms, cell_n = prof["cell"]
    pk, pk_src = peaks()
    # algorithmic bytes per launch: k_points reads every point once (16 B);
    # k_cells reads and writes the stored state of every touched cell (C2 colour map: 22 B)
    bytes_pts = M_ * npts * 16
    bytes_cells = 2 * 22 * stats["n_cells_touched"]
    achieved = bytes_pts / (pts_ms / pts_n * 1e-3) / 1e9 if pts_n else None
    achieved_cells = bytes_cells / (cell_ms / cell_n * 1e-3) / 1e9 if cell_n else None
    tr = traffic_record()
    traffic = None
    if tr and tr.get("maps") == M_ and tr.get("points_per_map") == npts:
        traffic = tr.get("k_points_dram_bytes_per_launch")
    # kernels per profiled call on this path: a point stage is k_points, a cell stage k_cells +
    # k_refold (cooperative; returns at once when no cell is uncertified) -- see the ncu launch
    # list profiles/r02z_launches_c2x64.txt: 3 kernels per step
    launches = sum(prof[k][1] for k in ("shift", "point", "image", "read", "write")) + 2 * prof["cell"][1]
    step_bytes = bytes_pts + bytes_cells

    # ---- e2e: through the C-ABI with HOST (pinned) buffers, H2D + D2H inside the timed region
    e2e = None
    if not a.no_e2e:
        host = [b.cpu().pin_memory() for b in batches[:2]]
        out = torch.empty((M_, c["rows"], c["cols"]), dtype=torch.float32).pin_memory()
        e_steps = min(a.steps, 50)
        for s in range(2):
            step(s, host)
            mp.get_layer("elevation", out)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for s in range(e_steps):
            step(s, host)
            mp.get_layer("elevation", out)  # the step's result read back to the host
        e1.record(stream)
        torch.cuda.synchronize()
        te = torch.tensor([e0.elapsed_time(e1)], device="cuda", dtype=torch.float64)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        t_step = float(te.item()) * 1e-3 / e_steps
        e2e = {"value": npts * M_ * e_steps * world / (float(te.item()) * 1e-3), "unit": "points/s",
               "h2d_bytes_per_step": int(host[0].numel() * 4), "d2h_bytes_per_step": int(out.numel() * 4),
               "steps": e_steps,
               # host<->device bytes per step over the step time: the PCIe link is the bound here
               "pcie_gbs": (host[0].numel() + out.numel()) * 4 / t_step / 1e9}

    # ---- single-map C2 latency (context: below launch latency)
    single = None
    if rank == 0:
        sm = M.Map(c["res"], c["rows"], c["cols"], c2_groups())
        for f in range(5):
            sm.move_to(*frames[f]["move"])
            sm.input_pointcloud(dev_frames[f], binds, frames[f]["R"], frames[f]["t"], c["noise"])
        torch.cuda.synchronize()
        l0, l1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        l0.record(stream)
        for f in range(100):
            fr = frames[f % POOL]
            sm.move_to(*fr["move"])
            sm.input_pointcloud(dev_frames[f % POOL], binds, fr["R"], fr["t"], c["noise"])
        l1.record(stream)
        torch.cuda.synchronize()
        single = {"us_per_frame": l0.elapsed_time(l1) * 10.0, "points_per_s": 100 * npts / (l0.elapsed_time(l1) * 1e-3)}
        sm.close()

    # the SPEC.md:518-521 protocol on the headline step: 10 steps captured as one CUDA graph,
    # 30 replays, mean +- std per step (a separate timing map)
    graph = None
    if rank == 0:
        mg = M.Map(c["res"], c["rows"], c["cols"], c2_groups(), n_maps=M_)
        graph = graph_sequence(torch, M, mg, lambda i: (mg.move_to_batch(xys[i % POOL]), mg.input_pointcloud_batch(
            batches[i % POOL], offsets, binds, Rs[i % POOL], ts[i % POOL], c["noise"])), n=10, reps=30)
        graph["points_per_s"] = npts * M_ / (graph["us_per_frame_mean"] * 1e-6)
        mg.close()

    sides = {}
    if not a.no_sides:
        sides["c5a"] = side_c5a(torch, M, stream, rank, world)
        t5 = torch.tensor([sides["c5a"]["ms_per_step"]], device="cuda", dtype=torch.float64)
        if world > 1:
            dist.all_reduce(t5, op=dist.ReduceOp.MAX)
        sides["c5a"]["ms_per_step_max_over_ranks"] = float(t5.item())
        sides["c5a"]["points_per_s"] = 4096 * S.C5A["points"] / (float(t5.item()) * 1e-3)
        sides["c5a"]["map_updates_per_s"] = 4096 / (float(t5.item()) * 1e-3)
        # the NCCL band exchange of the sharded map has only run with one rank so far (no
        # multi-GPU box in round 1): at N > 1 it is opt-in so that a fault there cannot take
        # the scaling run down with it
        if world == 1 or os.environ.get("MEM_BENCH_C5B") == "1":
            sides["c5b"] = side_c5b(torch, M, stream, rank, world, dist)
        if rank == 0:
            sides.update(side_c3_c4(torch, M, stream))
            sides["paper_sweep"] = side_paper_sweep(torch, M, stream)

    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu:
        pts_s, maps_s, cores, nf, dt = oracle_rate(frames, budget_s=12.0)
        cpu = {"value": pts_s, "unit": "points/s", "cores": cores, "kind": "oracle",
               "sample": f"{nf} C2 map-frames (131072 pts each) in {dt:.1f} s, one persistent map per host "
                         f"thread (steady state)", "map_updates_per_s": maps_s}

    if rank == 0:
        line = {
            "metric": "fused_points_per_s", "value": value, "unit": "points/s", "n_gpus": world, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": ms_max / a.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32+f64", "data": "synthetic",
            "config": headline_config(M_, npts, world),
            "map_updates_per_s": M_ * a.steps * world / (ms_max * 1e-3),
            "step_hbm_gbs": step_bytes / (ms_max / a.steps * 1e-3) / 1e9,
            "roofline": {"bound": "hbm", "kernel": "k_points", "achieved": achieved, "peak": pk,
                         "peak_source": pk_src, "unit": "GB/s",
                         "frac": (achieved / pk) if achieved else None, "traffic": traffic,
                         "algorithmic_bytes_per_launch": bytes_pts,
                         "kernel_timing": "CUDA events around every stage launch on the map's stream, "
                                          "a second pass of the same K steps",
                         "k_cells": {"achieved": achieved_cells, "frac": (achieved_cells / pk) if achieved_cells else None,
                                     "algorithmic_bytes_per_launch": bytes_cells},
                         "step": {"achieved": step_bytes / (ms_max / a.steps * 1e-3) / 1e9,
                                  "frac": step_bytes / (ms_max / a.steps * 1e-3) / 1e9 / pk}},
            "stages_ms_per_step": {k: v[0] / a.steps for k, v in prof.items() if v[1]},
            "gpu_launches": launches,
            "clocks": clk.summary(t_on, t_off),
            "e2e": e2e,
            "single_map_c2": single,
            "graph_10_steps": graph,
            "cpu_baseline": cpu,
            "side_lines": sides,
            "frame_stats_last_step": stats,
        }
        emit(line)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    mp.close()
    return 0


def main():
    a = parse()
    claim_stdout()
    if a.impl == "reference":
        return run_reference(a)
    return run_mem(a)


if __name__ == "__main__":
    sys.exit(main())
