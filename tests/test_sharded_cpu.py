"""CPU (gloo, world size 2 and 3) check of the sharded big map's decomposition (SURVEY §8(e)
C5b, include/mem.h "one big map sharded across ranks").

Each rank accumulates the statistics of its own shard of every frame's points against the
shared pre-frame state (oracle om_accumulate = steps 1-2 of SURVEY §8(c) N2), the statistics
are combined across ranks (sums for counts and f64 sums, max for class_max keys -- the merge
the library's k_merge does on the band each rank owns), each rank fuses its own row band
(om_fuse_rows = step 3) and the bands are all-gathered.  After every frame each rank's map
must equal one unsharded oracle fed all the points: integer layers and counters exactly,
fp32 layers within the north_star tolerance (the f64 sums are re-associated).

The second protocol (point routing, the library's default for sharded maps) is checked the
same way: points are sent to the owner of their cell's band and fused there, in global input
order, so the maps must equal the unsharded oracle bit for bit.
"""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

from oracle import oracle as O  # noqa: E402
from synth import scenes as S  # noqa: E402

GROUPS = [
    dict(name="feat", rule=O.AVERAGE, n_channels=3, w=0.5),
    dict(name="gf", rule=O.GAUSSIAN, n_channels=2, sigma_f2=0.2, mu0=0.1, sigma0_2=1.5),
    dict(name="cavg", rule=O.CLASS_AVERAGE, n_channels=4, w=0.3),
    dict(name="sem", rule=O.CLASS_BAYESIAN, n_channels=4, alpha0=1.0),
    dict(name="top", rule=O.CLASS_MAX, n_channels=4),
    dict(name="rgb", rule=O.COLOR, n_channels=3, w=0.5),
]
BINDS = [(0, 3, 0), (3, 2, 1), (5, 4, 2), (5, 4, 3), (5, 4, 4), (9, 1, 5)]
NOISE = dict(a=1e-3, b=1e-4, r_min=0.05, r_max=6.0, h_min=-3.0, h_max=1.0, tau2=4.0, v_out=0.02)
ROWS, COLS, RES = 36, 28, 0.1
LAYERS = (["elevation", "variance", "valid"] + [f"feat_{k}" for k in range(3)] + ["feat_observed"] +
          [f"gf_{k}" for k in range(2)] + [f"gf_var_{k}" for k in range(2)] + ["gf_observed"] +
          [f"cavg_{k}" for k in range(4)] + ["cavg_observed"] + [f"sem_alpha_{k}" for k in range(4)] +
          ["sem_observed", "top_label", "top_conf", "rgb_r", "rgb_g", "rgb_b", "rgb_observed"])
SIGN = np.uint64(1 << 63)


def cloud(f):
    rng = np.random.default_rng(900 + f)
    n = 4000 + 97 * f
    pts = S.random_cloud(900 + f, n, 13, ROWS, COLS, RES)
    p = rng.dirichlet(np.ones(4) * 0.7, n)
    tie = rng.uniform(size=n) < 0.1
    p[tie] = np.round(p[tie] * 4) / 4
    pts[:, 8:12] = p.astype(np.float32)
    pts[:, 12] = S.pack_rgb(rng.integers(0, 256, (n, 3)).astype(np.uint8))
    outl = rng.uniform(size=n) < 0.05
    pts[outl, 2] += 1.5
    return pts


def combine(arr, op):
    """in-place cross-rank merge of one statistics array (a numpy view into the oracle frame)."""
    if arr is None:
        return
    if arr.dtype == np.uint64:
        if op == "max":  # u64 order == int64 order of (x ^ 2^63)
            arr ^= SIGN
        t = torch.from_numpy(arr.view(np.int64))
        dist.all_reduce(t, op=dist.ReduceOp.MAX if op == "max" else dist.ReduceOp.SUM)
        if op == "max":
            arr ^= SIGN
    else:
        dist.all_reduce(torch.from_numpy(arr), op=dist.ReduceOp.SUM)


def worker(rank, world, port, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        shard = O.OracleMap(RES, ROWS, COLS, GROUPS)
        full = O.OracleMap(RES, ROWS, COLS, GROUPS)
        band = ROWS // world
        lo, hi = rank * band, (rank + 1) * band
        moves = [(0.0, 0.0), (0.15, -0.1), (0.4, 0.2), (0.4, 0.2), (-1.0, 0.5), (-0.95, 0.55)]
        worst = 0.0
        for f, (x, y) in enumerate(moves):
            shard.move_to(x, y)
            full.move_to(x, y)
            pts = cloud(f)
            cuts = np.linspace(0, len(pts), world + 1).astype(int)
            if f == 2:  # one rank without points
                cuts[1:] = np.maximum(cuts[1:], cuts[1]); cuts[1] = 0
            R, t = S.rot_z(0.4 * f), np.array([x + 0.02, y - 0.01, 1.0])
            fr = shard.accumulate(pts[cuts[rank]:cuts[rank + 1]], BINDS, R, t, NOISE)
            for arr, op in fr.arrays():
                combine(arr, op)
            cnt = torch.from_numpy(fr.counters.view(np.int64))
            dist.all_reduce(cnt)
            shard.fuse_rows(fr, lo, hi)
            for nm in LAYERS:  # all-gather the owned bands
                mine = torch.from_numpy(np.ascontiguousarray(shard.get_layer(nm)[lo:hi]))
                parts = [torch.empty_like(mine) for _ in range(world)]
                dist.all_gather(parts, mine)
                shard.set_layer(nm, torch.cat(parts).numpy())
            full.input_pointcloud(pts, BINDS, R, t, NOISE)
            st = np.array([shard.stats()[k] for k in O.STAT_NAMES], np.int64)
            touched = torch.tensor([st[7]])
            dist.all_reduce(touched)
            st[7] = int(touched[0])
            assert list(st) == [full.stats()[k] for k in O.STAT_NAMES], (f, st, full.stats())
            for nm in LAYERS:
                a, b = shard.get_layer(nm), full.get_layer(nm)
                assert np.array_equal(np.isnan(a), np.isnan(b)), (f, nm)
                if nm == "valid" or nm.endswith(("_observed", "_label")):
                    assert np.array_equal(a, b), (f, nm)
                else:
                    fin = ~np.isnan(b)
                    d = np.abs(a[fin].astype(np.float64) - b[fin])
                    assert np.all(d <= 1e-6 + 1e-5 * np.abs(b[fin])), (f, nm, d.max())
                    worst = max(worst, float(d.max()) if d.size else 0.0)
        assert full.get_layer("valid").sum() > 200
        dist.destroy_process_group()
        q.put((rank, "ok", worst))
    except Exception as e:  # report to the parent instead of hanging the other rank
        q.put((rank, f"{type(e).__name__}: {e}", None))
        raise


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world", [2, 3])
def test_band_decomposition_equals_unsharded(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    bad = [r for r in results if r[1] != "ok"]
    assert not bad, bad
    assert all(p.exitcode == 0 for p in procs)


def worker_route(rank, world, port, q):
    """point routing: each rank bins its shard, sends every in-window point to the owner of its
    cell's row band (all_gather_object), the owner accumulates what it received -- in rank order,
    i.e. the global input order -- and fuses its band; bands all-gathered.  Because every cell's
    points are summed in input order, the maps equal the unsharded oracle bit for bit."""
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        shard = O.OracleMap(RES, ROWS, COLS, GROUPS)
        full = O.OracleMap(RES, ROWS, COLS, GROUPS)
        band = ROWS // world
        lo, hi = rank * band, (rank + 1) * band
        moves = [(0.0, 0.0), (0.15, -0.1), (0.4, 0.2), (-1.0, 0.5)]
        for f, (x, y) in enumerate(moves):
            shard.move_to(x, y)
            full.move_to(x, y)
            pts = cloud(f)
            cuts = np.linspace(0, len(pts), world + 1).astype(int)
            R, t = S.rot_z(0.4 * f), np.array([x + 0.02, y - 0.01, 1.0])
            mine = pts[cuts[rank]:cuts[rank + 1]]
            fr, cell, code = shard.accumulate(mine, BINDS, R, t, NOISE, cells=True)
            drops = np.array([int(fr.counters[k]) for k in range(8)], np.int64)  # codes 1-4: this rank's drops
            owner = np.where(cell >= 0, (cell // COLS) // band, -1)
            out = [mine[owner == d] for d in range(world)]
            got = [None] * world
            dist.all_gather_object(got, out)
            recv = np.concatenate([got[p][rank] for p in range(world)])
            fo = shard.accumulate(recv, BINDS, R, t, NOISE)
            shard.fuse_rows(fo, lo, hi)
            for nm in LAYERS:
                part = torch.from_numpy(np.ascontiguousarray(shard.get_layer(nm)[lo:hi]))
                parts = [torch.empty_like(part) for _ in range(world)]
                dist.all_gather(parts, part)
                shard.set_layer(nm, torch.cat(parts).numpy())
            full.input_pointcloud(pts, BINDS, R, t, NOISE)
            st = shard.stats()
            mix = torch.tensor([drops[1], drops[2], drops[3], drops[4], st["n_inlier"], st["n_outlier"],
                                st["n_cells_touched"]], dtype=torch.int64)
            dist.all_reduce(mix)
            fs = full.stats()
            assert mix.tolist() == [fs["n_nonfinite"], fs["n_range"], fs["n_height"], fs["n_oob"], fs["n_inlier"],
                                    fs["n_outlier"], fs["n_cells_touched"]], (f, mix.tolist(), fs)
            for nm in LAYERS:
                a, b = shard.get_layer(nm), full.get_layer(nm)
                assert np.array_equal(a, b, equal_nan=True), (f, nm)
        dist.destroy_process_group()
        q.put((rank, "ok", 0.0))
    except Exception as e:
        q.put((rank, f"{type(e).__name__}: {e}", None))
        raise


@pytest.mark.parametrize("world", [2, 3])
def test_point_routing_equals_unsharded_bit_for_bit(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=worker_route, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    bad = [r for r in results if r[1] != "ok"]
    assert not bad, bad
