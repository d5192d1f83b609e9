"""GPU parity of the sharded big map against the CPU oracle.

One map, its points split across G shards (ragged, one shard sometimes empty).  The local
transport runs all G shards in this process on one device (include/mem.h); after each input
mem_shard_local_sync exchanges the row bands, merges and fuses them, and replicates the
state, so every shard must hold the map the oracle computes from all the points:
integer layers bit-exact, fp32 within the north_star tolerance (sums are re-associated
across shards).  The NCCL transport is exercised with one rank (the multi-rank exchange is
the same band protocol; its host-side decomposition is covered on CPU by test_sharded_cpu).
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from oracle import oracle as O  # noqa: E402
from paper_2309_16818_b200 import mem as M  # noqa: E402
from synth import scenes as S  # noqa: E402
from tests.helpers import compare_layers  # noqa: E402
from tests.test_parity_gpu import (ALL_BINDS, ALL_GROUPS, IMG_BINDS, IMG_GROUPS, NOISE_R,  # noqa: E402
                                   camera_looking_at, random_all_channels)


def split_points(n, G, rng, empty=None):
    if empty is None:
        cuts = np.sort(rng.integers(0, n + 1, G - 1))
        return np.concatenate([[0], cuts, [n]])
    # G - 1 non-trivial shards, then a zero-length range inserted for shard `empty`
    bounds = list(np.concatenate([[0], np.sort(rng.integers(0, n + 1, G - 2)), [n]]))
    bounds.insert(empty, bounds[empty])
    return np.asarray(bounds)


def make_shards(res, rows, cols, groups, G):
    return [M.Map.sharded(res, rows, cols, groups, r, G, debug_points=True) for r in range(G)]


def sync(shards):
    M.mem_shard_local_sync([s.h for s in shards])


def step_sharded(shards, o, pts, binds, R, t, noise, rng, empty=None):
    G = len(shards)
    b = split_points(len(pts), G, rng, empty)
    for r, s in enumerate(shards):
        s.input_pointcloud(torch.from_numpy(np.ascontiguousarray(pts[b[r]:b[r + 1]])).cuda(), binds, R, t, noise)
    sync(shards)
    cell, code = o.input_pointcloud(pts, binds, R, t, noise, debug=True)
    total = None
    for r, s in enumerate(shards):
        gc, gk = s.debug_codes()
        assert np.array_equal(gk, code[b[r]:b[r + 1]]), f"shard {r}: codes differ"
        assert np.array_equal(gc, cell[b[r]:b[r + 1]]), f"shard {r}: cells differ"
        st = s.stats()
        total = st if total is None else {k: total[k] + st[k] for k in st}
    assert total == o.stats(), (total, o.stats())


@pytest.mark.parametrize("G", [2, 4])
def test_local_shards_all_rules_with_shifts(G):
    rows, cols, res = 64, 48, 0.05
    shards = make_shards(res, rows, cols, ALL_GROUPS, G)
    o = O.OracleMap(res, rows, cols, ALL_GROUPS)
    rng = np.random.default_rng(7 + G)
    moves = [(0.0, 0.0), (0.12, 0.0), (0.31, -0.22), (-0.4, 0.05), (-0.4, 0.05), (3.0, 2.0), (2.95, 2.1),
             (2.7, 2.3), (2.5, 2.2), (2.52, 2.18)]
    for f, (x, y) in enumerate(moves):
        for s in shards:
            s.move_to(x, y)
        o.move_to(x, y)
        pts = random_all_channels(300 + f, 6000 + 211 * f, rows, cols, res)
        t = np.array([x + 0.01, y - 0.02, 1.0])
        step_sharded(shards, o, pts, ALL_BINDS, S.rot_z(0.3 * f), t, NOISE_R, rng, empty=f % G if f % 3 == 0 else None)
        for r, s in enumerate(shards):
            compare_layers(s, o, where=f"frame {f} shard {r}: ")


def test_local_shards_points_and_images():
    rows, cols, res, G = 60, 70, 0.05, 3
    shards = make_shards(res, rows, cols, IMG_GROUPS, G)
    o = O.OracleMap(res, rows, cols, IMG_GROUPS)
    rng = np.random.default_rng(91)
    noise = dict(a=1e-3, b=0.0, r_min=0.0, r_max=100.0, h_min=-10.0, h_max=10.0, tau2=9.0, v_out=0.01)
    K = np.array([[120.0, 0.5, 79.5], [0, 118.0, 59.5], [0, 0, 1.0]])
    for f in range(6):
        pts = S.random_cloud(500 + f, 20000, 3, rows, cols, res)
        step_sharded(shards, o, pts, [], np.eye(3), [0.0, 0.0, 1.0], noise, rng)
        eye = np.array([rng.uniform(-3, -2), rng.uniform(-1, 1), rng.uniform(1.0, 2.0)])
        R = camera_looking_at(eye, [rng.uniform(-0.5, 0.5), rng.uniform(-0.5, 0.5), 0.0])
        img = np.concatenate([S.softmax_image(rng.integers(0, 5, (120, 160)), 5, rng),
                              rng.normal(0, 1, (5, 120, 160)).astype(np.float32),
                              rng.uniform(0, 255, (3, 120, 160)).astype(np.float32)])
        for s in shards:
            s.input_image(torch.from_numpy(img).cuda(), IMG_BINDS, K, R, eye)
        sync(shards)
        o.input_image(img, IMG_BINDS, K, R, eye)
        for r, s in enumerate(shards):
            compare_layers(s, o, where=f"frame {f} shard {r}: ")
        if f == 2:
            for s in shards:
                s.move_to(0.33, -0.27)
            o.move_to(0.33, -0.27)
    assert (shards[1].get_layer("top_label") >= 0).sum() > 500


def test_local_shards_c2_full_size():
    c = S.C2
    G = 4
    groups = [dict(name="rgb", rule=M.MEM_COLOR, n_channels=3, w=c["w"])]
    shards = make_shards(c["res"], c["rows"], c["cols"], groups, G)
    o = O.OracleMap(c["res"], c["rows"], c["cols"], groups)
    rng = np.random.default_rng(5)
    for f in range(4):
        fr = S.c2_frame(f)
        for s in shards:
            s.move_to(*fr["move"])
        o.move_to(*fr["move"])
        step_sharded(shards, o, fr["points"], [(0, 1, 0)], fr["R"], fr["t"], c["noise"], rng)
        compare_layers(shards[f % G], o, where=f"frame {f}: ")


def test_nccl_single_rank():
    c = S.C1
    groups = [dict(name="feat", rule=M.MEM_AVERAGE, n_channels=1, w=c["w"])]
    uid = M.mem_nccl_unique_id()
    assert len(uid) == 128
    g = M.Map.sharded(c["res"], c["rows"], c["cols"], groups, 0, 1, nccl_id=uid, debug_points=True)
    o = O.OracleMap(c["res"], c["rows"], c["cols"], groups)
    for f in range(4):
        fr = S.c1_frame(f)
        g.move_to(*fr["move"])
        o.move_to(*fr["move"])
        g.input_pointcloud(torch.from_numpy(fr["points"]).cuda(), [(0, 1, 0)], fr["R"], fr["t"], c["noise"])
        o.input_pointcloud(fr["points"], [(0, 1, 0)], fr["R"], fr["t"], c["noise"])
        assert g.stats() == o.stats()
        compare_layers(g, o, where=f"frame {f}: ")


def test_sharded_errors():
    groups = [dict(name="feat", rule=M.MEM_AVERAGE, n_channels=1, w=0.5)]
    with pytest.raises(M.MemError):
        M.Map.sharded(0.1, 30, 20, groups, 0, 4)  # rows % nranks != 0
    with pytest.raises(M.MemError):
        M.Map.sharded(0.1, 32, 20, groups, 4, 4)  # rank out of range
    a = M.Map.sharded(0.1, 32, 20, groups, 0, 2)
    b = M.Map.sharded(0.1, 32, 20, groups, 1, 2)
    a.input_pointcloud(S.random_cloud(1, 100, 4, 32, 20, 0.1), [(0, 1, 0)], np.eye(3), [0, 0, 1.0], NOISE_R)
    with pytest.raises(M.MemError):
        M.mem_shard_local_sync([a.h, b.h])  # b did not take the frame
    with pytest.raises(M.MemError):
        M.mem_shard_local_sync([b.h, a.h])  # wrong rank order


def test_c5b_full_size_two_local_shards():
    """BASELINE configs[4] big map at full size (2000x2000, 4M points/frame) on 2 local shards;
    the oracle takes the union of the shards."""
    c = S.C5B
    G = 2
    groups = [dict(name="feat", rule=M.MEM_AVERAGE, n_channels=1, w=c["w"])]
    shards = [M.Map.sharded(c["res"], c["rows"], c["cols"], groups, r, G) for r in range(G)]
    o = O.OracleMap(c["res"], c["rows"], c["cols"], groups)
    for f in range(3):
        parts = [S.c5b_shard(f, r, G) for r in range(G)]
        for s, p in zip(shards, parts):
            s.move_to(*p["move"])
            s.input_pointcloud(torch.from_numpy(p["points"]).cuda(), [(0, 1, 0)], p["R"], p["t"], c["noise"])
        sync(shards)
        o.move_to(*parts[0]["move"])
        o.input_pointcloud(np.concatenate([p["points"] for p in parts]), [(0, 1, 0)], parts[0]["R"], parts[0]["t"],
                           c["noise"])
        total = None
        for s in shards:
            st = s.stats()
            total = st if total is None else {k: total[k] + st[k] for k in st}
        assert total == o.stats(), (total, o.stats())
        compare_layers(shards[f % G], o, where=f"frame {f}: ")
    assert o.stats()["n_outlier"] > 1000 and o.get_layer("valid").mean() > 0.9


# ---------------------------------------------------------------- point routing (default protocol)
def make_route_shards(res, rows, cols, groups, G):
    return [M.Map.sharded(res, rows, cols, groups, r, G) for r in range(G)]  # no debug codes: routing


def step_routed(shards, o, pts, binds, R, t, noise, rng, empty=None):
    G = len(shards)
    b = split_points(len(pts), G, rng, empty)
    for r, s in enumerate(shards):
        s.input_pointcloud(torch.from_numpy(np.ascontiguousarray(pts[b[r]:b[r + 1]])).cuda(), binds, R, t, noise)
    sync(shards)
    o.input_pointcloud(pts, binds, R, t, noise)
    total = None
    for s in shards:
        st = s.stats()
        total = st if total is None else {k: total[k] + st[k] for k in st}
    assert total == o.stats(), (total, o.stats())


@pytest.mark.parametrize("G", [2, 3, 4])
def test_routed_shards_all_rules_with_shifts(G):
    """point routing: every shard sends its in-window points to their band owner, which tests,
    accumulates and fuses them; counters summed over shards and every shard's layers equal the
    oracle fed all the points."""
    rows, cols, res = 60, 48, 0.05
    shards = make_route_shards(res, rows, cols, ALL_GROUPS, G)
    o = O.OracleMap(res, rows, cols, ALL_GROUPS)
    rng = np.random.default_rng(17 + G)
    moves = [(0.0, 0.0), (0.12, 0.0), (0.31, -0.22), (-0.4, 0.05), (3.0, 2.0), (2.95, 2.1), (2.7, 2.3)]
    for f, (x, y) in enumerate(moves):
        for s in shards:
            s.move_to(x, y)
        o.move_to(x, y)
        pts = random_all_channels(800 + f, 7000 + 131 * f, rows, cols, res)
        step_routed(shards, o, pts, ALL_BINDS, S.rot_z(0.3 * f), np.array([x + 0.01, y - 0.02, 1.0]), NOISE_R, rng,
                    empty=f % G if f % 3 == 0 else None)
        for r, s in enumerate(shards):
            compare_layers(s, o, where=f"routed frame {f} shard {r}: ")


def test_routed_shards_c5b_and_images():
    c = S.C5B
    G = 4
    groups = [dict(name="feat", rule=M.MEM_AVERAGE, n_channels=1, w=c["w"])]
    shards = make_route_shards(c["res"], c["rows"], c["cols"], groups, G)
    o = O.OracleMap(c["res"], c["rows"], c["cols"], groups)
    for f in range(2):
        parts = [S.c5b_shard(f, r, G) for r in range(G)]
        for s, p in zip(shards, parts):
            s.move_to(*p["move"])
            s.input_pointcloud(torch.from_numpy(p["points"]).cuda(), [(0, 1, 0)], p["R"], p["t"], c["noise"])
        sync(shards)
        o.move_to(*parts[0]["move"])
        o.input_pointcloud(np.concatenate([p["points"] for p in parts]), [(0, 1, 0)], parts[0]["R"], parts[0]["t"],
                           c["noise"])
        compare_layers(shards[f], o, where=f"routed C5b frame {f}: ")
    # images with occlusion on routed shards (every shard fuses its band)
    rows, cols, res = 60, 70, 0.05
    im_sh = make_route_shards(res, rows, cols, IMG_GROUPS, 3)
    oi = O.OracleMap(res, rows, cols, IMG_GROUPS)
    for s in im_sh:
        s.set_image_occlusion(True)
    oi.set_occlusion(True)
    rng = np.random.default_rng(5)
    noise = dict(a=1e-3, b=0.0, r_min=0.0, r_max=100.0, h_min=-10.0, h_max=10.0, tau2=9.0, v_out=0.01)
    K = np.array([[120.0, 0.5, 79.5], [0, 118.0, 59.5], [0, 0, 1.0]])
    for f in range(3):
        pts = S.random_cloud(600 + f, 20000, 3, rows, cols, res)
        step_routed(im_sh, oi, pts, [], np.eye(3), [0.0, 0.0, 1.0], noise, rng)
        eye = np.array([rng.uniform(-3, -2), rng.uniform(-1, 1), rng.uniform(1.0, 2.0)])
        R = camera_looking_at(eye, [rng.uniform(-0.5, 0.5), rng.uniform(-0.5, 0.5), 0.0])
        img = np.concatenate([S.softmax_image(rng.integers(0, 5, (120, 160)), 5, rng),
                              rng.normal(0, 1, (5, 120, 160)).astype(np.float32),
                              rng.uniform(0, 255, (3, 120, 160)).astype(np.float32)])
        for s in im_sh:
            s.input_image(torch.from_numpy(img).cuda(), IMG_BINDS, K, R, eye)
        sync(im_sh)
        oi.input_image(img, IMG_BINDS, K, R, eye)
        for r, s in enumerate(im_sh):
            compare_layers(s, oi, where=f"routed image frame {f} shard {r}: ")


def test_nccl_single_rank_c2():
    """one NCCL rank owns the whole map: the plain point pass on its band, vs the oracle."""
    c = S.C2
    groups = [dict(name="rgb", rule=M.MEM_COLOR, n_channels=3, w=c["w"])]
    g = M.Map.sharded(c["res"], c["rows"], c["cols"], groups, 0, 1, nccl_id=M.mem_nccl_unique_id())
    o = O.OracleMap(c["res"], c["rows"], c["cols"], groups)
    for f in range(3):
        fr = S.c2_frame(f)
        g.move_to(*fr["move"])
        o.move_to(*fr["move"])
        g.input_pointcloud(torch.from_numpy(fr["points"]).cuda(), [(0, 1, 0)], fr["R"], fr["t"], c["noise"])
        o.input_pointcloud(fr["points"], [(0, 1, 0)], fr["R"], fr["t"], c["noise"])
        assert g.stats() == o.stats()
        compare_layers(g, o, where=f"NCCL frame {f}: ")
