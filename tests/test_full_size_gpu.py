"""Full-size parity at the north_star bar: 10 chained frames of every benchmark configuration
against the CPU oracle, every layer BIT-identical (tests/helpers.compare_layers), plus the
path-invariance checks: the certified-atomic path, the small-map sort
kernel and the sort-by-cell pipeline must give the same bits, and a second run the same bits.
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

FRAMES = 10


def layers_of(g):
    return {nm: np.asarray(g.get_layer(nm)).copy() for nm in g.layer_names()}


def assert_same_bits(a, b, where):
    for nm in a:
        assert np.array_equal(a[nm].view(np.uint32), b[nm].view(np.uint32)), f"{where}: {nm} differs"


def c3_groups():
    c = S.C3
    return ([dict(name="sem", rule=M.MEM_CLASS_BAYESIAN, n_channels=c["n_classes"], alpha0=1.0),
             dict(name="top", rule=M.MEM_CLASS_MAX, n_channels=c["n_classes"])],
            [(0, c["n_classes"], 0), (0, c["n_classes"], 1)])


def test_c3_10_frames_full_size():
    """C3: three 640x480 depth clouds + the 20-class image per frame, 10 frames."""
    c = S.C3
    groups, binds = c3_groups()
    g = M.Map(c["res"], c["rows"], c["cols"], groups, debug_points=True)
    o = O.OracleMap(c["res"], c["rows"], c["cols"], groups)
    for f in range(FRAMES):
        fr = S.c3_frame(f)
        g.move_to(*fr["move"])
        o.move_to(*fr["move"])
        for cl in fr["clouds"]:
            g.input_pointcloud(torch.from_numpy(cl["points"]).cuda(), [], cl["R"], cl["t"], c["noise"])
            cell, code = o.input_pointcloud(cl["points"], [], cl["R"], cl["t"], c["noise"], debug=True)
            gc, gk = g.debug_codes()
            assert np.array_equal(gk, code) and np.array_equal(gc, cell), f"frame {f}: codes differ"
            assert g.stats() == o.stats()
        im = fr["image"]
        g.input_image(torch.from_numpy(im["img"]).cuda(), binds, im["K"], im["R"], im["t"])
        o.input_image(im["img"], binds, im["K"], im["R"], im["t"])
        compare_layers(g, o, where=f"C3 frame {f}: ")
    assert (g.get_layer("top_label") >= 0).sum() > 5000


def test_c4_10_images_with_pca_every_frame():
    """C4: geometry from one C3 frame, then 10 64-channel feature images, the PCA readout after
    every image (1e-4 on the [0, 1] outputs, reading D28)."""
    c, c3 = S.C4, S.C3
    groups = [dict(name="feat", rule=M.MEM_AVERAGE, n_channels=c["d"], w=c["w"])]
    g = M.Map(c["res"], c["rows"], c["cols"], groups)
    o = O.OracleMap(c["res"], c["rows"], c["cols"], groups)
    fr = S.c3_frame(0)
    g.move_to(*fr["move"])
    o.move_to(*fr["move"])
    for cl in fr["clouds"]:
        g.input_pointcloud(torch.from_numpy(cl["points"]).cuda(), [], cl["R"], cl["t"], c3["noise"])
        o.input_pointcloud(cl["points"], [], cl["R"], cl["t"], c3["noise"])
    for f in range(FRAMES):
        im = S.c4_image(f)
        g.input_image(torch.from_numpy(im["img"]).cuda(), [(0, c["d"], 0)], im["K"], im["R"], im["t"])
        o.input_image(im["img"], [(0, c["d"], 0)], im["K"], im["R"], im["t"])
        compare_layers(g, o, where=f"C4 image {f}: ")
        gp, op = np.asarray(g.pca_readout("feat", 3)), o.pca_readout("feat", 3)
        assert np.abs(gp - op).max() <= 1e-4, (f, np.abs(gp - op).max())
    assert g.get_layer("feat_observed").sum() > 5000


def test_c2x64_bench_configuration_10_steps_all_maps():
    """the headline step exactly as bench.py times it (64 C2 maps in one batched call, frames
    rotating through the 16-frame pool, map m at frame (step + m) % 16), 10 steps, EVERY map
    against its own oracle map, counters summed over the maps."""
    c = S.C2
    pool = [S.c2_frame(f) for f in range(16)]
    maps, npts = 64, pool[0]["points"].shape[0]
    groups = [dict(name="rgb", rule=M.MEM_COLOR, n_channels=3, w=c["w"])]
    gb = M.Map(c["res"], c["rows"], c["cols"], groups, n_maps=maps)
    oras = [O.OracleMap(c["res"], c["rows"], c["cols"], groups) for _ in range(maps)]
    dev = [torch.from_numpy(fr["points"]).cuda() for fr in pool]
    offsets = np.arange(maps + 1, dtype=np.int64) * npts
    for step in range(FRAMES):
        idx = [(step + m) % 16 for m in range(maps)]
        gb.move_to_batch(np.stack([pool[i]["move"] for i in idx]))
        gb.input_pointcloud_batch(torch.cat([dev[i] for i in idx]), offsets, [(0, 1, 0)],
                                  np.stack([pool[i]["R"] for i in idx]), np.stack([pool[i]["t"] for i in idx]),
                                  c["noise"])
        total = None
        for b in range(maps):
            fr = pool[idx[b]]
            oras[b].move_to(*fr["move"])
            oras[b].input_pointcloud(fr["points"], [(0, 1, 0)], fr["R"], fr["t"], c["noise"])
            st = oras[b].stats()
            total = st if total is None else {k: total[k] + st[k] for k in st}
        assert gb.stats() == total, (step, gb.stats(), total)
    for nm in gb.layer_names():
        lay = np.asarray(gb.get_layer(nm))
        for b in range(maps):
            o = oras[b].get_layer(nm)
            assert np.array_equal(lay[b].view(np.uint32), o.view(np.uint32)) or \
                np.array_equal(lay[b], o, equal_nan=True), (b, nm)


def test_c5a_full_batch_10_frames_first_and_last_map_of_every_shard():
    """C5a at full size: 4096 128x128 maps x 32,768 points per frame in one batched call, 10
    frames; checked against the oracle: the first and the last map of every shard of an 8-GPU
    split (512 maps each), 16 maps.  Map m is generated map m % 256 (as bench.py)."""
    c = S.C5A
    B, gen, P = 4096, 256, c["points"]
    groups = [dict(name="feat", rule=M.MEM_AVERAGE, n_channels=1, w=c["w"])]
    gb = M.Map(c["res"], c["rows"], c["cols"], groups, n_maps=B)
    check = sorted({s * 512 for s in range(8)} | {s * 512 + 511 for s in range(8)})
    oras = {b: O.OracleMap(c["res"], c["rows"], c["cols"], groups) for b in check}
    idx = np.arange(B) % gen
    offsets = np.arange(B + 1, dtype=np.int64) * P
    for f in range(FRAMES):
        bt = S.c5a_batch(f % 2, 0, gen)
        pts = bt["points"].reshape(gen, P, 4)
        dev = torch.from_numpy(pts).cuda()[torch.from_numpy(idx).cuda()].reshape(-1, 4).contiguous()
        gb.move_to_batch(bt["move"][idx])
        gb.input_pointcloud_batch(dev, offsets, [(0, 1, 0)], bt["R"][idx], bt["t"][idx], c["noise"])
        for b in check:
            k = b % gen
            oras[b].move_to(*bt["move"][k])
            oras[b].input_pointcloud(pts[k], [(0, 1, 0)], bt["R"][k], bt["t"][k], c["noise"])
    for nm in gb.layer_names():
        lay = np.asarray(gb.get_layer(nm))
        for b in check:
            assert np.array_equal(lay[b], oras[b].get_layer(nm), equal_nan=True), (b, nm)


def test_c5b_10_frames_full_size():
    """C5b: one 2000x2000 map, 4,194,304 points per frame, 10 frames; on one NCCL rank (the
    whole map) and on 2 local shards (point routing), both against the oracle."""
    c = S.C5B
    groups = [dict(name="feat", rule=M.MEM_AVERAGE, n_channels=1, w=c["w"])]
    one = M.Map.sharded(c["res"], c["rows"], c["cols"], groups, 0, 1, nccl_id=M.mem_nccl_unique_id())
    shards = [M.Map.sharded(c["res"], c["rows"], c["cols"], groups, r, 2) for r in range(2)]
    o = O.OracleMap(c["res"], c["rows"], c["cols"], groups)
    for f in range(FRAMES):
        parts = [S.c5b_shard(f, r, 2) for r in range(2)]
        allp = np.concatenate([p["points"] for p in parts])
        one.move_to(*parts[0]["move"])
        one.input_pointcloud(torch.from_numpy(allp).cuda(), [(0, 1, 0)], parts[0]["R"], parts[0]["t"], c["noise"])
        for s, p in zip(shards, parts):
            s.move_to(*p["move"])
            s.input_pointcloud(torch.from_numpy(p["points"]).cuda(), [(0, 1, 0)], p["R"], p["t"], c["noise"])
        M.mem_shard_local_sync([s.h for s in shards])
        o.move_to(*parts[0]["move"])
        o.input_pointcloud(allp, [(0, 1, 0)], parts[0]["R"], parts[0]["t"], c["noise"])
        assert one.stats() == o.stats(), f
    compare_layers(one, o, where="C5b one rank: ")
    compare_layers(shards[1], o, where="C5b shard 1 of 2: ")
    assert o.get_layer("valid").mean() > 0.9


@pytest.mark.parametrize("case", ["c2_colour", "c1_average", "c3_height", "c5a_small_maps"])
def test_paths_give_identical_bits(case):
    """Launch-path invariance: the default route (certified atomics, or the
    small-map sort kernel for batches of small maps) and the sort-by-cell pipeline
    (MEM_FLAG_FUSE_SORTED) must produce the same bits over 10 chained frames, and a second run
    of the default route the same bits again."""
    runs = []
    for sorted_, rep in ((False, 0), (True, 0), (False, 1)):
        if case == "c2_colour":
            c = S.C2
            g = M.Map(c["res"], c["rows"], c["cols"], [dict(name="rgb", rule=M.MEM_COLOR, n_channels=3, w=c["w"])],
                      fuse_sorted=sorted_)
            for f in range(FRAMES):
                fr = S.c2_frame(f)
                g.move_to(*fr["move"])
                g.input_pointcloud(torch.from_numpy(fr["points"]).cuda(), [(0, 1, 0)], fr["R"], fr["t"], c["noise"])
        elif case == "c1_average":
            c = S.C1
            g = M.Map(c["res"], c["rows"], c["cols"], [dict(name="feat", rule=M.MEM_AVERAGE, n_channels=1, w=c["w"])],
                      fuse_sorted=sorted_)
            for f in range(FRAMES):
                fr = S.c1_frame(f)
                g.move_to(*fr["move"])
                g.input_pointcloud(torch.from_numpy(fr["points"]).cuda(), [(0, 1, 0)], fr["R"], fr["t"], c["noise"])
        elif case == "c3_height":
            c = S.C3
            g = M.Map(c["res"], c["rows"], c["cols"], [], fuse_sorted=sorted_)
            for f in range(4):
                fr = S.c3_frame(f)
                g.move_to(*fr["move"])
                for cl in fr["clouds"]:
                    g.input_pointcloud(torch.from_numpy(cl["points"]).cuda(), [], cl["R"], cl["t"], c["noise"])
        else:
            c = S.C5A
            B = 96
            g = M.Map(c["res"], c["rows"], c["cols"], [dict(name="feat", rule=0, n_channels=1, w=c["w"])], n_maps=B,
                      fuse_sorted=sorted_)
            for f in range(4):
                bt = S.c5a_batch(f, 0, B)
                g.move_to_batch(bt["move"])
                g.input_pointcloud_batch(torch.from_numpy(bt["points"]).cuda(), bt["offsets"], [(0, 1, 0)], bt["R"],
                                         bt["t"], c["noise"])
        runs.append((layers_of(g), g.stats()))
    assert_same_bits(runs[0][0], runs[1][0], f"{case}: default vs sort pipeline")
    assert_same_bits(runs[0][0], runs[2][0], f"{case}: run to run")
    assert runs[0][1] == runs[1][1] == runs[2][1]


@pytest.mark.parametrize("rows,n,group", [(16, 20000, "average"), (4, 100000, "average"), (8, 50000, "colour"),
                                          (16, 20000, None), (2, 30000, None), (1, 40000, "average")])
def test_uncertified_cells_are_refolded_exactly(rows, n, group):
    run_uncertified(rows, n, group, sorted_=False)


@pytest.mark.parametrize("rows,n,group", [(16, 20000, "average"), (8, 50000, "colour"), (2, 30000, None)])
def test_uncertified_cells_through_the_sort_path(rows, n, group):
    """The same inputs through the sort pipeline (MEM_FLAG_FUSE_SORTED): mid and long cells whose
    certificate fails fold block-certified in input order (k_fuse), bit-exact."""
    run_uncertified(rows, n, group, sorted_=True)


def run_uncertified(rows, n, group, sorted_):
    """Cells whose height terms z/v span more binades than the certificate allows (z from 1e-12
    to 1 m in one cell) cannot be summed by atomics in an order-free way: they must be
    recomputed in input order (k_refold) and still equal the oracle bit for bit.
    Cells of up to 16384 points take the sorted-list path (block-certified fold), larger ones
    (1 x 1 map, 40k points) the whole-map walk; colour, 1-channel average and height only."""
    rng = np.random.default_rng(11 + rows)
    cols = rows
    res = 0.1
    half = rows * res / 2 - 0.01
    noise = dict(a=1e-4, b=0.0, r_min=0.0, r_max=100.0, h_min=-10.0, h_max=10.0, tau2=1e30, v_out=0.01)
    groups = {"average": [dict(name="feat", rule=M.MEM_AVERAGE, n_channels=1, w=0.5)],
              "colour": [dict(name="rgb", rule=M.MEM_COLOR, n_channels=3, w=0.5)], None: []}[group]
    binds = [] if group is None else [(0, 1, 0)]
    g = M.Map(res, rows, cols, groups, debug_points=True, fuse_sorted=sorted_)
    o = O.OracleMap(res, rows, cols, groups)
    for f in range(4):
        xy = rng.uniform(-half, half, (n, 2))
        z = rng.choice([1e-12, 1e-9, 1e-6, 1e-3, 1.0], n) * rng.choice([-1.0, 1.0], n) * rng.uniform(1, 2, n)
        feat = rng.choice([1e-20, 1e-10, 1.0, 1e10], n) * rng.uniform(1, 2, n)
        pts = np.stack([xy[:, 0], xy[:, 1], z - 1.0, feat], 1).astype(np.float32)
        if group == "colour":
            pts[:, 3] = S.pack_rgb(rng.integers(0, 256, (n, 3)).astype(np.uint8)).view(np.float32)
        g.input_pointcloud(torch.from_numpy(pts).cuda(), binds, np.eye(3), [0.0, 0.0, 1.0], noise)
        cell, code = o.input_pointcloud(pts, binds, np.eye(3), [0.0, 0.0, 1.0], noise, debug=True)
        gc, gk = g.debug_codes()
        assert np.array_equal(gk, code) and np.array_equal(gc, cell)
        assert g.stats() == o.stats()
        compare_layers(g, o, where=f"refold frame {f}: ")


def test_red_path_batch_of_more_than_128_maps():
    """More maps than ride in the kernel parameters (kInlineMaps = 128): frames, offsets and
    the warp-item prefix sums are staged in one parameter blob; maps too large for k_smap
    (130 x 130 cells) take the certified-RED path.  Ragged point counts, colour group, 3
    frames with moves; 6 maps checked against the oracle."""
    rng = np.random.default_rng(23)
    B, rows = 136, 130
    res = 0.1
    groups = [dict(name="rgb", rule=M.MEM_COLOR, n_channels=3, w=0.5)]
    noise = dict(a=1e-4, b=1e-5, r_min=0.0, r_max=50.0, h_min=-5.0, h_max=5.0, tau2=9.0, v_out=0.01)
    g = M.Map(res, rows, rows, groups, n_maps=B)
    check = [0, 1, 64, 127, 128, 135]
    oras = {b: O.OracleMap(res, rows, rows, groups) for b in check}
    for f in range(3):
        counts = rng.integers(0, 3000, B)
        offsets = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
        n = int(offsets[-1])
        xy = rng.uniform(-7.0, 7.0, (n, 2))
        z = 0.3 * np.sin(xy[:, 0]) + rng.normal(0, 0.02, n)
        pts = np.stack([xy[:, 0], xy[:, 1], z - 1.0, np.zeros(n)], 1).astype(np.float32)
        pts[:, 3] = S.pack_rgb(rng.integers(0, 256, (n, 3)).astype(np.uint8))
        moves = rng.uniform(-0.5, 0.5, (B, 2)) + 0.013
        R = np.tile(np.eye(3), (B, 1, 1))
        t = np.tile([0.0, 0.0, 1.0], (B, 1))
        g.move_to_batch(moves)
        g.input_pointcloud_batch(torch.from_numpy(pts).cuda(), offsets, [(0, 1, 0)], R, t, noise)
        for b in check:
            oras[b].move_to(*moves[b])
            oras[b].input_pointcloud(pts[offsets[b]:offsets[b + 1]], [(0, 1, 0)], np.eye(3), [0.0, 0.0, 1.0], noise)
    for nm in g.layer_names():
        lay = np.asarray(g.get_layer(nm))
        for b in check:
            assert np.array_equal(lay[b], oras[b].get_layer(nm), equal_nan=True), (b, nm)


def test_colour_map_beyond_the_packed_count_limit_takes_the_sort_path():
    """A colour call of more than 131,586 points per map cannot use the packed colour count word
    of the RED path (b | n << 25 | n_out << 43): it is fused by the sort pipeline, with the same
    bits as the oracle -- two LiDAR frames merged into one 262,144-point call, 3 calls."""
    c = S.C2
    groups = [dict(name="rgb", rule=M.MEM_COLOR, n_channels=3, w=c["w"])]
    g = M.Map(c["res"], c["rows"], c["cols"], groups)
    o = O.OracleMap(c["res"], c["rows"], c["cols"], groups)
    for f in range(3):
        a, b = S.c2_frame(2 * f), S.c2_frame(2 * f + 1)
        pts = np.concatenate([a["points"], b["points"]]).astype(np.float32)
        g.move_to(*a["move"])
        o.move_to(*a["move"])
        g.input_pointcloud(torch.from_numpy(pts).cuda(), [(0, 1, 0)], a["R"], a["t"], c["noise"])
        o.input_pointcloud(pts, [(0, 1, 0)], a["R"], a["t"], c["noise"])
        assert g.stats() == o.stats()
    compare_layers(g, o, where="colour, 262,144 points per call: ")
