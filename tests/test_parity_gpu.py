"""GPU parity: libmem (CUDA, through the C-ABI) vs the CPU oracle on the same seeded inputs.

Integer outputs (per-point cell + code, counters, valid, observed flags, class_max labels,
ring/shift indexing) must be bit-exact; fp32 layers within 1e-5 rel / 1e-6 abs after 10
fused frames (north_star).
"""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from oracle import oracle as O  # noqa: E402
from paper_2309_16818_b200 import mem as M  # noqa: E402
from synth import scenes as S  # noqa: E402
from tests.helpers import compare_layers, copy_state_to_oracle  # noqa: E402


def make_pair(res, rows, cols, groups, debug=True):
    g = M.Map(res, rows, cols, groups, debug_points=debug)
    o = O.OracleMap(res, rows, cols, groups)
    return g, o


def step_points(g, o, pts, binds, R, t, noise, check_codes=True, device=True):
    src = torch.from_numpy(pts).cuda() if device else pts
    g.input_pointcloud(src, binds, R, t, noise)
    oc = o.input_pointcloud(pts, binds, R, t, noise, debug=check_codes)
    if check_codes:
        cell, code = g.debug_codes()
        assert np.array_equal(code, oc[1]), f"codes differ at {np.argwhere(code != oc[1])[:5].ravel()}"
        assert np.array_equal(cell, oc[0]), f"cells differ at {np.argwhere(cell != oc[0])[:5].ravel()}"
    gs, os_ = g.stats(), o.stats()
    assert gs == os_, (gs, os_)
    return gs


# ---------------------------------------------------------------- C1 (configs[0])
def test_c1_chained_10_frames():
    c = S.C1
    groups = [dict(name="feat", rule=M.MEM_AVERAGE, n_channels=1, w=c["w"])]
    g, o = make_pair(c["res"], c["rows"], c["cols"], groups)
    for f in range(c["frames"]):
        fr = S.c1_frame(f)
        g.move_to(*fr["move"])
        o.move_to(*fr["move"])
        assert tuple(g.center()[0]) == o.center()
        st = step_points(g, o, fr["points"], [(0, 1, 0)], fr["R"], fr["t"], c["noise"])
        assert st["n_outlier"] > 0 or f == 0
        compare_layers(g, o, where=f"frame {f}: ")


# ---------------------------------------------------------------- all six rules, ragged map
ALL_GROUPS = [
    dict(name="feat", rule=M.MEM_AVERAGE, n_channels=3, w=0.5),
    dict(name="gf", rule=M.MEM_GAUSSIAN, n_channels=2, sigma_f2=0.2, mu0=0.1, sigma0_2=1.5),
    dict(name="cavg", rule=M.MEM_CLASS_AVERAGE, n_channels=4, w=0.3),
    dict(name="sem", rule=M.MEM_CLASS_BAYESIAN, n_channels=4, alpha0=1.0),
    dict(name="top", rule=M.MEM_CLASS_MAX, n_channels=4),
    dict(name="rgb", rule=M.MEM_COLOR, n_channels=3, w=0.5),
]
ALL_BINDS = [(0, 3, 0), (3, 2, 1), (5, 4, 2), (5, 4, 3), (5, 4, 4), (9, 1, 5)]
NOISE_R = dict(a=1e-3, b=1e-4, r_min=0.05, r_max=6.0, h_min=-3.0, h_max=1.0, tau2=4.0, v_out=0.02)


def random_all_channels(seed, n, rows, cols, res):
    rng = np.random.default_rng(seed)
    pts = S.random_cloud(seed, n, 13, rows, cols, res, channel_kind="feature")
    p = rng.dirichlet(np.ones(4) * 0.7, n)
    tie = rng.uniform(size=n) < 0.1
    p[tie] = np.round(p[tie] * 4) / 4  # exact ties exercise the lowest-index rule (D19)
    pts[:, 8:12] = p.astype(np.float32)
    pts[:, 12] = S.pack_rgb(rng.integers(0, 256, (n, 3)).astype(np.uint8))
    bad = rng.uniform(size=n) < 0.01
    pts[bad, 3] = np.nan  # D31: non-finite channel skips only that group
    outl = rng.uniform(size=n) < 0.03
    pts[outl, 2] += 1.5
    return pts


@pytest.mark.parametrize("rows,cols,res", [(37, 53, 0.1), (64, 64, 0.05)])
def test_all_rules_chained_with_shifts(rows, cols, res):
    g, o = make_pair(res, rows, cols, ALL_GROUPS)
    moves = [(0.0, 0.0), (0.12, 0.0), (0.31, -0.22), (-0.4, 0.05), (-0.4, 0.05), (3.0, 2.0), (2.95, 2.1),
             (2.7, 2.3), (2.5, 2.2), (2.52, 2.18)]
    for f, (x, y) in enumerate(moves):
        g.move_to(x, y)
        o.move_to(x, y)
        pts = random_all_channels(100 + f, 5000 + 137 * f, rows, cols, res)
        R = S.rot_z(0.3 * f)
        t = np.array([x + 0.01, y - 0.02, 1.0])
        step_points(g, o, pts, ALL_BINDS, R, t, NOISE_R)
        compare_layers(g, o, where=f"frame {f}: ")


# ---------------------------------------------------------------- C2 (configs[1]) full size
def test_c2_lidar_10_frames():
    c = S.C2
    groups = [dict(name="rgb", rule=M.MEM_COLOR, n_channels=3, w=c["w"])]
    g, o = make_pair(c["res"], c["rows"], c["cols"], groups)
    for f in range(c["frames"]):
        fr = S.c2_frame(f)
        g.move_to(*fr["move"])
        o.move_to(*fr["move"])
        step_points(g, o, fr["points"], [(0, 1, 0)], fr["R"], fr["t"], c["noise"])
        compare_layers(g, o, where=f"frame {f}: ")
    assert g.get_layer("valid").sum() > 5000


def test_host_buffers_equal_device_buffers():
    """the e2e path (host pointers through the C-ABI) gives bit-identical maps."""
    c = S.C2
    groups = [dict(name="rgb", rule=M.MEM_COLOR, n_channels=3, w=c["w"])]
    a = M.Map(c["res"], c["rows"], c["cols"], groups)
    b = M.Map(c["res"], c["rows"], c["cols"], groups)
    for f in range(3):
        fr = S.c2_frame(f)
        for m, dev in ((a, True), (b, False)):
            m.move_to(*fr["move"])
            m.input_pointcloud(torch.from_numpy(fr["points"]).cuda() if dev else fr["points"], [(0, 1, 0)],
                               fr["R"], fr["t"], c["noise"])
    for nm in a.layer_names():
        assert np.array_equal(a.get_layer(nm), b.get_layer(nm), equal_nan=True), nm


# ---------------------------------------------------------------- image path
def camera_looking_at(eye, target):
    """R (camera->map): z_c toward target, x_c right, y_c down."""
    z = np.asarray(target, float) - np.asarray(eye, float)
    z /= np.linalg.norm(z)
    up = np.array([0.0, 0.0, 1.0])
    x = np.cross(z, up)
    x /= np.linalg.norm(x)
    y = np.cross(z, x)
    return np.stack([x, y, z], 1)


IMG_GROUPS = [
    dict(name="sem", rule=M.MEM_CLASS_BAYESIAN, n_channels=5, alpha0=1.0),
    dict(name="top", rule=M.MEM_CLASS_MAX, n_channels=5),
    dict(name="feat", rule=M.MEM_AVERAGE, n_channels=3, w=0.5),
    dict(name="gf", rule=M.MEM_GAUSSIAN, n_channels=2, sigma_f2=0.3, mu0=0.0, sigma0_2=1.0),
    dict(name="rgb", rule=M.MEM_COLOR, n_channels=3, w=0.5),
    dict(name="cavg", rule=M.MEM_CLASS_AVERAGE, n_channels=5, w=0.4),
]
IMG_BINDS = [(0, 5, 0), (0, 5, 1), (5, 3, 2), (8, 2, 3), (10, 3, 4), (0, 5, 5)]


def test_image_fusion_chained():
    rows, cols, res = 60, 70, 0.05
    g, o = make_pair(res, rows, cols, IMG_GROUPS)
    rng = np.random.default_rng(41)
    noise = dict(a=1e-3, b=0.0, r_min=0.0, r_max=100.0, h_min=-10.0, h_max=10.0, tau2=9.0, v_out=0.01)
    K = np.array([[120.0, 0.5, 79.5], [0, 118.0, 59.5], [0, 0, 1.0]])
    for f in range(10):
        pts = S.random_cloud(200 + f, 20000, 3, rows, cols, res)
        step_points(g, o, pts, [], np.eye(3), [0.0, 0.0, 1.0], noise)
        eye = np.array([rng.uniform(-3, -2), rng.uniform(-1, 1), rng.uniform(1.0, 2.0)])
        R = camera_looking_at(eye, [rng.uniform(-0.5, 0.5), rng.uniform(-0.5, 0.5), 0.0])
        img = np.concatenate([S.softmax_image(rng.integers(0, 5, (120, 160)), 5, rng),
                              rng.normal(0, 1, (5, 120, 160)).astype(np.float32),
                              rng.uniform(0, 255, (3, 120, 160)).astype(np.float32)])
        img[5, rng.integers(0, 120, 50), rng.integers(0, 160, 50)] = np.nan
        src = torch.from_numpy(img).cuda() if f % 2 == 0 else img
        g.input_image(src, IMG_BINDS, K, R, eye)
        o.input_image(img, IMG_BINDS, K, R, eye)
        compare_layers(g, o, where=f"frame {f}: ")
        if f == 4:
            g.move_to(0.33, -0.27)
            o.move_to(0.33, -0.27)
    assert (g.get_layer("top_label") >= 0).sum() > 500



@pytest.mark.gpu
def test_image_fusion_wide_groups():
    """Groups wider than k_image's 16-channel load batch (ragged last batch), every per-channel
    rule, a NaN in the second batch (D21 skips the whole group), class_max ties across batches."""
    rows, cols, res = 40, 50, 0.05
    groups = [dict(name="gw", rule=M.MEM_GAUSSIAN, n_channels=19, sigma_f2=0.3, mu0=0.0, sigma0_2=1.0),
              dict(name="ca", rule=M.MEM_CLASS_AVERAGE, n_channels=21, w=0.4),
              dict(name="av", rule=M.MEM_AVERAGE, n_channels=17, w=0.5),
              dict(name="db", rule=M.MEM_CLASS_BAYESIAN, n_channels=33, alpha0=1.0),
              dict(name="mx", rule=M.MEM_CLASS_MAX, n_channels=33)]
    binds = [(0, 19, 0), (19, 21, 1), (40, 17, 2), (57, 33, 3), (57, 33, 4)]
    g, o = make_pair(res, rows, cols, groups)
    rng = np.random.default_rng(77)
    noise = dict(a=1e-3, b=0.0, r_min=0.0, r_max=100.0, h_min=-10.0, h_max=10.0, tau2=9.0, v_out=0.01)
    K = np.array([[120.0, 0.0, 79.5], [0, 120.0, 59.5], [0, 0, 1.0]])
    for f in range(4):
        step_points(g, o, S.random_cloud(300 + f, 15000, 3, rows, cols, res), [], np.eye(3), [0.0, 0.0, 1.0], noise)
        eye = np.array([rng.uniform(-3, -2), rng.uniform(-1, 1), rng.uniform(1.0, 2.0)])
        R = camera_looking_at(eye, [rng.uniform(-0.3, 0.3), rng.uniform(-0.3, 0.3), 0.0])
        img = rng.normal(0, 1, (90, 120, 160)).astype(np.float32)
        img[57:90] = np.round(rng.uniform(0, 3, (33, 120, 160))).astype(np.float32)  # many ties
        img[17, rng.integers(0, 120, 40), rng.integers(0, 160, 40)] = np.nan  # gaussian, 2nd batch
        img[75, rng.integers(0, 120, 40), rng.integers(0, 160, 40)] = np.inf  # class groups
        g.input_image(torch.from_numpy(img).cuda(), binds, K, R, eye)
        o.input_image(img, binds, K, R, eye)
        compare_layers(g, o, where=f"frame {f}: ")


# ---------------------------------------------------------------- batched maps
def test_batched_equals_single_and_oracle():
    rows, cols, res = 48, 40, 0.1
    B = 5
    groups = [dict(name="feat", rule=M.MEM_AVERAGE, n_channels=1, w=0.5),
              dict(name="rgb", rule=M.MEM_COLOR, n_channels=3, w=0.5)]
    gb = M.Map(res, rows, cols, groups, n_maps=B)
    singles = [M.Map(res, rows, cols, groups) for _ in range(B)]
    oras = [O.OracleMap(res, rows, cols, groups) for _ in range(2)]
    rng = np.random.default_rng(43)
    binds = [(0, 1, 0), (1, 1, 1)]
    for f in range(4):
        counts = rng.integers(0, 3000, B)
        counts[f % B] = 0  # an empty map in the batch
        clouds = []
        for b in range(B):
            p = S.random_cloud(1000 * f + b, int(counts[b]), 5, rows, cols, res)
            p[:, 4] = S.pack_rgb(rng.integers(0, 256, (len(p), 3)).astype(np.uint8))
            clouds.append(p)
        off = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
        allp = np.concatenate(clouds) if off[-1] else np.zeros((0, 5), np.float32)
        Rs = np.stack([S.rot_z(0.1 * b + f) for b in range(B)])
        ts = np.stack([[0.05 * b, -0.03 * f, 1.0] for b in range(B)])
        xy = np.stack([[0.1 * f * (b + 1), -0.07 * f] for b in range(B)])
        gb.move_to_batch(xy)
        gb.input_pointcloud_batch(torch.from_numpy(allp).cuda(), off, binds, Rs, ts, NOISE_R)
        for b in range(B):
            singles[b].move_to(*xy[b])
            singles[b].input_pointcloud(clouds[b], binds, Rs[b], ts[b], NOISE_R)
        for b in range(2):
            oras[b].move_to(*xy[b])
            oras[b].input_pointcloud(clouds[b], binds, Rs[b], ts[b], NOISE_R)
    for nm in gb.layer_names():
        allb = gb.get_layer(nm)
        for b in range(B):
            assert np.array_equal(allb[b], singles[b].get_layer(nm), equal_nan=True), (nm, b)
    for b in range(2):
        compare_layers(singles[b], oras[b], where=f"map {b}: ")


# ---------------------------------------------------------------- single-step parity, run-twice identity
def test_single_step_parity_and_determinism():
    c = S.C2
    groups = [dict(name="rgb", rule=M.MEM_COLOR, n_channels=3, w=c["w"])]
    runs = []
    for rep in range(2):
        g = M.Map(c["res"], c["rows"], c["cols"], groups, debug_points=True)
        for f in range(6):
            fr = S.c2_frame(f)
            g.move_to(*fr["move"])
            if f == 5 and rep == 0:  # single step from the GPU's own pre-frame state
                o = O.OracleMap(c["res"], c["rows"], c["cols"], groups)
                o.move_to(*fr["move"])
                copy_state_to_oracle(g, o)
                step_points(g, o, fr["points"], [(0, 1, 0)], fr["R"], fr["t"], c["noise"])
                compare_layers(g, o, where="single step: ")
            else:
                g.input_pointcloud(torch.from_numpy(fr["points"]).cuda(), [(0, 1, 0)], fr["R"], fr["t"], c["noise"])
        runs.append({nm: g.get_layer(nm) for nm in g.layer_names()})
    for nm in runs[0]:
        assert np.array_equal(runs[0][nm], runs[1][nm], equal_nan=True), nm  # run-twice bit identity


# ---------------------------------------------------------------- edge cases
def test_edge_cases():
    noise = dict(a=1e-2, b=0.0, r_min=0.0, r_max=100.0, h_min=-10.0, h_max=10.0, tau2=9.0, v_out=0.01)
    groups = [dict(name="f", rule=M.MEM_AVERAGE, n_channels=1, w=0.5)]
    # 1x1 map
    g, o = make_pair(0.5, 1, 1, groups)
    pts = np.array([[0.1, 0.1, -1.0, 2.0], [0.3, 0.0, -1.0, 3.0], [np.nan, 0, 0, 1.0]], np.float32)
    step_points(g, o, pts, [(0, 1, 0)], np.eye(3), [0, 0, 1.0], noise)
    compare_layers(g, o)
    # empty cloud: map unchanged, stats zero
    before = {nm: g.get_layer(nm) for nm in g.layer_names()}
    g.input_pointcloud(np.zeros((0, 4), np.float32), [(0, 1, 0)], np.eye(3), [0, 0, 1.0], noise)
    assert g.stats()["n_input"] == 0
    for nm, v in before.items():
        assert np.array_equal(g.get_layer(nm), v, equal_nan=True)
    # all non-finite / all out of bounds
    g, o = make_pair(0.1, 16, 16, groups)
    for pts in (np.full((1000, 4), np.nan, np.float32),
                np.tile(np.array([[50.0, 0.0, -1.0, 1.0]], np.float32), (777, 1))):
        step_points(g, o, pts, [(0, 1, 0)], np.eye(3), [0, 0, 1.0], noise)
        compare_layers(g, o)
    # one point per cell on a dense grid (no within-cell aggregation), odd tail
    g, o = make_pair(0.25, 33, 31, groups)
    ii, jj = np.meshgrid(np.arange(33), np.arange(31), indexing="ij")
    pts = np.stack([(ii.ravel() + 0.5 - 16.5) * 0.25, (jj.ravel() + 0.5 - 15.5) * 0.25,
                    np.full(ii.size, -1.0), np.arange(ii.size, dtype=float)], 1).astype(np.float32)
    step_points(g, o, pts, [(0, 1, 0)], np.eye(3), [0, 0, 1.0], noise)
    compare_layers(g, o)
    assert g.get_layer("valid").all()
    # many points in one cell (heavy atomic contention)
    g, o = make_pair(1.0, 4, 4, groups)
    rng = np.random.default_rng(47)
    pts = np.concatenate([rng.uniform(0.01, 0.99, (100000, 2)), rng.normal(-1, 0.01, (100000, 1)),
                          rng.normal(0, 1, (100000, 1))], 1).astype(np.float32)
    step_points(g, o, pts, [(0, 1, 0)], np.eye(3), [0, 0, 1.0], noise)
    compare_layers(g, o)


def test_errors_and_info():
    g = M.Map(0.1, 10, 12, [dict(name="f", rule=M.MEM_AVERAGE, n_channels=1, w=0.5)])
    with pytest.raises(M.MemError) as e:
        R = np.eye(3)
        R[0, 1] = 0.01
        g.input_pointcloud(np.zeros((3, 4), np.float32), [(0, 1, 0)], R, [0, 0, 0], NOISE_R)
    assert e.value.status == M.MEM_EPOSE
    with pytest.raises(M.MemError) as e:
        g.input_pointcloud(np.zeros((3, 4), np.float32), [(1, 1, 0)], np.eye(3), [0, 0, 0], NOISE_R)
    assert e.value.status == M.MEM_EINVAL
    with pytest.raises(M.MemError) as e:
        g.get_layer("nope")
    assert e.value.status == M.MEM_ENOTFOUND
    with pytest.raises(M.MemError) as e:
        M.Map(0.1, 10, 10, [dict(name="a", rule=M.MEM_AVERAGE), dict(name="a", rule=M.MEM_AVERAGE)])
    assert e.value.status == M.MEM_EDUPNAME
    with pytest.raises(M.MemError) as e:
        M.Map(0.1, 10, 10, [dict(name="c", rule=M.MEM_CLASS_BAYESIAN, n_channels=1)])
    assert e.value.status == M.MEM_ERULE
    # memory accounting: each fp32 layer is rows x cols x 4 bytes
    base = M.Map(0.04, 200, 200, [])
    one = M.Map(0.04, 200, 200, [dict(name="f", rule=M.MEM_AVERAGE, n_channels=1, w=0.5)])
    assert one.footprint() - base.footprint() == 160000 + 40000  # + 1-byte observed flag
    assert "elevation" in base.layer_names() and "f_observed" in one.layer_names()


def test_uniform_batch_sweep_vs_oracle():
    """uniform batches (every map the same point count) take the fused sweep kernel; every map
    must match its own oracle map (codes bit-exact via stats, layers within tolerance)."""
    rows, cols, res = 40, 36, 0.1
    B, n = 9, 4000
    groups = [dict(name="feat", rule=M.MEM_AVERAGE, n_channels=1, w=0.5),
              dict(name="rgb", rule=M.MEM_COLOR, n_channels=3, w=0.5)]
    gb = M.Map(res, rows, cols, groups, n_maps=B, debug_points=True)
    oras = [O.OracleMap(res, rows, cols, groups) for _ in range(B)]
    rng = np.random.default_rng(53)
    binds = [(0, 1, 0), (1, 1, 1)]
    for f in range(6):
        clouds = []
        for b in range(B):
            p = S.random_cloud(7000 * f + b, n, 5, rows, cols, res)
            p[:, 4] = S.pack_rgb(rng.integers(0, 256, (n, 3)).astype(np.uint8))
            p[rng.uniform(size=n) < 0.05, 2] += 1.0  # outliers
            clouds.append(p)
        off = np.arange(B + 1, dtype=np.int64) * n
        Rs = np.stack([S.rot_z(0.2 * b - 0.3 * f) for b in range(B)])
        ts = np.stack([[0.03 * b, 0.02 * f, 1.0] for b in range(B)])
        xy = np.stack([[0.13 * f * (b % 3 + 1), -0.11 * f] for b in range(B)])
        gb.move_to_batch(xy)
        gb.input_pointcloud_batch(torch.from_numpy(np.concatenate(clouds)).cuda(), off, binds, Rs, ts, NOISE_R)
        cell, code = gb.debug_codes()
        tot = dict.fromkeys(O.STAT_NAMES, 0)
        for b in range(B):
            oras[b].move_to(*xy[b])
            oc, ok = oras[b].input_pointcloud(clouds[b], binds, Rs[b], ts[b], NOISE_R, debug=True)
            assert np.array_equal(code[b * n:(b + 1) * n], ok), (f, b)
            assert np.array_equal(cell[b * n:(b + 1) * n], oc), (f, b)
            for k, v in oras[b].stats().items():
                tot[k] += v
        assert gb.stats() == tot
    for b in range(B):
        for nm in gb.layer_names():
            g = gb.get_layer(nm)[b]
            o = oras[b].get_layer(nm)
            assert np.array_equal(np.isnan(g), np.isnan(o)), (b, nm)
            fin = ~np.isnan(o)
            if nm.endswith("_observed") or nm == "valid":
                assert np.array_equal(g, o), (b, nm)
            else:
                assert np.all(np.abs(g[fin].astype(np.float64) - o[fin]) <= 1e-6 + 1e-5 * np.abs(o[fin])), (b, nm)


# ---------------------------------------------------------------- C3 / C4 (configs[2], configs[3]) full size
def test_c3_rgbd_semantic_full_size():
    """three 640x480 depth clouds (stride 3) + a 20-class softmax image per frame, class_bayesian
    and class_max from the same channels."""
    c = S.C3
    groups = [dict(name="sem", rule=M.MEM_CLASS_BAYESIAN, n_channels=c["n_classes"], alpha0=1.0),
              dict(name="top", rule=M.MEM_CLASS_MAX, n_channels=c["n_classes"])]
    binds = [(0, c["n_classes"], 0), (0, c["n_classes"], 1)]
    g, o = make_pair(c["res"], c["rows"], c["cols"], groups)
    for f in range(3):
        fr = S.c3_frame(f)
        g.move_to(*fr["move"])
        o.move_to(*fr["move"])
        for cl in fr["clouds"]:
            step_points(g, o, cl["points"], [], cl["R"], cl["t"], c["noise"])
        im = fr["image"]
        g.input_image(torch.from_numpy(im["img"]).cuda(), binds, im["K"], im["R"], im["t"])
        o.input_image(im["img"], binds, im["K"], im["R"], im["t"])
        compare_layers(g, o, where=f"C3 frame {f}: ")
    assert (g.get_layer("top_label") >= 0).sum() > 5000


def test_c4_feature_image_full_size():
    """64-channel 480x640 feature image, 64 x average(w=0.5)."""
    c, c3 = S.C4, S.C3
    groups = [dict(name="feat", rule=M.MEM_AVERAGE, n_channels=c["d"], w=c["w"])]
    g, o = make_pair(c["res"], c["rows"], c["cols"], groups)
    fr = S.c3_frame(0)
    g.move_to(*fr["move"])
    o.move_to(*fr["move"])
    for cl in fr["clouds"]:
        step_points(g, o, cl["points"], [], cl["R"], cl["t"], c3["noise"], check_codes=False)
    for f in range(3):
        im = S.c4_image(f)
        g.input_image(torch.from_numpy(im["img"]).cuda(), [(0, c["d"], 0)], im["K"], im["R"], im["t"])
        o.input_image(im["img"], [(0, c["d"], 0)], im["K"], im["R"], im["t"])
    compare_layers(g, o, where="C4: ")
    assert g.get_layer("feat_observed").sum() > 5000
    # PCA readout (a14): top-3 components min-max scaled, 1e-4 abs on [0, 1] outputs (D28)
    gp, op = np.asarray(g.pca_readout("feat", 3)), o.pca_readout("feat", 3)
    assert np.abs(gp - op).max() <= 1e-4, np.abs(gp - op).max()
    assert (gp[:, g.get_layer("feat_observed") == 0] == 0).all()


def test_pca_readout_random_and_degenerate():
    rng = np.random.default_rng(71)
    rows, cols, d = 33, 47, 6
    groups = [dict(name="f", rule=M.MEM_AVERAGE, n_channels=d, w=0.5)]
    for case in ("random", "constant", "rank2"):
        g, o = make_pair(0.1, rows, cols, groups)
        if case == "random":
            f = (rng.normal(0, 1, (d, 1, 1)) * rng.normal(0, 1, (d, rows, cols)) + rng.normal(0, 1, (d, 1, 1)))
        elif case == "constant":
            f = np.full((d, rows, cols), 0.25)
        else:
            base = rng.normal(0, 1, (2, rows, cols))
            f = np.einsum("kd,krc->drc", rng.normal(0, 1, (2, d)), base)
        obs = (rng.uniform(size=(rows, cols)) < 0.8).astype(np.float32)
        for k in range(d):
            g.set_layer(f"f_{k}", f[k].astype(np.float32))
            o.set_layer(f"f_{k}", f[k].astype(np.float32))
        g.set_layer("f_observed", obs)
        o.set_layer("f_observed", obs)
        gp, op = np.asarray(g.pca_readout("f", 3)), o.pca_readout("f", 3)
        assert np.abs(gp - op).max() <= 1e-4, (case, np.abs(gp - op).max())
        if case == "constant":
            assert (gp == 0).all()
        if case == "rank2":
            assert (gp[2] == 0).all()  # beyond the rank: zero-filled


# ---------------------------------------------------------------- C5a (configs[4]) batched maps
def test_c5a_batched_maps_subset():
    """C5a shape (128x128 @ 0.1 m maps, 32,768 points each, height + average), 24 maps x 4 frames
    in one batched call per frame; every 8th map checked against its own oracle."""
    c = S.C5A
    B = 24
    groups = [dict(name="feat", rule=M.MEM_AVERAGE, n_channels=1, w=c["w"])]
    gb = M.Map(c["res"], c["rows"], c["cols"], groups, n_maps=B)
    check = list(range(0, B, 8))
    oras = {b: O.OracleMap(c["res"], c["rows"], c["cols"], groups) for b in check}
    for f in range(4):
        bt = S.c5a_batch(f, 0, B)
        gb.move_to_batch(bt["move"])
        gb.input_pointcloud_batch(torch.from_numpy(bt["points"]).cuda(), bt["offsets"], [(0, 1, 0)], bt["R"],
                                  bt["t"], c["noise"])
        for b in check:
            oras[b].move_to(*bt["move"][b])
            oras[b].input_pointcloud(bt["points"][bt["offsets"][b]:bt["offsets"][b + 1]], [(0, 1, 0)], bt["R"][b],
                                     bt["t"][b], c["noise"])
    for b in check:
        for nm in gb.layer_names():
            g, o = gb.get_layer(nm)[b], oras[b].get_layer(nm)
            assert np.array_equal(np.isnan(g), np.isnan(o)), (b, nm)
            fin = ~np.isnan(o)
            if nm in ("valid", "feat_observed"):
                assert np.array_equal(g, o), (b, nm)
            else:
                assert np.all(np.abs(g[fin].astype(np.float64) - o[fin]) <= 1e-6 + 1e-5 * np.abs(o[fin])), (b, nm)
        assert (gb.get_layer("valid")[b] > 0).sum() > 8000


@pytest.mark.parametrize("stride,offset", [(5, 0), (4, 1), (4, 0)])
def test_colour_group_any_stride_and_alignment(stride, offset):
    """a single colour group with xyz + rgb + intensity (stride 5), or a
    stride-4 cloud in a device buffer that is not 16-B aligned, must fuse exactly like the
    aligned float4 case (C2 LiDAR, 4 chained frames with shifts, vs the oracle)."""
    c = S.C2
    g, o = make_pair(c["res"], c["rows"], c["cols"], [dict(name="rgb", rule=M.MEM_COLOR, n_channels=3, w=c["w"])])
    for f in range(4):
        fr = S.c2_frame(f)
        pts = fr["points"]
        if stride == 5:
            pts = np.concatenate([pts, np.full((len(pts), 1), 7.0, np.float32)], 1)
        buf = torch.zeros(len(pts) * stride + offset, dtype=torch.float32, device="cuda")
        buf[offset:] = torch.from_numpy(np.ascontiguousarray(pts).reshape(-1)).cuda()
        src = buf[offset:].view(len(pts), stride)
        g.move_to(*fr["move"])
        o.move_to(*fr["move"])
        g.input_pointcloud(src, [(0, 1, 0)], fr["R"], fr["t"], c["noise"])
        oc = o.input_pointcloud(np.ascontiguousarray(pts), [(0, 1, 0)], fr["R"], fr["t"], c["noise"], debug=True)
        cell, code = g.debug_codes()
        assert np.array_equal(code, oc[1]) and np.array_equal(cell, oc[0])
        assert g.stats() == o.stats()
        compare_layers(g, o, where=f"stride {stride} offset {offset} frame {f}: ")
    assert (g.get_layer("rgb_r") > 0).sum() > 1000


def test_injected_state_then_fusion():
    """state written through mem_set_layer (valid first, as mem.h asks) then one fused frame:
    per-point codes (the Mahalanobis gate reads the injected h / s2) and every layer must match
    the oracle; variance written on invalid cells reads back as NaN."""
    c = S.C2
    groups = [dict(name="rgb", rule=M.MEM_COLOR, n_channels=3, w=c["w"])]
    g, o = make_pair(c["res"], c["rows"], c["cols"], groups)
    for f in range(3):  # the oracle alone builds a state
        fr = S.c2_frame(f)
        o.move_to(*fr["move"])
        o.input_pointcloud(fr["points"], [(0, 1, 0)], fr["R"], fr["t"], c["noise"])
    g.move_to(*S.c2_frame(2)["move"])
    assert tuple(g.center()[0]) == o.center()
    # checkpoint restore in layer_names() order through set_layers, which writes "valid"
    # first (variance before valid would be lost)
    g.set_layers({nm: o.get_layer(nm) for nm in g.layer_names()})
    compare_layers(g, o, where="injected: ")
    var = np.full((c["rows"], c["cols"]), 0.5, np.float32)
    h = g.get_layer("valid")
    g2 = M.Map(c["res"], c["rows"], c["cols"], groups)
    g2.set_layer("valid", h)
    g2.set_layer("variance", var)
    v2 = np.asarray(g2.get_layer("variance"))
    assert np.isnan(v2[h == 0]).all() and (v2[h == 1] == 0.5).all()
    fr = S.c2_frame(3)
    g.move_to(*fr["move"])
    o.move_to(*fr["move"])
    step_points(g, o, fr["points"], [(0, 1, 0)], fr["R"], fr["t"], c["noise"])
    compare_layers(g, o, where="after one frame: ")


# ---------------------------------------------------------------- NEXT-1 occlusion
def test_image_occlusion_random_terrain():
    """Bresenham occlusion on blocky + sloped terrain with unknown cells,
    several cameras (inside and outside the map), all rules: every layer vs the oracle, and
    the occlusion must actually remove cells the frustum alone would fuse."""
    rows, cols, res = 90, 70, 0.05
    g, o = make_pair(res, rows, cols, IMG_GROUPS)
    g.set_image_occlusion(True, 1e-4)
    o.set_occlusion(True, 1e-4)
    ref = O.OracleMap(res, rows, cols, IMG_GROUPS)  # same inputs, frustum only
    rng = np.random.default_rng(123)
    x = (np.arange(rows) + 0.5 - rows / 2) * res
    y = (np.arange(cols) + 0.5 - cols / 2) * res
    X, Y = np.meshgrid(x, y, indexing="ij")
    elev = 0.1 * np.sin(2 * X) * np.cos(3 * Y)
    for _ in range(8):
        r, c = rng.integers(5, rows - 12), rng.integers(5, cols - 12)
        elev[r:r + rng.integers(2, 8), c:c + rng.integers(2, 10)] += rng.uniform(0.3, 1.2)
    valid = (rng.uniform(size=(rows, cols)) > 0.05).astype(np.float32)
    for m in (g, o, ref):
        m.set_layer("valid", valid)
        m.set_layer("elevation", np.where(valid > 0, elev, np.nan).astype(np.float32))
        m.set_layer("variance", np.where(valid > 0, 0.01, np.nan).astype(np.float32))
    K = np.array([[150.0, 0.3, 79.5], [0, 148.0, 59.5], [0, 0, 1.0]])
    eyes = [(-1.9, 0.1, 1.2), (-3.0, -0.4, 1.6), (0.2, -2.2, 1.0), (1.9, 1.5, 2.0), (0.03, 0.02, 1.5)]
    for f, eye in enumerate(eyes):
        eye = np.array(eye)
        R = camera_looking_at(eye, [rng.uniform(-0.5, 0.5), rng.uniform(-0.5, 0.5), 0.0]) if f < 4 else \
            camera_looking_at(eye, [0.8, 0.3, 0.0])
        img = np.concatenate([S.softmax_image(rng.integers(0, 5, (120, 160)), 5, rng),
                              rng.normal(0, 1, (5, 120, 160)).astype(np.float32),
                              rng.uniform(0, 255, (3, 120, 160)).astype(np.float32)])
        g.input_image(torch.from_numpy(img).cuda(), IMG_BINDS, K, R, eye)
        o.input_image(img, IMG_BINDS, K, R, eye)
        ref.input_image(img, IMG_BINDS, K, R, eye)
        compare_layers(g, o, where=f"camera {f}: ")
    seen, seen_ref = g.get_layer("sem_observed"), ref.get_layer("sem_observed")
    assert (seen <= seen_ref).all() and (seen_ref - seen).sum() > 200 and seen.sum() > 1000


def test_c3_with_occlusion_full_size():
    c = S.C3
    groups = [dict(name="sem", rule=M.MEM_CLASS_BAYESIAN, n_channels=c["n_classes"], alpha0=1.0),
              dict(name="top", rule=M.MEM_CLASS_MAX, n_channels=c["n_classes"])]
    binds = [(0, c["n_classes"], 0), (0, c["n_classes"], 1)]
    g, o = make_pair(c["res"], c["rows"], c["cols"], groups)
    g.set_image_occlusion(True)
    o.set_occlusion(True)
    for f in range(2):
        fr = S.c3_frame(f)
        g.move_to(*fr["move"])
        o.move_to(*fr["move"])
        for cl in fr["clouds"]:
            step_points(g, o, cl["points"], [], cl["R"], cl["t"], c["noise"])
        im = fr["image"]
        g.input_image(torch.from_numpy(im["img"]).cuda(), binds, im["K"], im["R"], im["t"])
        o.input_image(im["img"], binds, im["K"], im["R"], im["t"])
        compare_layers(g, o, where=f"C3+occlusion frame {f}: ")
    assert (g.get_layer("top_label") >= 0).sum() > 5000


# ---------------------------------------------------------------- NEXT-3 plugins
def test_plugins_vs_oracle():
    """normals, traversability and semantic argmax (include/mem.h NEXT-3) on a fused random
    map with holes, after shifts (the ring is unrolled): bit-exact labels, fp32 tolerance."""
    rows, cols, res = 64, 48, 0.05
    g, o = make_pair(res, rows, cols, ALL_GROUPS)
    for f, (x, y) in enumerate([(0.0, 0.0), (0.12, -0.07), (0.31, 0.2)]):
        g.move_to(x, y)
        o.move_to(x, y)
        pts = random_all_channels(700 + f, 9000, rows, cols, res)
        step_points(g, o, pts, ALL_BINDS, S.rot_z(0.2 * f), np.array([x, y, 1.0]), NOISE_R)
    tol = lambda a, b: np.array_equal(np.isnan(a), np.isnan(b)) and np.all(
        np.abs(a[~np.isnan(b)] - b[~np.isnan(b)]) <= 1e-6 + 1e-5 * np.abs(b[~np.isnan(b)]))
    gn, on = np.asarray(g.normals()), o.normals()
    assert tol(gn, on) and (~np.isnan(on[2])).sum() > 1000
    for smax, stepmax in ((0.7, 0.2), (1.2, 0.05)):
        assert tol(np.asarray(g.traversability(smax, stepmax)), o.traversability(smax, stepmax))
    for grp in ("cavg", "sem", "top"):
        ga, oa = np.asarray(g.semantic_argmax(grp)), o.semantic_argmax(grp)
        assert np.array_equal(ga[0], oa[0]), grp
        assert tol(ga[1], oa[1]), grp
        assert (oa[0] >= 0).sum() > 1000
    with pytest.raises(M.MemError):
        g.semantic_argmax("feat")
    d = torch.empty((3, rows, cols), device="cuda")
    g.normals(out=d)
    assert tol(d.cpu().numpy(), on)


# ---------------------------------------------------------------- NEXT-4 paper-shaped workload
@pytest.mark.parametrize("rule,L", [(M.MEM_AVERAGE, 4), (M.MEM_CLASS_BAYESIAN, 20)])
def test_paper_cloud_full_size(rule, L):
    """the 230,400-point semantic cloud of the paper's performance setup."""
    c = S.PAPER
    groups = [dict(name="sem", rule=rule, n_channels=L, w=0.5, alpha0=1.0)]
    g, o = make_pair(c["res"], c["rows"], c["cols"], groups)
    for f in range(2):
        cl = S.paper_cloud(L, f)
        g.move_to(*cl["move"])
        o.move_to(*cl["move"])
        step_points(g, o, cl["points"], [(0, L, 0)], cl["R"], cl["t"], c["noise"])
        compare_layers(g, o, where=f"paper cloud L={L} frame {f}: ")
    assert g.get_layer("sem_observed").sum() > 5000


# ---------------------------------------------------------------- NEXT-2 top-k class input
def topk_channels(rng, n, K, k, bad_frac=0.02):
    """(n, 2k) pairs: distinct ids mostly, some repeated ids, some invalid ids / NaN."""
    ids = np.stack([rng.choice(K, k, replace=False) for _ in range(n)]).astype(np.float32)
    rep = rng.uniform(size=n) < 0.05
    ids[rep, 1] = ids[rep, 0]  # a repeated id: its probabilities add up
    p = rng.dirichlet(np.ones(k + 1), n)[:, :k].astype(np.float32)
    tie = rng.uniform(size=n) < 0.1
    p[tie] = np.round(p[tie] * 4) / 4  # exact ties exercise the lowest-index rule of class_max
    bad = rng.uniform(size=n) < bad_frac
    ids[bad, 0] = np.where(rng.uniform(size=bad.sum()) < 0.5, K + 2, 1.5)  # out of range / not integer
    nanm = rng.uniform(size=n) < bad_frac
    p[nanm, -1] = np.nan
    return np.stack([ids, p], 2).reshape(n, 2 * k)


TOPK_GROUPS = [dict(name="d", rule=M.MEM_CLASS_BAYESIAN, n_channels=9, alpha0=0.5),
               dict(name="a", rule=M.MEM_CLASS_AVERAGE, n_channels=9, w=0.4),
               dict(name="x", rule=M.MEM_CLASS_MAX, n_channels=9)]


def test_topk_points_and_images_vs_oracle():
    rows, cols, res, K, k = 50, 44, 0.05, 8, 3
    g, o = make_pair(res, rows, cols, TOPK_GROUPS)
    rng = np.random.default_rng(61)
    noise = dict(a=1e-3, b=0.0, r_min=0.0, r_max=100.0, h_min=-10.0, h_max=10.0, tau2=9.0, v_out=0.01)
    binds = [(0, 2 * k, gi, k) for gi in range(3)]
    Kimg = np.array([[120.0, 0.0, 79.5], [0, 118.0, 59.5], [0, 0, 1.0]])
    for f in range(4):
        pts = S.random_cloud(900 + f, 15000, 3, rows, cols, res)
        pts = np.concatenate([pts, topk_channels(rng, len(pts), K, k)], 1).astype(np.float32)
        step_points(g, o, pts, binds, np.eye(3), [0.0, 0.0, 1.0], noise)
        compare_layers(g, o, where=f"top-k points frame {f}: ")
        eye = np.array([rng.uniform(-3, -2), rng.uniform(-1, 1), rng.uniform(1.0, 2.0)])
        R = camera_looking_at(eye, [rng.uniform(-0.5, 0.5), rng.uniform(-0.5, 0.5), 0.0])
        img = np.ascontiguousarray(topk_channels(rng, 120 * 160, K, k).T.reshape(2 * k, 120, 160))
        g.input_image(torch.from_numpy(img).cuda(), binds, Kimg, R, eye)
        o.input_image(img, binds, Kimg, R, eye)
        compare_layers(g, o, where=f"top-k image frame {f}: ")
    assert (g.get_layer("x_label") >= 0).sum() > 1000
    with pytest.raises(M.MemError):  # top-k needs a class rule
        M.Map(res, rows, cols, [dict(name="f", rule=M.MEM_AVERAGE, n_channels=9)]).input_pointcloud(
            pts, [(0, 2 * k, 0, k)], np.eye(3), [0.0, 0.0, 1.0], noise)


# ---------------------------------------------------------------- k_smap (small maps, sort by cell)
def test_deterministic_small_maps_are_bit_exact():
    """MEM_FLAG_DETERMINISTIC: maps of <= 16384 cells with <= 65535 points take k_smap, which
    sums every cell's points in input order with the oracle's formulas: every layer must equal
    the oracle bit for bit (C1 with moves, a batch of C5a maps with shifts), per-point codes and
    counters too."""
    c = S.C1
    groups = [dict(name="feat", rule=M.MEM_AVERAGE, n_channels=1, w=c["w"])]
    g = M.Map(c["res"], c["rows"], c["cols"], groups, debug_points=True, deterministic=True)
    o = O.OracleMap(c["res"], c["rows"], c["cols"], groups)
    for f in range(c["frames"]):
        fr = S.c1_frame(f)
        g.move_to(*fr["move"])
        o.move_to(*fr["move"])
        step_points(g, o, fr["points"], [(0, 1, 0)], fr["R"], fr["t"], c["noise"])
        for nm in g.layer_names():
            assert np.array_equal(np.asarray(g.get_layer(nm)), o.get_layer(nm), equal_nan=True), (f, nm)
    c5 = S.C5A
    nmaps = 12
    gb = M.Map(c5["res"], c5["rows"], c5["cols"], [dict(name="feat", rule=0, n_channels=1, w=c5["w"])],
               n_maps=nmaps, deterministic=True)
    oras = [O.OracleMap(c5["res"], c5["rows"], c5["cols"], [dict(name="feat", rule=0, n_channels=1, w=c5["w"])])
            for _ in range(nmaps)]
    for f in range(3):
        bt = S.c5a_batch(f, 100, nmaps)
        gb.move_to_batch(bt["move"])
        gb.input_pointcloud_batch(torch.from_numpy(bt["points"]).cuda(), bt["offsets"], [(0, 1, 0)], bt["R"], bt["t"],
                                  c5["noise"])
        P = c5["points"]
        for b in range(nmaps):
            oras[b].move_to(*bt["move"][b])
            oras[b].input_pointcloud(bt["points"][b * P:(b + 1) * P], [(0, 1, 0)], bt["R"][b], bt["t"][b], c5["noise"])
    for nm in gb.layer_names():
        lay = np.asarray(gb.get_layer(nm))
        for b in range(nmaps):
            assert np.array_equal(lay[b], oras[b].get_layer(nm), equal_nan=True), (b, nm)


def test_deterministic_dense_cells_bit_exact():
    """cells with far more than 256 points (here ~2,000 in one cell and a
    few hundred in its neighbours, with z spanning many binades so that the fp64 sums are not
    exact) must still be summed in input order: every layer bit-identical to the oracle, over
    5 frames, and identical across two runs."""
    rows, cols, res = 32, 32, 0.1
    groups = [dict(name="feat", rule=M.MEM_AVERAGE, n_channels=1, w=0.5)]
    noise = dict(a=1e-4, b=1e-4, r_min=0.0, r_max=50.0, h_min=-5.0, h_max=5.0, tau2=9.0, v_out=0.01)
    outs = []
    for run in range(2):
        rng = np.random.default_rng(42)
        g = M.Map(res, rows, cols, groups, n_maps=64, deterministic=True)
        o = O.OracleMap(res, rows, cols, groups)
        for f in range(5):
            n = 6000
            xy = np.where(rng.uniform(size=(n, 1)) < 0.4, rng.normal(0.05, 0.01, (n, 2)), rng.uniform(-1.6, 1.6, (n, 2)))
            z = rng.normal(0.0, 1.0, n) * 10.0 ** rng.uniform(-8, 0, n)
            feat = rng.normal(0, 1, n) * 10.0 ** rng.uniform(-6, 3, n)
            pts = np.stack([xy[:, 0], xy[:, 1], z - 1.0, feat], 1).astype(np.float32)
            allp = np.tile(pts, (64, 1))
            offs = np.arange(65, dtype=np.int64) * n
            g.input_pointcloud_batch(torch.from_numpy(allp).cuda(), offs, [(0, 1, 0)], np.tile(np.eye(3), (64, 1, 1)),
                                     np.tile([0.0, 0.0, 1.0], (64, 1)), noise)
            o.input_pointcloud(pts, [(0, 1, 0)], np.eye(3), [0.0, 0.0, 1.0], noise)
        lay = {nm: np.asarray(g.get_layer(nm)) for nm in g.layer_names()}
        for nm, v in lay.items():
            for b in (0, 63):
                assert np.array_equal(v[b], o.get_layer(nm), equal_nan=True), (run, nm, b)
        outs.append(lay)
    for nm in outs[0]:
        assert np.array_equal(outs[0][nm], outs[1][nm], equal_nan=True), nm


@pytest.mark.parametrize("rule", ["color", "average"])
def test_deterministic_batch_without_debug_outputs_is_bit_exact(rule):
    """k_smap without per-point debug outputs (its production variant: the point's cell comes
    from its sorted position, z and v are recomputed) on a batch of 64 maps of 64x64 cells with
    up to 60,000 points each, dense and sparse maps, colour or average (with NaN features),
    moves every frame: every layer bit-identical to the oracle, counters equal."""
    rows, cols, res, B = 64, 64, 0.1, 64
    if rule == "color":
        groups = [dict(name="rgb", rule=M.MEM_COLOR, n_channels=3, w=0.4)]
    else:
        groups = [dict(name="feat", rule=M.MEM_AVERAGE, n_channels=1, w=0.4)]
    gb = M.Map(res, rows, cols, groups, n_maps=B, deterministic=True)
    oras = [O.OracleMap(res, rows, cols, groups) for _ in range(B)]
    rng = np.random.default_rng(31)
    for f in range(3):
        sizes = rng.integers(0, 60000, B)
        sizes[0], sizes[1] = 0, 60000
        clouds = []
        for b in range(B):
            p = S.random_cloud(1000 * f + b, int(sizes[b]), 4, rows, cols, res)
            if rule == "color":
                p[:, 3] = S.pack_rgb(rng.integers(0, 256, (len(p), 3)).astype(np.uint8))
            else:
                p[rng.uniform(size=len(p)) < 0.03, 3] = np.nan
            p[rng.uniform(size=len(p)) < 0.02, 2] += 2.0  # outliers
            clouds.append(p)
        offs = np.concatenate([[0], np.cumsum([len(p) for p in clouds])]).astype(np.int64)
        moves = rng.uniform(-0.3, 0.3, (B, 2)) * f
        Rs = np.stack([S.rot_z(0.1 * f + 0.01 * b) for b in range(B)])
        ts = np.stack([[moves[b, 0] + 0.01, moves[b, 1] - 0.02, 1.0] for b in range(B)])
        gb.move_to_batch(moves)
        gb.input_pointcloud_batch(torch.from_numpy(np.concatenate(clouds)).cuda(), offs, [(0, 1, 0)], Rs, ts, NOISE_R)
        for b in range(B):
            oras[b].move_to(*moves[b])
            oras[b].input_pointcloud(clouds[b], [(0, 1, 0)], Rs[b], ts[b], NOISE_R)
        st = gb.stats()
        for k in O.STAT_NAMES:
            assert st[k] == sum(o.stats()[k] for o in oras), (f, k)
    for nm in gb.layer_names():
        lay = np.asarray(gb.get_layer(nm))
        for b in range(B):
            assert np.array_equal(lay[b], oras[b].get_layer(nm), equal_nan=True), (rule, b, nm)
    assert sum((np.asarray(gb.get_layer("valid"))[b] > 0).sum() for b in range(B)) > 100000


def test_c5a_bench_configuration_sampled():
    """C5a exactly as bench.py's side line runs it: 4096 maps (256 generated maps tiled) in one
    batched call per step, k_smap with its full grid (one CTA per SM, each CTA walking ~28
    maps with its shared memory reused), frames alternating with moves; 3 steps.  Sampled maps
    (first and later maps of a CTA, the last map) are bit-identical to their own oracle."""
    c = S.C5A
    total, P = 4096, c["points"]
    pool = [S.c5a_batch(f, 0, 256) for f in range(2)]
    idx = np.arange(total) % 256
    dev = [torch.from_numpy(fr["points"].reshape(256, P, 4)[idx].reshape(-1, 4)).cuda() for fr in pool]
    offsets = np.arange(total + 1, dtype=np.int64) * P
    groups = [dict(name="feat", rule=M.MEM_AVERAGE, n_channels=1, w=c["w"])]
    gb = M.Map(c["res"], c["rows"], c["cols"], groups, n_maps=total)
    sample = [0, 147, 148, 296, 2049, 4095]
    oras = {b: O.OracleMap(c["res"], c["rows"], c["cols"], groups) for b in sample}
    for step in range(3):
        fr = pool[step % 2]
        gb.move_to_batch(fr["move"][idx])
        gb.input_pointcloud_batch(dev[step % 2], offsets, [(0, 1, 0)], fr["R"][idx], fr["t"][idx], c["noise"])
        for b in sample:
            g = idx[b]
            oras[b].move_to(*fr["move"][g])
            oras[b].input_pointcloud(fr["points"][g * P:(g + 1) * P], [(0, 1, 0)], fr["R"][g], fr["t"][g], c["noise"])
    for nm in gb.layer_names():
        lay = np.asarray(gb.get_layer(nm))
        for b in sample:
            assert np.array_equal(lay[b], oras[b].get_layer(nm), equal_nan=True), (b, nm)
    assert all((np.asarray(gb.get_layer("valid"))[b] > 0).sum() > 8000 for b in sample)


def test_deterministic_flag_falls_back_beyond_limits():
    """MEM_FLAG_DETERMINISTIC on inputs k_smap does not take (too many points per map, a
    multi-group map) fuses through the default path, still within the parity bar."""
    rows, cols, res = 40, 36, 0.1
    groups = [dict(name="feat", rule=M.MEM_AVERAGE, n_channels=1, w=0.5)]
    g = M.Map(res, rows, cols, groups, deterministic=True)
    o = O.OracleMap(res, rows, cols, groups)
    pts = S.random_cloud(4242, 70000, 4, rows, cols, res)  # > 65535 points
    step_points(g, o, pts, [(0, 1, 0)], np.eye(3), [0.0, 0.0, 1.0], NOISE_R, check_codes=False)
    compare_layers(g, o, where="70k points: ")
    g2 = M.Map(res, rows, cols, ALL_GROUPS, deterministic=True)
    o2 = O.OracleMap(res, rows, cols, ALL_GROUPS)
    step_points(g2, o2, random_all_channels(77, 5000, rows, cols, res), ALL_BINDS, np.eye(3), [0.0, 0.0, 1.0],
                NOISE_R, check_codes=False)
    compare_layers(g2, o2, where="all rules: ")


def test_c2x64_bench_configuration_sampled():
    """the headline step exactly as bench.py times it: 64 C2 maps batched in one call (one
    wave, colour fast path, frames rotating through the 16-frame pool with map m at frame
    (step + m) % 16); 3 steps; 6 sampled maps compared against their own oracle maps
    (counters of the sampled maps via per-map oracle sums, every layer)."""
    c = S.C2
    pool = [S.c2_frame(f) for f in range(16)]
    maps, npts = 64, pool[0]["points"].shape[0]
    groups = [dict(name="rgb", rule=M.MEM_COLOR, n_channels=3, w=c["w"])]
    gb = M.Map(c["res"], c["rows"], c["cols"], groups, n_maps=maps)
    sample = [0, 1, 17, 31, 50, 63]
    oras = {b: O.OracleMap(c["res"], c["rows"], c["cols"], groups) for b in sample}
    dev = [torch.from_numpy(fr["points"]).cuda() for fr in pool]
    offsets = np.arange(maps + 1, dtype=np.int64) * npts
    for step in range(3):
        idx = [(step + m) % 16 for m in range(maps)]
        gb.move_to_batch(np.stack([pool[i]["move"] for i in idx]))
        gb.input_pointcloud_batch(torch.cat([dev[i] for i in idx]), offsets, [(0, 1, 0)],
                                  np.stack([pool[i]["R"] for i in idx]), np.stack([pool[i]["t"] for i in idx]),
                                  c["noise"])
        for b in sample:
            fr = pool[idx[b]]
            oras[b].move_to(*fr["move"])
            oras[b].input_pointcloud(fr["points"], [(0, 1, 0)], fr["R"], fr["t"], c["noise"])
    for nm in gb.layer_names():
        lay = np.asarray(gb.get_layer(nm))
        for b in sample:
            o = oras[b].get_layer(nm)
            g = lay[b]
            assert np.array_equal(np.isnan(g), np.isnan(o)), (b, nm)
            fin = ~np.isnan(o)
            if nm.endswith("_observed") or nm == "valid":
                assert np.array_equal(g, o), (b, nm)
            else:
                assert np.all(np.abs(g[fin].astype(np.float64) - o[fin]) <= 1e-6 + 1e-5 * np.abs(o[fin])), (b, nm)
