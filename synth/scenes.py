"""Seeded synthetic scenes and sensors for the MEM hot path (SURVEY.md §8(d) recipes).

This module is the ONLY code shared by the oracle side and the CUDA side of the tests:
it makes input bytes (points, images, poses, trajectories) and holds none of the
method's arithmetic (no binning, no filtering, no fusion).  Every generator takes an
explicit seed and returns float32 arrays in the layouts the C-ABI takes:

* point cloud: (N, stride) float32, AoS, xyz in the SENSOR frame then channels;
  a packed colour channel is 0x00RRGGBB bit-cast into float32 (reading D20);
* image: (C, H, W) float32, CHW;
* pose: R (3x3 float64, sensor->map), t (3, float64).

Scenes are 2.5D analytic height fields: a ground plane z = 0 plus
axis-aligned boxes and one ramp, each with a class id and an RGB colour.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

GROUND_CLASS = 0


@dataclass
class Box:
    x0: float
    x1: float
    y0: float
    y1: float
    height: float
    cls: int
    rgb: tuple


@dataclass
class Ramp:
    """Inclined patch z = slope * (x - x0) over [x0, x1] x [y0, y1] (top surface only)."""
    x0: float
    x1: float
    y0: float
    y1: float
    slope: float
    cls: int
    rgb: tuple


@dataclass
class Scene:
    boxes: list = field(default_factory=list)
    ramps: list = field(default_factory=list)
    ground_rgb: tuple = (90, 140, 60)
    ground_rgb2: tuple = (110, 160, 80)  # checker texture on the ground (1 m squares)

    # ---- height field and per-location attributes (world frame) ----
    def height(self, x, y):
        x = np.asarray(x, np.float64)
        y = np.asarray(y, np.float64)
        h = np.zeros(np.broadcast(x, y).shape)
        for b in self.boxes:
            inside = (x >= b.x0) & (x < b.x1) & (y >= b.y0) & (y < b.y1)
            h = np.where(inside, np.maximum(h, b.height), h)
        for r in self.ramps:
            inside = (x >= r.x0) & (x < r.x1) & (y >= r.y0) & (y < r.y1)
            h = np.where(inside, np.maximum(h, r.slope * (x - r.x0)), h)
        return h

    def attributes(self, x, y, z):
        """class id and rgb (uint8 x3) of the surface point (x, y, z)."""
        x = np.asarray(x, np.float64)
        y = np.asarray(y, np.float64)
        checker = ((np.floor(x) + np.floor(y)) % 2 == 0)
        cls = np.full(x.shape, GROUND_CLASS, np.int32)
        rgb = np.where(checker[..., None], np.array(self.ground_rgb), np.array(self.ground_rgb2))
        for r in self.ramps:
            inside = (x >= r.x0) & (x < r.x1) & (y >= r.y0) & (y < r.y1) & (z > 0.02)
            cls = np.where(inside, r.cls, cls)
            rgb = np.where(inside[..., None], np.array(r.rgb), rgb)
        for b in self.boxes:
            # points on or in the box (its top or its sides)
            inside = (x >= b.x0 - 1e-6) & (x <= b.x1 + 1e-6) & (y >= b.y0 - 1e-6) & (y <= b.y1 + 1e-6) & (z > 0.02)
            cls = np.where(inside, b.cls, cls)
            rgb = np.where(inside[..., None], np.array(b.rgb), rgb)
        return cls, rgb.astype(np.uint8)

    # ---- analytic ray casting (sensor simulation, not the method) ----
    def raycast(self, o, d, t_max=100.0):
        """first hit distance along unit rays d (N,3) from origin o (3,); inf if none."""
        o = np.asarray(o, np.float64)
        d = np.asarray(d, np.float64)
        n = d.shape[0]
        best = np.full(n, np.inf)
        with np.errstate(divide="ignore", invalid="ignore"):
            # ground plane z = 0
            t = -o[2] / d[:, 2]
            ok = (d[:, 2] < 0) & (t > 0)
            best = np.where(ok, np.minimum(best, t), best)
            for b in self.boxes:
                lo = np.array([b.x0, b.y0, 0.0])
                hi = np.array([b.x1, b.y1, b.height])
                t1 = (lo - o) / d
                t2 = (hi - o) / d
                tmin = np.nanmax(np.minimum(t1, t2), axis=1)
                tmax = np.nanmin(np.maximum(t1, t2), axis=1)
                ok = (tmax >= tmin) & (tmin > 0)
                best = np.where(ok, np.minimum(best, tmin), best)
            for r in self.ramps:
                # plane z = slope (x - x0)  <=>  slope*x - z = slope*x0
                nrm = np.array([r.slope, 0.0, -1.0])
                den = d @ nrm
                t = (r.slope * r.x0 - o @ nrm) / den
                p = o + t[:, None] * d
                ok = (t > 0) & (p[:, 0] >= r.x0) & (p[:, 0] < r.x1) & (p[:, 1] >= r.y0) & (p[:, 1] < r.y1)
                best = np.where(ok, np.minimum(best, t), best)
        best = np.where(best <= t_max, best, np.inf)
        return best


def rot_z(yaw):
    c, s = math.cos(yaw), math.sin(yaw)
    return np.array([[c, -s, 0.0], [s, c, 0.0], [0.0, 0.0, 1.0]])


def rot_y(a):
    c, s = math.cos(a), math.sin(a)
    return np.array([[c, 0.0, s], [0.0, 1.0, 0.0], [-s, 0.0, c]])


def rot_x(a):
    c, s = math.cos(a), math.sin(a)
    return np.array([[1.0, 0.0, 0.0], [0.0, c, -s], [0.0, s, c]])


def pack_rgb(rgb_u8):
    """(N,3) uint8 -> (N,) float32 whose bits are 0x00RRGGBB (reading D20)."""
    rgb = rgb_u8.astype(np.uint32)
    bits = (rgb[:, 0] << 16) | (rgb[:, 1] << 8) | rgb[:, 2]
    return bits.astype(np.uint32).view(np.float32)


def assert_tie_guard(x, res, guard=0.05):
    """every trajectory position must stay >= `guard` cell from a snap tie (D14)."""
    f = x / res + 0.5
    frac = f - math.floor(f)
    assert min(frac, 1.0 - frac) >= guard, f"position {x} within {guard} cell of a snap tie"


# --------------------------------------------------------------------------------------
# C1: 64x64 @ 0.1 m, plane + box, uniform points, 1 average-fused feature
# --------------------------------------------------------------------------------------
C1 = dict(res=0.1, rows=64, cols=64, n_points=10_000, frames=10, w=0.5,
          noise=dict(a=1e-4, b=1e-4, r_min=0.1, r_max=10.0, h_min=-3.0, h_max=0.5, tau2=9.0, v_out=0.01))


def c1_scene():
    return Scene(boxes=[Box(0.5, 1.5, -0.5, 0.5, 0.4, 1, (200, 30, 30))])


def c1_frame(frame, seed=1, n_points=C1["n_points"]):
    """One C1 frame: returns dict(points (N,4) f32 sensor frame, R, t, move=(x, y))."""
    rng = np.random.default_rng([seed, frame])
    scene = c1_scene()
    sensor = np.array([0.12 * frame, 0.0, 1.5])
    assert_tie_guard(sensor[0], C1["res"])
    assert_tie_guard(sensor[1], C1["res"])
    xy = sensor[:2] + rng.uniform(-3.4, 3.4, size=(n_points, 2))
    z = scene.height(xy[:, 0], xy[:, 1]) + rng.normal(0.0, 0.01, n_points)
    feat = (scene.height(xy[:, 0], xy[:, 1]) > 0.2).astype(np.float64) + rng.normal(0.0, 0.05, n_points)
    kind = rng.uniform(size=n_points)
    z = np.where(kind < 0.01, z + rng.uniform(0.5, 1.0, n_points), z)  # 1% outliers
    p = np.stack([xy[:, 0], xy[:, 1], z], 1) - sensor  # R = I
    far = (kind >= 0.01) & (kind < 0.015)
    p[far] *= 20.0  # 0.5% beyond r_max
    nanm = (kind >= 0.015) & (kind < 0.02)
    p[nanm, rng.integers(0, 3, nanm.sum())] = np.nan  # 0.5% non-finite
    pts = np.concatenate([p, feat[:, None]], 1).astype(np.float32)
    return dict(points=pts, R=np.eye(3), t=sensor.copy(), move=(sensor[0], sensor[1]))


# --------------------------------------------------------------------------------------
# C2: 200x200 @ 0.04 m, 128x1024 LiDAR with packed RGB, colour fusion, shift on motion
# --------------------------------------------------------------------------------------
C2 = dict(res=0.04, rows=200, cols=200, rings=128, azimuths=1024, frames=10, w=0.5,
          noise=dict(a=1e-4, b=2.5e-5, r_min=0.3, r_max=60.0, h_min=-2.5, h_max=1.0, tau2=9.0, v_out=0.01))


def c2_scene(seed=2):
    rng = np.random.default_rng([seed, 999])
    boxes = []
    colours = [(200, 40, 40), (40, 40, 200), (220, 200, 40), (160, 60, 200)]
    for k, (cx, cy) in enumerate([(2.0, 1.0), (-1.5, 2.2), (1.0, -2.5), (-2.5, -1.0)]):
        sx, sy = rng.uniform(0.4, 0.9, 2)
        boxes.append(Box(cx - sx, cx + sx, cy - sy, cy + sy, float(rng.uniform(0.2, 0.8)), 1 + k, colours[k]))
    ramps = [Ramp(3.0, 5.0, -1.0, 1.0, 0.25, 5, (130, 130, 130))]
    return Scene(boxes=boxes, ramps=ramps)


def c2_pose(frame):
    """trajectory: 0.046 m/frame along heading 30 deg, +0.1 rad/frame yaw, 1.0 m high.

    The trajectory repeats every 16 frames (the robot jumps back to the start, a large
    shift), because the tie guard cannot hold for longer straight runs at this speed."""
    frame = frame % 16
    x0, y0 = 0.0, 0.005
    hd = math.radians(30.0)
    x = x0 + 0.046 * frame * math.cos(hd)
    y = y0 + 0.046 * frame * math.sin(hd)
    assert_tie_guard(x, C2["res"])
    assert_tie_guard(y, C2["res"])
    return rot_z(0.1 * frame), np.array([x, y, 1.0])


def lidar_dirs(rings, azimuths, elev_deg=(-22.5, 22.5), az_offset=0.0):
    el = np.radians(np.linspace(elev_deg[0], elev_deg[1], rings))
    az = az_offset + 2.0 * math.pi * np.arange(azimuths) / azimuths
    el, az = np.meshgrid(el, az, indexing="ij")  # ring-major: row = ring
    d = np.stack([np.cos(el) * np.cos(az), np.cos(el) * np.sin(az), np.sin(el)], -1)
    return d.reshape(-1, 3)


def lidar_frame(scene, R, t, rng, rings, azimuths, noise_a, noise_b, outlier_frac=0.005, with_rgb=True,
                feature=None):
    """simulate an organised LiDAR scan; no-return rays are NaN. Returns (N, 4) float32."""
    d_s = lidar_dirs(rings, azimuths, az_offset=float(rng.uniform(0, 2 * math.pi / azimuths)))
    d_w = d_s @ R.T
    rng_t = scene.raycast(t, d_w)
    hit = np.isfinite(rng_t)
    r_true = np.where(hit, rng_t, 0.0)
    sigma = np.sqrt(noise_a + noise_b * r_true ** 2)
    r_meas = r_true + rng.normal(0.0, 1.0, r_true.shape) * sigma
    p_s = d_s * r_meas[:, None]
    pw = t + d_w * r_true[:, None]
    out = rng.uniform(size=r_true.shape) < outlier_frac
    p_s[out, 2] += rng.uniform(0.3, 1.0, out.sum())
    p_s[~hit] = np.nan
    if with_rgb:
        _, rgb = scene.attributes(pw[:, 0], pw[:, 1], pw[:, 2])
        ch = pack_rgb(rgb)
    else:
        ch = (feature(pw) if feature is not None else np.zeros(len(p_s))).astype(np.float32)
    pts = np.empty((p_s.shape[0], 4), np.float32)
    pts[:, :3] = p_s.astype(np.float32)
    pts[:, 3] = ch
    return pts


def c2_frame(frame, seed=2):
    rng = np.random.default_rng([seed, frame])
    scene = c2_scene(seed)
    R, t = c2_pose(frame)
    pts = lidar_frame(scene, R, t, rng, C2["rings"], C2["azimuths"], C2["noise"]["a"], C2["noise"]["b"])
    return dict(points=pts, R=R, t=t, move=(t[0], t[1]))


# --------------------------------------------------------------------------------------
# small random cases for parity tests (several tiles + ragged tails)
# --------------------------------------------------------------------------------------
def random_cloud(seed, n, stride, rows, cols, res, centre=(0.0, 0.0), z_sigma=0.05, nan_frac=0.02,
                 channel_kind="feature", n_classes=0, sensor_h=1.0):
    """uniform points over (slightly more than) the window; sensor frame with R = I at (centre, sensor_h)."""
    rng = np.random.default_rng(seed)
    ex, ey = rows * res / 2 * 1.1, cols * res / 2 * 1.1
    x = rng.uniform(-ex, ex, n)
    y = rng.uniform(-ey, ey, n)
    z = 0.3 * np.sin(x) * np.cos(y) + rng.normal(0, z_sigma, n)
    pts = np.zeros((n, stride), np.float32)
    pts[:, 0] = x
    pts[:, 1] = y
    pts[:, 2] = z - sensor_h
    nanm = rng.uniform(size=n) < nan_frac
    pts[nanm, 0] = np.nan
    if stride > 3:
        if channel_kind == "feature":
            pts[:, 3:] = rng.normal(0, 1, (n, stride - 3))
        elif channel_kind == "probs":
            k = n_classes
            logits = rng.normal(0, 1, (n, k))
            p = np.exp(logits)
            p /= p.sum(1, keepdims=True)
            pts[:, 3:3 + k] = p
        elif channel_kind == "rgb":
            pts[:, 3] = pack_rgb(rng.integers(0, 256, (n, 3)).astype(np.uint8))
    return pts


def softmax_image(labels, n_classes, rng, scale=4.0):
    """(H,W) int labels -> (K,H,W) float32 softmax of scale*onehot + N(0,1) logits (C3 recipe)."""
    H, W = labels.shape
    logits = rng.normal(0.0, 1.0, (n_classes, H, W))
    logits[labels, np.arange(H)[:, None], np.arange(W)[None, :]] += scale
    logits -= logits.max(0, keepdims=True)
    e = np.exp(logits)
    return (e / e.sum(0, keepdims=True)).astype(np.float32)


# --------------------------------------------------------------------------------------
# cameras (D17: optical axis +z_c, x right, y down; R = camera -> map)
# --------------------------------------------------------------------------------------
def camera_looking_at(eye, target):
    z = np.asarray(target, float) - np.asarray(eye, float)
    z /= np.linalg.norm(z)
    up = np.array([0.0, 0.0, 1.0])
    x = np.cross(z, up)
    x /= np.linalg.norm(x)
    y = np.cross(z, x)
    return np.stack([x, y, z], 1)


def camera_yaw_pitch(eye, yaw, pitch_down):
    """camera at `eye` looking along heading `yaw`, tilted `pitch_down` rad below horizontal."""
    d = np.array([math.cos(yaw) * math.cos(pitch_down), math.sin(yaw) * math.cos(pitch_down), -math.sin(pitch_down)])
    return camera_looking_at(eye, np.asarray(eye, float) + d)


def pinhole_rays(W, H, fx, fy, cx, cy):
    """unit ray directions (H*W, 3) in the camera frame, row-major over (v, u)."""
    u, v = np.meshgrid(np.arange(W, dtype=np.float64), np.arange(H, dtype=np.float64))
    d = np.stack([(u - cx) / fx, (v - cy) / fy, np.ones_like(u)], -1).reshape(-1, 3)
    return d / np.linalg.norm(d, axis=1, keepdims=True)


def depth_frame(scene, R, t, rng, W=640, H=480, f=385.0, noise_a=1e-6, noise_b=4e-6):
    """depth camera cloud (H*W, 3) float32 in the camera frame; no-hit pixels are NaN."""
    d_c = pinhole_rays(W, H, f, f, W / 2.0, H / 2.0)
    d_w = d_c @ R.T
    rng_t = scene.raycast(t, d_w, t_max=20.0)
    hit = np.isfinite(rng_t)
    r = np.where(hit, rng_t, 0.0)
    r_meas = r + rng.normal(0.0, 1.0, r.shape) * np.sqrt(noise_a + noise_b * r ** 2)
    p = d_c * r_meas[:, None]
    p[~hit] = np.nan
    return p.astype(np.float32), hit, (t + d_w * r[:, None])


# --------------------------------------------------------------------------------------
# C3: 250x250 @ 0.04 m, three 640x480 depth clouds + a 20-class softmax image
# --------------------------------------------------------------------------------------
C3 = dict(res=0.04, rows=250, cols=250, n_classes=20, frames=10, W=640, H=480, f=385.0, cam_h=0.7,
          pitch=math.radians(30.0),
          noise=dict(a=1e-6, b=4e-6, r_min=0.2, r_max=8.0, h_min=-1.5, h_max=1.5, tau2=9.0, v_out=0.01))


def c3_scene(seed=3):
    rng = np.random.default_rng([seed, 999])
    boxes = []
    for k in range(9):
        cx, cy = rng.uniform(-4.5, 4.5, 2)
        sx, sy = rng.uniform(0.2, 0.6, 2)
        boxes.append(Box(cx - sx, cx + sx, cy - sy, cy + sy, float(rng.uniform(0.1, 0.7)), 1 + k,
                         tuple(int(c) for c in rng.integers(0, 256, 3))))
    ramps = [Ramp(1.5, 3.5, 2.5, 4.0, 0.2, 10, (120, 120, 120))]
    return Scene(boxes=boxes, ramps=ramps)


def c3_frame(frame, seed=3, cameras=3):
    """three depth clouds (yaw 0, +-120 deg) and the front camera's 20-class softmax image."""
    rng = np.random.default_rng([seed, frame])
    scene = c3_scene(seed)
    c = C3
    x0, y0 = 0.009 + 0.029 * frame, 0.009 - 0.013 * frame
    assert_tie_guard(x0, c["res"])
    assert_tie_guard(y0, c["res"])
    heading = 0.05 * frame
    K = np.array([[c["f"], 0.0, c["W"] / 2.0], [0.0, c["f"], c["H"] / 2.0], [0.0, 0.0, 1.0]])
    clouds = []
    for k, dy in enumerate((0.0, 2 * math.pi / 3, -2 * math.pi / 3)[:cameras]):
        eye = np.array([x0, y0, c["cam_h"]])
        R = camera_yaw_pitch(eye, heading + dy, c["pitch"])
        pts, hit, pw = depth_frame(scene, R, eye, rng, c["W"], c["H"], c["f"], c["noise"]["a"], c["noise"]["b"])
        clouds.append(dict(points=pts, R=R, t=eye))
        if k == 0:
            cls, _ = scene.attributes(pw[:, 0], pw[:, 1], pw[:, 2])
            labels = np.where(hit, cls, 0).reshape(c["H"], c["W"])
            img = softmax_image(labels, c["n_classes"], rng)
            image = dict(img=img, K=K, R=R, t=eye)
    return dict(clouds=clouds, image=image, move=(x0, y0))


# --------------------------------------------------------------------------------------
# C4: 250x250 @ 0.04 m, 64-channel feature image (one C3 depth frame for geometry first)
# --------------------------------------------------------------------------------------
C4 = dict(res=0.04, rows=250, cols=250, d=64, frames=10, W=640, H=480, w=0.5)


def c4_class_features(seed=4, n_classes=20, d=64):
    rng = np.random.default_rng([seed, 12345])
    v = rng.normal(0.0, 1.0, (n_classes, d))
    return v / np.linalg.norm(v, axis=1, keepdims=True)


def c4_image(frame, seed=4):
    """64 x 480 x 640 feature image from the C3 front camera at frame 0: per-class unit vector +
    N(0, 0.1^2) per channel."""
    rng = np.random.default_rng([seed, frame])
    scene = c3_scene(3)
    c3 = c3_frame(0)
    im = c3["image"]
    d_c = pinhole_rays(C3["W"], C3["H"], C3["f"], C3["f"], C3["W"] / 2.0, C3["H"] / 2.0)
    d_w = d_c @ im["R"].T
    t = scene.raycast(im["t"], d_w, t_max=20.0)
    hit = np.isfinite(t)
    pw = im["t"] + d_w * np.where(hit, t, 0.0)[:, None]
    cls, _ = scene.attributes(pw[:, 0], pw[:, 1], pw[:, 2])
    cls = np.where(hit, cls, 0).reshape(C3["H"], C3["W"])
    feats = c4_class_features(seed)
    img = feats[cls].transpose(2, 0, 1) + rng.normal(0.0, 0.1, (C4["d"], C3["H"], C3["W"]))
    return dict(img=img.astype(np.float32), K=im["K"], R=im["R"], t=im["t"])


# --------------------------------------------------------------------------------------
# C5a: batched learning workload, B independent 128x128 @ 0.1 m maps x 32,768 points
# --------------------------------------------------------------------------------------
C5A = dict(res=0.1, rows=128, cols=128, points=32768, w=0.5, n_boxes=3,
           noise=dict(a=1e-4, b=1e-4, r_min=0.1, r_max=12.0, h_min=-3.0, h_max=1.0, tau2=9.0, v_out=0.01))


def c5a_batch(frame, first_map, n_maps, seed=1000, points=C5A["points"]):
    """points (n_maps*points, 4) f32 [x y z feature] in each map's sensor frame, per-map R (n,3,3),
    t (n,3), move (n,2).  Map m: its own plane + 3 boxes (seed 1000 + m), sensor 1.5 m high at a
    per-map start moving 0.07 m/frame along its own heading with yaw += 0.05 rad/frame; points
    uniform over +-7 m around the sensor (the window is +-6.4 m), z = height + N(0, 0.02^2), 1%
    outliers, 0.5% NaN; feature = box id / 3 + N(0, 0.05^2)."""
    nb, P = C5A["n_boxes"], points
    maps = np.arange(first_map, first_map + n_maps)
    # per-map scene parameters (deterministic in the map id)
    bx = np.empty((n_maps, nb, 5))
    heading = np.empty(n_maps)
    start = np.empty((n_maps, 2))
    for i, mm in enumerate(maps):
        r = np.random.default_rng([seed + int(mm), 7])
        c = r.uniform(-5, 5, (nb, 2))
        sz = r.uniform(0.3, 1.2, (nb, 2))
        bx[i, :, 0], bx[i, :, 1] = c[:, 0] - sz[:, 0], c[:, 0] + sz[:, 0]
        bx[i, :, 2], bx[i, :, 3] = c[:, 1] - sz[:, 1], c[:, 1] + sz[:, 1]
        bx[i, :, 4] = r.uniform(0.2, 0.9, nb)
        heading[i] = r.uniform(0, 2 * math.pi)
        start[i] = r.uniform(-0.5, 0.5, 2)
    rng = np.random.default_rng([seed, frame, first_map, n_maps])
    pos = start + 0.07 * frame * np.stack([np.cos(heading), np.sin(heading)], 1)
    # keep every snap >= 0.05 cell from a tie (D14 tie guard): nudge by a quarter cell if needed
    for ax in range(2):
        q = pos[:, ax] / C5A["res"] + 0.5
        fr = q - np.floor(q)
        bad = np.minimum(fr, 1 - fr) < 0.05
        pos[bad, ax] += 0.25 * C5A["res"]
    yaw = heading + 0.05 * frame
    xy = pos[:, None, :] + rng.uniform(-7.0, 7.0, (n_maps, P, 2))
    h = np.zeros((n_maps, P))
    fid = np.zeros((n_maps, P))
    for k in range(nb):
        inside = ((xy[..., 0] >= bx[:, None, k, 0]) & (xy[..., 0] < bx[:, None, k, 1]) &
                  (xy[..., 1] >= bx[:, None, k, 2]) & (xy[..., 1] < bx[:, None, k, 3]))
        h = np.where(inside, np.maximum(h, bx[:, None, k, 4]), h)
        fid = np.where(inside, k + 1, fid)
    z = h + rng.normal(0.0, 0.02, h.shape)
    kind = rng.uniform(size=h.shape)
    z = np.where(kind < 0.01, z + rng.uniform(0.5, 1.0, h.shape), z)
    t = np.concatenate([pos, np.full((n_maps, 1), 1.5)], 1)
    c, s = np.cos(yaw), np.sin(yaw)
    R = np.zeros((n_maps, 3, 3))
    R[:, 0, 0], R[:, 0, 1], R[:, 1, 0], R[:, 1, 1], R[:, 2, 2] = c, -s, s, c, 1.0
    d = np.stack([xy[..., 0] - t[:, None, 0], xy[..., 1] - t[:, None, 1], z - 1.5], -1)
    p = np.einsum("mji,mpj->mpi", R, d)  # R^T (world - t)
    nanm = (kind >= 0.01) & (kind < 0.015)
    p[nanm, 0] = np.nan
    feat = fid / 3.0 + rng.normal(0.0, 0.05, h.shape)
    pts = np.concatenate([p, feat[..., None]], -1).astype(np.float32).reshape(-1, 4)
    return dict(points=pts, R=R, t=t, move=pos.copy(), offsets=np.arange(n_maps + 1, dtype=np.int64) * P)


# --------------------------------------------------------------------------------------
# C5b: one 2000x2000 map @ 0.04 m (80 m), 4M points/frame, point-sharded
# --------------------------------------------------------------------------------------
C5B = dict(res=0.04, rows=2000, cols=2000, points=4_194_304, w=0.5, sensor_h=20.0,
           noise=dict(a=1e-4, b=2e-6, r_min=0.5, r_max=80.0, h_min=-25.0, h_max=-15.0, tau2=9.0, v_out=0.01))


def c5b_pose(frame):
    """a virtual elevated sensor 20 m above the map centre drifting 0.042 m/frame (1.05 cells)
    along +x and 0.0412 m/frame (1.03 cells) along +y with yaw 0.02 rad/frame; the snap
    fractions stay >= 0.05 cell from a tie for 12 frames (asserted)."""
    frame = frame % 12
    x, y = -0.01 + 0.042 * frame, -0.008 + 0.0412 * frame
    assert_tie_guard(x, C5B["res"])
    assert_tie_guard(y, C5B["res"])
    return rot_z(0.02 * frame), np.array([x, y, C5B["sensor_h"]])


def c5b_terrain(x, y):
    """smooth rolling terrain plus a 10 x 10 grid of 2 m blocks (0.6 m high)."""
    h = 0.4 * np.sin(x / 6.0) * np.cos(y / 9.0) + 0.01 * x
    blk = ((np.floor(x / 8.0) + np.floor(y / 8.0)) % 2 == 0) & (np.mod(x, 8.0) < 2.0) & (np.mod(y, 8.0) < 2.0)
    return h + 0.6 * blk, blk


def c5b_shard(frame, rank, nranks, seed=5, points=C5B["points"]):
    """rank's contiguous shard [rank*n/G, (rank+1)*n/G) of frame `frame`'s 4M points, (n/G, 4)
    float32 [x y z feature] in the sensor frame: (x, y) uniform over +-41 m around the map
    centre (the window is +-40 m; ~2.5% fall outside), z = terrain + N(0, 0.02^2), 1% outliers
    (+U[0.5, 1]), 0.5% NaN; feature = block indicator + N(0, 0.05^2).  The shards of one frame
    are drawn from per-shard seeds, so any G gives the same union only for the same G."""
    R, t = c5b_pose(frame)
    n = points // nranks
    rng = np.random.default_rng([seed, frame, rank, nranks])
    cx, cy = np.floor(t[0] / C5B["res"] + 0.5) * C5B["res"], np.floor(t[1] / C5B["res"] + 0.5) * C5B["res"]
    x = cx + rng.uniform(-41.0, 41.0, n)
    y = cy + rng.uniform(-41.0, 41.0, n)
    h, blk = c5b_terrain(x, y)
    z = h + rng.normal(0.0, 0.02, n)
    kind = rng.uniform(size=n)
    z = np.where(kind < 0.01, z + rng.uniform(0.5, 1.0, n), z)
    d = np.stack([x - t[0], y - t[1], z - t[2]], 1)
    p = d @ R  # R^T (world - t)
    p[(kind >= 0.01) & (kind < 0.015), 0] = np.nan
    feat = blk + rng.normal(0.0, 0.05, n)
    return dict(points=np.concatenate([p, feat[:, None]], 1).astype(np.float32), R=R, t=t, move=(t[0], t[1]))


# --------------------------------------------------------------------------------------
# PAPER: the performance setup of PAPER.md:404-408 / Table II / Fig. 6:
# 250x250 @ 0.04 m map, one ZED-2i-like 360x640 RGB-D camera -> a 230,400-point semantic cloud
# whose channels are L class probabilities (softmax of 4 onehot + N(0,1) over L classes)
# --------------------------------------------------------------------------------------
PAPER = dict(res=0.04, rows=250, cols=250, W=640, H=360, f=340.0, cam_h=0.7, pitch=math.radians(25.0),
             layers=(1, 2, 4, 8, 16, 20), noise=C3["noise"])


def paper_cloud(n_layers, frame=0, seed=6):
    """(230400, 3 + L) float32 [x y z p_0..p_{L-1}] in the camera frame (no-return pixels NaN),
    R, t, move.  The class of a point is the scene's object id modulo L."""
    c = PAPER
    rng = np.random.default_rng([seed, frame, n_layers])
    scene = c3_scene(3)
    x0, y0 = 0.009 + 0.029 * frame, 0.009 - 0.013 * frame
    assert_tie_guard(x0, c["res"])
    assert_tie_guard(y0, c["res"])
    eye = np.array([x0, y0, c["cam_h"]])
    R = camera_yaw_pitch(eye, 0.05 * frame, c["pitch"])
    pts, hit, pw = depth_frame(scene, R, eye, rng, c["W"], c["H"], c["f"], c["noise"]["a"], c["noise"]["b"])
    cls, _ = scene.attributes(pw[:, 0], pw[:, 1], pw[:, 2])
    cls = np.where(hit, cls, 0) % n_layers
    logits = 4.0 * np.eye(n_layers)[cls] + rng.normal(0.0, 1.0, (len(cls), n_layers))
    p = np.exp(logits - logits.max(1, keepdims=True))
    p /= p.sum(1, keepdims=True)
    return dict(points=np.concatenate([pts, p.astype(np.float32)], 1), R=R, t=eye, move=(x0, y0))
