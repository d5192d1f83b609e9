"""ctypes wrapper of the CPU oracle (oracle/mem_oracle.c).

TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs may import this module.  The product package
(paper_2309_16818_b200) never imports it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "mem_oracle.c")
LIB = os.path.join(HERE, "libmem_oracle.so")
# D29: IEEE fp32/fp64, round-to-nearest, no FMA contraction, no fast-math.
CFLAGS = ["-O2", "-std=c11", "-fPIC", "-shared", "-ffp-contract=off", "-fno-fast-math", "-fopenmp"]

AVERAGE, GAUSSIAN, CLASS_AVERAGE, CLASS_BAYESIAN, CLASS_MAX, COLOR = range(6)
INLIER, OUTLIER, NONFINITE, RANGE, HEIGHT, OOB = range(6)
STAT_NAMES = ["n_input", "n_nonfinite", "n_range", "n_height", "n_oob", "n_inlier", "n_outlier",
              "n_cells_touched"]


class _Spec(C.Structure):
    _fields_ = [("name", C.c_char_p), ("rule", C.c_int), ("n_channels", C.c_int), ("w", C.c_float),
                ("sigma_f2", C.c_float), ("mu0", C.c_float), ("sigma0_2", C.c_float), ("alpha0", C.c_float)]


class _Bind(C.Structure):
    _fields_ = [("ch_offset", C.c_int), ("n_ch", C.c_int), ("group", C.c_int), ("topk", C.c_int)]


class _Noise(C.Structure):
    _fields_ = [(n, C.c_float) for n in ("a", "b", "r_min", "r_max", "h_min", "h_max", "tau2", "v_out")]


def build(force=False):
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        subprocess.check_call(["gcc", *CFLAGS, "-o", LIB, SRC, "-lm"])
    return LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(LIB)
        vp = C.c_void_p
        L.om_create.restype = vp
        L.om_create.argtypes = [C.c_float, C.c_int, C.c_int, C.POINTER(_Spec), C.c_int, C.POINTER(C.c_int)]
        L.om_destroy.argtypes = [vp]
        L.om_input_pointcloud.argtypes = [vp, vp, C.c_long, C.c_int, C.POINTER(_Bind), C.c_int,
                                          C.POINTER(C.c_double), C.POINTER(C.c_double), C.POINTER(_Noise),
                                          vp, vp]
        L.om_input_image.argtypes = [vp, vp, C.c_int, C.c_int, C.c_int, C.POINTER(_Bind), C.c_int,
                                     C.POINTER(C.c_double), C.POINTER(C.c_double), C.POINTER(C.c_double)]
        L.om_move_to.argtypes = [vp, C.c_double, C.c_double]
        L.om_get_layer.argtypes = [vp, C.c_char_p, vp]
        L.om_set_layer.argtypes = [vp, C.c_char_p, vp]
        L.om_get_stats.argtypes = [vp, vp]
        L.om_get_center.argtypes = [vp, vp]
        L.om_pca_readout.argtypes = [vp, C.c_char_p, C.c_int, vp]
        L.om_bresenham.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, vp, vp, C.c_int]
        L.om_set_occlusion.argtypes = [vp, C.c_int, C.c_float]
        L.om_plugin_normals.argtypes = [vp, vp]
        L.om_plugin_traversability.argtypes = [vp, C.c_float, C.c_float, vp]
        L.om_plugin_semantic_argmax.argtypes = [vp, C.c_char_p, vp]
        L.om_accumulate.restype = vp
        L.om_accumulate.argtypes = L.om_input_pointcloud.argtypes + [C.POINTER(C.c_int)]
        L.om_fuse_rows.argtypes = [vp, vp, C.c_int, C.c_int]
        L.om_frame_free.argtypes = [vp]
        L.om_frame_array.restype = vp
        L.om_frame_array.argtypes = [vp, C.c_int, C.c_int, C.POINTER(C.c_long)]
        _lib = L
    return _lib


def _dbl(a, n):
    a = np.ascontiguousarray(np.asarray(a, np.float64).reshape(-1))
    assert a.size == n
    return a, a.ctypes.data_as(C.POINTER(C.c_double))


class OracleError(RuntimeError):
    def __init__(self, status, what):
        super().__init__(f"{what}: oracle status {status}")
        self.status = status


def make_binds(bindings):
    arr = (_Bind * max(1, len(bindings)))()
    for i, b in enumerate(bindings):  # (ch_offset, n_ch, group[, topk])
        arr[i] = _Bind(*b)
    return arr


def bresenham(a, b):
    """intermediate cells (exclusive of both endpoints) of the 8-connected line a -> b."""
    cap = 4 * (abs(a[0] - b[0]) + abs(a[1] - b[1])) + 8
    rr, cc = np.empty(cap, np.int32), np.empty(cap, np.int32)
    n = lib().om_bresenham(int(a[0]), int(a[1]), int(b[0]), int(b[1]), rr.ctypes.data, cc.ctypes.data, cap)
    return list(zip(rr[:n].tolist(), cc[:n].tolist()))


class OracleFrame:
    """one frame's per-cell sufficient statistics (om_accumulate), as writable numpy views:
    n_in, n_out (u64), P, S (f64), and per binding b: count[b] (u64), sums[b] (f64,
    [n_ch][cells]), keys[b] (u64 class_max keys or None); counters (u64[8])."""

    _FIELDS = {0: ("n_in", np.uint64), 1: ("n_out", np.uint64), 2: ("P", np.float64), 3: ("S", np.float64)}

    def __init__(self, handle, nb):
        self._h = handle
        L = lib()

        def view(field, b, dtype):
            n = C.c_long(0)
            ptr = L.om_frame_array(self._h, field, b, C.byref(n))
            if not ptr or n.value == 0:
                return None
            return np.ctypeslib.as_array(C.cast(ptr, C.POINTER(C.c_uint64 if dtype == np.uint64 else C.c_double)),
                                         (n.value,))

        for f, (name, dt) in self._FIELDS.items():
            setattr(self, name, view(f, 0, dt))
        self.count = [view(4, b, np.uint64) for b in range(nb)]
        self.sums = [view(5, b, np.float64) for b in range(nb)]
        self.keys = [view(6, b, np.uint64) for b in range(nb)]
        self.counters = view(7, 0, np.uint64)

    def arrays(self):
        """every statistic array with its merge operation ('sum' or 'max')"""
        out = [(self.n_in, "sum"), (self.n_out, "sum"), (self.P, "sum"), (self.S, "sum")]
        for c, s, k in zip(self.count, self.sums, self.keys):
            out += [(c, "sum"), (s, "sum")]
            if k is not None:
                out.append((k, "max"))
        return out

    def __del__(self):
        if getattr(self, "_h", None):
            lib().om_frame_free(self._h)
            self._h = None


class OracleMap:
    """One map of the oracle. groups: list of dicts(name, rule, n_channels, w, sigma_f2, mu0, sigma0_2, alpha0)."""

    def __init__(self, res, rows, cols, groups=()):
        L = lib()
        self.rows, self.cols, self.res = rows, cols, res
        self._names = [g["name"].encode() for g in groups]
        specs = (_Spec * max(1, len(groups)))()
        for i, g in enumerate(groups):
            specs[i] = _Spec(self._names[i], g["rule"], g.get("n_channels", 1), g.get("w", 1.0),
                             g.get("sigma_f2", 1.0), g.get("mu0", 0.0), g.get("sigma0_2", 1.0),
                             g.get("alpha0", 1.0))
        st = C.c_int(0)
        self._h = L.om_create(C.c_float(res), rows, cols, specs, len(groups), C.byref(st))
        if not self._h:
            raise OracleError(st.value, "om_create")

    def __del__(self):
        if getattr(self, "_h", None):
            lib().om_destroy(self._h)
            self._h = None

    def input_pointcloud(self, pts, bindings, R, t, noise, debug=False):
        pts = np.ascontiguousarray(pts, np.float32)
        n, stride = pts.shape
        Rr, Rp = _dbl(R, 9)
        tt, tp = _dbl(t, 3)
        nz = _Noise(**noise)
        cell = np.empty(n, np.int32) if debug else None
        code = np.empty(n, np.uint8) if debug else None
        st = lib().om_input_pointcloud(self._h, pts.ctypes.data, n, stride, make_binds(bindings), len(bindings),
                                       Rp, tp, C.byref(nz), cell.ctypes.data if debug else None,
                                       code.ctypes.data if debug else None)
        if st != 0:
            raise OracleError(st, "om_input_pointcloud")
        return (cell, code) if debug else None

    def accumulate(self, pts, bindings, R, t, noise, cells=False):
        """steps 1-2 only (per-point filtering and binning against the current state); with
        cells=True also returns every point's logical cell (-1 = dropped) and code."""
        pts = np.ascontiguousarray(pts, np.float32)
        n, stride = pts.shape
        Rr, Rp = _dbl(R, 9)
        tt, tp = _dbl(t, 3)
        nz = _Noise(**noise)
        st = C.c_int(0)
        cell = np.empty(max(n, 1), np.int32) if cells else None
        code = np.empty(max(n, 1), np.uint8) if cells else None
        h = lib().om_accumulate(self._h, pts.ctypes.data, n, stride, make_binds(bindings), len(bindings), Rp, tp,
                                C.byref(nz), cell.ctypes.data if cells else None, code.ctypes.data if cells else None,
                                C.byref(st))
        if not h:
            raise OracleError(st.value, "om_accumulate")
        fr = OracleFrame(h, len(bindings))
        return (fr, cell[:n], code[:n]) if cells else fr

    def fuse_rows(self, frame, row_lo, row_hi):
        """step 3 on rows [row_lo, row_hi)."""
        st = lib().om_fuse_rows(self._h, frame._h, row_lo, row_hi)
        if st != 0:
            raise OracleError(st, "om_fuse_rows")

    def normals(self):
        out = np.empty((3, self.rows, self.cols), np.float32)
        lib().om_plugin_normals(self._h, out.ctypes.data)
        return out

    def traversability(self, slope_max, step_max):
        """slope_max (rad): cos(slope_max) is rounded once to fp32 (reading D36)."""
        out = np.empty((self.rows, self.cols), np.float32)
        st = lib().om_plugin_traversability(self._h, C.c_float(float(np.float32(np.cos(slope_max)))),
                                            C.c_float(step_max), out.ctypes.data)
        if st != 0:
            raise OracleError(st, "om_plugin_traversability")
        return out

    def semantic_argmax(self, group):
        out = np.empty((2, self.rows, self.cols), np.float32)
        st = lib().om_plugin_semantic_argmax(self._h, group.encode(), out.ctypes.data)
        if st != 0:
            raise OracleError(st, "om_plugin_semantic_argmax")
        return out

    def set_occlusion(self, enable=True, eps_occ=1e-4):
        lib().om_set_occlusion(self._h, int(enable), C.c_float(eps_occ))

    def input_image(self, img, bindings, K, R, t):
        img = np.ascontiguousarray(img, np.float32)
        Cc, H, W = img.shape
        Kr, Kp = _dbl(K, 9)
        Rr, Rp = _dbl(R, 9)
        tt, tp = _dbl(t, 3)
        st = lib().om_input_image(self._h, img.ctypes.data, Cc, H, W, make_binds(bindings), len(bindings),
                                  Kp, Rp, tp)
        if st != 0:
            raise OracleError(st, "om_input_image")

    def move_to(self, x, y):
        st = lib().om_move_to(self._h, C.c_double(x), C.c_double(y))
        if st != 0:
            raise OracleError(st, "om_move_to")

    def get_layer(self, name):
        out = np.empty((self.rows, self.cols), np.float32)
        st = lib().om_get_layer(self._h, name.encode(), out.ctypes.data)
        if st != 0:
            raise OracleError(st, f"om_get_layer({name})")
        return out

    def set_layer(self, name, values):
        v = np.ascontiguousarray(np.broadcast_to(np.asarray(values, np.float32), (self.rows, self.cols)))
        st = lib().om_set_layer(self._h, name.encode(), v.ctypes.data)
        if st != 0:
            raise OracleError(st, f"om_set_layer({name})")

    def pca_readout(self, group, k=3):
        out = np.empty((k, self.rows, self.cols), np.float32)
        st = lib().om_pca_readout(self._h, group.encode(), k, out.ctypes.data)
        if st != 0:
            raise OracleError(st, f"om_pca_readout({group})")
        return out

    def stats(self):
        out = np.zeros(8, np.uint64)
        lib().om_get_stats(self._h, out.ctypes.data)
        return dict(zip(STAT_NAMES, (int(x) for x in out)))

    def center(self):
        out = np.zeros(2, np.int64)
        lib().om_get_center(self._h, out.ctypes.data)
        return int(out[0]), int(out[1])
