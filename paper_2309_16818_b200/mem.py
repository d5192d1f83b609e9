"""Thin Python binding of libmem (include/mem.h) -- argument marshalling only.

Every step of the fusion path runs in the CUDA kernels of libmem.so; this module converts
numpy arrays / torch tensors to pointers and status codes to exceptions.  It never falls
back to anything: if libmem.so is missing, importing this module raises ImportError, and
without a CUDA device every call raises MemError(MEM_ECUDA).

The functions carry the C names (mem_create, mem_input_pointcloud, ...); `Map` wraps a
handle for convenience.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# MEM_LIB: a variant build of the same sources (tests/test_launch_config_gpu.py only)
LIB_PATH = os.environ.get("MEM_LIB") or os.path.join(HERE, "libmem.so")

MEM_OK, MEM_EINVAL, MEM_EDUPNAME, MEM_ENOTFOUND, MEM_ERULE, MEM_EPOSE, MEM_ECUDA, MEM_ENOMEM, MEM_ECOMM = (
    0, -1, -2, -3, -4, -5, -6, -7, -8)
MEM_AVERAGE, MEM_GAUSSIAN, MEM_CLASS_AVERAGE, MEM_CLASS_BAYESIAN, MEM_CLASS_MAX, MEM_COLOR = range(6)
CODE_INLIER, CODE_OUTLIER, CODE_NONFINITE, CODE_RANGE, CODE_HEIGHT, CODE_OOB = range(6)
MEM_FLAG_DEBUG_POINTS = 1
MEM_FLAG_DETERMINISTIC = 2
MEM_FLAG_FUSE_SORTED = 4
RULES = dict(average=MEM_AVERAGE, gaussian=MEM_GAUSSIAN, class_average=MEM_CLASS_AVERAGE,
             class_bayesian=MEM_CLASS_BAYESIAN, class_max=MEM_CLASS_MAX, color=MEM_COLOR)
STAT_NAMES = ["n_input", "n_nonfinite", "n_range", "n_height", "n_oob", "n_inlier", "n_outlier", "n_cells_touched"]

# the exported C-ABI (checked by tests/test_abi.py against include/mem.h)
EXPORTS = ["mem_create", "mem_create_batch", "mem_destroy", "mem_set_stream", "mem_synchronize",
           "mem_input_pointcloud", "mem_input_pointcloud_batch", "mem_input_image", "mem_input_image_batch",
           "mem_move_to", "mem_move_to_batch", "mem_get_layer", "mem_set_layer", "mem_get_layer_names",
           "mem_memory_footprint", "mem_get_info", "mem_get_center", "mem_frame_stats", "mem_debug_point_codes",
           "mem_profile", "mem_profile_read", "mem_pca_readout", "mem_nccl_unique_id", "mem_create_sharded",
           "mem_shard_local_sync", "mem_set_image_occlusion", "mem_plugin_normals",
           "mem_plugin_traversability", "mem_plugin_semantic_argmax", "mem_last_error", "mem_version"]
STAGES = ["shift", "point", "cell", "image", "read", "write", "h2d", "d2h"]


class mem_layer_spec(C.Structure):
    _fields_ = [("name", C.c_char_p), ("rule", C.c_int), ("n_channels", C.c_int), ("w", C.c_float),
                ("sigma_f2", C.c_float), ("mu0", C.c_float), ("sigma0_2", C.c_float), ("alpha0", C.c_float)]


class mem_binding(C.Structure):  # bindings are given as (ch_offset, n_ch, group[, topk]) tuples
    _fields_ = [("ch_offset", C.c_int), ("n_ch", C.c_int), ("group", C.c_int), ("topk", C.c_int)]


class mem_noise(C.Structure):
    _fields_ = [(n, C.c_float) for n in ("a", "b", "r_min", "r_max", "h_min", "h_max", "tau2", "v_out")]


class mem_stats(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in STAT_NAMES]


class MemError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"libmem status {status}: {msg}")
        self.status = status


if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is not built (python -m paper_2309_16818_b200.build); "
                      "libmem has no CPU fallback")

_lib = C.CDLL(LIB_PATH)
_vp = C.c_void_p
_P = C.POINTER
_sig = {
    "mem_create": [C.c_float, C.c_int, C.c_int, _P(mem_layer_spec), C.c_int, C.c_uint, _vp, _P(_vp)],
    "mem_create_batch": [C.c_int, C.c_float, C.c_int, C.c_int, _P(mem_layer_spec), C.c_int, C.c_uint, _vp, _P(_vp)],
    "mem_destroy": [_vp],
    "mem_set_stream": [_vp, _vp],
    "mem_synchronize": [_vp],
    "mem_input_pointcloud": [_vp, _vp, C.c_int64, C.c_int, _P(mem_binding), C.c_int, _P(C.c_double),
                             _P(C.c_double), _P(mem_noise)],
    "mem_input_pointcloud_batch": [_vp, _vp, _P(C.c_int64), C.c_int, _P(mem_binding), C.c_int, _P(C.c_double),
                                   _P(C.c_double), _P(mem_noise)],
    "mem_input_image": [_vp, _vp, C.c_int, C.c_int, C.c_int, _P(mem_binding), C.c_int, _P(C.c_double),
                        _P(C.c_double), _P(C.c_double)],
    "mem_input_image_batch": [_vp, _vp, C.c_int, C.c_int, C.c_int, _P(mem_binding), C.c_int, _P(C.c_double),
                              _P(C.c_double), _P(C.c_double)],
    "mem_move_to": [_vp, C.c_double, C.c_double],
    "mem_move_to_batch": [_vp, _P(C.c_double)],
    "mem_get_layer": [_vp, C.c_char_p, _vp],
    "mem_set_layer": [_vp, C.c_char_p, _vp],
    "mem_get_layer_names": [_vp, C.c_char_p, C.c_size_t],
    "mem_memory_footprint": [_vp, _P(C.c_uint64)],
    "mem_get_info": [_vp, _P(C.c_int), _P(C.c_int), _P(C.c_int), _P(C.c_float)],
    "mem_get_center": [_vp, _P(C.c_int64)],
    "mem_frame_stats": [_vp, _P(mem_stats)],
    "mem_debug_point_codes": [_vp, _vp, _vp],
    "mem_profile": [_vp, C.c_int],
    "mem_pca_readout": [_vp, C.c_char_p, C.c_int, _vp],
    "mem_nccl_unique_id": [_vp],
    "mem_create_sharded": [C.c_float, C.c_int, C.c_int, _P(mem_layer_spec), C.c_int, C.c_uint, _vp, _vp, C.c_int,
                           C.c_int, _P(_vp)],
    "mem_shard_local_sync": [_P(_vp), C.c_int],
    "mem_set_image_occlusion": [_vp, C.c_int, C.c_float],
    "mem_plugin_normals": [_vp, _vp],
    "mem_plugin_traversability": [_vp, C.c_float, C.c_float, _vp],
    "mem_plugin_semantic_argmax": [_vp, C.c_char_p, _vp],
    "mem_profile_read": [_vp, _P(C.c_double), _P(C.c_uint64), C.c_int],
}
for _n, _a in _sig.items():
    getattr(_lib, _n).argtypes = _a
    getattr(_lib, _n).restype = C.c_int
_lib.mem_last_error.restype = C.c_char_p
_lib.mem_last_error.argtypes = []
_lib.mem_version.restype = C.c_char_p
_lib.mem_version.argtypes = []


def mem_last_error():
    return _lib.mem_last_error().decode()


def mem_version():
    return _lib.mem_version().decode()


def _check(status, what):
    if status != MEM_OK:
        raise MemError(status, f"{what}: {mem_last_error()}")


# ---------------------------------------------------------------- marshalling helpers
def _ptr(x):
    """data pointer of a numpy array / torch tensor (contiguity checked) or an int address."""
    if x is None:
        return None
    if isinstance(x, int):
        return x
    if isinstance(x, np.ndarray):
        assert x.flags["C_CONTIGUOUS"], "array must be C-contiguous"
        return x.ctypes.data
    if hasattr(x, "data_ptr"):  # torch.Tensor
        assert x.is_contiguous(), "tensor must be contiguous"
        return x.data_ptr()
    raise TypeError(f"unsupported buffer type {type(x)}")


_DT = {"float32": (np.float32, "torch.float32"), "int64": (np.int64, "torch.int64")}


def _buf(x, dtype, min_elems=None, what="buffer"):
    """_ptr of an array / tensor after checking its element type and size: a
    float64 cloud or a too-small output buffer is refused instead of being read as garbage
    or written out of bounds."""
    if x is None or isinstance(x, int):
        return _ptr(x)
    npd, thd = _DT[dtype]
    if isinstance(x, np.ndarray):
        ok, n = x.dtype == npd, x.size
    elif hasattr(x, "data_ptr"):
        ok, n = str(x.dtype) == thd, x.numel()
    else:
        raise TypeError(f"unsupported buffer type {type(x)}")
    if not ok:
        raise TypeError(f"{what}: expected {dtype}, got {x.dtype}")
    if min_elems is not None and n < min_elems:
        raise ValueError(f"{what}: {n} elements, need at least {min_elems}")
    return _ptr(x)


def _dbl(a, n):
    """n doubles as a ctypes array (a copy: ~1 us, where ndarray.ctypes.data_as costs ~5 us)."""
    arr = np.asarray(a, np.float64)
    if arr.size != n:
        raise ValueError(f"expected {n} doubles, got {arr.size}")
    if not arr.flags["C_CONTIGUOUS"]:
        arr = np.ascontiguousarray(arr)
    buf = (C.c_double * n).from_buffer_copy(arr)
    return buf, buf


def _binds(bindings):
    arr = (mem_binding * max(1, len(bindings)))()
    for i, b in enumerate(bindings):
        arr[i] = mem_binding(*b)
    return arr


def _noise(noise):
    return mem_noise(**noise) if isinstance(noise, dict) else noise


def _stream_ptr(stream):
    if stream is None:
        try:
            import torch
            if torch.cuda.is_available():
                return torch.cuda.current_stream().cuda_stream
        except ImportError:
            pass
        return None
    return stream if isinstance(stream, int) else stream.cuda_stream


# ---------------------------------------------------------------- C-named functions
def _specs(groups):
    names = [g["name"].encode() for g in groups]
    specs = (mem_layer_spec * max(1, len(groups)))()
    for i, g in enumerate(groups):
        rule = RULES[g["rule"]] if isinstance(g["rule"], str) else g["rule"]
        specs[i] = mem_layer_spec(names[i], rule, g.get("n_channels", 3 if rule == MEM_COLOR else 1),
                                  g.get("w", 1.0), g.get("sigma_f2", 1.0), g.get("mu0", 0.0),
                                  g.get("sigma0_2", 1.0), g.get("alpha0", 1.0))
    return specs, names


def mem_nccl_unique_id():
    buf = C.create_string_buffer(128)
    _check(_lib.mem_nccl_unique_id(buf), "mem_nccl_unique_id")
    return buf.raw


def mem_create_sharded(resolution, rows, cols, groups, rank, nranks, nccl_id=None, flags=0, stream=None):
    specs, names = _specs(groups)
    h = _vp()
    idb = C.create_string_buffer(nccl_id, 128) if nccl_id is not None else None
    _check(_lib.mem_create_sharded(resolution, rows, cols, specs, len(groups), flags, _stream_ptr(stream), idb, rank,
                                   nranks, C.byref(h)), "mem_create_sharded")
    return h.value


def mem_shard_local_sync(handles):
    arr = (_vp * len(handles))(*handles)
    _check(_lib.mem_shard_local_sync(arr, len(handles)), "mem_shard_local_sync")


def mem_create(resolution, rows, cols, groups=(), flags=0, stream=None, n_maps=1):
    names = [g["name"].encode() for g in groups]
    specs = (mem_layer_spec * max(1, len(groups)))()
    for i, g in enumerate(groups):
        rule = RULES[g["rule"]] if isinstance(g["rule"], str) else g["rule"]
        specs[i] = mem_layer_spec(names[i], rule, g.get("n_channels", 3 if rule == MEM_COLOR else 1),
                                  g.get("w", 1.0), g.get("sigma_f2", 1.0), g.get("mu0", 0.0),
                                  g.get("sigma0_2", 1.0), g.get("alpha0", 1.0))
    h = _vp()
    if n_maps == 1:
        st = _lib.mem_create(resolution, rows, cols, specs, len(groups), flags, _stream_ptr(stream), C.byref(h))
    else:
        st = _lib.mem_create_batch(n_maps, resolution, rows, cols, specs, len(groups), flags, _stream_ptr(stream),
                                   C.byref(h))
    _check(st, "mem_create")
    return h.value


def mem_destroy(h):
    _check(_lib.mem_destroy(h), "mem_destroy")


def mem_input_pointcloud(h, pts, bindings, R, t, noise, n=None, stride=None):
    if n is None:
        n, stride = pts.shape
    _, Rp = _dbl(R, 9)
    _, tp = _dbl(t, 3)
    nz = _noise(noise)
    _check(_lib.mem_input_pointcloud(h, _buf(pts, "float32", n * stride, "points"), n, stride, _binds(bindings), len(bindings), Rp, tp, C.byref(nz)),
           "mem_input_pointcloud")


def mem_input_pointcloud_batch(h, pts, offsets, bindings, R, t, noise, stride=None, n_maps=None):
    off = np.ascontiguousarray(np.asarray(offsets, np.int64))
    n_maps = len(off) - 1
    stride = stride if stride is not None else pts.shape[-1]
    _, Rp = _dbl(R, 9 * n_maps)
    _, tp = _dbl(t, 3 * n_maps)
    nz = _noise(noise)
    _check(_lib.mem_input_pointcloud_batch(h, _buf(pts, "float32", int(off[-1]) * stride, "points"), off.ctypes.data_as(_P(C.c_int64)), stride,
                                           _binds(bindings), len(bindings), Rp, tp, C.byref(nz)),
           "mem_input_pointcloud_batch")


def mem_input_image(h, img, bindings, K, R, t):
    Cc, H, W = img.shape[-3:]
    _, Kp = _dbl(K, 9)
    _, Rp = _dbl(R, 9)
    _, tp = _dbl(t, 3)
    _check(_lib.mem_input_image(h, _buf(img, "float32", Cc * H * W, "image"), Cc, H, W, _binds(bindings), len(bindings), Kp, Rp, tp),
           "mem_input_image")


def mem_input_image_batch(h, img, bindings, K, R, t):
    B, Cc, H, W = img.shape
    _, Kp = _dbl(K, 9 * B)
    _, Rp = _dbl(R, 9 * B)
    _, tp = _dbl(t, 3 * B)
    _check(_lib.mem_input_image_batch(h, _buf(img, "float32", B * Cc * H * W, "image"), Cc, H, W, _binds(bindings), len(bindings), Kp, Rp, tp),
           "mem_input_image_batch")


def mem_move_to(h, x, y):
    _check(_lib.mem_move_to(h, float(x), float(y)), "mem_move_to")


def mem_move_to_batch(h, xy):
    arr = np.ascontiguousarray(np.asarray(xy, np.float64).reshape(-1))
    _check(_lib.mem_move_to_batch(h, arr.ctypes.data_as(_P(C.c_double))), "mem_move_to_batch")


def mem_get_info(h):
    b, r, c, res = C.c_int(), C.c_int(), C.c_int(), C.c_float()
    _check(_lib.mem_get_info(h, C.byref(b), C.byref(r), C.byref(c), C.byref(res)), "mem_get_info")
    return b.value, r.value, c.value, res.value


def mem_get_layer(h, name, out=None):
    B, H, W, _ = mem_get_info(h)
    if out is None:
        out = np.empty((B, H, W) if B > 1 else (H, W), np.float32)
    _check(_lib.mem_get_layer(h, name.encode(), _buf(out, "float32", B * H * W, "out")), f"mem_get_layer({name})")
    return out


def mem_set_layer(h, name, src):
    B, H, W, _ = mem_get_info(h)
    if isinstance(src, (int, float)):
        src = np.full((B, H, W), src, np.float32)
    _check(_lib.mem_set_layer(h, name.encode(), _buf(src, "float32", B * H * W, "src")), f"mem_set_layer({name})")


def mem_set_layers(h, layers):
    """restores a state {name: array} in a safe order: "valid" first, then the rest (an
    invalid cell stores no variance, so writing "variance" before "valid" would lose it;
    ADVICE r1)."""
    names = sorted(layers, key=lambda nm: 0 if nm == "valid" else 1)
    for nm in names:
        mem_set_layer(h, nm, layers[nm])


def mem_get_layer_names(h):
    buf = C.create_string_buffer(1 << 16)
    _check(_lib.mem_get_layer_names(h, buf, len(buf)), "mem_get_layer_names")
    return buf.value.decode().split()


def mem_memory_footprint(h):
    v = C.c_uint64()
    _check(_lib.mem_memory_footprint(h, C.byref(v)), "mem_memory_footprint")
    return v.value


def mem_get_center(h):
    B = mem_get_info(h)[0]
    out = np.zeros(2 * B, np.int64)
    _check(_lib.mem_get_center(h, out.ctypes.data_as(_P(C.c_int64))), "mem_get_center")
    return out.reshape(B, 2)


def mem_frame_stats(h):
    s = mem_stats()
    _check(_lib.mem_frame_stats(h, C.byref(s)), "mem_frame_stats")
    return {n: int(getattr(s, n)) for n in STAT_NAMES}


def mem_debug_point_codes(h, n):
    cell = np.empty(n, np.int32)
    code = np.empty(n, np.uint8)
    _check(_lib.mem_debug_point_codes(h, cell.ctypes.data, code.ctypes.data), "mem_debug_point_codes")
    return cell, code


def mem_pca_readout(h, group, k=3, out=None):
    B, H, W, _ = mem_get_info(h)
    if out is None:
        out = np.empty((B, k, H, W) if B > 1 else (k, H, W), np.float32)
    _check(_lib.mem_pca_readout(h, group.encode(), k, _buf(out, "float32", k * H * W, "out")), f"mem_pca_readout({group})")
    return out


def mem_profile(h, enable):
    _check(_lib.mem_profile(h, int(enable)), "mem_profile")


def mem_profile_read(h, reset=False):
    ms = (C.c_double * len(STAGES))()
    cnt = (C.c_uint64 * len(STAGES))()
    _check(_lib.mem_profile_read(h, ms, cnt, int(reset)), "mem_profile_read")
    return {s: (float(ms[i]), int(cnt[i])) for i, s in enumerate(STAGES)}


def mem_synchronize(h):
    _check(_lib.mem_synchronize(h), "mem_synchronize")


def mem_set_stream(h, stream):
    _check(_lib.mem_set_stream(h, _stream_ptr(stream)), "mem_set_stream")


class Map:
    """Owning wrapper of a mem_map handle (one map, or n_maps batched maps)."""

    def __init__(self, resolution, rows, cols, groups=(), n_maps=1, debug_points=False, stream=None, _handle=None,
                 deterministic=False, fuse_sorted=False):
        self.rows, self.cols, self.res, self.n_maps = rows, cols, resolution, n_maps
        flags = ((MEM_FLAG_DEBUG_POINTS if debug_points else 0) | (MEM_FLAG_DETERMINISTIC if deterministic else 0)
                 | (MEM_FLAG_FUSE_SORTED if fuse_sorted else 0))
        self.h = _handle if _handle is not None else mem_create(resolution, rows, cols, groups, flags, stream, n_maps)
        self._last_n = 0

    def _plugin(self, planes, call, *args, out=None):
        shape = (planes, self.n_maps, self.rows, self.cols) if self.n_maps > 1 else (planes, self.rows, self.cols)
        if out is None:
            out = np.empty(shape, np.float32)
        ptr = out.data_ptr() if hasattr(out, "data_ptr") else out.ctypes.data
        _check(call(self.h, *args, C.c_void_p(ptr)), call.__name__)
        return out

    def normals(self, out=None):
        """NEXT-3: normal_x, normal_y, normal_z planes (include/mem.h)."""
        return self._plugin(3, _lib.mem_plugin_normals, out=out)

    def traversability(self, slope_max, step_max, out=None):
        r = self._plugin(1, _lib.mem_plugin_traversability, C.c_float(slope_max), C.c_float(step_max), out=out)
        return r[0] if out is None else r

    def semantic_argmax(self, group, out=None):
        """NEXT-3: class_id, confidence planes of a class group."""
        return self._plugin(2, _lib.mem_plugin_semantic_argmax, group.encode(), out=out)

    def set_image_occlusion(self, enable=True, eps_occ=1e-4):
        """NEXT-1: Bresenham occlusion test for the following image inputs (include/mem.h)."""
        _check(_lib.mem_set_image_occlusion(self.h, int(enable), eps_occ), "mem_set_image_occlusion")

    @classmethod
    def sharded(cls, resolution, rows, cols, groups, rank, nranks, nccl_id=None, debug_points=False, stream=None):
        """rank `rank` of a big map sharded over `nranks` ranks (NCCL when nccl_id is given, else
        a local shard for single-process emulation; see include/mem.h)."""
        h = mem_create_sharded(resolution, rows, cols, groups, rank, nranks, nccl_id,
                               MEM_FLAG_DEBUG_POINTS if debug_points else 0, stream)
        return cls(resolution, rows, cols, groups, _handle=h)

    def close(self):
        if getattr(self, "h", None):
            mem_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def input_pointcloud(self, pts, bindings, R, t, noise):
        self._last_n = int(pts.shape[0])
        mem_input_pointcloud(self.h, pts, bindings, R, t, noise)

    def input_pointcloud_batch(self, pts, offsets, bindings, R, t, noise):
        self._last_n = int(offsets[-1])
        mem_input_pointcloud_batch(self.h, pts, offsets, bindings, R, t, noise)

    def input_image(self, img, bindings, K, R, t):
        mem_input_image(self.h, img, bindings, K, R, t)

    def input_image_batch(self, img, bindings, K, R, t):
        mem_input_image_batch(self.h, img, bindings, K, R, t)

    def move_to(self, x, y):
        mem_move_to(self.h, x, y)

    def move_to_batch(self, xy):
        mem_move_to_batch(self.h, xy)

    def get_layer(self, name, out=None):
        return mem_get_layer(self.h, name, out)

    def set_layer(self, name, src):
        mem_set_layer(self.h, name, src)

    def set_layers(self, layers):
        """checkpoint restore: {name: array} written "valid" first (see mem_set_layers)."""
        mem_set_layers(self.h, layers)

    def layer_names(self):
        return mem_get_layer_names(self.h)

    def footprint(self):
        return mem_memory_footprint(self.h)

    def center(self):
        return mem_get_center(self.h)

    def stats(self):
        return mem_frame_stats(self.h)

    def debug_codes(self):
        return mem_debug_point_codes(self.h, self._last_n)

    def synchronize(self):
        mem_synchronize(self.h)

    def pca_readout(self, group, k=3, out=None):
        return mem_pca_readout(self.h, group, k, out)

    def profile(self, enable=True):
        mem_profile(self.h, enable)

    def profile_read(self, reset=False):
        return mem_profile_read(self.h, reset)
