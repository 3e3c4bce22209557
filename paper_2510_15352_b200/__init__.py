"""Python binding of libgg (include/gg.h) — argument marshalling only.

Every step of the render path runs in the CUDA kernels of libgg.so
(csrc/).  This module never computes anything of the method itself and has
no CPU fallback: if libgg.so is missing or the device is not a CUDA GPU,
calls raise.  PyTorch is used for device memory (the caching allocator is
passed to libgg through the gg_allocator hook), streams and tensors.

The functions keep the C names (gg_create, gg_load_scene, gg_render, ...)
and accept torch tensors / numpy arrays in place of raw pointers.
`Renderer` is a small convenience object over the same calls.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("GG_LIB") or os.path.join(_HERE, "libgg.so")   # GG_LIB: an alternative in-tree build (A/B runs)

GG_OK, GG_E_INVALID, GG_E_NONFINITE, GG_E_OOM, GG_E_CUDA, GG_E_BAD_SCENE, GG_E_CAPACITY, GG_E_UNSUPPORTED = range(8)
GG_KEEP_INTERMEDIATES = 1
GG_COUNTERS = 2
GG_ASYNC = 4
GG_TIGHT_TILES = 8          # opacity-aware tile rects (reading R35)
GG_ELLIPSE_TILES = 16       # + ellipse-intersects-tile masks (reading R37)
(GG_DUMP_TILE_COUNTS, GG_DUMP_SORTED_TILE, GG_DUMP_SORTED_ZBITS, GG_DUMP_SORTED_GIDS, GG_DUMP_RANGES,
 GG_DUMP_COUNTERS, GG_DUMP_N_EVAL, GG_DUMP_PROJ) = range(8)

# every symbol include/gg.h declares
EXPORTS = ["gg_default_opts", "gg_create", "gg_destroy", "gg_load_scene", "gg_unload_scene", "gg_reserve",
           "gg_render", "gg_render_host", "gg_render_blur", "gg_blur_poses", "gg_checksum", "gg_check_errors", "gg_debug_dump", "gg_get_counters",
           "gg_launch_count", "gg_set_timing", "gg_get_stage_ms", "gg_last_error", "gg_status_string",
           "gg_read_ply", "gg_load_ply", "gg_ply_error", "gg_reserve_async", "gg_dino_input", "gg_get_stage_times",
           "gg_render_host_async", "gg_host_sync",
           "gg_chunk_envs"]


class GGError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{_status_name(status)}: {msg}")
        self.status = status


class gg_render_opts(C.Structure):
    _fields_ = [("near_plane", C.c_float), ("far_plane", C.c_float), ("background", C.c_float * 3),
                ("sh_degree", C.c_int32), ("rgb_format", C.c_int32), ("flags", C.c_uint32),
                ("debug_env", C.c_int32)]


ALLOC_FN = C.CFUNCTYPE(C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p)
FREE_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_void_p, C.c_void_p)


class gg_allocator(C.Structure):
    _fields_ = [("alloc", ALLOC_FN), ("free", FREE_FN), ("user", C.c_void_p)]


_lib = None


def load_library(path: str = LIB_PATH):
    """Load libgg.so; raises (no fallback) if it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"libgg.so not built at {path}: run paper_2510_15352_b200/build.sh "
                          "(or __graft_entry__.build()); there is no CPU fallback")
    L = C.CDLL(path)
    vp, i32, i64 = C.c_void_p, C.c_int32, C.c_int64
    fp = C.c_void_p
    L.gg_default_opts.argtypes = [C.POINTER(gg_render_opts)]
    L.gg_default_opts.restype = None
    L.gg_create.argtypes = [C.c_int, C.POINTER(gg_allocator), C.POINTER(vp)]
    L.gg_destroy.argtypes = [vp]
    L.gg_load_scene.argtypes = [vp, i64, i32, fp, fp, fp, fp, fp, C.POINTER(i32)]
    L.gg_unload_scene.argtypes = [vp, i32]
    L.gg_reserve.argtypes = [vp, i32, i32, i32, i32]
    L.gg_reserve_async.argtypes = [vp, i32, i32, i32, i32, C.c_float, C.c_float]
    L.gg_render.argtypes = [vp, i32, vp, vp, vp, i32, i32, C.POINTER(gg_render_opts), vp, vp, vp, vp]
    L.gg_render_host.argtypes = [vp, i32, vp, vp, vp, i32, i32, C.POINTER(gg_render_opts), vp, vp, vp, vp]
    L.gg_render_host_async.argtypes = [vp, i32, vp, vp, vp, i32, i32, C.POINTER(gg_render_opts), vp, vp, vp, vp]
    L.gg_host_sync.argtypes = [vp]
    L.gg_render_blur.argtypes = [vp, i32, vp, vp, vp, vp, vp, C.c_float, i32, i32, i32, C.POINTER(gg_render_opts),
                                 vp, vp, vp, vp]
    L.gg_blur_poses.argtypes = [vp, i32, vp, vp, vp, C.c_float, i32, vp, vp]
    L.gg_checksum.argtypes = [vp, i32, i32, i32, vp, i32, vp, vp, vp]
    L.gg_dino_input.argtypes = [vp, i32, i32, i32, vp, i32, vp, vp]
    L.gg_check_errors.argtypes = [vp, vp]
    L.gg_debug_dump.argtypes = [vp, i32, vp, i64, C.POINTER(i64)]
    L.gg_get_counters.argtypes = [vp, i32, vp]
    L.gg_launch_count.argtypes = [vp]
    L.gg_launch_count.restype = i64
    L.gg_chunk_envs.argtypes = [vp]
    L.gg_chunk_envs.restype = i32
    L.gg_set_timing.argtypes = [vp, i32]
    L.gg_get_stage_ms.argtypes = [vp, C.POINTER(C.c_float)]
    L.gg_get_stage_times.argtypes = [vp, C.POINTER(C.c_float), i32]
    L.gg_last_error.argtypes = [vp]
    L.gg_last_error.restype = C.c_char_p
    L.gg_status_string.argtypes = [C.c_int]
    L.gg_status_string.restype = C.c_char_p
    L.gg_read_ply.argtypes = [C.c_char_p, C.POINTER(i64), C.POINTER(i32), vp, vp, vp, vp, vp]
    L.gg_load_ply.argtypes = [vp, C.c_char_p, C.POINTER(i32)]
    L.gg_ply_error.argtypes = []
    L.gg_ply_error.restype = C.c_char_p
    for name in EXPORTS:
        if name not in ("gg_default_opts", "gg_launch_count", "gg_last_error", "gg_status_string", "gg_ply_error",
                        "gg_chunk_envs"):
            getattr(L, name).restype = C.c_int
    _lib = L
    return L


def _status_name(s: int) -> str:
    try:
        return load_library().gg_status_string(s).decode()
    except Exception:
        return f"status {s}"


def _check(ctx, status: int):
    if status != GG_OK:
        msg = load_library().gg_last_error(ctx).decode() if ctx else ""
        raise GGError(status, msg)


def _ptr(x) -> int | None:
    """Raw address of a torch tensor / numpy array (None passes NULL)."""
    if x is None:
        return None
    if isinstance(x, np.ndarray):
        if not x.flags["C_CONTIGUOUS"]:
            raise ValueError("array must be C-contiguous")
        return x.ctypes.data
    if hasattr(x, "data_ptr"):
        if not x.is_contiguous():
            raise ValueError("tensor must be contiguous")
        return x.data_ptr()
    raise TypeError(f"cannot take the address of {type(x)}")


def _stream_handle(stream) -> int:
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


def default_opts(**kw) -> gg_render_opts:
    o = gg_render_opts()
    load_library().gg_default_opts(C.byref(o))
    for k, v in kw.items():
        if k == "background":
            o.background = (C.c_float * 3)(*v)
        else:
            setattr(o, k, v)
    return o


# ---------------------------------------------------------------- C names

def torch_allocator(device: int) -> tuple[gg_allocator, tuple]:
    """gg_allocator routed to the PyTorch caching allocator of `device`."""
    import torch

    def _alloc(size, stream, user):
        try:
            return int(torch.cuda.caching_allocator_alloc(int(size), device, int(stream or 0)))
        except Exception:
            return 0

    def _free(ptr, stream, user):
        torch.cuda.caching_allocator_delete(int(ptr))

    a, f = ALLOC_FN(_alloc), FREE_FN(_free)
    return gg_allocator(a, f, None), (a, f)


def gg_create(device: int = 0, allocator: gg_allocator | None = None):
    L = load_library()
    h = C.c_void_p()
    _check(None, L.gg_create(device, C.byref(allocator) if allocator is not None else None, C.byref(h)))
    return h


def gg_destroy(ctx):
    _check(ctx, load_library().gg_destroy(ctx))


def gg_load_scene(ctx, n, sh_degree, means, scales, quats, opacities, sh) -> int:
    out = C.c_int32(-1)
    _check(ctx, load_library().gg_load_scene(ctx, int(n), int(sh_degree), _ptr(means), _ptr(scales), _ptr(quats),
                                             _ptr(opacities), _ptr(sh), C.byref(out)))
    return out.value


def gg_unload_scene(ctx, scene_id: int):
    _check(ctx, load_library().gg_unload_scene(ctx, int(scene_id)))


def gg_reserve(ctx, max_envs: int, width: int, height: int, chunk_envs: int = 0):
    _check(ctx, load_library().gg_reserve(ctx, max_envs, width, height, chunk_envs))


def gg_reserve_async(ctx, max_envs: int, width: int, height: int, chunk_envs: int = 0,
                     max_visible_frac: float = 0.6, keys_per_visible: float = 4.0):
    _check(ctx, load_library().gg_reserve_async(ctx, max_envs, width, height, chunk_envs, max_visible_frac,
                                                keys_per_visible))


def gg_render(ctx, n_envs, scene_ids, viewmats, intrinsics, width, height, opts=None, rgb=None, depth=None,
              alpha=None, stream=None):
    o = opts if opts is not None else default_opts()
    _check(ctx, load_library().gg_render(ctx, int(n_envs), _ptr(scene_ids), _ptr(viewmats), _ptr(intrinsics),
                                         int(width), int(height), C.byref(o), _ptr(rgb), _ptr(depth), _ptr(alpha),
                                         _stream_handle(stream)))


def gg_render_host(ctx, n_envs, scene_ids, viewmats, intrinsics, width, height, opts=None, rgb=None, depth=None,
                   alpha=None, stream=None):
    o = opts if opts is not None else default_opts()
    _check(ctx, load_library().gg_render_host(ctx, int(n_envs), _ptr(scene_ids), _ptr(viewmats), _ptr(intrinsics),
                                              int(width), int(height), C.byref(o), _ptr(rgb), _ptr(depth),
                                              _ptr(alpha), _stream_handle(stream)))


def gg_render_host_async(ctx, n_envs, scene_ids, viewmats, intrinsics, width, height, opts=None, rgb=None,
                         depth=None, alpha=None, stream=None):
    """gg_render_host without the final wait: host buffers are valid after gg_host_sync."""
    o = opts if opts is not None else default_opts()
    _check(ctx, load_library().gg_render_host_async(ctx, int(n_envs), _ptr(scene_ids), _ptr(viewmats),
                                                    _ptr(intrinsics), int(width), int(height), C.byref(o), _ptr(rgb),
                                                    _ptr(depth), _ptr(alpha), _stream_handle(stream)))


def gg_host_sync(ctx):
    _check(ctx, load_library().gg_host_sync(ctx))


def gg_render_blur(ctx, n_envs, scene_ids, viewmats, intrinsics, lin_vel, ang_vel, shutter, K, width, height,
                   opts=None, rgb=None, depth=None, alpha=None, stream=None):
    o = opts if opts is not None else default_opts()
    _check(ctx, load_library().gg_render_blur(ctx, int(n_envs), _ptr(scene_ids), _ptr(viewmats), _ptr(intrinsics),
                                              _ptr(lin_vel), _ptr(ang_vel), float(shutter), int(K), int(width),
                                              int(height), C.byref(o), _ptr(rgb), _ptr(depth), _ptr(alpha),
                                              _stream_handle(stream)))


def gg_blur_poses(ctx, n_envs, viewmats, lin_vel, ang_vel, shutter, K, out, stream=None):
    _check(ctx, load_library().gg_blur_poses(ctx, int(n_envs), _ptr(viewmats), _ptr(lin_vel), _ptr(ang_vel),
                                             float(shutter), int(K), _ptr(out), _stream_handle(stream)))


def gg_checksum(ctx, n_envs, width, height, rgb, rgb_format, depth, out, stream=None):
    _check(ctx, load_library().gg_checksum(ctx, int(n_envs), int(width), int(height), _ptr(rgb), int(rgb_format),
                                           _ptr(depth), _ptr(out), _stream_handle(stream)))


def gg_dino_input(ctx, n_envs, width, height, rgb, size, out, stream=None):
    """u8 [E,H,W,3] device frames -> bf16 [E,3,size,size] DinoV2 input (R36)."""
    _check(ctx, load_library().gg_dino_input(ctx, int(n_envs), int(width), int(height), _ptr(rgb), int(size),
                                             _ptr(out), _stream_handle(stream)))


def gg_check_errors(ctx, stream=None):
    _check(ctx, load_library().gg_check_errors(ctx, _stream_handle(stream)))


def gg_debug_dump(ctx, kind: int) -> np.ndarray:
    L = load_library()
    n = C.c_int64(0)
    _check(ctx, L.gg_debug_dump(ctx, kind, None, 0, C.byref(n)))
    dt = {GG_DUMP_SORTED_ZBITS: np.uint32, GG_DUMP_COUNTERS: np.int64, GG_DUMP_PROJ: np.float32}.get(kind, np.int32)
    a = np.zeros(n.value, dtype=dt)
    if n.value:
        _check(ctx, L.gg_debug_dump(ctx, kind, a.ctypes.data, n.value, C.byref(n)))
    return a


def gg_get_counters(ctx, n_envs: int) -> np.ndarray:
    a = np.zeros((n_envs, 4), np.int64)
    _check(ctx, load_library().gg_get_counters(ctx, n_envs, a.ctypes.data))
    return a


def gg_chunk_envs(ctx) -> int:
    return int(load_library().gg_chunk_envs(ctx))


def gg_launch_count(ctx) -> int:
    return int(load_library().gg_launch_count(ctx))


def gg_set_timing(ctx, enable: bool):
    _check(ctx, load_library().gg_set_timing(ctx, 1 if enable else 0))


def gg_get_stage_ms(ctx) -> tuple[float, float, float]:
    a = (C.c_float * 3)()
    _check(ctx, load_library().gg_get_stage_ms(ctx, a))
    return tuple(a)


STAGES = ("cull", "project", "depth_sort", "placement", "raster")


def gg_get_stage_times(ctx, n: int = 5) -> tuple:
    """Finer per-stage ms of the last timed render (STAGES order)."""
    a = (C.c_float * n)()
    _check(ctx, load_library().gg_get_stage_times(ctx, a, n))
    return tuple(a)


def gg_read_ply(path: str):
    """Parse a 3DGS PLY into activated numpy arrays (means, scales, quats, opacities, sh, degree)."""
    L = load_library()
    n, d = C.c_int64(0), C.c_int32(0)
    st = L.gg_read_ply(path.encode(), C.byref(n), C.byref(d), None, None, None, None, None)
    if st != GG_OK:
        raise GGError(st, L.gg_ply_error().decode())
    N, K = n.value, (d.value + 1) ** 2
    m, s, q = np.zeros((N, 3), np.float32), np.zeros((N, 3), np.float32), np.zeros((N, 4), np.float32)
    o, sh = np.zeros(N, np.float32), np.zeros((N, K, 3), np.float32)
    st = L.gg_read_ply(path.encode(), C.byref(n), C.byref(d), m.ctypes.data, s.ctypes.data, q.ctypes.data,
                       o.ctypes.data, sh.ctypes.data)
    if st != GG_OK:
        raise GGError(st, L.gg_ply_error().decode())
    return m, s, q, o, sh, d.value


def gg_load_ply(ctx, path: str) -> int:
    out = C.c_int32(-1)
    st = load_library().gg_load_ply(ctx, path.encode(), C.byref(out))
    if st != GG_OK:
        msg = load_library().gg_ply_error().decode() or load_library().gg_last_error(ctx).decode()
        raise GGError(st, msg)
    return out.value


def gg_ply_error() -> str:
    return load_library().gg_ply_error().decode()


def gg_last_error(ctx) -> str:
    return load_library().gg_last_error(ctx).decode()


def gg_status_string(s: int) -> str:
    return load_library().gg_status_string(s).decode()


# ---------------------------------------------------------------- convenience

class Renderer:
    """One context on one CUDA device, memory from the torch caching allocator."""

    def __init__(self, device: int = 0, use_torch_allocator: bool = True):
        import torch
        if not torch.cuda.is_available():
            raise RuntimeError("paper_2510_15352_b200 needs a CUDA device (no CPU fallback)")
        self.device = device
        self._keep = None
        alloc = None
        if use_torch_allocator:
            alloc, self._keep = torch_allocator(device)
        with torch.cuda.device(device):
            self.ctx = gg_create(device, alloc)

    def load_scene(self, means, scales, quats, opacities, sh, sh_degree: int) -> int:
        return gg_load_scene(self.ctx, means.shape[0], sh_degree, means, scales, quats, opacities, sh)

    def render(self, scene_ids, viewmats, intrinsics, width, height, rgb=None, depth=None, alpha=None,
               stream=None, **opt_kw):
        gg_render(self.ctx, scene_ids.shape[0], scene_ids, viewmats, intrinsics, width, height,
                  default_opts(**opt_kw), rgb, depth, alpha, stream)

    def close(self):
        if getattr(self, "ctx", None):
            gg_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
