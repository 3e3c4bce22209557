"""CPU oracle for the batched 3DGS render path — TEST INFRASTRUCTURE.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` /
`--impl reference` legs may import this package.  The product path
(`paper_2510_15352_b200`) never imports it, and it never imports the product.

The arithmetic lives in `gg_oracle.cpp` (plain C++, f32 canonical projection
+ f64 compositing; see its header and DESIGN.md §2).  This module only
marshals numpy arrays through ctypes.

Parity pins live in tests/test_oracle_*.py (closed forms, Monte-Carlo,
finite differences, SH quadrature vs scipy, brute force, invariants).
Parity unpinned: agreement with the paper's own renderer (its code, scenes
and camera parameters are not available).
"""
from __future__ import annotations

import ctypes as C
import math
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libgg_oracle.so")

MODE_A = 0          # f32 canonical projection, f64 compositing (defines integer parity)
MODE_B = 1          # f64 projection (diagnostic)
F_NO_EARLY_OUT = 1
F_UNTRUNCATED = 2
F_PLAIN = 4
F_TIGHT = 8         # work-reduction variant: opacity-aware tile rects (R35)
F_ELLIPSE = 16      # work-reduction variant: ellipse ∩ tile masks on tight rects (R37)
F_INTEGER_ONLY = 32 # stop after O3: integer artefacts only (image outputs empty)

K_RGB, K_DEPTH, K_ALPHA, K_NEVAL, K_NCONTRIB, K_EXEMPT = 0, 1, 2, 3, 4, 5
K_TILE_COUNTS, K_SORTED_TILE, K_SORTED_ZBITS, K_SORTED_GID, K_RANGES = 6, 7, 8, 9, 10
K_PROJ, K_RGB8 = 11, 12

_DT = {K_RGB: np.float64, K_DEPTH: np.float64, K_ALPHA: np.float64, K_NEVAL: np.int32,
       K_NCONTRIB: np.int32, K_EXEMPT: np.uint8, K_TILE_COUNTS: np.int32, K_SORTED_TILE: np.int32,
       K_SORTED_ZBITS: np.uint32, K_SORTED_GID: np.int32, K_RANGES: np.int32, K_PROJ: np.float32,
       K_RGB8: np.uint8}


class _Opts(C.Structure):
    _fields_ = [("near_plane", C.c_float), ("far_plane", C.c_float), ("background", C.c_double * 3),
                ("sh_degree", C.c_int32), ("mode", C.c_int32), ("flags", C.c_int32)]


_lib = None


def build() -> None:
    subprocess.check_call(["sh", os.path.join(_HERE, "build.sh")])


def lib():
    global _lib
    if _lib is None:
        src = os.path.join(_HERE, "gg_oracle.cpp")
        if not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
            build()
        L = C.CDLL(_LIB_PATH)
        vp, fp, dp = C.c_void_p, C.POINTER(C.c_float), C.POINTER(C.c_double)
        L.or_scene_create.restype = vp
        L.or_scene_create.argtypes = [C.c_int64, C.c_int32, fp, fp, fp, fp, fp]
        L.or_scene_free.argtypes = [vp]
        L.or_scene_cov3.argtypes = [vp, fp, dp]
        L.or_sh_basis.argtypes = [C.c_int32, dp, dp]
        L.or_num_threads.restype = C.c_int
        L.or_set_threads.argtypes = [C.c_int]
        L.or_render_env.restype = vp
        L.or_render_env.argtypes = [vp, fp, fp, C.c_int32, C.c_int32, C.POINTER(_Opts)]
        L.or_result_len.restype = C.c_int64
        L.or_result_len.argtypes = [vp, C.c_int32]
        L.or_result_copy.argtypes = [vp, C.c_int32, vp]
        L.or_result_free.argtypes = [vp]
        _lib = L
    return _lib


def _f32(a):
    a = np.ascontiguousarray(a, dtype=np.float32)
    return a, a.ctypes.data_as(C.POINTER(C.c_float))


class OracleScene:
    """O1 (per-Gaussian preprocessing) done at construction."""

    def __init__(self, means, scales, quats, opacities, sh, sh_degree: int):
        self._keep = []
        ptrs = []
        for a in (means, scales, quats, opacities, sh):
            arr, p = _f32(a)
            self._keep.append(arr)
            ptrs.append(p)
        self.n = int(self._keep[0].shape[0])
        self.sh_degree = int(sh_degree)
        self._h = lib().or_scene_create(self.n, self.sh_degree, *ptrs)
        if not self._h:
            raise ValueError("or_scene_create failed")

    @classmethod
    def from_inputs(cls, s) -> "OracleScene":
        return cls(s.means, s.scales, s.quats, s.opacities, s.sh, s.sh_degree)

    def cov3(self):
        o32 = np.zeros((self.n, 6), np.float32)
        o64 = np.zeros((self.n, 6), np.float64)
        lib().or_scene_cov3(self._h, o32.ctypes.data_as(C.POINTER(C.c_float)),
                            o64.ctypes.data_as(C.POINTER(C.c_double)))
        return o32, o64

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.or_scene_free(self._h)
            self._h = None


@dataclass
class EnvResult:
    width: int
    height: int
    rgb: np.ndarray          # [H,W,3] f64, pre-quantisation (C + T bg)
    rgb8: np.ndarray         # [H,W,3] u8 (O5)
    depth: np.ndarray        # [H,W] f64
    alpha: np.ndarray        # [H,W] f64
    n_eval: np.ndarray       # [H,W] i32
    n_contrib: np.ndarray    # [H,W] i32
    exempt: np.ndarray       # [H,W] bool
    tile_counts: np.ndarray  # [N] i32 (0 if culled)
    sorted_tile: np.ndarray  # [K] i32
    sorted_zbits: np.ndarray # [K] u32
    sorted_gid: np.ndarray   # [K] i32
    ranges: np.ndarray       # [TY*TX, 2] i32
    proj: np.ndarray         # [N,16] f32: vis,u,v,A,B,C,z,r,x0,x1,y0,y1,r,g,b,o


def render_env(scene: OracleScene, viewmat, intr, width: int, height: int, *, near: float = 0.01,
               far: float = 1e10, background=(0.0, 0.0, 0.0), sh_degree: int = -1, mode: int = MODE_A,
               flags: int = 0) -> EnvResult:
    """O1-O5 for one environment's camera."""
    L = lib()
    v, vp = _f32(np.asarray(viewmat).reshape(16))
    k, kp = _f32(np.asarray(intr).reshape(4))
    o = _Opts(near, far, (C.c_double * 3)(*background), sh_degree, mode, flags)
    h = L.or_render_env(scene._h, vp, kp, width, height, C.byref(o))
    if not h:
        raise ValueError("or_render_env failed (bad size or sh_degree)")
    try:
        def get(kind):
            n = L.or_result_len(h, kind)
            a = np.empty(n, dtype=_DT[kind])
            if n:
                L.or_result_copy(h, kind, a.ctypes.data_as(C.c_void_p))
            return a
        H, W = (height, width) if not (flags & F_INTEGER_ONLY) else (0, 0)
        return EnvResult(width, height,
                         get(K_RGB).reshape(H, W, 3), get(K_RGB8).reshape(H, W, 3),
                         get(K_DEPTH).reshape(H, W), get(K_ALPHA).reshape(H, W),
                         get(K_NEVAL).reshape(H, W), get(K_NCONTRIB).reshape(H, W),
                         get(K_EXEMPT).reshape(H, W).astype(bool), get(K_TILE_COUNTS),
                         get(K_SORTED_TILE), get(K_SORTED_ZBITS), get(K_SORTED_GID),
                         get(K_RANGES).reshape(-1, 2), get(K_PROJ).reshape(-1, 16))
    finally:
        L.or_result_free(h)


def sh_basis(degree: int, direction) -> np.ndarray:
    d = np.ascontiguousarray(direction, np.float64)
    out = np.zeros(16, np.float64)
    lib().or_sh_basis(degree, d.ctypes.data_as(C.POINTER(C.c_double)),
                      out.ctypes.data_as(C.POINTER(C.c_double)))
    return out[:(degree + 1) ** 2]


def num_threads() -> int:
    return int(lib().or_num_threads())


def use_all_cores() -> int:
    """Run the oracle on every host core available to this process (torchrun
    sets OMP_NUM_THREADS=1 per rank; the CPU baseline must not inherit that)."""
    import os
    n = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
    lib().or_set_threads(n)
    return num_threads()


# ---------------------------------------------------------------- motion blur
# SPEC.md:221-229 render_with_motion_blur; §3.3.  Readings
# R32-R34: t_i = shutter ((i + 0.5)/K - 0.5); sample pose i
# rotates the camera about its centre by the world-frame axis-angle vector
# w t_i and moves the centre by v t_i; uniform 1/K average of the linear
# colours (and alphas); depth from the centre sample, i.e. the nominal pose
# t = 0 the offsets are centred on ("depth taken from the center
# sample", "offsets centered on the nominal pose") = the caller's
# view matrix, for odd and even K alike.

def _rodrigues(rv):
    rv = np.asarray(rv, np.float64)
    th = float(np.linalg.norm(rv))
    if th == 0.0:
        return np.eye(3)
    k = rv / th
    Kx = np.array([[0.0, -k[2], k[1]], [k[2], 0.0, -k[0]], [-k[1], k[0], 0.0]])
    return np.eye(3) + np.sin(th) * Kx + (1.0 - np.cos(th)) * (Kx @ Kx)


def blur_poses(viewmat, lin_vel, ang_vel, shutter: float, K: int) -> np.ndarray:
    """The K sample view matrices [K,4,4] (f64) of one camera."""
    V = np.asarray(viewmat, np.float64).reshape(4, 4)
    Rcw, t = V[:3, :3], V[:3, 3]
    C = -Rcw.T @ t
    v = np.asarray(lin_vel, np.float64)
    w = np.asarray(ang_vel, np.float64)
    out = np.zeros((K, 4, 4))
    for i in range(K):
        ti = float(np.float32(shutter)) * ((i + 0.5) / K - 0.5)
        Rwc = _rodrigues(w * ti) @ Rcw.T
        Ci = C + v * ti
        out[i, :3, :3] = Rwc.T
        out[i, :3, 3] = -Rwc.T @ Ci
        out[i, 3, 3] = 1.0
    return out


@dataclass
class BlurResult:
    rgb: np.ndarray      # [H,W,3] f64 uniform average of the samples' linear colours
    rgb8: np.ndarray     # [H,W,3] u8
    depth: np.ndarray    # [H,W] depth of the nominal pose (t = 0)
    alpha: np.ndarray    # [H,W] average alpha
    exempt: np.ndarray   # [H,W] any sample's near-miss flag
    depth_alpha: np.ndarray   # [H,W] alpha of the depth's sample
    samples: list


def render_blur_env(scene: OracleScene, viewmat, intr, width: int, height: int, lin_vel, ang_vel,
                    shutter: float, K: int, **kw) -> BlurResult:
    if K < 1:
        raise ValueError("K must be >= 1 (SPEC.md:226)")
    poses = blur_poses(viewmat, lin_vel, ang_vel, shutter, K)
    samples = [render_env(scene, np.float32(p), intr, width, height, **kw) for p in poses]
    rgb = np.mean([s.rgb for s in samples], axis=0)
    alpha = np.mean([s.alpha for s in samples], axis=0)
    rgb8 = np.rint(np.clip(rgb, 0.0, 1.0) * 255.0).astype(np.uint8)   # numpy rint = half-to-even
    nominal = render_env(scene, np.asarray(viewmat, np.float32), intr, width, height, **kw)   # t = 0
    exempt = np.any([s.exempt for s in samples] + [nominal.exempt], axis=0)
    return BlurResult(rgb, rgb8, nominal.depth, alpha, exempt, nominal.alpha, samples)


# ---------------------------------------------------------------- DinoV2 input
# SURVEY §8(f) row 4 ("fused render -> DinoV2 input (224^2 resize, normalise,
# bf16 planar)"); PAPER.md:253 feeds DinoV2 "the raw RGB frame".  Reading R36
# (DESIGN.md): the whole u8 frame is resized to S x S by bilinear
# interpolation with half-pixel centres (src = (dst + 0.5) * in/out - 0.5,
# clamped at 0; the upper neighbour clamped to the last pixel), no
# antialiasing; values u8/255 are normalised with the ImageNet mean/std
# DinoV2 was trained with; output is channel-planar [3, S, S].
IMAGENET_MEAN = (0.485, 0.456, 0.406)
IMAGENET_STD = (0.229, 0.224, 0.225)


def _bilinear_axis(n_in: int, n_out: int):
    """Per output index: (lower index, upper index, upper weight), f64."""
    scale = n_in / n_out
    lo = np.zeros(n_out, np.int64)
    hi = np.zeros(n_out, np.int64)
    w = np.zeros(n_out, np.float64)
    for d in range(n_out):
        src = max((d + 0.5) * scale - 0.5, 0.0)
        i0 = int(math.floor(src))
        i0 = min(i0, n_in - 1)
        lo[d] = i0
        hi[d] = min(i0 + 1, n_in - 1)
        w[d] = src - i0
    return lo, hi, w


def dino_input(rgb_u8, size: int = 224) -> np.ndarray:
    """[H, W, 3] u8 frame -> [3, size, size] f64 normalised DinoV2 input."""
    img = np.asarray(rgb_u8, np.float64) / 255.0
    H, W = img.shape[0], img.shape[1]
    ylo, yhi, wy = _bilinear_axis(H, size)
    xlo, xhi, wx = _bilinear_axis(W, size)
    out = np.zeros((3, size, size), np.float64)
    for c in range(3):
        ch = img[:, :, c]
        top = ch[ylo][:, xlo] * (1.0 - wx)[None, :] + ch[ylo][:, xhi] * wx[None, :]
        bot = ch[yhi][:, xlo] * (1.0 - wx)[None, :] + ch[yhi][:, xhi] * wx[None, :]
        v = top * (1.0 - wy)[:, None] + bot * wy[:, None]
        out[c] = (v - IMAGENET_MEAN[c]) / IMAGENET_STD[c]
    return out
