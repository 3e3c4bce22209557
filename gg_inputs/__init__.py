"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This module only *constructs inputs* (Gaussian parameters, camera poses,
scene bindings).  It holds none of the method's arithmetic: no projection,
no covariance, no binning, no compositing.  Both `oracle/` and
`paper_2510_15352_b200/` consume what it returns; neither imports the other.

Recipe:
  * base seed 2510015352; each object draws from
    numpy.random.Generator(PCG64(SeedSequence([BASE, kind, index]))).
  * `room_scene` is shaped like the paper's workloads: an indoor room
    (§3.1 indoor scans), a staircase (PAPER.md:232, :264 stairs),
    an obstacle field with a yellow floor patch (§4.3).
  * `cameras` places robot-mounted pinhole cameras at A1 body height (0.32 m)
    or T1 head height (1.20 m), 90 deg HFoV (the paper
    gives none), OpenCV axes, world->camera row-major 4x4 view matrices.

All arrays are float32, C-contiguous.  Gaussian inputs are *activated*
(scales in metres > 0, opacity in [0,1], quaternion (w,x,y,z) unnormalised
allowed), matching the gg_load_scene contract (include/gg.h).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

BASE_SEED = 2510015352

# object kinds for SeedSequence([BASE_SEED, kind, index])
KIND_ROOM = 1
KIND_CAMERAS = 2
KIND_CLOUD = 3
KIND_BINDING = 4
KIND_FIXTURE = 5

YELLOW_PATCH = (0.9, 0.8, 0.1)   # PAPER.md:274 (yellow floor patch), SURVEY §8(d).1


def rng(kind: int, index: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence([BASE_SEED, kind, index])))


@dataclass
class Scene:
    """Activated Gaussian parameters of one scene (gg_load_scene inputs)."""
    means: np.ndarray        # [n,3] f32, metres, world frame (z up)
    scales: np.ndarray       # [n,3] f32, > 0, metres (per-axis std-dev)
    quats: np.ndarray        # [n,4] f32, (w,x,y,z), any non-zero norm
    opacities: np.ndarray    # [n]   f32, in [0,1]
    sh: np.ndarray           # [n,(d+1)^2,3] f32, coefficient-major
    sh_degree: int
    # free-floor description used only to place cameras (not a render input)
    free_boxes: list = field(default_factory=list)   # list of (xmin,xmax,ymin,ymax) obstacles
    half_extent: float = 6.0

    @property
    def n(self) -> int:
        return int(self.means.shape[0])


@dataclass
class Cameras:
    viewmats: np.ndarray     # [E,4,4] f32, world->camera, OpenCV (+x right, +y down, +z fwd)
    intrinsics: np.ndarray   # [E,4] f32, fx, fy, cx, cy in pixels
    width: int
    height: int

    @property
    def n(self) -> int:
        return int(self.viewmats.shape[0])


# ---------------------------------------------------------------------------
# small helpers (input construction only)
# ---------------------------------------------------------------------------

def _quat_from_frames(R: np.ndarray) -> np.ndarray:
    """Quaternion (w,x,y,z) whose rotation matrix has the given columns.

    Input construction: turns a sampled local frame into the quaternion the
    loader expects.  Shepperd's branch-free-ish method, vectorised.
    """
    m00, m01, m02 = R[:, 0, 0], R[:, 0, 1], R[:, 0, 2]
    m10, m11, m12 = R[:, 1, 0], R[:, 1, 1], R[:, 1, 2]
    m20, m21, m22 = R[:, 2, 0], R[:, 2, 1], R[:, 2, 2]
    tr = m00 + m11 + m22
    q = np.empty((R.shape[0], 4), dtype=np.float64)
    c0 = tr > 0
    s = np.sqrt(np.maximum(tr + 1.0, 1e-30)) * 2
    q[c0] = np.stack([0.25 * s, (m21 - m12) / s, (m02 - m20) / s, (m10 - m01) / s], 1)[c0]
    c1 = (~c0) & (m00 > m11) & (m00 > m22)
    s = np.sqrt(np.maximum(1.0 + m00 - m11 - m22, 1e-30)) * 2
    q[c1] = np.stack([(m21 - m12) / s, 0.25 * s, (m01 + m10) / s, (m02 + m20) / s], 1)[c1]
    c2 = (~c0) & (~c1) & (m11 > m22)
    s = np.sqrt(np.maximum(1.0 + m11 - m00 - m22, 1e-30)) * 2
    q[c2] = np.stack([(m02 - m20) / s, (m01 + m10) / s, 0.25 * s, (m12 + m21) / s], 1)[c2]
    c3 = (~c0) & (~c1) & (~c2)
    s = np.sqrt(np.maximum(1.0 + m22 - m00 - m11, 1e-30)) * 2
    q[c3] = np.stack([(m10 - m01) / s, (m02 + m20) / s, (m12 + m21) / s, 0.25 * s], 1)[c3]
    return q


def _random_unit_quats(g: np.random.Generator, n: int) -> np.ndarray:
    q = g.normal(size=(n, 4))
    return q / np.linalg.norm(q, axis=1, keepdims=True)


def _dc_coeff(rgb: np.ndarray) -> np.ndarray:
    """DC SH coefficient that encodes albedo `rgb` (inverse of the degree-0
    basis value 1/(2*sqrt(pi)) with the +0.5 offset)."""
    return (rgb - 0.5) * (2.0 * math.sqrt(math.pi))


def _sh_block(g: np.random.Generator, n: int, degree: int, rgb: np.ndarray) -> np.ndarray:
    k = (degree + 1) ** 2
    sh = np.zeros((n, k, 3), dtype=np.float64)
    sh[:, 0, :] = _dc_coeff(rgb)
    for l in range(1, degree + 1):
        sd = 0.08 / (l + 1)
        sh[:, l * l:(l + 1) * (l + 1), :] = g.normal(0.0, sd, size=(n, 2 * l + 1, 3))
    return sh


# ---------------------------------------------------------------------------
# room scenes (SURVEY §8(d).1 "Scene generator room(seed, N, d)")
# ---------------------------------------------------------------------------

def _room_quads(g: np.random.Generator, L: float, stairs: bool):
    """Axis-aligned rectangles (origin, U, V, normal, base colour, kind)."""
    h = L / 2
    quads = []

    def add(o, U, V, n, col, kind=0):
        quads.append((np.array(o, float), np.array(U, float), np.array(V, float),
                      np.array(n, float), np.array(col, float), kind))

    # floor (kind 1: checker + patch), walls 3 m high, no ceiling
    add((-h, -h, 0), (L, 0, 0), (0, L, 0), (0, 0, 1), g.uniform(0.35, 0.75, 3), 1)
    wall_h = 3.0
    add((-h, -h, 0), (L, 0, 0), (0, 0, wall_h), (0, 1, 0), g.uniform(0.3, 0.9, 3))
    add((-h, h, 0), (L, 0, 0), (0, 0, wall_h), (0, -1, 0), g.uniform(0.3, 0.9, 3))
    add((-h, -h, 0), (0, L, 0), (0, 0, wall_h), (1, 0, 0), g.uniform(0.3, 0.9, 3))
    add((h, -h, 0), (0, L, 0), (0, 0, wall_h), (-1, 0, 0), g.uniform(0.3, 0.9, 3))

    obstacles = []
    if stairs:
        # 6 steps, rise 0.17 m, run 0.30 m, width 2 m, against the -y wall
        x0 = g.uniform(-h + 0.5, h - 2.5)
        y0 = -h
        col = g.uniform(0.3, 0.8, 3)
        for s in range(6):
            z = 0.17 * (s + 1)
            ys = y0 + 0.30 * s
            add((x0, ys, z - 0.17), (2.0, 0, 0), (0, 0, 0.17), (0, -1, 0), col * 0.85)  # riser
            add((x0, ys, z), (2.0, 0, 0), (0, 0.30 * (6 - s), 0), (0, 0, 1), col)        # tread (top)
        obstacles.append((x0 - 0.3, x0 + 2.3, y0, y0 + 1.8 + 0.3))

    n_boxes = int(g.integers(10, 41))
    for _ in range(n_boxes):
        sx, sy, sz = g.uniform(0.2, 1.0, 3)
        cx = g.uniform(-h + 0.6, h - 0.6)
        cy = g.uniform(-h + 0.6, h - 0.6)
        col = g.uniform(0.15, 0.95, 3)
        bx0, by0 = cx - sx / 2, cy - sy / 2
        add((bx0, by0, sz), (sx, 0, 0), (0, sy, 0), (0, 0, 1), col)          # top
        add((bx0, by0, 0), (sx, 0, 0), (0, 0, sz), (0, -1, 0), col * 0.9)    # -y face
        add((bx0, by0 + sy, 0), (sx, 0, 0), (0, 0, sz), (0, 1, 0), col * 0.9)
        add((bx0, by0, 0), (0, sy, 0), (0, 0, sz), (-1, 0, 0), col * 0.8)
        add((bx0 + sx, by0, 0), (0, sy, 0), (0, 0, sz), (1, 0, 0), col * 0.8)
        obstacles.append((bx0 - 0.3, bx0 + sx + 0.3, by0 - 0.3, by0 + sy + 0.3))

    # yellow 1 x 1.5 m floor patch
    px = g.uniform(-h + 1.0, h - 2.0)
    py = g.uniform(-h + 1.0, h - 2.5)
    patch = (px, px + 1.0, py, py + 1.5)
    return quads, obstacles, patch


def room_scene(index: int, n: int, sh_degree: int = 0, L: float | None = None,
               stairs: bool | None = None) -> Scene:
    """Seeded synthetic indoor room with `n` Gaussians.

    95% surfels sampled proportional to surface area with 1 cm normal jitter,
    5% floaters uniform in the volume.  Scales from the surface spacing
    h = sqrt(area / N_surf); opacity 80% Beta(8,1.5), 20% U(0.02,0.6).
    """
    g = rng(KIND_ROOM, index)
    if L is None:
        L = float(g.uniform(10.0, 16.0))
    if stairs is None:
        stairs = bool(g.uniform() < 0.5)
    quads, obstacles, patch = _room_quads(g, L, stairs)
    areas = np.array([np.linalg.norm(np.cross(q[1], q[2])) for q in quads])
    n_surf = int(round(0.95 * n))
    n_float = n - n_surf
    spacing = math.sqrt(areas.sum() / max(n_surf, 1))

    qi = g.choice(len(quads), size=n_surf, p=areas / areas.sum())
    a = g.uniform(size=n_surf)
    b = g.uniform(size=n_surf)
    O = np.stack([quads[i][0] for i in range(len(quads))])
    U = np.stack([quads[i][1] for i in range(len(quads))])
    V = np.stack([quads[i][2] for i in range(len(quads))])
    N = np.stack([quads[i][3] for i in range(len(quads))])
    C = np.stack([quads[i][4] for i in range(len(quads))])
    K = np.array([quads[i][5] for i in range(len(quads))])
    pos = O[qi] + a[:, None] * U[qi] + b[:, None] * V[qi]
    nrm = N[qi]
    pos = pos + nrm * g.normal(0.0, 0.01, size=(n_surf, 1))

    # tangent frame with random twist: columns (t1, t2, n)
    Uh = U[qi] / np.linalg.norm(U[qi], axis=1, keepdims=True)
    t2 = np.cross(nrm, Uh)
    tw = g.uniform(0, 2 * math.pi, size=n_surf)
    c, s = np.cos(tw)[:, None], np.sin(tw)[:, None]
    e1 = c * Uh + s * t2
    e2 = -s * Uh + c * t2
    Rm = np.stack([e1, e2, nrm], axis=2)          # columns
    q_surf = _quat_from_frames(Rm)
    sig_t = np.exp(g.normal(math.log(0.7 * spacing), 0.35, size=(n_surf, 2)))
    sig_n = 0.15 * sig_t.mean(axis=1, keepdims=True)
    s_surf = np.concatenate([sig_t, sig_n], axis=1)

    # procedural albedo: 0.25 m checker x smooth value noise, yellow patch
    base = C[qi]
    ck = (np.floor(pos[:, 0] / 0.25) + np.floor(pos[:, 1] / 0.25) + np.floor(pos[:, 2] / 0.25)) % 2
    ph = g.uniform(0, 2 * math.pi, size=6)
    noise = (np.sin(3.1 * pos[:, 0] + ph[0]) * np.sin(2.7 * pos[:, 1] + ph[1])
             + 0.5 * np.sin(7.3 * pos[:, 2] + ph[2]) * np.sin(5.9 * pos[:, 0] + ph[3])
             + 0.25 * np.sin(13.1 * pos[:, 1] + ph[4]) * np.sin(11.7 * pos[:, 2] + ph[5]))
    shade = 0.8 + 0.12 * noise / 1.75
    floor_ck = np.where(K[qi] == 1, 0.75 + 0.25 * ck, 1.0)
    rgb = base * (shade * floor_ck)[:, None]
    in_patch = ((K[qi] == 1) & (pos[:, 0] >= patch[0]) & (pos[:, 0] <= patch[1])
                & (pos[:, 1] >= patch[2]) & (pos[:, 1] <= patch[3]))
    rgb[in_patch] = np.array(YELLOW_PATCH) * shade[in_patch, None]
    rgb = np.clip(rgb, 0.0, 1.0)

    # floaters
    hL = L / 2
    f_pos = np.stack([g.uniform(-hL, hL, n_float), g.uniform(-hL, hL, n_float),
                      g.uniform(0.0, 3.0, n_float)], 1)
    f_s = np.exp(g.normal(math.log(2 * spacing), 0.5, size=(n_float, 1))) * np.ones((1, 3))
    f_q = _random_unit_quats(g, n_float)
    f_rgb = g.uniform(0.1, 0.9, size=(n_float, 3))

    means = np.concatenate([pos, f_pos])
    scales = np.concatenate([s_surf, f_s])
    quats = np.concatenate([q_surf, f_q])
    colors = np.concatenate([rgb, f_rgb])
    op = np.where(g.uniform(size=n) < 0.8, g.beta(8.0, 1.5, size=n), g.uniform(0.02, 0.6, size=n))
    # interleave surfels and floaters so gid order carries no structure
    perm = g.permutation(n)
    sh = _sh_block(g, n, sh_degree, colors[perm])
    sc = Scene(means=np.ascontiguousarray(means[perm], np.float32),
               scales=np.ascontiguousarray(scales[perm], np.float32),
               quats=np.ascontiguousarray(quats[perm], np.float32),
               opacities=np.ascontiguousarray(op[perm], np.float32),
               sh=np.ascontiguousarray(sh, np.float32),
               sh_degree=sh_degree, free_boxes=obstacles, half_extent=hL)
    return sc


# ---------------------------------------------------------------------------
# cameras
# ---------------------------------------------------------------------------

def look_viewmat(center, yaw: float, pitch: float, roll: float) -> np.ndarray:
    """World->camera 4x4 (OpenCV axes) for a camera at `center` (world z up)
    looking along yaw/pitch, rolled about its optical axis.  Input
    construction (pose of the robot-mounted camera)."""
    f = np.array([math.cos(pitch) * math.cos(yaw), math.cos(pitch) * math.sin(yaw), math.sin(pitch)])
    up = np.array([0.0, 0.0, 1.0])
    xr = np.cross(f, up)
    xr /= np.linalg.norm(xr)
    yd = np.cross(f, xr)
    cr, sr = math.cos(roll), math.sin(roll)
    x2 = cr * xr + sr * yd
    y2 = -sr * xr + cr * yd
    Rwc = np.stack([x2, y2, f], axis=1)      # camera axes in world coords (columns)
    Rcw = Rwc.T
    t = -Rcw @ np.asarray(center, float)
    M = np.eye(4)
    M[:3, :3] = Rcw
    M[:3, 3] = t
    return M


def pinhole(width: int, height: int) -> np.ndarray:
    """90 deg horizontal FoV pinhole (the paper states none): fx=fy=W/2, c=centre."""
    return np.array([width / 2.0, width / 2.0, width / 2.0, height / 2.0])


def cameras(index: int, n_envs: int, width: int, height: int, scene: Scene | None = None,
            half_extent: float = 6.0, obstacles=None) -> Cameras:
    """Robot-mounted cameras placed on the free floor of a room.

    height 0.32 m (A1 body camera) or 1.20 m (T1 head camera,
    PAPER.md:269) 50/50; yaw U[0,2pi), pitch U[-30,-5] deg, roll N(0,2 deg).
    """
    g = rng(KIND_CAMERAS, index)
    if scene is not None:
        half_extent = scene.half_extent
        obstacles = scene.free_boxes
    obstacles = obstacles or []
    lim = half_extent - 0.5
    V = np.empty((n_envs, 4, 4))
    for e in range(n_envs):
        for _ in range(1000):
            x, y = g.uniform(-lim, lim, 2)
            if not any(b[0] <= x <= b[1] and b[2] <= y <= b[3] for b in obstacles):
                break
        z = 0.32 if g.uniform() < 0.5 else 1.20
        yaw = g.uniform(0, 2 * math.pi)
        pitch = math.radians(g.uniform(-30.0, -5.0))
        roll = math.radians(g.normal(0.0, 2.0))
        V[e] = look_viewmat((x, y, z), yaw, pitch, roll)
    K = np.tile(pinhole(width, height), (n_envs, 1))
    return Cameras(viewmats=np.ascontiguousarray(V, np.float32),
                   intrinsics=np.ascontiguousarray(K, np.float32), width=width, height=height)


def scene_binding(index: int, n_envs: int, n_scenes: int) -> np.ndarray:
    """Uniform random env -> scene binding."""
    g = rng(KIND_BINDING, index)
    return np.ascontiguousarray(g.integers(0, n_scenes, size=n_envs), np.int32)


def round_robin(n_envs: int, n_scenes: int) -> np.ndarray:
    """SPEC.md:78-86 register_scenes: env e -> scene e mod M."""
    return (np.arange(n_envs) % n_scenes).astype(np.int32)


# ---------------------------------------------------------------------------
# tiny adversarial / random fixtures (SURVEY §8(d).1 fixtures)
# ---------------------------------------------------------------------------

def random_cloud(index: int, n: int, sh_degree: int = 0) -> Scene:
    """<=512 Gaussians in a 2 m cube 4 m ahead of a camera at the origin
    looking down +z (SPEC.md:518 acceptance suite)."""
    g = rng(KIND_CLOUD, index)
    means = np.stack([g.uniform(-1, 1, n), g.uniform(-1, 1, n), g.uniform(3, 5, n)], 1)
    scales = np.exp(g.normal(math.log(0.06), 0.6, size=(n, 3)))
    quats = g.normal(size=(n, 4))
    op = g.uniform(0.0, 1.0, n)
    op[g.uniform(size=n) < 0.05] = 0.0
    op[g.uniform(size=n) < 0.05] = 1.0
    rgb = g.uniform(0.0, 1.0, (n, 3))
    sh = _sh_block(g, n, sh_degree, rgb)
    return Scene(np.float32(means), np.float32(scales), np.float32(quats), np.float32(op),
                 np.ascontiguousarray(sh, np.float32), sh_degree)


def cloud_cameras(index: int, n_envs: int, width: int = 64, height: int = 64) -> Cameras:
    """Cameras near the origin looking roughly down +z at a random_cloud."""
    g = rng(KIND_CAMERAS, 10_000 + index)
    V = np.empty((n_envs, 4, 4))
    for e in range(n_envs):
        c = g.normal(0.0, 0.3, 3)
        M = np.eye(4)
        # small random rotation about a random axis
        ax = g.normal(size=3)
        ax /= np.linalg.norm(ax)
        ang = g.normal(0, 0.12)
        Kx = np.array([[0, -ax[2], ax[1]], [ax[2], 0, -ax[0]], [-ax[1], ax[0], 0]])
        Rr = np.eye(3) + math.sin(ang) * Kx + (1 - math.cos(ang)) * (Kx @ Kx)
        M[:3, :3] = Rr
        M[:3, 3] = -Rr @ c
        V[e] = M
    fx = g.uniform(0.8, 1.2, n_envs) * width
    K = np.stack([fx, fx * g.uniform(0.9, 1.1, n_envs),
                  width / 2 + g.normal(0, 2, n_envs), height / 2 + g.normal(0, 2, n_envs)], 1)
    return Cameras(np.float32(V), np.float32(K), width, height)


def single_gaussian(mean, scale, opacity, rgb, quat=(1.0, 0.0, 0.0, 0.0), sh_degree: int = 0) -> Scene:
    """One Gaussian with DC colour `rgb` (closed-form fixtures)."""
    k = (sh_degree + 1) ** 2
    sh = np.zeros((1, k, 3))
    sh[0, 0] = _dc_coeff(np.asarray(rgb, float))
    return Scene(np.float32([mean]), np.float32([scale if np.ndim(scale) else [scale] * 3]),
                 np.float32([quat]), np.float32([opacity]), np.float32(sh), sh_degree)


def concat(scenes) -> Scene:
    d = max(s.sh_degree for s in scenes)
    k = (d + 1) ** 2
    shs = []
    for s in scenes:
        pad = np.zeros((s.n, k, 3), np.float32)
        pad[:, :s.sh.shape[1]] = s.sh
        shs.append(pad)
    return Scene(np.concatenate([s.means for s in scenes]), np.concatenate([s.scales for s in scenes]),
                 np.concatenate([s.quats for s in scenes]), np.concatenate([s.opacities for s in scenes]),
                 np.concatenate(shs), d)


def identity_cameras(n_envs: int, width: int, height: int, fx: float, fy: float | None = None,
                     cx: float | None = None, cy: float | None = None) -> Cameras:
    """Cameras at the world origin with identity rotation (camera frame = world)."""
    V = np.tile(np.eye(4), (n_envs, 1, 1))
    fy = fx if fy is None else fy
    cx = width / 2 if cx is None else cx
    cy = height / 2 if cy is None else cy
    K = np.tile(np.array([fx, fy, cx, cy]), (n_envs, 1))
    return Cameras(np.float32(V), np.float32(K), width, height)


# ---------------------------------------------------------------------------
# the BASELINE.json configs (SURVEY §8(d).1 "Per config")
# ---------------------------------------------------------------------------

CONFIGS = {
    # name: (n_scenes, n_gauss, sh_degree, n_envs, W, H, depth, L, stairs)
    "c1": dict(n_scenes=1, n_gauss=20_000, sh_degree=0, n_envs=4, width=64, height=48, depth=True),
    "c2": dict(n_scenes=1, n_gauss=500_000, sh_degree=3, n_envs=1024, width=320, height=240, depth=False),
    "c3": dict(n_scenes=1, n_gauss=1_000_000, sh_degree=3, n_envs=4096, width=640, height=480, depth=True),
    "c4": dict(n_scenes=256, n_gauss=1_000_000, sh_degree=0, n_envs=4096, width=640, height=480, depth=True),
    "c5": dict(n_scenes=2500, n_gauss=500_000, sh_degree=0, n_envs=32768, width=640, height=480, depth=True),
}


def config_scene(cfg: str, scene_index: int = 0, n_gauss: int | None = None, sh_degree: int | None = None) -> Scene:
    c = CONFIGS[cfg]
    n = c["n_gauss"] if n_gauss is None else n_gauss
    d = c["sh_degree"] if sh_degree is None else sh_degree
    fixed = c["n_scenes"] == 1
    # c1-c3 fix L = 12 m and always include the staircase
    return room_scene(scene_index, n, d, L=12.0 if fixed else None, stairs=True if fixed else None)


def config_cameras(cfg: str, scene: Scene, n_envs: int | None = None, index: int = 0) -> Cameras:
    c = CONFIGS[cfg]
    return cameras(index, c["n_envs"] if n_envs is None else n_envs, c["width"], c["height"], scene)


# ---------------------------------------------------------------------------
# Benchmark workloads (bench.py and the full-size parity tests share them)
# ---------------------------------------------------------------------------

def _room_job(args3):
    k, n, d = args3
    return room_scene(100 + k, n, d)


class Workload:
    """The seeded inputs of one BASELINE config as bench.py renders them.

    One scene (c1-c3: `config_scene`) or S rooms `room_scene(100 + k, ...)`
    with a seeded uniform env->scene binding over the GLOBAL env set
    (c4/c5).  Every input is a function of the global env
    index, never of the rank or world size, so a rank-sliced multi-GPU run
    renders exactly the envs of a single-GPU run of the same global set
    (SURVEY §8(e) determinism checks): the poses of the envs of block
    b = e // POSE_BLOCK bound to scene k in pose set s are drawn from
    rng(KIND_CAMERAS, pose_index(s, b, k)), in env order, in scene k.

    `env_range` = [a, b) materialises only those envs (a rank's slice).
    `scenes()` generates the rooms in parallel and streams them (c5's 2,500
    rooms never sit in host memory at once), placing the cameras of scene k's
    envs as it goes by; `place(k, free_boxes, half_extent)` does the same from
    a scene's floor description alone (ranks that receive scenes by broadcast);
    `scene(k)` regenerates one scene on its own (same seed, same arrays).
    """
    POSE_BLOCK = 32

    def __init__(self, cfg: str, n_envs: int | None = None, n_sets: int = 1, env_range=None,
                 n_scenes: int | None = None, n_gauss: int | None = None, sh_degree: int | None = None):
        c = CONFIGS[cfg]
        self.cfg = cfg
        self.n_total = c["n_envs"] if n_envs is None else n_envs
        self.a, self.b = env_range if env_range is not None else (0, self.n_total)
        self.n_envs = self.b - self.a
        self.n_sets = n_sets
        self.width, self.height = c["width"], c["height"]
        self.n_gauss = c["n_gauss"] if n_gauss is None else n_gauss
        self.sh_degree = c["sh_degree"] if sh_degree is None else sh_degree
        self.n_scenes = n_scenes or (c["n_scenes"] if cfg in ("c4", "c5") else 1)
        S = self.n_scenes
        self.glob_binding = scene_binding(7, self.n_total, S) if S > 1 else np.zeros(self.n_total, np.int32)
        self.binding = np.ascontiguousarray(self.glob_binding[self.a:self.b])
        self.viewmats = np.empty((n_sets, self.n_envs, 4, 4), np.float32)
        self.intrinsics = np.tile(pinhole(self.width, self.height).astype(np.float32), (self.n_envs, 1))

    @staticmethod
    def pose_index(s: int, block: int, k: int) -> int:
        return (s << 40) | (block << 16) | k

    def scene(self, k: int) -> Scene:
        if self.n_scenes == 1:
            return config_scene(self.cfg, n_gauss=self.n_gauss, sh_degree=self.sh_degree)
        return _room_job((k, self.n_gauss, self.sh_degree))

    def place(self, k: int, free_boxes, half_extent: float):
        """Cameras of this slice's envs bound to scene k (all pose sets)."""
        idx = np.flatnonzero(self.binding == k) + self.a        # global envs of this slice bound to k
        if not idx.size:
            return
        PB = self.POSE_BLOCK
        for blk in np.unique(idx // PB):
            lo, hi = int(blk) * PB, min(self.n_total, (int(blk) + 1) * PB)
            blk_envs = lo + np.flatnonzero(self.glob_binding[lo:hi] == k)   # all of the block's envs on k
            mine = (blk_envs >= self.a) & (blk_envs < self.b)
            for s_ in range(self.n_sets):
                cams = cameras(self.pose_index(s_, int(blk), k), blk_envs.size, self.width, self.height,
                               half_extent=half_extent, obstacles=list(free_boxes))
                self.viewmats[s_, blk_envs[mine] - self.a] = cams.viewmats[mine]

    def scenes(self, n_proc: int | None = None):
        """Yield (k, scene) for k = 0..S-1 in order (parallel host generation)."""
        S = self.n_scenes
        if S == 1:
            sc = self.scene(0)
            self.place(0, sc.free_boxes, sc.half_extent)
            yield 0, sc
            return
        import concurrent.futures as cf
        import os
        if n_proc is None:
            n_proc = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 4)
            n_proc = max(1, min(16, n_proc))
        job = (self.n_gauss, self.sh_degree)
        with cf.ProcessPoolExecutor(n_proc) as ex:
            futs = {k: ex.submit(_room_job, (k,) + job) for k in range(min(S, 2 * n_proc))}
            for k in range(S):
                sc = futs.pop(k).result()
                nxt = k + 2 * n_proc
                if nxt < S:
                    futs[nxt] = ex.submit(_room_job, (nxt,) + job)
                self.place(k, sc.free_boxes, sc.half_extent)
                yield k, sc

    def cameras(self, s: int = 0) -> Cameras:
        return Cameras(self.viewmats[s], self.intrinsics, self.width, self.height)


MAX_FREE_BOXES = 64


def pack_floor(scene: Scene) -> np.ndarray:
    """A scene's camera-placement description (half extent, obstacle boxes) as
    a fixed-size float64 vector, for broadcast to ranks that only receive the
    scene's Gaussians."""
    v = np.zeros(2 + 4 * MAX_FREE_BOXES, np.float64)
    boxes = list(scene.free_boxes)[:MAX_FREE_BOXES]
    v[0], v[1] = scene.half_extent, len(boxes)
    for i, b in enumerate(boxes):
        v[2 + 4 * i: 6 + 4 * i] = b
    return v


def unpack_floor(v) -> tuple:
    v = np.asarray(v, np.float64)
    n = int(v[1])
    return [tuple(float(x) for x in v[2 + 4 * i: 6 + 4 * i]) for i in range(n)], float(v[0])


# ---------------------------------------------------------------------------
# 3DGS PLY writer (input construction for the PLY-reader tests): stores the
# *raw* parameters the 3DGS format holds (log scales, opacity logits,
# channel-major f_rest).
# ---------------------------------------------------------------------------

def write_3dgs_ply(path: str, scene: Scene) -> None:
    import struct
    n, d = scene.n, scene.sh_degree
    K = (d + 1) ** 2
    names = ["x", "y", "z", "nx", "ny", "nz", "f_dc_0", "f_dc_1", "f_dc_2"]
    names += [f"f_rest_{i}" for i in range(3 * (K - 1))]
    names += ["opacity", "scale_0", "scale_1", "scale_2", "rot_0", "rot_1", "rot_2", "rot_3"]
    op = np.clip(scene.opacities.astype(np.float64), 1e-7, 1 - 1e-7)
    cols = [scene.means.astype(np.float64), np.zeros((n, 3)), scene.sh[:, 0, :].astype(np.float64)]
    rest = scene.sh[:, 1:, :].astype(np.float64).transpose(0, 2, 1).reshape(n, -1)   # channel-major
    cols += [rest, np.log(op / (1 - op))[:, None], np.log(scene.scales.astype(np.float64)),
             scene.quats.astype(np.float64)]
    data = np.concatenate(cols, axis=1).astype("<f4")
    assert data.shape[1] == len(names)
    with open(path, "wb") as f:
        hdr = "ply\nformat binary_little_endian 1.0\nelement vertex %d\n" % n
        hdr += "".join(f"property float {nm}\n" for nm in names) + "end_header\n"
        f.write(hdr.encode())
        f.write(data.tobytes())
    del struct
