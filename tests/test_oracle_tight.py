"""Pins for the oracle's opacity-aware tile-rect variant (F_TIGHT, DESIGN.md
reading R35; SURVEY §8(f) row 3 "opacity-aware footprints").

What fixes it independently of its own formula:
  * closed form — an axis-aligned Gaussian on the optical axis has conic
    diag(1/a, 1/c) with a = (fx sx / z)^2 + 0.3, c = (fy sy / z)^2 + 0.3, so
    alpha >= 1/255 exactly on |dx| <= sqrt(2 ln(255 o) a), |dy| <= sqrt(2 ln(255 o) c);
  * brute force — every pixel where some Gaussian reaches alpha >= 1/255 (f64,
    from the dumped f32 record) lies inside that Gaussian's tight rect;
  * invariance — images are bit-identical with and without the variant (a
    dropped tile never held a blending pixel) and the lists are the
    order-preserving filter of the paper's lists.
"""
import math

import numpy as np

import gg_inputs as gi
import oracle as orc


def _render(scene, cams, e, W, H, flags=0):
    s = orc.OracleScene.from_inputs(scene)
    return orc.render_env(s, cams.viewmats[e], cams.intrinsics[e], W, H, flags=flags)


def test_tight_closed_form_axis_aligned():
    W = H = 256
    z, sx, sy, o = 4.0, 0.25, 0.5, 0.05
    sc = gi.single_gaussian((0.0, 0.0, z), (sx, sy, 0.1), o, (0.8, 0.2, 0.1))
    cams = gi.identity_cameras(1, W, H, fx=128.0)
    r0 = _render(sc, cams, 0, W, H)
    rt = _render(sc, cams, 0, W, H, flags=orc.F_TIGHT)
    a = (128.0 * sx / z) ** 2 + 0.3
    c = (128.0 * sy / z) ** 2 + 0.3
    q = 2.0 * math.log(255.0 * o)
    ex, ey = math.sqrt(q * a), math.sqrt(q * c)            # 18.09, 36.12 px around (128, 128)
    # tiles whose pixel centres 16t+0.5 .. 16t+15.5 reach [128 - e, 128 + e]
    tx = [t for t in range(16) if 16 * t + 15.5 >= 128 - ex and 16 * t + 0.5 <= 128 + ex]
    ty = [t for t in range(16) if 16 * t + 15.5 >= 128 - ey and 16 * t + 0.5 <= 128 + ey]
    assert (tx[0], tx[-1] + 1, ty[0], ty[-1] + 1) == (6, 10, 5, 11)
    assert tuple(rt.proj[0, 8:12].astype(int)) == (6, 10, 5, 11)
    assert rt.tile_counts[0] == 4 * 6
    # the paper's 3-sigma circle rect is larger (r = ceil(3 sqrt(c)) = 49 px)
    assert tuple(r0.proj[0, 8:12].astype(int)) == (4, 12, 4, 12)
    assert np.array_equal(rt.rgb, r0.rgb) and np.array_equal(rt.depth, r0.depth)


def test_tight_empty_below_cutoff_opacity():
    # o < 1/255: alpha < 1/255 everywhere -> no tiles, image = background
    sc = gi.single_gaussian((0.0, 0.0, 3.0), 0.2, 0.9 / 255.0, (1.0, 1.0, 1.0))
    cams = gi.identity_cameras(1, 64, 64, fx=32.0)
    r0 = _render(sc, cams, 0, 64, 64)
    rt = _render(sc, cams, 0, 64, 64, flags=orc.F_TIGHT)
    assert r0.tile_counts[0] > 0 and rt.tile_counts[0] == 0
    assert rt.sorted_gid.size == 0
    assert np.array_equal(rt.rgb, r0.rgb) and np.all(rt.alpha == 0)


def _check_pair(r0, rt, n):
    assert np.array_equal(rt.rgb, r0.rgb)
    assert np.array_equal(rt.depth, r0.depth)
    assert np.array_equal(rt.alpha, r0.alpha)
    assert np.array_equal(rt.exempt, r0.exempt)
    assert np.all(rt.n_eval <= r0.n_eval)
    assert np.all(rt.tile_counts <= r0.tile_counts)
    # tight rect inside the paper rect
    vis = rt.tile_counts > 0
    p0, pt = r0.proj[vis], rt.proj[vis]
    assert np.all(pt[:, 8] >= p0[:, 8]) and np.all(pt[:, 9] <= p0[:, 9])
    assert np.all(pt[:, 10] >= p0[:, 10]) and np.all(pt[:, 11] <= p0[:, 11])
    # lists: order-preserving filter of the paper lists by tight-rect membership
    TX = (r0.width + 15) // 16
    tx, ty = r0.sorted_tile % TX, r0.sorted_tile // TX
    g = r0.sorted_gid
    keep = (rt.proj[g, 8] <= tx) & (tx < rt.proj[g, 9]) & (rt.proj[g, 10] <= ty) & (ty < rt.proj[g, 11])
    assert np.array_equal(rt.sorted_gid, g[keep])
    assert np.array_equal(rt.sorted_tile, r0.sorted_tile[keep])
    assert np.array_equal(rt.sorted_zbits, r0.sorted_zbits[keep])
    assert rt.sorted_gid.size == int(rt.tile_counts.sum())


def _bruteforce_conservative(rt, W, H):
    """Every pixel with alpha >= 1/255 (f64 from the dumped f32 record) is
    inside the Gaussian's tight rect."""
    px = np.arange(W) + 0.5
    py = np.arange(H) + 0.5
    for gidx in np.flatnonzero(rt.proj[:, 0] == 1):
        p = rt.proj[gidx].astype(np.float64)
        u, v, A, B, C, o = p[1], p[2], p[3], p[4], p[5], p[15]
        dx = u - px[None, :]
        dy = v - py[:, None]
        q = np.maximum(A * dx * dx + 2 * B * dx * dy + C * dy * dy, 0.0)
        alpha = np.minimum(0.99, o * np.exp(-0.5 * q))
        ys, xs = np.nonzero(alpha >= 1.0 / 255.0)
        if xs.size == 0:
            continue
        tx, ty = xs // 16, ys // 16
        assert tx.min() >= p[8] and tx.max() < p[9], (gidx, tx.min(), tx.max(), p[8:12])
        assert ty.min() >= p[10] and ty.max() < p[11], (gidx, ty.min(), ty.max(), p[8:12])


def test_tight_random_clouds_identical_and_conservative():
    W = H = 64
    for idx in range(4):
        sc = gi.random_cloud(idx, 400, sh_degree=idx % 2)
        cams = gi.cloud_cameras(idx, 2, W, H)
        for e in range(2):
            r0 = _render(sc, cams, e, W, H)
            rt = _render(sc, cams, e, W, H, flags=orc.F_TIGHT)
            _check_pair(r0, rt, sc.means.shape[0])
            _bruteforce_conservative(rt, W, H)


def test_tight_room_scene_reduces_keys():
    sc = gi.config_scene("c1")
    cams = gi.config_cameras("c1", sc)
    W, H = cams.width, cams.height
    r0 = _render(sc, cams, 0, W, H)
    rt = _render(sc, cams, 0, W, H, flags=orc.F_TIGHT)
    _check_pair(r0, rt, sc.means.shape[0])
    assert rt.sorted_gid.size < r0.sorted_gid.size
