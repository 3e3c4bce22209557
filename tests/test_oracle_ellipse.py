"""Pins for the oracle's ellipse ∩ tile variant (F_ELLIPSE, DESIGN.md reading
R37; SURVEY §8(f) row 3 "ellipse∩tile tests"), independent of its formula:
  * brute force — every pixel where a Gaussian reaches alpha >= 1/255 (f64,
    from the dumped f32 record) lies in a kept tile of that Gaussian;
  * exactness — tiles whose pixel-centre rectangle is clearly outside the
    ellipse (f64 minimum of q over the rectangle above 1.05 q_max) are dropped,
    and a 45-degree needle's far bbox corners are among them;
  * invariance — images bit-identical to the paper's and the tight lists, and
    the lists an order-preserving filter of the tight ones.
"""
import math

import numpy as np

import gg_inputs as gi
import oracle as orc
from test_oracle_tight import _bruteforce_conservative, _render


def _qmin_rect_f64(u, v, A, B, C, x0, x1, y0, y1):
    """min over [x0,x1]x[y0,y1] (pixel-centre coords) of A dx^2 + 2B dx dy + C dy^2, f64, by dense sampling
    of the boundary plus the interior test (a convex quadratic's minimum lies on the boundary unless the
    centre is inside)."""
    if x0 <= u <= x1 and y0 <= v <= y1:
        return 0.0
    t = np.linspace(0.0, 1.0, 2001)
    pts = [(x0 + (x1 - x0) * t, np.full_like(t, y0)), (x0 + (x1 - x0) * t, np.full_like(t, y1)),
           (np.full_like(t, x0), y0 + (y1 - y0) * t), (np.full_like(t, x1), y0 + (y1 - y0) * t)]
    best = math.inf
    for px, py in pts:
        dx, dy = px - u, py - v
        best = min(best, float((A * dx * dx + 2 * B * dx * dy + C * dy * dy).min()))
    return best


def _check_exact(rt, W, H):
    """Dropped-vs-kept against the f64 geometry for every <= 32-tile rect."""
    TX = (W + 15) // 16
    kept = {}
    for t, g in zip(rt.sorted_tile, rt.sorted_gid):
        kept.setdefault(int(g), set()).add(int(t))
    dropped_clear = 0
    for gidx in np.flatnonzero(rt.proj[:, 0] == 1):
        p = rt.proj[gidx].astype(np.float64)
        u, v, A, B, C, o = p[1], p[2], p[3], p[4], p[5], p[15]
        x0, x1, y0, y1 = (int(p[8]), int(p[9]), int(p[10]), int(p[11]))
        if (x1 - x0) * (y1 - y0) > 32:
            continue
        qmax = 2.0 * math.log(255.0 * o)
        for ty in range(y0, y1):
            for tx in range(x0, x1):
                q = _qmin_rect_f64(u, v, A, B, C, 16 * tx + 0.5, 16 * tx + 15.5, 16 * ty + 0.5, 16 * ty + 15.5)
                if q > 1.05 * qmax + 1e-2:
                    assert ty * TX + tx not in kept.get(int(gidx), set()), (gidx, tx, ty, q, qmax)
                    dropped_clear += 1
    return dropped_clear


def test_ellipse_needle_drops_far_corners():
    # a 45-degree needle: long axis along the image diagonal, thin across it
    W = H = 128
    c, s = math.cos(math.pi / 8), math.sin(math.pi / 8)          # quaternion for 45 deg about z
    sc = gi.single_gaussian((0.0, 0.0, 4.0), (0.6, 0.03, 0.03), 0.95, (0.5, 0.5, 0.5), quat=(c, 0.0, 0.0, s))
    cams = gi.identity_cameras(1, W, H, fx=64.0)
    rt = _render(sc, cams, 0, W, H, flags=orc.F_TIGHT)
    re = _render(sc, cams, 0, W, H, flags=orc.F_ELLIPSE)
    assert re.tile_counts[0] < rt.tile_counts[0]
    assert _check_exact(re, W, H) >= 2
    assert np.array_equal(re.rgb, rt.rgb) and np.array_equal(re.depth, rt.depth)
    _bruteforce_conservative(re, W, H)


def test_ellipse_random_clouds_identical_and_conservative():
    W = H = 64
    for idx in range(4):
        sc = gi.random_cloud(40 + idx, 400, sh_degree=idx % 2)
        cams = gi.cloud_cameras(40 + idx, 2, W, H)
        for e in range(2):
            rt = _render(sc, cams, e, W, H, flags=orc.F_TIGHT)
            re = _render(sc, cams, e, W, H, flags=orc.F_ELLIPSE)
            r0 = _render(sc, cams, e, W, H)
            for a in ("rgb", "depth", "alpha", "exempt"):
                assert np.array_equal(getattr(re, a), getattr(rt, a))
                assert np.array_equal(getattr(re, a), getattr(r0, a))
            assert np.all(re.tile_counts <= rt.tile_counts)
            # lists: order-preserving filter of the tight lists
            keep = np.isin(rt.sorted_tile.astype(np.int64) * 10**6 + rt.sorted_gid,
                           re.sorted_tile.astype(np.int64) * 10**6 + re.sorted_gid)
            assert np.array_equal(rt.sorted_gid[keep], re.sorted_gid)
            assert np.array_equal(rt.sorted_tile[keep], re.sorted_tile)
            assert re.sorted_gid.size == int(re.tile_counts.sum())
            _bruteforce_conservative(re, W, H)
            _check_exact(re, W, H)


def test_ellipse_room_scene_reduces_keys():
    sc = gi.config_scene("c1")
    cams = gi.config_cameras("c1", sc)
    W, H = cams.width, cams.height
    rt = _render(sc, cams, 0, W, H, flags=orc.F_TIGHT)
    re = _render(sc, cams, 0, W, H, flags=orc.F_ELLIPSE)
    assert re.sorted_gid.size < rt.sorted_gid.size
    assert np.array_equal(re.rgb, rt.rgb)
