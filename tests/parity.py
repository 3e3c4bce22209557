"""Helpers for GPU-vs-oracle parity tests (tolerances from BASELINE.json north_star).

  * integer artefacts (tile counts, sorted (tile, depth bits, gid) lists,
    tile ranges): bit-exact
  * RGB: max-abs per channel <= 2e-3 on [0,1] (u8 output: |u8/255 - rgb_or|)
  * depth: relative error <= 1e-4 where the oracle's alpha > 0, exactly 0
    where it is 0
  * alpha: abs <= 2e-3
  * at most 0.01% of pixels may fail, and only pixels the oracle flagged as
    threshold near-misses (DESIGN.md §3 "exempt pixels")
"""
from __future__ import annotations

import numpy as np

RGB_TOL = 2e-3
DEPTH_RTOL = 1e-4
ALPHA_TOL = 2e-3
EXEMPT_BUDGET = 1e-4


def pixel_failures(rgb_gpu, depth_gpu, alpha_gpu, o, rgb_is_u8=True):
    """Boolean [H,W] mask of pixels outside tolerance (before exemptions)."""
    ref = np.clip(o.rgb, 0.0, 1.0)
    if rgb_gpu is not None:
        g = rgb_gpu.astype(np.float64) / 255.0 if rgb_is_u8 else np.clip(rgb_gpu.astype(np.float64), 0, 1)
        bad = np.abs(g - ref).max(axis=-1) > RGB_TOL
    else:
        bad = np.zeros(o.alpha.shape, bool)
    if depth_gpu is not None:
        d = depth_gpu.astype(np.float64)
        # the depth's own accumulated alpha (motion blur: the centre sample's)
        pos = getattr(o, "depth_alpha", o.alpha) > 0
        rel = np.where(pos, np.abs(d - o.depth) / np.where(pos, o.depth, 1.0), 0.0)
        bad |= pos & (rel > DEPTH_RTOL)
        bad |= (~pos) & (d != 0.0)
    if alpha_gpu is not None:
        bad |= np.abs(alpha_gpu.astype(np.float64) - o.alpha) > ALPHA_TOL
    return bad


class Tally:
    def __init__(self):
        self.pixels = 0
        self.fail_exempt = 0
        self.fail_hard = 0
        self.max_rgb = 0.0
        self.max_depth_rel = 0.0

    def add(self, rgb_gpu, depth_gpu, alpha_gpu, o, rgb_is_u8=True):
        bad = pixel_failures(rgb_gpu, depth_gpu, alpha_gpu, o, rgb_is_u8)
        self.pixels += bad.size
        self.fail_exempt += int((bad & o.exempt).sum())
        self.fail_hard += int((bad & ~o.exempt).sum())
        ok = ~bad
        if rgb_gpu is not None and ok.any():
            g = rgb_gpu.astype(np.float64) / 255.0 if rgb_is_u8 else rgb_gpu.astype(np.float64)
            self.max_rgb = max(self.max_rgb, float(np.abs(g - np.clip(o.rgb, 0, 1)).max(axis=-1)[ok].max()))
        if depth_gpu is not None:
            pos = (getattr(o, "depth_alpha", o.alpha) > 0) & ok
            if pos.any():
                rel = np.abs(depth_gpu.astype(np.float64)[pos] - o.depth[pos]) / o.depth[pos]
                self.max_depth_rel = max(self.max_depth_rel, float(rel.max()))
        return bad

    def check(self):
        assert self.fail_hard == 0, f"{self.fail_hard} non-exempt pixels outside tolerance ({self})"
        budget = int(np.floor(EXEMPT_BUDGET * self.pixels))
        assert self.fail_exempt <= budget, f"{self.fail_exempt} exempt failures > budget {budget} ({self})"

    def __repr__(self):
        return (f"Tally(pixels={self.pixels}, exempt_fail={self.fail_exempt}, hard_fail={self.fail_hard}, "
                f"max_rgb={self.max_rgb:.3g}, max_depth_rel={self.max_depth_rel:.3g})")


def check_integer_dumps(gg, ctx, o, n_gauss):
    """Bit-exact comparison of the debug env's integer artefacts."""
    tc = gg.gg_debug_dump(ctx, gg.GG_DUMP_TILE_COUNTS)
    assert tc.shape[0] == n_gauss
    assert np.array_equal(tc, o.tile_counts), f"tile counts differ at {np.flatnonzero(tc != o.tile_counts)[:10]}"
    st = gg.gg_debug_dump(ctx, gg.GG_DUMP_SORTED_TILE)
    sz = gg.gg_debug_dump(ctx, gg.GG_DUMP_SORTED_ZBITS)
    sg = gg.gg_debug_dump(ctx, gg.GG_DUMP_SORTED_GIDS)
    assert st.shape == o.sorted_tile.shape, (st.shape, o.sorted_tile.shape)
    assert np.array_equal(st, o.sorted_tile)
    assert np.array_equal(sz, o.sorted_zbits)
    assert np.array_equal(sg, o.sorted_gid)
    rg = gg.gg_debug_dump(ctx, gg.GG_DUMP_RANGES).reshape(-1, 2)
    assert np.array_equal(rg, o.ranges)
    # projected record floats of visible Gaussians: bit-identical u, v, conic, z
    pj = gg.gg_debug_dump(ctx, gg.GG_DUMP_PROJ).reshape(-1, 16)
    vis = o.proj[:, 0] == 1
    assert np.array_equal(pj[:, 0] == 1, vis)
    for col in (1, 2, 3, 4, 5, 6, 8, 9, 10, 11):
        assert np.array_equal(pj[vis, col].view(np.uint32), o.proj[vis, col].view(np.uint32)), col
    assert np.allclose(pj[vis, 12:15], o.proj[vis, 12:15], atol=2e-6)
