"""Pins for the oracle's motion blur (readings R32-R34), -m "not gpu"."""
import numpy as np
import pytest
from scipy.spatial.transform import Rotation

import gg_inputs as gi
import oracle


def test_blur_poses_vs_scipy():
    rng = np.random.default_rng(0)
    sc = gi.room_scene(1, 1000, 0, L=12.0, stairs=True)
    V = gi.cameras(1, 1, 64, 48, sc).viewmats[0].astype(np.float64)
    v, w = rng.normal(size=3), rng.normal(size=3) * 2
    shutter, K = 0.02, 5
    P = oracle.blur_poses(V, v, w, shutter, K)
    C = -V[:3, :3].T @ V[:3, 3]
    for i in range(K):
        t = float(np.float32(shutter)) * ((i + 0.5) / K - 0.5)
        Rwc = Rotation.from_rotvec(w * t).as_matrix() @ V[:3, :3].T
        assert np.allclose(P[i, :3, :3], Rwc.T, atol=1e-12)
        # centre moved by v t
        assert np.allclose(-P[i, :3, :3].T @ P[i, :3, 3], C + v * t, atol=1e-12)
    # symmetric sample times: the middle sample of odd K is the static pose
    assert np.allclose(P[K // 2], V, atol=1e-12)
    # K = 1 and zero velocity: static pose
    assert np.allclose(oracle.blur_poses(V, v, w, shutter, 1)[0], V, atol=1e-12)
    assert np.allclose(oracle.blur_poses(V, 0 * v, 0 * w, shutter, 4), V[None], atol=1e-12)


def _setup():
    sc = gi.random_cloud(77, 300)
    cams = gi.cloud_cameras(77, 1)
    return oracle.OracleScene.from_inputs(sc), cams


def test_blur_static_cases_equal_plain_render():
    osc, cams = _setup()
    base = oracle.render_env(osc, cams.viewmats[0], cams.intrinsics[0], 64, 64)
    b1 = oracle.render_blur_env(osc, cams.viewmats[0], cams.intrinsics[0], 64, 64, [0.3, 0, 0], [0, 0.5, 0], 0.03, 1)
    assert np.array_equal(b1.rgb, base.rgb) and np.array_equal(b1.depth, base.depth)
    b0 = oracle.render_blur_env(osc, cams.viewmats[0], cams.intrinsics[0], 64, 64, [0, 0, 0], [0, 0, 0], 0.03, 4)
    assert np.allclose(b0.rgb, base.rgb, atol=1e-15) and np.array_equal(b0.depth, base.depth)
    with pytest.raises(ValueError):
        oracle.render_blur_env(osc, cams.viewmats[0], cams.intrinsics[0], 64, 64, [0, 0, 0], [0, 0, 0], 0.03, 0)


def test_blur_is_convex_combination_and_blurs():
    osc, cams = _setup()
    b = oracle.render_blur_env(osc, cams.viewmats[0], cams.intrinsics[0], 64, 64, [2.0, 0, 0], [0, 0, 3.0], 0.05, 4)
    lo = np.min([s.rgb for s in b.samples], axis=0)
    hi = np.max([s.rgb for s in b.samples], axis=0)
    assert np.all(b.rgb >= lo - 1e-12) and np.all(b.rgb <= hi + 1e-12)
    base = oracle.render_env(osc, cams.viewmats[0], cams.intrinsics[0], 64, 64)
    assert np.abs(b.rgb - base.rgb).max() > 1e-3       # motion changes the image
    # depth from the nominal pose t = 0 ("center sample"), not from an offset sample of even K
    assert np.array_equal(b.depth, base.depth)
    assert not np.array_equal(b.depth, b.samples[2].depth)
    b5 = oracle.render_blur_env(osc, cams.viewmats[0], cams.intrinsics[0], 64, 64, [2.0, 0, 0], [0, 0, 3.0], 0.05, 5)
    assert np.array_equal(b5.depth, base.depth)
