"""Depth-only render mode (the paper's depth-only
baseline): gg_render with rgb = NULL skips the SH colour and
the colour accumulation; depth and alpha must be bit-identical to the RGB+D
render (same pass decisions and weights), in sync and async mode, and the
depth must match the oracle (-m gpu)."""
import numpy as np
import pytest

import gg_inputs as gi
import oracle
from parity import Tally
from test_gpu_parity import dev, load

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def gg():
    import paper_2510_15352_b200 as m
    m.load_library()
    return m


@pytest.fixture()
def R(gg):
    r = gg.Renderer(0)
    yield r
    r.close()


def _render(gg, r, ids, cams, with_rgb, flags=0):
    E, W, H = cams.n, cams.width, cams.height
    rgb = torch.zeros((E, H, W, 3), dtype=torch.uint8, device="cuda") if with_rgb else None
    depth = torch.full((E, H, W), -1.0, dtype=torch.float32, device="cuda")
    alpha = torch.full((E, H, W), -1.0, dtype=torch.float32, device="cuda")
    r.render(dev(np.asarray(ids, np.int32)), dev(cams.viewmats), dev(cams.intrinsics), W, H, rgb=rgb, depth=depth,
             alpha=alpha, flags=flags)
    gg.gg_check_errors(r.ctx)
    torch.cuda.synchronize()
    return depth.cpu().numpy(), alpha.cpu().numpy()


@pytest.mark.parametrize("flags_name", ["", "GG_TIGHT_TILES"])
def test_depth_only_equals_rgbd(gg, R, flags_name):
    flags = getattr(gg, flags_name) if flags_name else 0
    scs = [gi.random_cloud(900 + k, 200 + 50 * k, sh_degree=3 - k) for k in range(3)]
    sids = [load(R, sc) for sc in scs]
    cams = gi.cloud_cameras(900, 24, 70, 50)
    ids = [sids[k % 3] for k in range(cams.n)]
    d1, a1 = _render(gg, R, ids, cams, True, flags)
    d0, a0 = _render(gg, R, ids, cams, False, flags)
    assert np.array_equal(d0, d1) and np.array_equal(a0, a1)
    # depth vs the oracle on a few envs
    t = Tally()
    for e in (0, 7, 23):
        k = e % 3
        o = oracle.render_env(oracle.OracleScene.from_inputs(scs[k]), cams.viewmats[e], cams.intrinsics[e],
                              cams.width, cams.height)
        t.add(None, d0[e], a0[e], o)
    t.check()


def test_depth_only_c1_async(gg, R):
    sc = gi.config_scene("c1")
    cams = gi.config_cameras("c1", sc, n_envs=32)
    sid = load(R, sc)
    gg.gg_reserve_async(R.ctx, cams.n, cams.width, cams.height)
    d1, a1 = _render(gg, R, [sid] * cams.n, cams, True)
    d0, a0 = _render(gg, R, [sid] * cams.n, cams, False, gg.GG_ASYNC)
    assert np.array_equal(d0, d1) and np.array_equal(a0, a1)
