"""GG_TIGHT_TILES / GG_ELLIPSE_TILES (work-reduction variants, DESIGN.md
readings R35, R37) on the GPU: integer artefacts bit-exact against the
oracle's F_TIGHT / F_ELLIPSE, images bit-identical to the paper-rect render,
async mode equal to sync (-m gpu)."""
import numpy as np
import pytest

import gg_inputs as gi
import oracle
from parity import Tally, check_integer_dumps
from test_gpu_parity import _adversarial, dev, load, parity_envs, render

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


def _same_images(a, b):
    for x, y in zip(a, b):
        if x is not None:
            assert np.array_equal(x, y)


VARIANTS = [("tight", {"tight": True}), ("ellipse", {"ellipse": True})]


@pytest.mark.parametrize("name,var", VARIANTS)
def test_tight_c1_and_clouds(gg, R, name, var):
    cases = [(gi.config_scene("c1"), None)]
    cases += [(gi.random_cloud(2000 + k, 150 + 60 * k, sh_degree=k % 4), k) for k in range(6)]
    for sc, k in cases:
        if k is None:
            cams = gi.config_cameras("c1", sc)
        else:
            cams = gi.cloud_cameras(2000 + k, 3, *((70, 50) if k % 2 else (64, 64)))
        sid = load(R, sc)
        t = Tally()
        imgs_t = parity_envs(gg, R, {sid: sc}, [sid] * cams.n, cams, range(cams.n), t, **var)
        t.check()
        imgs_p = render(gg, R, [sid] * cams.n, cams)
        _same_images(imgs_t, imgs_p)
        gg.gg_unload_scene(R.ctx, sid)


@pytest.mark.parametrize("name,var", VARIANTS)
def test_tight_adversarial(gg, R, name, var):
    sc = _adversarial()
    cams = gi.identity_cameras(2, 70, 50, 64.0)
    cams.intrinsics[1] = [40.0, 44.0, 33.3, 27.1]
    sid = load(R, sc)
    t = Tally()
    imgs_t = parity_envs(gg, R, {sid: sc}, [sid] * 2, cams, range(2), t, **var)
    t.check()
    _same_images(imgs_t, render(gg, R, [sid] * 2, cams))


@pytest.mark.parametrize("gflag,oflag", [("GG_TIGHT_TILES", "F_TIGHT"), ("GG_ELLIPSE_TILES", "F_ELLIPSE")])
def test_tight_c3_subset_identical_and_fewer_keys(gg, R, gflag, oflag):
    """512 envs of the bench workload: images bit-identical, keys fewer, one
    env's lists bit-exact against the oracle's F_TIGHT."""
    sc = gi.config_scene("c3")
    cams = gi.config_cameras("c3", sc, n_envs=512)
    sid = load(R, sc)
    ids = [sid] * cams.n
    a = render(gg, R, ids, cams, want_alpha=False, flags=gg.GG_COUNTERS)
    c0 = gg.gg_get_counters(R.ctx, cams.n)
    b = render(gg, R, ids, cams, want_alpha=False, flags=gg.GG_COUNTERS | getattr(gg, gflag))
    c1 = gg.gg_get_counters(R.ctx, cams.n)
    _same_images(a, b)
    k0, k1 = c0[:, 3].sum(), c1[:, 3].sum()
    assert k1 < 0.9 * k0, (k0, k1)
    assert np.array_equal(c0[:, 2], c1[:, 2])           # same visible records
    assert np.all(c1[:, 0] <= c0[:, 0])                 # n_eval never grows
    assert np.array_equal(c0[:, 1], c1[:, 1])           # n_contrib identical
    e = 301
    render(gg, R, ids, cams, want_alpha=False, flags=gg.GG_KEEP_INTERMEDIATES | getattr(gg, gflag), debug_env=e)
    o = oracle.render_env(oracle.OracleScene.from_inputs(sc), cams.viewmats[e], cams.intrinsics[e], cams.width,
                          cams.height, flags=getattr(oracle, oflag))
    check_integer_dumps(gg, R.ctx, o, sc.n)


@pytest.mark.parametrize("gflag", ["GG_TIGHT_TILES", "GG_ELLIPSE_TILES"])
def test_tight_async_matches_sync(gg, R, gflag):
    sc = gi.config_scene("c1")
    cams = gi.config_cameras("c1", sc, n_envs=64)
    sid = load(R, sc)
    gg.gg_reserve_async(R.ctx, cams.n, cams.width, cams.height)
    a = render(gg, R, [sid] * cams.n, cams, flags=getattr(gg, gflag))
    b = render(gg, R, [sid] * cams.n, cams, flags=getattr(gg, gflag) | gg.GG_ASYNC)
    _same_images(a, b)
