"""Motion blur on the GPU (gg_render_blur) vs its definition and the oracle (-m gpu)."""
import numpy as np
import pytest

import gg_inputs as gi
import oracle
from parity import Tally

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def gg():
    import paper_2510_15352_b200 as m
    m.load_library()
    return m


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _setup(gg, seed=5, E=6, W=64, H=48):
    sc = gi.config_scene("c1")
    cams = gi.cameras(seed, E, W, H, sc)
    r = gg.Renderer(0)
    sid = r.load_scene(dev(sc.means), dev(sc.scales), dev(sc.quats), dev(sc.opacities), dev(sc.sh), sc.sh_degree)
    rng = np.random.default_rng(seed)
    lin = np.float32(rng.normal(0, 1.0, (E, 3)))
    ang = np.float32(rng.normal(0, 2.0, (E, 3)))
    return sc, cams, r, sid, lin, ang


def _outs(E, H, W, fmt):
    rgb = torch.zeros((E, H, W, 3), dtype=torch.uint8 if fmt == 0 else torch.float32, device="cuda")
    return rgb, torch.zeros((E, H, W), device="cuda"), torch.zeros((E, H, W), device="cuda")


def _blur(gg, r, sid, cams, lin, ang, shutter, K, fmt=0):
    E, W, H = cams.n, cams.width, cams.height
    rgb, dep, al = _outs(E, H, W, fmt)
    gg.gg_render_blur(r.ctx, E, dev(np.full(E, sid, np.int32)), dev(cams.viewmats), dev(cams.intrinsics), dev(lin),
                      dev(ang), shutter, K, W, H, gg.default_opts(rgb_format=fmt), rgb, dep, al)
    torch.cuda.synchronize()
    return rgb.cpu().numpy(), dep.cpu().numpy(), al.cpu().numpy()


def _plain(gg, r, sid, vm, cams, fmt=0):
    E, W, H = vm.shape[0], cams.width, cams.height
    rgb, dep, al = _outs(E, H, W, fmt)
    intr = np.tile(cams.intrinsics[:1], (E, 1))
    r.render(dev(np.full(E, sid, np.int32)), dev(vm), dev(intr), W, H, rgb=rgb, depth=dep, alpha=al, rgb_format=fmt)
    torch.cuda.synchronize()
    return rgb.cpu().numpy(), dep.cpu().numpy(), al.cpu().numpy()


def test_poses_match_oracle_definition(gg):
    sc, cams, r, sid, lin, ang = _setup(gg)
    K = 4
    out = torch.zeros((cams.n, K, 4, 4), device="cuda")
    gg.gg_blur_poses(r.ctx, cams.n, dev(cams.viewmats), dev(lin), dev(ang), 0.02, K, out)
    torch.cuda.synchronize()
    got = out.cpu().numpy()
    for e in range(cams.n):
        ref = oracle.blur_poses(cams.viewmats[e], lin[e], ang[e], 0.02, K)
        assert np.allclose(got[e], ref, atol=2e-7, rtol=1e-6)
    r.close()


def test_static_cases_bit_exact(gg):
    sc, cams, r, sid, lin, ang = _setup(gg)
    for fmt in (0, 1):
        base = _plain(gg, r, sid, cams.viewmats, cams, fmt)
        k1 = _blur(gg, r, sid, cams, lin, ang, 0.03, 1, fmt)
        z4 = _blur(gg, r, sid, cams, 0 * lin, 0 * ang, 0.03, 4, fmt)
        for a, b, c in zip(base, k1, z4):
            assert np.array_equal(a, b) and np.array_equal(a, c)
    r.close()


def test_average_of_sample_renders_bit_exact(gg):
    """the K=4 blend equals the float mean of the four offset renders
    (in the R34 order: m = x0 + ((x1-x0) + (x2-x0) + (x3-x0)) / 4), depth from the nominal pose (t = 0)."""
    sc, cams, r, sid, lin, ang = _setup(gg)
    K, E = 4, cams.n
    poses = torch.zeros((E, K, 4, 4), device="cuda")
    gg.gg_blur_poses(r.ctx, E, dev(cams.viewmats), dev(lin), dev(ang), 0.03, K, poses)
    torch.cuda.synchronize()
    pv = poses.cpu().numpy()
    rgb_b, dep_b, al_b = _blur(gg, r, sid, cams, lin, ang, 0.03, K, fmt=1)
    for e in range(E):
        s_rgb, s_dep, s_al = _plain(gg, r, sid, pv[e], cams, fmt=1)
        for out, x in ((rgb_b[e], s_rgb), (al_b[e], s_al)):
            acc = x[1] - x[0]
            for i in range(2, K):
                acc = acc + (x[i] - x[0])
            m = x[0] + acc / np.float32(K)
            assert np.array_equal(out, m)
        lo, hi = s_rgb.min(axis=0), s_rgb.max(axis=0)
        assert np.all(rgb_b[e] >= lo) and np.all(rgb_b[e] <= hi)    # convex combination
    base = _plain(gg, r, sid, cams.viewmats, cams, fmt=1)
    assert np.array_equal(dep_b, base[1])        # depth of the nominal pose t = 0, even K
    r.close()


@pytest.mark.parametrize("K", [3, 4])
def test_blur_oracle_parity(gg, K):
    sc, cams, r, sid, lin, ang = _setup(gg, seed=9, E=4)
    shutter = 0.02
    rgb, dep, al = _blur(gg, r, sid, cams, lin, ang, shutter, K)
    osc = oracle.OracleScene.from_inputs(sc)
    t = Tally()
    for e in range(cams.n):
        o = oracle.render_blur_env(osc, cams.viewmats[e], cams.intrinsics[e], cams.width, cams.height, lin[e], ang[e],
                                   shutter, K)
        t.add(rgb[e], dep[e], al[e], o)
    print(t)
    t.check()
    r.close()


def test_blur_honours_tile_list_flags(gg):
    """gg_render_blur keeps GG_TIGHT_TILES / GG_ELLIPSE_TILES; both
    list variants give images identical to the paper's rects (R35, R37)."""
    sc, cams, r, sid, lin, ang = _setup(gg, seed=11, E=5)
    E, W, H = cams.n, cams.width, cams.height
    outs = []
    for flags in (0, gg.GG_TIGHT_TILES, gg.GG_ELLIPSE_TILES):
        rgb, dep, al = _outs(E, H, W, 0)
        gg.gg_render_blur(r.ctx, E, dev(np.full(E, sid, np.int32)), dev(cams.viewmats), dev(cams.intrinsics),
                          dev(lin), dev(ang), 0.02, 3, W, H, gg.default_opts(flags=flags), rgb, dep, al)
        torch.cuda.synchronize()
        outs.append((rgb.cpu().numpy(), dep.cpu().numpy(), al.cpu().numpy()))
    for o in outs[1:]:
        for a, b in zip(outs[0], o):
            assert np.array_equal(a, b)
    r.close()
