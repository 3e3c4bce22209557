"""Full-size parity on sampled envs, in the launch configuration bench.py
times (all envs of the config in one gg_render, default chunking), -m gpu.

c3 (BASELINE.json configs[2], the bench workload): 1M Gaussians SH3, 4,096
envs, 640x480 RGB+D.  c2: 500k SH3, 1,024 envs, 320x240 RGB.  c4-lite: the
multi-scene random binding of c4 at reduced scale (8 scenes x 250k, 512 envs)
— generating 256 x 1M scenes on the host takes minutes, so the full c4 is a
bench option, not a test.
"""
import numpy as np
import pytest

import gg_inputs as gi
import oracle
from parity import Tally, check_integer_dumps

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def gg():
    import paper_2510_15352_b200 as m
    m.load_library()
    return m


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _run(gg, scenes, ids, cams, sample, depth=True, ints_env=None, flags=0, oflags=0):
    r = gg.Renderer(0)
    try:
        sid_map = {}
        for k, sc in scenes.items():
            sid_map[k] = r.load_scene(dev(sc.means), dev(sc.scales), dev(sc.quats), dev(sc.opacities), dev(sc.sh),
                                      sc.sh_degree)
        dev_ids = dev(np.array([sid_map[int(i)] for i in ids], np.int32))
        E, W, H = cams.n, cams.width, cams.height
        rgb = torch.empty((E, H, W, 3), dtype=torch.uint8, device="cuda")
        dep = torch.empty((E, H, W), dtype=torch.float32, device="cuda") if depth else None
        vm, K = dev(cams.viewmats), dev(cams.intrinsics)
        r.render(dev_ids, vm, K, W, H, rgb=rgb, depth=dep, flags=flags)
        gg.gg_check_errors(r.ctx)
        torch.cuda.synchronize()
        t = Tally()
        osc = {}
        for e in sample:
            k = int(ids[e])
            if k not in osc:
                osc[k] = oracle.OracleScene.from_inputs(scenes[k])
            o = oracle.render_env(osc[k], cams.viewmats[e], cams.intrinsics[e], W, H, flags=oflags)
            t.add(rgb[e].cpu().numpy(), None if dep is None else dep[e].cpu().numpy(), None, o)
            if e == ints_env:
                # integer artefacts of this env from a second full-batch render
                r.render(dev_ids, vm, K, W, H, rgb=rgb, depth=dep, flags=gg.GG_KEEP_INTERMEDIATES | flags,
                         debug_env=e)
                torch.cuda.synchronize()
                check_integer_dumps(gg, r.ctx, o, scenes[k].n)
        print(t)
        t.check()
    finally:
        r.close()


def test_c3_sampled(gg):
    sc = gi.config_scene("c3")
    cams = gi.config_cameras("c3", sc)
    _run(gg, {0: sc}, np.zeros(cams.n, np.int32), cams, [0, 1111, 2047, 4095], ints_env=2047)


def test_c3_sampled_bench_lists(gg):
    """The configuration bench.py times: all 4,096 envs in one render with the
    opacity-aware tile rects (GG_TIGHT_TILES, reading R35)."""
    sc = gi.config_scene("c3")
    cams = gi.config_cameras("c3", sc)
    _run(gg, {0: sc}, np.zeros(cams.n, np.int32), cams, [7, 2500, 4000], ints_env=2500,
         flags=gg.GG_TIGHT_TILES, oflags=oracle.F_TIGHT)


def test_c2_sampled(gg):
    sc = gi.config_scene("c2")
    cams = gi.config_cameras("c2", sc)
    _run(gg, {0: sc}, np.zeros(cams.n, np.int32), cams, [3, 700, 1023], depth=False, ints_env=700)


def test_c4_lite_multi_scene(gg):
    scenes = {k: gi.room_scene(100 + k, 250_000, 0) for k in range(8)}
    E = 512
    ids = gi.scene_binding(7, E, 8)
    vms = [gi.cameras(5000 + e, 1, 640, 480, scenes[int(ids[e])]).viewmats[0] for e in range(E)]
    cams = gi.Cameras(np.stack(vms), np.tile(gi.pinhole(640, 480).astype(np.float32), (E, 1)), 640, 480)
    _run(gg, scenes, ids, cams, [0, 255, 511], ints_env=255)
