"""Rate-decoupled loop (examples/rate_decoupled_loop.py):
the graph-captured render replayed every `decimation` control steps gives the
frames a direct render of those poses gives, and holds them in between (-m gpu)."""
import os
import sys

import numpy as np
import pytest

import gg_inputs as gi

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "examples"))


def test_rate_decoupled_graph_loop():
    import paper_2510_15352_b200 as gg
    from rate_decoupled_loop import RateDecoupledRenderer, advance
    sc = gi.config_scene("c1")
    E, W, H = 24, 64, 48
    r = gg.Renderer(0)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    sid = r.load_scene(t(sc.means), t(sc.scales), t(sc.quats), t(sc.opacities), t(sc.sh), sc.sh_degree)
    cams = gi.cameras(4, E, W, H, sc)
    ids, K = t(np.full(E, sid, np.int32)), t(cams.intrinsics)
    vm = t(cams.viewmats)
    rr = RateDecoupledRenderer(r.ctx, ids, vm, K, W, H, dino_size=32)
    held = None
    for k in range(7):
        vm = advance(vm, 1.0 / 50.0, speed=2.0)
        if k % 3 == 0:
            rr.render(vm)
            torch.cuda.synchronize()
            rgb = torch.empty((E, H, W, 3), dtype=torch.uint8, device="cuda")
            dep = torch.empty((E, H, W), dtype=torch.float32, device="cuda")
            gg.gg_render(r.ctx, E, ids, vm, K, W, H, gg.default_opts(flags=gg.GG_TIGHT_TILES), rgb, dep, None)
            dino = torch.empty((E, 3, 32, 32), dtype=torch.bfloat16, device="cuda")
            gg.gg_dino_input(r.ctx, E, W, H, rgb, 32, dino)
            torch.cuda.synchronize()
            assert torch.equal(rr.rgb, rgb) and torch.equal(rr.depth, dep) and torch.equal(rr.dino, dino)
            if held is not None:
                assert not torch.equal(held, rr.rgb)       # the cameras moved
            held = rr.rgb.clone()
        else:
            assert torch.equal(rr.rgb, held)               # frames held between camera steps
    gg.gg_check_errors(r.ctx)
    r.close()
