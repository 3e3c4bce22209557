"""Sync-free render mode (GG_ASYNC, gg_reserve_async) and CUDA-graph capture (-m gpu)."""
import numpy as np
import pytest

import gg_inputs as gi

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def gg():
    import paper_2510_15352_b200 as m
    m.load_library()
    return m


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _outs(E, H, W):
    return (torch.zeros((E, H, W, 3), dtype=torch.uint8, device="cuda"), torch.zeros((E, H, W), device="cuda"),
            torch.zeros((E, H, W), device="cuda"))


def _render(gg, r, ids, vm, K, W, H, flags=0):
    E = vm.shape[0]
    rgb, dep, al = _outs(E, H, W)
    gg.gg_render(r.ctx, E, ids, vm, K, W, H, gg.default_opts(flags=flags), rgb, dep, al)
    gg.gg_check_errors(r.ctx)
    torch.cuda.synchronize()
    return rgb.cpu().numpy(), dep.cpu().numpy(), al.cpu().numpy()


def test_async_equals_sync_mixed_scenes(gg):
    r = gg.Renderer(0)
    scenes = [gi.room_scene(40 + k, 20_000, (k % 2) * 3, L=None, stairs=None) for k in range(3)]
    sids = [r.load_scene(dev(s.means), dev(s.scales), dev(s.quats), dev(s.opacities), dev(s.sh), s.sh_degree)
            for s in scenes]
    E, W, H = 70, 96, 64                      # 70 envs: groups of 16 with a ragged tail, mixed scenes
    bind = gi.scene_binding(11, E, 3)
    vms = np.stack([gi.cameras(300 + e, 1, W, H, scenes[int(bind[e])]).viewmats[0] for e in range(E)])
    K = dev(np.tile(gi.pinhole(W, H).astype(np.float32), (E, 1)))
    ids = dev(np.array([sids[int(b)] for b in bind], np.int32))
    vm = dev(vms)
    gg.gg_reserve(r.ctx, E, W, H, 32)         # sync mode: chunks of 32 (scene-sorted)
    a = _render(gg, r, ids, vm, K, W, H)
    gg.gg_reserve_async(r.ctx, E, W, H, 48, 0.9, 6.0)
    b = _render(gg, r, ids, vm, K, W, H, flags=gg.GG_ASYNC)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)
    r.close()


def test_async_graph_capture_replay(gg):
    r = gg.Renderer(0)
    sc = gi.config_scene("c1")
    sid = r.load_scene(dev(sc.means), dev(sc.scales), dev(sc.quats), dev(sc.opacities), dev(sc.sh), sc.sh_degree)
    E, W, H = 16, 64, 48
    cams_a = gi.cameras(1, E, W, H, sc)
    cams_b = gi.cameras(2, E, W, H, sc)
    ids = dev(np.full(E, sid, np.int32))
    K = dev(cams_a.intrinsics)
    vm = dev(cams_a.viewmats)                  # static input of the graph
    rgb, dep, al = _outs(E, H, W)
    gg.gg_reserve_async(r.ctx, E, W, H, 0, 0.9, 6.0)
    opts = gg.default_opts(flags=gg.GG_ASYNC)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):                 # warm-up outside the capture
        gg.gg_render(r.ctx, E, ids, vm, K, W, H, opts, rgb, dep, al, stream=s)
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        gg.gg_render(r.ctx, E, ids, vm, K, W, H, opts, rgb, dep, al, stream=s)
    for cams in (cams_b, cams_a):
        vm.copy_(dev(cams.viewmats))
        g.replay()
        torch.cuda.synchronize()
        ref = _render(gg, r, ids, dev(cams.viewmats), K, W, H)
        assert np.array_equal(rgb.cpu().numpy(), ref[0])
        assert np.array_equal(dep.cpu().numpy(), ref[1])
        assert np.array_equal(al.cpu().numpy(), ref[2])
    r.close()


def test_async_capacity_overflow_is_reported(gg):
    r = gg.Renderer(0)
    sc = gi.config_scene("c1")
    sid = r.load_scene(dev(sc.means), dev(sc.scales), dev(sc.quats), dev(sc.opacities), dev(sc.sh), sc.sh_degree)
    E, W, H = 4, 64, 48
    cams = gi.cameras(3, E, W, H, sc)
    gg.gg_reserve_async(r.ctx, E, W, H, 0, 0.001, 1.0)   # far too small
    rgb, dep, al = _outs(E, H, W)
    gg.gg_render(r.ctx, E, dev(np.full(E, sid, np.int32)), dev(cams.viewmats), dev(cams.intrinsics), W, H,
                 gg.default_opts(flags=gg.GG_ASYNC), rgb, dep, al)
    with pytest.raises(gg.GGError) as ei:
        gg.gg_check_errors(r.ctx)
    assert ei.value.status == gg.GG_E_CAPACITY
    assert float(al.abs().max()) == 0.0          # the invalid chunk renders as background
    r.close()
