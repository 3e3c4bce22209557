"""Sync-free render mode (GG_ASYNC, gg_reserve_async) and CUDA-graph capture (-m gpu)."""
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
    # and the sync-free render against the oracle, every env
    osc = [oracle.OracleScene.from_inputs(s) for s in scenes]
    intr = np.tile(gi.pinhole(W, H).astype(np.float32), (E, 1))
    t = Tally()
    for e in range(E):
        o = oracle.render_env(osc[int(bind[e])], vms[e], intr[e], W, H)
        t.add(b[0][e], b[1][e], b[2][e], o)
    print(t)
    t.check()
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
    osc = oracle.OracleScene.from_inputs(sc)
    for cams in (cams_b, cams_a):
        vm.copy_(dev(cams.viewmats))
        g.replay()
        torch.cuda.synchronize()
        got = (rgb.cpu().numpy(), dep.cpu().numpy(), al.cpu().numpy())
        t = Tally()                                  # the replayed graph against the oracle
        for e in range(E):
            t.add(got[0][e], got[1][e], got[2][e],
                  oracle.render_env(osc, cams.viewmats[e], cams.intrinsics[e], W, H))
        print(t)
        t.check()
        ref = _render(gg, r, ids, dev(cams.viewmats), K, W, H)
        for x, y in zip(got, ref):
            assert np.array_equal(x, y)
    r.close()


def test_graph_survives_sync_renders_and_scene_loads(gg):
    """a graph captured over a GG_ASYNC render must stay valid when
    sync renders (which grow their own workspace) and scene loads happen
    between replays."""
    r = gg.Renderer(0)
    sc = gi.config_scene("c1")
    sid = r.load_scene(dev(sc.means), dev(sc.scales), dev(sc.quats), dev(sc.opacities), dev(sc.sh), sc.sh_degree)
    E, W, H = 8, 64, 48
    cams = gi.cameras(4, E, W, H, sc)
    ids = dev(np.full(E, sid, np.int32))
    K, vm = dev(cams.intrinsics), dev(cams.viewmats)
    rgb, dep, al = _outs(E, H, W)
    gg.gg_reserve_async(r.ctx, E, W, H, 0, 0.9, 6.0)
    opts = gg.default_opts(flags=gg.GG_ASYNC)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        gg.gg_render(r.ctx, E, ids, vm, K, W, H, opts, rgb, dep, al, stream=s)
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        gg.gg_render(r.ctx, E, ids, vm, K, W, H, opts, rgb, dep, al, stream=s)
    g.replay()
    torch.cuda.synchronize()
    first = (rgb.cpu().numpy(), dep.cpu().numpy(), al.cpu().numpy())
    # a much larger sync render (its workspace grows) and another scene load
    big = gi.room_scene(9, 200_000, 3)
    bid = r.load_scene(dev(big.means), dev(big.scales), dev(big.quats), dev(big.opacities), dev(big.sh), 3)
    cb = gi.cameras(5, 64, 320, 240, big)
    _render(gg, r, dev(np.full(64, bid, np.int32)), dev(cb.viewmats), dev(cb.intrinsics), 320, 240)
    rgb.zero_(); dep.zero_(); al.zero_()
    g.replay()
    torch.cuda.synchronize()
    for x, y in zip(first, (rgb.cpu().numpy(), dep.cpu().numpy(), al.cpu().numpy())):
        assert np.array_equal(x, y)
    r.close()


def test_calibrated_reservation(gg):
    """gg_reserve_async(-h): capacities from a synchronous render at the same
    size; refused without one; the sync-free render then equals the sync one."""
    r = gg.Renderer(0)
    sc = gi.config_scene("c1")
    sid = r.load_scene(dev(sc.means), dev(sc.scales), dev(sc.quats), dev(sc.opacities), dev(sc.sh), sc.sh_degree)
    E, W, H = 24, 64, 48
    cams = gi.cameras(8, E, W, H, sc)
    ids, vm, K = dev(np.full(E, sid, np.int32)), dev(cams.viewmats), dev(cams.intrinsics)
    with pytest.raises(gg.GGError) as ei:
        gg.gg_reserve_async(r.ctx, E, W, H, 0, -1.5, 0.0)
    assert ei.value.status == gg.GG_E_INVALID
    a = _render(gg, r, ids, vm, K, W, H)
    gg.gg_reserve_async(r.ctx, E, W, H, 0, -1.5, 0.0)
    b = _render(gg, r, ids, vm, K, W, H, flags=gg.GG_ASYNC)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)
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


def test_calibrated_capacity_overflow_is_reported(gg):
    """A calibrated reservation (capacity-sized grids of the sync kernels) that
    the next poses outgrow: the chunk is flagged, renders as background, and
    gg_check_errors reports GG_E_CAPACITY (no out-of-bounds work)."""
    r = gg.Renderer(0)
    sc = gi.config_scene("c1")
    sid = r.load_scene(dev(sc.means), dev(sc.scales), dev(sc.quats), dev(sc.opacities), dev(sc.sh), sc.sh_degree)
    E, W, H = 8, 64, 48
    cams = gi.cameras(5, E, W, H, sc)
    ids, K = dev(np.full(E, sid, np.int32)), dev(cams.intrinsics)
    same = np.repeat(cams.viewmats[:1], E, axis=0)   # every env: env 0's view (V0 visible each)
    away = same.copy()
    away[1:, 2, 3] -= 1e4                     # envs 1.. see nothing (every Gaussian behind the camera)
    _render(gg, r, ids, dev(away), K, W, H)   # calibrates: mean V0 / 8, max V0 -> capacity 1.5 * 4 V0
    gg.gg_reserve_async(r.ctx, E, W, H, 0, -1.5, 0.0)
    rgb, dep, al = _outs(E, H, W)
    gg.gg_render(r.ctx, E, ids, dev(same), K, W, H, gg.default_opts(flags=gg.GG_ASYNC), rgb, dep, al)   # 8 V0
    with pytest.raises(gg.GGError) as ei:
        gg.gg_check_errors(r.ctx)
    assert ei.value.status == gg.GG_E_CAPACITY
    assert float(al.abs().max()) == 0.0
    r.close()
