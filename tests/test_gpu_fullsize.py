"""Full-size parity on sampled envs, in the launch configuration bench.py
times (all envs of the config in one gg_render, default chunking, the
workload's own seeded inputs via gg_inputs.Workload), -m gpu.

Every BASELINE.json config (north_star: "bit-exact binning/sort and
in-tolerance RGB+depth versus the CPU oracle on every config"):

  c2  500k Gaussians SH3, 1,024 envs, 320x240 RGB
  c3  1M SH3, 4,096 envs, 640x480 RGB+D (the bench workload), with the
      opacity-aware lists bench.py renders and with the paper's 3-sigma rects,
      sync and sync-free (GG_ASYNC, replayed from a CUDA graph)
  c4  256 scenes x 1M SH0, 4,096 envs, seeded random binding
  c5  one GPU's share: 2,500 scenes x 0.5M SH0, 4,096 envs
  (c1 is checked in full by test_gpu_parity.py)

Samples: 8 envs compared image by image with the oracle and
64 envs whose integer artefacts (tile counts, sorted (tile, depth bits, gid)
lists, ranges, projected records) must be bit-identical.
"""
import numpy as np
import pytest

import gg_inputs as gi
import oracle
from parity import Tally, check_integer_dumps

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

N_IMAGE, N_INT = 8, 64


@pytest.fixture(scope="module")
def gg():
    import paper_2510_15352_b200 as m
    m.load_library()
    return m


@pytest.fixture(autouse=True)
def _release_cache():
    yield
    torch.cuda.synchronize()
    torch.cuda.empty_cache()


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def samples(E, n, seed):
    """n distinct envs spread over [0, E): the first, the last and a seeded draw."""
    if n <= 0:
        return []
    if n >= E:
        return list(range(E))
    if n <= 2:
        return [0, E - 1][:n]
    rest = np.random.default_rng(seed).choice(np.arange(1, E - 1), n - 2, replace=False)
    return sorted({0, E - 1, *(int(x) for x in rest)})


def load_workload(r, wl, keep):
    """Stream the workload's scenes onto the GPU; keep host copies of `keep`."""
    sid, kept = {}, {}
    for k, sc in wl.scenes():
        sid[k] = r.load_scene(dev(sc.means), dev(sc.scales), dev(sc.quats), dev(sc.opacities), dev(sc.sh),
                              sc.sh_degree)
        if k in keep:
            kept[k] = sc
    return sid, kept


def run_workload(gg, wl, flags=0, oflags=0, depth=True, n_image=N_IMAGE, n_int=N_INT, mode="sync"):
    E, W, H = wl.n_envs, wl.width, wl.height
    img_envs = samples(E, n_image, 1)
    int_envs = samples(E, n_int, 2)
    r = gg.Renderer(0)
    try:
        keep = {int(wl.binding[e]) for e in img_envs + int_envs}
        sid, kept = load_workload(r, wl, keep)
        ids = dev(np.array([sid[int(k)] for k in wl.binding], np.int32))
        vm, K = dev(wl.viewmats[0]), dev(wl.intrinsics)
        rgb = torch.empty((E, H, W, 3), dtype=torch.uint8, device="cuda")
        dep = torch.empty((E, H, W), dtype=torch.float32, device="cuda") if depth else None
        if mode == "sync":
            r.render(ids, vm, K, W, H, rgb=rgb, depth=dep, flags=flags)
        else:
            # bench.py --mode graph: capacities calibrated by a synchronous render (as the
            # bench does), the GG_ASYNC render captured once in a CUDA graph, poses
            # copied into the captured input, replayed
            r.render(ids, dev(wl.viewmats[1 % wl.n_sets]), K, W, H, flags=flags)
            gg.gg_reserve_async(r.ctx, E, W, H, 0, -1.5, 0.0)
            vm_static = dev(wl.viewmats[1 % wl.n_sets])
            opts = gg.default_opts(flags=flags | gg.GG_ASYNC)
            s = torch.cuda.Stream()
            s.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(s):
                gg.gg_render(r.ctx, E, ids, vm_static, K, W, H, opts, rgb, dep, None, stream=s)
            torch.cuda.current_stream().wait_stream(s)
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                gg.gg_render(r.ctx, E, ids, vm_static, K, W, H, opts, rgb, dep, None, stream=s)
            vm_static.copy_(vm)
            g.replay()
        gg.gg_check_errors(r.ctx)
        torch.cuda.synchronize()
        rgb_h = {e: rgb[e].cpu().numpy() for e in img_envs}
        dep_h = {e: dep[e].cpu().numpy() for e in img_envs} if depth else {}
        osc = {}

        def oscene(k):
            if k not in osc:
                osc.clear()                      # one oracle scene at a time (host memory)
                osc[k] = oracle.OracleScene.from_inputs(kept[k])
            return osc[k]

        t = Tally()
        for e in sorted(img_envs, key=lambda e: int(wl.binding[e])):
            k = int(wl.binding[e])
            o = oracle.render_env(oscene(k), wl.viewmats[0][e], wl.intrinsics[e], W, H, flags=oflags)
            t.add(rgb_h[e], dep_h.get(e), None, o)
        print(t)
        t.check()
        # integer artefacts, each from a full-batch render in the same launch configuration
        for e in sorted(int_envs, key=lambda e: int(wl.binding[e])):
            k = int(wl.binding[e])
            r.render(ids, vm, K, W, H, rgb=rgb, depth=dep, flags=gg.GG_KEEP_INTERMEDIATES | flags, debug_env=e)
            torch.cuda.synchronize()
            o = oracle.render_env(oscene(k), wl.viewmats[0][e], wl.intrinsics[e], W, H,
                                  flags=oflags | oracle.F_INTEGER_ONLY)
            check_integer_dumps(gg, r.ctx, o, kept[k].n)
        return t
    finally:
        r.close()


def test_c3_sampled_bench_lists(gg):
    """The configuration bench.py times: 4,096 envs in one render with the
    opacity-aware tile rects (GG_TIGHT_TILES, reading R35)."""
    run_workload(gg, gi.Workload("c3", n_sets=2), flags=gg.GG_TIGHT_TILES, oflags=oracle.F_TIGHT)


def test_c3_sampled_paper_lists(gg):
    run_workload(gg, gi.Workload("c3"), n_int=16)


def test_c3_graph_replay_sampled(gg):
    """bench.py --mode graph: the sync-free GG_ASYNC render replayed from a CUDA
    graph (device-built tables, bounded LOOP grids) against the oracle."""
    run_workload(gg, gi.Workload("c3", n_sets=2), flags=gg.GG_TIGHT_TILES, oflags=oracle.F_TIGHT, mode="graph",
                 n_int=0)


def test_c2_sampled(gg):
    run_workload(gg, gi.Workload("c2"), flags=gg.GG_TIGHT_TILES, oflags=oracle.F_TIGHT, depth=False)


def test_c4_sampled(gg):
    """256 scenes x 1M Gaussians SH0, 4,096 envs, seeded uniform binding."""
    run_workload(gg, gi.Workload("c4", n_envs=4096), flags=gg.GG_TIGHT_TILES, oflags=oracle.F_TIGHT)


def test_c5_share_sampled(gg):
    """One GPU's share of c5: 2,500 scenes x 0.5M SH0 (75 GB of scenes), 4,096
    envs (~1.6 envs per scene: env groups of 1-2 envs)."""
    run_workload(gg, gi.Workload("c5", n_envs=4096), flags=gg.GG_TIGHT_TILES, oflags=oracle.F_TIGHT)


def test_c3_blur_sampled(gg):
    """Motion blur at the bench's scale (bench.py --blur 3): 4,096 envs x 3
    sample cameras through the fused raster average (R32-R34), 4 envs
    compared with the oracle's blur (three renders and the nominal pose each)."""
    wl = gi.Workload("c3")
    E, W, H = wl.n_envs, wl.width, wl.height
    r = gg.Renderer(0)
    try:
        (k, sc), = list(wl.scenes())
        sid = r.load_scene(dev(sc.means), dev(sc.scales), dev(sc.quats), dev(sc.opacities), dev(sc.sh), sc.sh_degree)
        g = gi.rng(gi.KIND_CAMERAS, 777)
        lin = np.float32(g.normal(0.0, 0.5, (E, 3)))
        ang = np.float32(g.normal(0.0, 1.0, (E, 3)))
        rgb = torch.empty((E, H, W, 3), dtype=torch.uint8, device="cuda")
        dep = torch.empty((E, H, W), dtype=torch.float32, device="cuda")
        gg.gg_render_blur(r.ctx, E, dev(np.full(E, sid, np.int32)), dev(wl.viewmats[0]), dev(wl.intrinsics), dev(lin),
                          dev(ang), 0.01, 3, W, H, gg.default_opts(flags=gg.GG_TIGHT_TILES), rgb, dep, None)
        gg.gg_check_errors(r.ctx)
        torch.cuda.synchronize()
        osc = oracle.OracleScene.from_inputs(sc)
        t = Tally()
        for e in samples(E, 4, 3):
            o = oracle.render_blur_env(osc, wl.viewmats[0][e], wl.intrinsics[e], W, H, lin[e], ang[e], 0.01, 3,
                                       flags=oracle.F_TIGHT)
            t.add(rgb[e].cpu().numpy(), dep[e].cpu().numpy(), None, o)
        print(t)
        t.check()
    finally:
        r.close()
