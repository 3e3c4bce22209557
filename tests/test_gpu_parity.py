"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle (-m gpu).

Integer artefacts bit-exact; images within the north-star tolerances with
the 0.01% exempt-pixel budget (tests/parity.py).
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


@pytest.fixture()
def R(gg):
    r = gg.Renderer(0)
    yield r
    r.close()


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def load(r, sc):
    return r.load_scene(dev(sc.means), dev(sc.scales), dev(sc.quats), dev(sc.opacities), dev(sc.sh), sc.sh_degree)


def render(gg, r, ids, cams, want_depth=True, want_alpha=True, fmt=0, **kw):
    E, W, H = cams.n, cams.width, cams.height
    rgb = torch.zeros((E, H, W, 3), dtype=torch.uint8 if fmt == 0 else torch.float32, device="cuda")
    depth = torch.zeros((E, H, W), dtype=torch.float32, device="cuda") if want_depth else None
    alpha = torch.zeros((E, H, W), dtype=torch.float32, device="cuda") if want_alpha else None
    r.render(dev(np.asarray(ids, np.int32)), dev(cams.viewmats), dev(cams.intrinsics), W, H, rgb=rgb, depth=depth,
             alpha=alpha, rgb_format=fmt, **kw)
    gg.gg_check_errors(r.ctx)
    torch.cuda.synchronize()
    return (rgb.cpu().numpy(), None if depth is None else depth.cpu().numpy(),
            None if alpha is None else alpha.cpu().numpy())


def parity_envs(gg, r, scenes, sids, cams, envs, tally, ints=True, sh_degree=-1, background=(0.0, 0.0, 0.0),
                tight=False, ellipse=False, **kw):
    """Render all envs on the GPU; compare `envs` with the oracle (and their
    integer artefacts, one debug render per env).  tight: GG_TIGHT_TILES on
    the GPU, F_TIGHT in the oracle (reading R35); ellipse: GG_ELLIPSE_TILES /
    F_ELLIPSE (reading R37)."""
    kw["background"] = background
    gflag = gg.GG_ELLIPSE_TILES if ellipse else (gg.GG_TIGHT_TILES if tight else 0)
    oflag = oracle.F_ELLIPSE if ellipse else (oracle.F_TIGHT if tight else 0)
    rgb, depth, alpha = render(gg, r, sids, cams, sh_degree=sh_degree, flags=gflag, **kw)
    oscenes = {}
    for e in envs:
        s = int(sids[e])
        if s not in oscenes:
            oscenes[s] = oracle.OracleScene.from_inputs(scenes[s])
        o = oracle.render_env(oscenes[s], cams.viewmats[e], cams.intrinsics[e], cams.width, cams.height,
                              sh_degree=sh_degree, background=tuple(float(np.float32(b)) for b in background),
                              flags=oflag, near=float(np.float32(kw.get("near_plane", 0.01))),
                              far=float(np.float32(kw.get("far_plane", 1e10))))
        tally.add(rgb[e], depth[e], alpha[e], o)
        if ints:
            render(gg, r, sids, cams, sh_degree=sh_degree,
                   flags=gg.GG_KEEP_INTERMEDIATES | gg.GG_COUNTERS | gflag, debug_env=e, **kw)
            check_integer_dumps(gg, r.ctx, o, scenes[s].n)
            neval = gg.gg_debug_dump(r.ctx, gg.GG_DUMP_N_EVAL).reshape(cams.height, cams.width)
            same = ~o.exempt
            assert np.array_equal(neval[same], o.n_eval[same]), "n_eval differs on non-exempt pixels"
    return rgb, depth, alpha


def test_c1_full(gg, R):
    sc = gi.config_scene("c1")
    cams = gi.config_cameras("c1", sc)
    sid = load(R, sc)
    t = Tally()
    parity_envs(gg, R, {sid: sc}, [sid] * cams.n, cams, range(cams.n), t)
    t.check()
    print(t)


def test_near_far_cull_boundaries(gg, R):
    """The GPU's cull predicate on the f32 boundary values (test_oracle_pins
    near_far_fixture): tile counts bit-exact with the oracle, images in tolerance."""
    from test_oracle_pins import FAR32, NEAR32, near_far_fixture
    sc, expect, _ = near_far_fixture()
    cams = gi.identity_cameras(1, 64, 48, 32.0)
    sid = load(R, sc)
    t = Tally()
    parity_envs(gg, R, {sid: sc}, [sid], cams, [0], t, near_plane=float(NEAR32), far_plane=float(FAR32))
    t.check()
    tc = gg.gg_debug_dump(R.ctx, gg.GG_DUMP_TILE_COUNTS)
    assert ((tc > 0) == expect).all()


@pytest.mark.parametrize("near,far,passes", [(4.0, 4.4, 2), (0.01, 1e10, 3), (1e-30, 1e10, 4)])
def test_depth_pass_counts(gg, R, near, far, passes):
    """The depth-sort key is z bits - bits(near) (every record has near < z <= far),
    so [near, far] fixes the number of 10-bit passes: a thin slab of the cloud
    sorts in 2 passes, an extreme span in 4.  Lists and images match the
    oracle run with the same planes."""
    span = int(np.float32(far).view(np.uint32)) - int(np.float32(near).view(np.uint32))
    assert (span.bit_length() + 9) // 10 == passes
    sc = gi.random_cloud(1500, 400, sh_degree=1)
    cams = gi.cloud_cameras(1500, 3)
    sid = load(R, sc)
    t = Tally()
    parity_envs(gg, R, {sid: sc}, [sid] * 3, cams, range(3), t, near_plane=near, far_plane=far)
    t.check()


@pytest.mark.parametrize("seed", range(12))
def test_random_clouds(gg, R, seed):
    """SPEC.md:518 suite: random scenes <= 512 splats, 64x64 (and 70x50 partial
    tiles), random cameras, all SH degrees."""
    d = seed % 4
    sc = gi.random_cloud(1000 + seed, 64 + 37 * seed, sh_degree=d)
    W, H = (70, 50) if seed % 3 == 2 else (64, 64)
    cams = gi.cloud_cameras(1000 + seed, 3, W, H)
    sid = load(R, sc)
    t = Tally()
    bg = (0.1, 0.5, 0.9) if seed % 2 else (0.0, 0.0, 0.0)
    parity_envs(gg, R, {sid: sc}, [sid] * 3, cams, range(3), t, background=bg)
    t.check()


def _adversarial():
    """Near-plane straddlers, behind-camera, full-image, exact depth ties,
    u-r on a tile boundary, near-zero scale, opacity 0 and 1."""
    parts = []
    rng = np.random.default_rng(77)
    for k in range(20):   # straddle the near plane (0.01 m)
        parts.append(gi.single_gaussian((rng.uniform(-0.02, 0.02), rng.uniform(-0.02, 0.02), 0.01 + rng.normal(0, 0.004)),
                                        0.01, 0.7, rng.uniform(0, 1, 3)))
    for k in range(10):   # behind the camera
        parts.append(gi.single_gaussian((rng.uniform(-1, 1), rng.uniform(-1, 1), -rng.uniform(0.1, 3)), 0.2, 0.9,
                                        rng.uniform(0, 1, 3)))
    parts.append(gi.single_gaussian((0, 0, 3.0), 3.0, 0.3, (0.2, 0.7, 0.4)))    # covers every tile
    for k in range(5):    # exact depth ties (duplicates)
        g = gi.single_gaussian((rng.uniform(-0.5, 0.5), rng.uniform(-0.5, 0.5), 2.5), 0.05, 0.8, rng.uniform(0, 1, 3))
        parts += [g, g, g]
    # u - r on a multiple of 16: f=64, z=4, u = 32 + 64 x/4; choose x so u = 20 (r = 4 -> u - r = 16)
    parts.append(gi.single_gaussian(((20 - 32) * 4 / 64, 0.0, 4.0), 1e-4, 0.9, (1, 0, 0)))
    for k in range(10):   # near-zero scales (r = 3), opacity 0 / 1
        parts.append(gi.single_gaussian((rng.uniform(-0.8, 0.8), rng.uniform(-0.6, 0.6), rng.uniform(1, 4)),
                                        1e-8, float(k % 2), rng.uniform(0, 1, 3)))
    parts.append(gi.random_cloud(78, 200))
    return gi.concat(parts)


def test_adversarial_fixtures(gg, R):
    sc = _adversarial()
    cams = gi.identity_cameras(2, 70, 50, 64.0)
    cams.intrinsics[1] = [40.0, 44.0, 33.3, 27.1]
    sid = load(R, sc)
    t = Tally()
    parity_envs(gg, R, {sid: sc}, [sid] * 2, cams, range(2), t)
    t.check()


def test_determinism_batch_and_rgb_only(gg, R):
    """run twice bit-identical; batch == singles;
    RGB of RGB+D == RGB-only; chunking does not change the result."""
    a = gi.random_cloud(500, 400)
    b = gi.random_cloud(501, 300, sh_degree=2)
    sa, sb = load(R, a), load(R, b)
    cams = gi.cloud_cameras(500, 64)
    ids = np.where(np.arange(64) % 2 == 0, sa, sb).astype(np.int32)
    r1 = render(gg, R, ids, cams)
    r2 = render(gg, R, ids, cams)
    for x, y in zip(r1, r2):
        assert np.array_equal(x, y)
    for e in (0, 1, 17, 63):
        one = gi.Cameras(cams.viewmats[e:e + 1], cams.intrinsics[e:e + 1], cams.width, cams.height)
        s = render(gg, R, ids[e:e + 1], one)
        for x, y in zip(r1, s):
            assert np.array_equal(x[e], y[0])
    rgb_only, _, _ = render(gg, R, ids, cams, want_depth=False, want_alpha=False)
    assert np.array_equal(rgb_only, r1[0])
    gg.gg_reserve(R.ctx, 64, cams.width, cams.height, 5)     # chunks of 5 envs
    r3 = render(gg, R, ids, cams)
    for x, y in zip(r1, r3):
        assert np.array_equal(x, y)
    # the counters walk (256-thread reference kernel) gives bit-identical images
    r4 = render(gg, R, ids, cams, flags=gg.GG_COUNTERS)
    for x, y in zip(r1, r4):
        assert np.array_equal(x, y)


def test_multi_scene_random_binding(gg, R):
    scenes = {}
    for k in range(4):
        sc = gi.room_scene(10 + k, 30_000, k % 2 * 3, L=None, stairs=None)
        scenes[load(R, sc)] = sc
    keys = sorted(scenes)
    ids = np.array(keys)[gi.scene_binding(3, 24, 4)]
    cams_list = [gi.cameras(100 + e, 1, 96, 64, scenes[int(ids[e])]) for e in range(24)]
    cams = gi.Cameras(np.concatenate([c.viewmats for c in cams_list]),
                      np.concatenate([c.intrinsics for c in cams_list]), 96, 64)
    t = Tally()
    parity_envs(gg, R, scenes, ids, cams, [0, 5, 11, 23], t)
    t.check()


def test_f32_rgb_format(gg, R):
    sc = gi.random_cloud(600, 300, sh_degree=1)
    cams = gi.cloud_cameras(600, 2)
    sid = load(R, sc)
    rgb, depth, alpha = render(gg, R, [sid, sid], cams, fmt=1)
    osc = oracle.OracleScene.from_inputs(sc)
    t = Tally()
    for e in range(2):
        o = oracle.render_env(osc, cams.viewmats[e], cams.intrinsics[e], 64, 64)
        t.add(rgb[e], depth[e], alpha[e], o, rgb_is_u8=False)
    t.check()


def test_render_host_matches_device(gg, R):
    sc = gi.random_cloud(700, 300)
    cams = gi.cloud_cameras(700, 9)
    sid = load(R, sc)
    ref = render(gg, R, [sid] * 9, cams)
    E, W, H = 9, 64, 64
    rgb = torch.zeros((E, H, W, 3), dtype=torch.uint8).pin_memory()
    depth = torch.zeros((E, H, W), dtype=torch.float32).pin_memory()
    alpha = torch.zeros((E, H, W), dtype=torch.float32).pin_memory()
    gg.gg_reserve(R.ctx, 9, W, H, 4)
    gg.gg_render_host(R.ctx, E, np.full(E, sid, np.int32), cams.viewmats, cams.intrinsics, W, H, None,
                      rgb, depth, alpha)
    assert np.array_equal(rgb.numpy(), ref[0])
    assert np.array_equal(depth.numpy(), ref[1])
    assert np.array_equal(alpha.numpy(), ref[2])


def test_render_host_multi_scene_slices(gg, R):
    """gg_render_host with a random binding to 3 scenes (processing order !=
    caller order) and chunks of 512 envs streamed in raster slices: the host
    frames equal the device render."""
    scs = [gi.random_cloud(710 + k, 120 + 40 * k, sh_degree=k) for k in range(3)]
    sids = [load(R, sc) for sc in scs]
    E, W, H = 600, 32, 32
    cams = gi.cloud_cameras(710, E, W, H)
    ids = np.array(sids, np.int32)[gi.rng(gi.KIND_CAMERAS, 711).integers(0, 3, E)]
    gg.gg_reserve(R.ctx, E, W, H, 512)
    ref = render(gg, R, ids, cams)
    rgb = torch.zeros((E, H, W, 3), dtype=torch.uint8).pin_memory()
    depth = torch.zeros((E, H, W), dtype=torch.float32).pin_memory()
    alpha = torch.zeros((E, H, W), dtype=torch.float32).pin_memory()
    gg.gg_render_host(R.ctx, E, ids, cams.viewmats, cams.intrinsics, W, H, None, rgb, depth, alpha)
    assert np.array_equal(rgb.numpy(), ref[0])
    assert np.array_equal(depth.numpy(), ref[1])
    assert np.array_equal(alpha.numpy(), ref[2])


def test_render_host_async_pipelined(gg, R):
    """gg_render_host_async: 4 back-to-back calls with different poses into 4
    host frame sets (the two device staging slots are reused while earlier
    frames may still be copying out), then gg_host_sync: every set equals the
    device render of its poses."""
    scs = [gi.random_cloud(720 + k, 200, sh_degree=k) for k in range(2)]
    sids = [load(R, sc) for sc in scs]
    E, W, H = 300, 48, 32
    ids = np.array(sids, np.int32)[gi.rng(gi.KIND_CAMERAS, 721).integers(0, 2, E)]
    gg.gg_reserve(R.ctx, E, W, H, 128)
    poses = [gi.cloud_cameras(730 + k, E, W, H) for k in range(4)]
    refs = [render(gg, R, ids, c) for c in poses]
    outs = [(torch.zeros((E, H, W, 3), dtype=torch.uint8).pin_memory(),
             torch.zeros((E, H, W), dtype=torch.float32).pin_memory(),
             torch.zeros((E, H, W), dtype=torch.float32).pin_memory()) for _ in poses]
    for c, o in zip(poses, outs):
        gg.gg_render_host_async(R.ctx, E, ids, c.viewmats, c.intrinsics, W, H, None, *o)
    gg.gg_host_sync(R.ctx)
    for ref, o in zip(refs, outs):
        for a, b in zip(ref, o):
            assert np.array_equal(a, b.numpy())


def test_chunk_halving_when_workspace_allocation_fails(gg):
    """A chunk whose record workspace cannot be allocated is redone in halves:
    with an allocator that refuses blocks above 1 MB, a 512-env chunk (~1.6 MB
    of rec0) falls back to smaller chunks and the frames are unchanged."""
    import ctypes as C
    sc = gi.random_cloud(740, 300)
    E, W, H = 512, 64, 64
    cams = gi.cloud_cameras(740, E, W, H)
    r_ref = gg.Renderer(0)
    try:
        sid = load(r_ref, sc)
        gg.gg_reserve(r_ref.ctx, E, W, H, 512)
        ref = render(gg, r_ref, [sid] * E, cams)
    finally:
        r_ref.close()
    base, keep = gg.torch_allocator(0)
    LIMIT = 1 << 20

    def _alloc(size, stream, user):
        return 0 if size > LIMIT else base.alloc(size, stream, user)

    fa = gg.ALLOC_FN(_alloc)
    lim = gg.gg_allocator(fa, base.free, None)
    ctx = gg.gg_create(0, lim)
    try:
        sid = gg.gg_load_scene(ctx, sc.n, sc.sh_degree, dev(sc.means), dev(sc.scales), dev(sc.quats),
                               dev(sc.opacities), dev(sc.sh))
        gg.gg_reserve(ctx, E, W, H, 512)
        out = [torch.zeros((E, H, W, 3), dtype=torch.uint8, device="cuda"),
               torch.zeros((E, H, W), device="cuda"), torch.zeros((E, H, W), device="cuda")]
        gg.gg_render(ctx, E, dev(np.full(E, sid, np.int32)), dev(cams.viewmats), dev(cams.intrinsics), W, H, None,
                     *out)
        gg.gg_check_errors(ctx)
        torch.cuda.synchronize()
        for a, b in zip(ref, out):
            assert np.array_equal(a, b.cpu().numpy())
    finally:
        gg.gg_destroy(ctx)
    del keep, fa


def test_errors(gg, R):
    sc = gi.random_cloud(800, 10)
    with pytest.raises(gg.GGError) as ei:
        bad = sc.means.copy()
        bad[3, 1] = np.nan
        gg.gg_load_scene(R.ctx, 10, 0, dev(bad), dev(sc.scales), dev(sc.quats), dev(sc.opacities), dev(sc.sh))
    assert ei.value.status == gg.GG_E_NONFINITE and "record 3" in str(ei.value)
    with pytest.raises(gg.GGError) as ei:
        s2 = sc.scales.copy()
        s2[7, 0] = 0.0
        gg.gg_load_scene(R.ctx, 10, 0, sc.means, s2, sc.quats, sc.opacities, sc.sh)   # host pointers
    assert ei.value.status == gg.GG_E_INVALID and "record 7" in str(ei.value)
    with pytest.raises(gg.GGError) as ei:
        gg.gg_load_scene(R.ctx, 0, 0, sc.means, sc.scales, sc.quats, sc.opacities, sc.sh)
    assert ei.value.status == gg.GG_E_INVALID
    sid = gg.gg_load_scene(R.ctx, 10, 0, sc.means, sc.scales, sc.quats, sc.opacities, sc.sh)   # host ok
    cams = gi.cloud_cameras(800, 2)
    with pytest.raises(gg.GGError) as ei:
        render(gg, R, [sid, sid + 5], cams)
    assert ei.value.status == gg.GG_E_BAD_SCENE


def test_counters_match_oracle(gg, R):
    sc = gi.config_scene("c1")
    cams = gi.config_cameras("c1", sc)
    sid = load(R, sc)
    render(gg, R, [sid] * cams.n, cams, flags=gg.GG_COUNTERS)
    cnt = gg.gg_get_counters(R.ctx, cams.n)
    osc = oracle.OracleScene.from_inputs(sc)
    for e in range(cams.n):
        o = oracle.render_env(osc, cams.viewmats[e], cams.intrinsics[e], cams.width, cams.height)
        assert cnt[e, 3] == len(o.sorted_gid)
        assert abs(cnt[e, 0] - o.n_eval.sum()) <= 0.001 * o.n_eval.sum()
        assert abs(cnt[e, 1] - o.n_contrib.sum()) <= 0.001 * o.n_contrib.sum()


def test_ply_scene_renders_like_arrays(gg, R, tmp_path):
    """gg_load_ply (native PLY reader + load) renders bit-identically to
    loading the reader's activated arrays through gg_load_scene."""
    sc = gi.random_cloud(900, 200, sh_degree=2)
    p = tmp_path / "s.ply"
    gi.write_3dgs_ply(str(p), sc)
    sid_ply = gg.gg_load_ply(R.ctx, str(p))
    m, s, q, o, sh, d = gg.gg_read_ply(str(p))
    sid_arr = gg.gg_load_scene(R.ctx, m.shape[0], d, m, s, q, o, sh)
    cams = gi.cloud_cameras(900, 2)
    a = render(gg, R, [sid_ply, sid_ply], cams)
    b = render(gg, R, [sid_arr, sid_arr], cams)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)


@pytest.mark.parametrize("W,H", [(1280, 960), (1, 1), (17, 3)])
def test_image_sizes(gg, R, W, H):
    """> 2048 tiles (the 13-bit placement path), and degenerate tiny images."""
    sc = gi.random_cloud(1300, 300, sh_degree=1)
    cams = gi.cloud_cameras(1300, 2, W, H)
    sid = load(R, sc)
    t = Tally()
    parity_envs(gg, R, {sid: sc}, [sid] * 2, cams, range(2), t)
    t.check()
    t2 = Tally()
    parity_envs(gg, R, {sid: sc}, [sid] * 2, cams, range(2), t2, tight=True)
    t2.check()
