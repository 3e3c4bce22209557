"""Pins for the CPU oracle against things other than itself (-m "not gpu").

Each test pins one step of DESIGN.md §2 (O1-O5) to a closed form, a value
SPEC.md prints (tests/golden/spec_examples.json), an independent library
routine (scipy rotations / spherical harmonics, numpy sampling), brute force,
or an invariant — chosen so a dropped term, wrong sign/index or transposed
operand in the oracle fails at least one of them.
"""
import json
import math
import os

import numpy as np
import pytest
from scipy.spatial.transform import Rotation
import scipy.special as sps

import gg_inputs as gi
import oracle

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))
PROJ_VIS, PROJ_U, PROJ_V, PROJ_A, PROJ_B, PROJ_C, PROJ_Z, PROJ_R = 0, 1, 2, 3, 4, 5, 6, 7
PROJ_X0, PROJ_X1, PROJ_Y0, PROJ_Y1, PROJ_COL, PROJ_O = 8, 9, 10, 11, slice(12, 15), 15


def render(scene, cams, e=0, **kw):
    os_ = oracle.OracleScene.from_inputs(scene)
    return oracle.render_env(os_, cams.viewmats[e], cams.intrinsics[e], cams.width, cams.height, **kw)


def sigma2_from_conic(row):
    A, B, C = float(row[PROJ_A]), float(row[PROJ_B]), float(row[PROJ_C])
    return np.linalg.inv(np.array([[A, B], [B, C]]))


# ---------------------------------------------------------------- O1 -------

def test_cov3_identity_and_isotropic():
    g = GOLD["isotropic_cov3"]
    s = gi.single_gaussian((0, 0, 5), g["s"], 0.5, (0.5, 0.5, 0.5))
    c32, c64 = oracle.OracleScene.from_inputs(s).cov3()
    assert np.allclose(c64[0], [g["expect_diag"], 0, 0, g["expect_diag"], 0, g["expect_diag"]], atol=1e-15)
    # isotropic under a random rotation: still s^2 I
    rng = np.random.default_rng(1)
    q = rng.normal(size=4)
    s2 = gi.single_gaussian((0, 0, 5), 0.3, 0.5, (0.5, 0.5, 0.5), quat=q)
    _, c = oracle.OracleScene.from_inputs(s2).cov3()
    assert np.allclose(c[0], [0.09, 0, 0, 0.09, 0, 0.09], atol=1e-14)


def test_cov3_matches_scipy_rotation():
    """Sigma3 = R diag(s^2) R^T with R from scipy (independent quaternion code)."""
    rng = np.random.default_rng(2)
    n = 200
    q = rng.normal(size=(n, 4)) * rng.uniform(0.2, 5.0, size=(n, 1))   # unnormalised
    sc = np.exp(rng.normal(-2, 1, size=(n, 3)))
    scene = gi.Scene(np.zeros((n, 3), np.float32), np.float32(sc), np.float32(q),
                     np.full(n, 0.5, np.float32), np.zeros((n, 1, 3), np.float32), 0)
    _, c64 = oracle.OracleScene.from_inputs(scene).cov3()
    q32 = np.float32(q).astype(np.float64)
    R = Rotation.from_quat(np.stack([q32[:, 1], q32[:, 2], q32[:, 3], q32[:, 0]], 1)).as_matrix()
    S = R @ (np.float32(sc).astype(np.float64)[:, :, None] ** 2 * np.eye(3)[None]) @ R.transpose(0, 2, 1)
    ref = np.stack([S[:, 0, 0], S[:, 0, 1], S[:, 0, 2], S[:, 1, 1], S[:, 1, 2], S[:, 2, 2]], 1)
    assert np.allclose(c64, ref, rtol=1e-10, atol=1e-14 * np.abs(ref).max())
    # eigenvalues are s^2
    for i in range(10):
        M = np.array([[c64[i, 0], c64[i, 1], c64[i, 2]], [c64[i, 1], c64[i, 3], c64[i, 4]],
                      [c64[i, 2], c64[i, 4], c64[i, 5]]])
        assert np.allclose(np.sort(np.linalg.eigvalsh(M)), np.sort(np.float32(sc[i]).astype(float) ** 2),
                           rtol=1e-9, atol=1e-15)


def test_cov3_sign_and_axis_swap():
    """q and -q give bit-identical f32 Sigma3; a 90 deg z-rotation swaps xx and yy."""
    base = dict(mean=(0, 0, 5), opacity=0.5, rgb=(0.5, 0.5, 0.5))
    s1 = gi.single_gaussian(scale=[0.1, 0.3, 0.2], quat=(0.3, -0.4, 0.5, 0.7), **base)
    s2 = gi.single_gaussian(scale=[0.1, 0.3, 0.2], quat=(-0.3, 0.4, -0.5, -0.7), **base)
    a, _ = oracle.OracleScene.from_inputs(s1).cov3()
    b, _ = oracle.OracleScene.from_inputs(s2).cov3()
    assert np.array_equal(a.view(np.uint32), b.view(np.uint32))
    h = math.sqrt(0.5)
    s3 = gi.single_gaussian(scale=[0.1, 0.3, 0.2], quat=(h, 0, 0, h), **base)
    _, c = oracle.OracleScene.from_inputs(s3).cov3()
    assert c[0, 0] == pytest.approx(0.09, rel=1e-6) and c[0, 3] == pytest.approx(0.01, rel=1e-6)
    assert c[0, 5] == pytest.approx(0.04, rel=1e-6)


# ---------------------------------------------------------------- O2 -------

def test_project_on_axis_golden():
    g = GOLD["project_on_axis"]
    gg = GOLD["isotropic_cov2_closed_form"]
    s = gi.single_gaussian(g["mean_cam"], gg["s"], 0.8, (0.2, 0.4, 0.6))
    cams = gi.identity_cameras(1, 64, 64, g["fx"], g["fy"], g["cx"], g["cy"])
    r = render(s, cams)
    p = r.proj[0]
    assert p[PROJ_VIS] == 1
    assert (p[PROJ_U], p[PROJ_V]) == tuple(g["expect_uv"])
    S2 = sigma2_from_conic(p)
    assert S2[0, 0] == pytest.approx(gg["expect_a"], rel=1e-6)
    assert S2[1, 1] == pytest.approx(gg["expect_a"], rel=1e-6)
    assert abs(S2[0, 1]) < 1e-9
    assert int(p[PROJ_R]) == gg["expect_r"]
    assert [int(p[PROJ_X0]), int(p[PROJ_X1])] == gg["expect_x_tiles_on_64_wide"]
    assert p[PROJ_Z] == 5.0


def test_project_mean_matches_pinhole():
    """u,v = K (R mu + t) / z for random points and real room cameras."""
    sc = gi.room_scene(3, 4000, 0, L=12.0, stairs=True)
    cams = gi.cameras(3, 3, 640, 480, sc)
    os_ = oracle.OracleScene.from_inputs(sc)
    for e in range(3):
        r = oracle.render_env(os_, cams.viewmats[e], cams.intrinsics[e], 640, 480)
        V = cams.viewmats[e].astype(np.float64)
        fx, fy, cx, cy = cams.intrinsics[e].astype(np.float64)
        p = sc.means.astype(np.float64) @ V[:3, :3].T + V[:3, 3]
        vis = r.proj[:, PROJ_VIS] == 1
        assert vis.sum() > 100
        assert np.all(p[vis, 2] > 0.01)
        u = fx * p[vis, 0] / p[vis, 2] + cx
        v = fy * p[vis, 1] / p[vis, 2] + cy
        # f32 canonical vs f64: error grows as p_z -> near; compare where z > 0.3
        far = p[vis, 2] > 0.3
        assert far.sum() > 100
        assert np.allclose(r.proj[vis, PROJ_U][far], u[far], rtol=1e-5, atol=2e-3)
        assert np.allclose(r.proj[vis, PROJ_V][far], v[far], rtol=1e-5, atol=2e-3)
        assert np.allclose(r.proj[vis, PROJ_U], u, rtol=1e-3)
        assert np.allclose(r.proj[vis, PROJ_Z], p[vis, 2], rtol=1e-6, atol=4e-6)
        # everything in front and on screen (centre inside) is visible
        inside = (p[:, 2] > 0.05)
        uu = fx * p[:, 0] / np.where(inside, p[:, 2], 1) + cx
        vv = fy * p[:, 1] / np.where(inside, p[:, 2], 1) + cy
        on = inside & (uu > 1) & (uu < 639) & (vv > 1) & (vv < 479)
        assert np.all(vis[on])
        # behind the near plane never visible
        assert not np.any(vis[p[:, 2] <= 0.0])


NEAR32, FAR32 = np.float32(0.01), np.float32(100.0)


def near_far_fixture():
    """Gaussians on the optical axis of an identity camera at the cull
    boundaries.  With R = I, t = 0 the canonical p_z = ((0 mu_x + 0 mu_y) +
    1 mu_z) + 0 is mu_z exactly, so each z below is the f32 value the
    predicate p_z <= near or p_z > far sees."""
    zs = [np.nextafter(NEAR32, np.float32(0)), NEAR32, np.nextafter(NEAR32, np.float32(1)),
          np.float32(5.0), FAR32, np.nextafter(FAR32, np.float32(1e9)), np.float32(-1.0)]
    expect = [False, False, True, True, True, False, False]
    gs = [gi.single_gaussian([0.0, 0.0, float(z)], max(1e-3, float(z) * 1e-2) if z > 0 else 0.01, 0.8,
                             [0.5, 0.5, 0.5]) for z in zs]
    return gi.concat(gs), np.array(expect), np.array(zs, np.float32)


def test_near_far_cull_boundaries():
    """Visible iff near < p_z <= far, decided on the f32 value: z = near and
    nextafter(near, 0) are culled, nextafter(near, +inf) is kept; z = far is
    kept, nextafter(far, +inf) culled; behind the camera culled."""
    sc, expect, zs = near_far_fixture()
    assert sc.means[:, 2].tobytes() == zs.tobytes()
    cams = gi.identity_cameras(1, 64, 48, 32.0)
    os_ = oracle.OracleScene.from_inputs(sc)
    r = oracle.render_env(os_, cams.viewmats[0], cams.intrinsics[0], 64, 48, near=float(NEAR32), far=float(FAR32))
    vis = r.proj[:, PROJ_VIS] == 1
    assert vis.tolist() == expect.tolist()
    assert np.all(r.tile_counts[expect] > 0) and np.all(r.tile_counts[~expect] == 0)
    assert np.array_equal(r.proj[expect, PROJ_Z], zs[expect])     # depth bits = mu_z
    # shifting the planes by one ulp flips exactly the boundary Gaussians
    r2 = oracle.render_env(os_, cams.viewmats[0], cams.intrinsics[0], 64, 48,
                           near=float(np.nextafter(NEAR32, np.float32(0))), far=float(np.nextafter(FAR32, np.float32(0))))
    vis2 = r2.proj[:, PROJ_VIS] == 1
    assert vis2.tolist() == [False, True, True, True, False, False, False]


def test_cov2_monte_carlo():
    """cov2d within 2% Frobenius of 1e5 Monte-Carlo projected
    samples (s/z <= 0.02), dilation removed.  Samples use scipy's rotation."""
    rng = np.random.default_rng(7)
    for trial in range(6):
        z = rng.uniform(3, 6)
        mean = np.array([rng.uniform(-0.8, 0.8), rng.uniform(-0.6, 0.6), z])
        sc = rng.uniform(0.2, 1.0, 3) * 0.02 * z / 1.0
        sc = np.minimum(sc, 0.02 * z)
        q = rng.normal(size=4)
        s = gi.single_gaussian(mean, sc, 0.5, (0.5, 0.5, 0.5), quat=q)
        cams = gi.identity_cameras(1, 200, 160, 180.0, 170.0, 100.0, 80.0)
        r = render(s, cams)
        assert r.proj[0, PROJ_VIS] == 1
        S2 = sigma2_from_conic(r.proj[0]) - 0.3 * np.eye(2)
        qf = np.float32(q).astype(float)
        R = Rotation.from_quat([qf[1], qf[2], qf[3], qf[0]]).as_matrix()
        L = R @ np.diag(np.float32(sc).astype(float))
        X = mean + rng.normal(size=(100_000, 3)) @ L.T
        uv = np.stack([180.0 * X[:, 0] / X[:, 2] + 100.0, 170.0 * X[:, 1] / X[:, 2] + 80.0], 1)
        emp = np.cov(uv.T)
        assert np.linalg.norm(emp - S2) / np.linalg.norm(emp) < 0.02, trial


def _fd_jacobian(p, fx, fy, h=1e-6):
    def proj(q):
        return np.array([fx * q[0] / q[2], fy * q[1] / q[2]])
    J = np.zeros((2, 3))
    for k in range(3):
        e = np.zeros(3)
        e[k] = h
        J[:, k] = (proj(p + e) - proj(p - e)) / (2 * h)
    return J


def test_jacobian_finite_difference_mode_b():
    """Mode B (f64): Sigma2 - 0.3I == J_fd W Sigma3 W^T J_fd^T for on-screen
    Gaussians (Jacobian clamp inactive), J_fd by central differences."""
    rng = np.random.default_rng(11)
    sc = gi.random_cloud(5, 64)
    cams = gi.cloud_cameras(5, 2)
    os_ = oracle.OracleScene.from_inputs(sc)
    _, c64 = os_.cov3()
    checked = 0
    for e in range(2):
        r = oracle.render_env(os_, cams.viewmats[e], cams.intrinsics[e], 64, 64, mode=oracle.MODE_B)
        V = cams.viewmats[e].astype(np.float64)
        fx, fy = cams.intrinsics[e, :2].astype(np.float64)
        for i in range(sc.n):
            if r.proj[i, PROJ_VIS] != 1:
                continue
            p = V[:3, :3] @ sc.means[i].astype(np.float64) + V[:3, 3]
            if not (0 < r.proj[i, PROJ_U] < 64 and 0 < r.proj[i, PROJ_V] < 64):
                continue
            Jf = _fd_jacobian(p, fx, fy)
            S3 = np.array([[c64[i, 0], c64[i, 1], c64[i, 2]], [c64[i, 1], c64[i, 3], c64[i, 4]],
                           [c64[i, 2], c64[i, 4], c64[i, 5]]])
            T = Jf @ V[:3, :3]
            ref = T @ S3 @ T.T + 0.3 * np.eye(2)
            got = sigma2_from_conic(r.proj[i])   # conic stored as f32: rel ~1e-7
            assert np.allclose(got, ref, rtol=2e-5, atol=1e-6 * np.abs(ref).max()), (e, i)
            checked += 1
    assert checked > 20
    del rng


def test_jacobian_clamp_offscreen():
    """Reading R4: far off-screen Gaussians use the clamped x' (gsplat form);
    the on-screen part of the Jacobian is unchanged."""
    W, H, f = 64, 64, 64.0
    cams = gi.identity_cameras(1, W, H, f)
    z = 2.0
    lim = (W - W / 2) / f + 0.3 * (0.5 * W / f)       # 0.65
    x = 3.0 * z                                       # tx = 3 >> lim
    s = gi.single_gaussian((x, 0, z), [0.5, 0.5, 0.5], 0.9, (0.5, 0.5, 0.5))
    r = render(s, cams, mode=oracle.MODE_B)
    p = r.proj[0]
    # centre far right of the image -> culled by the rect unless r is large
    S2 = None if p[PROJ_VIS] != 1 else sigma2_from_conic(p)
    # closed form with clamped x' = lim*z
    J = np.array([[f / z, 0, -f * (lim * z) / z ** 2], [0, f / z, 0]])
    ref = J @ (0.25 * np.eye(3)) @ J.T + 0.3 * np.eye(2)
    if S2 is not None:
        assert np.allclose(S2, ref, rtol=1e-5)
    # a visible variant: big Gaussian just outside the right edge
    # just past the clamp (tx = 0.7 > 0.65): J uses x' = 0.65 z
    s2 = gi.single_gaussian((0.7 * z, 0, z), [0.5, 0.5, 0.5], 0.9, (0.5, 0.5, 0.5))
    r2 = render(s2, cams, mode=oracle.MODE_B)
    assert r2.proj[0, PROJ_VIS] == 1
    J2 = np.array([[f / z, 0, -f * (lim * z) / z ** 2], [0, f / z, 0]])
    ref2 = J2 @ (0.25 * np.eye(3)) @ J2.T + 0.3 * np.eye(2)
    assert np.allclose(sigma2_from_conic(r2.proj[0]), ref2, rtol=1e-5)
    # inside the clamp (tx = 0.6): unclamped J
    s3 = gi.single_gaussian((0.6 * z, 0, z), [0.5, 0.5, 0.5], 0.9, (0.5, 0.5, 0.5))
    r3 = render(s3, cams, mode=oracle.MODE_B)
    J3 = np.array([[f / z, 0, -f * (0.6 * z) / z ** 2], [0, f / z, 0]])
    ref3 = J3 @ (0.25 * np.eye(3)) @ J3.T + 0.3 * np.eye(2)
    assert np.allclose(sigma2_from_conic(r3.proj[0]), ref3, rtol=1e-5)


def test_radius_closed_form_sweep():
    """Isotropic on-axis: lambda1 = sigma^2 + sqrt(0.1) (reading R6), r = ceil(3 sqrt(lambda1))."""
    cams = gi.identity_cameras(1, 256, 256, 100.0, cx=128, cy=128)
    for s in np.linspace(0.001, 0.6, 37):
        sig2 = (100.0 * float(np.float32(s)) / 5.0) ** 2 + 0.3
        lam = sig2 + math.sqrt(0.1)
        x = 3 * math.sqrt(lam)
        if abs(x - round(x)) < 1e-4:
            continue
        r = render(gi.single_gaussian((0, 0, 5), s, 0.5, (0.5, 0.5, 0.5)), cams)
        assert int(r.proj[0, PROJ_R]) == math.ceil(x), s
    # zero-ish scale -> Sigma2 = 0.3 I -> r = ceil(3 sqrt(0.3 + 0.316)) = 3
    r = render(gi.single_gaussian((0, 0, 5), 1e-9, 0.5, (0.5, 0.5, 0.5)), cams)
    assert int(r.proj[0, PROJ_R]) == 3


def test_rect_brute_force_and_tile_counts():
    """SPEC.md:144 per-tile sets == brute-force footprint-intersection scan;
    tile counts == rect area; culled Gaussians count 0."""
    sc = gi.random_cloud(9, 400)
    cams = gi.cloud_cameras(9, 3, 70, 50)            # partial edge tiles
    os_ = oracle.OracleScene.from_inputs(sc)
    for e in range(3):
        r = oracle.render_env(os_, cams.viewmats[e], cams.intrinsics[e], 70, 50)
        TX, TY = 5, 4
        members = {t: set() for t in range(TX * TY)}
        for i in range(sc.n):
            p = r.proj[i]
            if p[PROJ_VIS] != 1:
                assert r.tile_counts[i] == 0
                continue
            u, v, rr = float(p[PROJ_U]), float(p[PROJ_V]), float(p[PROJ_R])
            cnt = 0
            for ty in range(TY):
                for tx in range(TX):
                    if 16 * tx < u + rr and 16 * tx + 16 > u - rr and 16 * ty < v + rr and 16 * ty + 16 > v - rr:
                        members[ty * TX + tx].add(i)
                        cnt += 1
            assert cnt == r.tile_counts[i] > 0
        for t in range(TX * TY):
            a, b = r.ranges[t]
            assert set(r.sorted_gid[a:b].tolist()) == members[t]
            assert np.all(r.sorted_tile[a:b] == t)


def test_sorted_lists_independent_lexsort():
    """O3 order == numpy lexsort on (tile, f32 depth bits, gid) of brute-force pairs."""
    sc = gi.random_cloud(12, 300)
    sc.means[7] = sc.means[3]          # exact depth tie (duplicate)
    sc.means[8] = sc.means[3]
    cams = gi.cloud_cameras(12, 1)
    r = render(sc, cams)
    pairs = []
    for i in range(sc.n):
        p = r.proj[i]
        if p[PROJ_VIS] != 1:
            continue
        zb = np.float32(p[PROJ_Z]).view(np.uint32)
        for ty in range(int(p[PROJ_Y0]), int(p[PROJ_Y1])):
            for tx in range(int(p[PROJ_X0]), int(p[PROJ_X1])):
                pairs.append((ty * 4 + tx, int(zb), i))
    pairs = np.array(pairs, dtype=np.int64)
    order = np.lexsort((pairs[:, 2], pairs[:, 1], pairs[:, 0]))
    assert np.array_equal(r.sorted_tile, pairs[order, 0])
    assert np.array_equal(r.sorted_zbits.astype(np.int64), pairs[order, 1])
    assert np.array_equal(r.sorted_gid, pairs[order, 2])


def test_bin_full_image_and_depth_order_golden():
    g = GOLD["bin_full_image"]
    cams = gi.identity_cameras(1, g["width"], g["height"], 32.0)
    big = gi.single_gaussian((0, 0, 3), 2.0, 0.5, (0.5, 0.5, 0.5))
    r = render(big, cams)
    assert r.tile_counts[0] == g["expect_tiles"]
    assert np.all(r.ranges[:, 1] - r.ranges[:, 0] == 1)
    d = GOLD["bin_depth_order"]["depths"]
    two = gi.concat([gi.single_gaussian((0, 0, d[0]), 1.0, 0.5, (1, 0, 0)),
                     gi.single_gaussian((0, 0, d[1]), 0.5, 0.5, (0, 1, 0))])
    r = render(two, cams)
    for t in range(4):
        a, b = r.ranges[t]
        assert list(r.sorted_gid[a:b]) == [1, 0]


# ---------------------------------------------------------------- colour ---

def test_dc_colour_decodes_albedo():
    """DC -> RGB via 0.2820948 c + 0.5 (clamped).  The generator
    encodes albedo with 2 sqrt(pi) = 1/C0; decoding must return it."""
    rng = np.random.default_rng(3)
    rgb = rng.uniform(0, 1, 3)
    s = gi.single_gaussian((0, 0, 4), 0.05, 0.9, rgb)
    r = render(s, gi.identity_cameras(1, 32, 32, 32.0))
    assert np.allclose(r.proj[0, PROJ_COL], rgb, atol=1e-6)
    # clamp: out-of-range DC
    s.sh[0, 0] = [10.0, -10.0, 0.0]
    r = render(s, gi.identity_cameras(1, 32, 32, 32.0))
    assert np.allclose(r.proj[0, PROJ_COL], [1.0, 0.0, 0.5], atol=1e-7)


def _real_sh_scipy(l, m, theta, phi):
    if m < 0:
        return math.sqrt(2) * sps.sph_harm_y(l, -m, theta, phi).imag
    if m == 0:
        return sps.sph_harm_y(l, 0, theta, phi).real
    return math.sqrt(2) * sps.sph_harm_y(l, m, theta, phi).real


def test_sh_basis_orthonormal_quadrature():
    """The 16 basis functions are orthonormal over S^2 (Gauss-Legendre x
    uniform-phi quadrature, exact for these polynomials)."""
    xs, ws = np.polynomial.legendre.leggauss(12)
    nphi = 24
    G = np.zeros((16, 16))
    for ct, w in zip(xs, ws):
        st = math.sqrt(1 - ct * ct)
        for k in range(nphi):
            ph = 2 * math.pi * k / nphi
            Y = oracle.sh_basis(3, [st * math.cos(ph), st * math.sin(ph), ct])
            G += w * (2 * math.pi / nphi) * np.outer(Y, Y)
    assert np.allclose(G, np.eye(16), atol=1e-12)


def test_sh_basis_matches_scipy_legendre():
    """Signs/indices vs scipy's associated-Legendre SH with the 3DGS real
    convention (-1)^m (k = l^2 + l + m)."""
    rng = np.random.default_rng(5)
    for _ in range(50):
        th, ph = math.acos(rng.uniform(-1, 1)), rng.uniform(0, 2 * math.pi)
        Y = oracle.sh_basis(3, [math.sin(th) * math.cos(ph), math.sin(th) * math.sin(ph), math.cos(th)])
        ref = [_real_sh_scipy(l, m, th, ph) for l in range(4) for m in range(-l, l + 1)]
        assert np.allclose(Y, ref, atol=1e-12)
    # dir = +z: only m = 0 terms survive
    Y = oracle.sh_basis(3, [0, 0, 1])
    nz = [k for k in range(16) if abs(Y[k]) > 1e-15]
    assert nz == [0, 2, 6, 12]


def test_sh_colour_view_dependent():
    """Rendered colour (d=3) == clamp(0.5 + sum_k Y_k(dir) f_k) with Y from
    scipy, dir = unit(mu - camera centre) in the world frame."""
    sc = gi.random_cloud(21, 40, sh_degree=3)
    cams = gi.cloud_cameras(21, 2)
    os_ = oracle.OracleScene.from_inputs(sc)
    n_ok = 0
    for e in range(2):
        V = cams.viewmats[e].astype(np.float64)
        Cc = -V[:3, :3].T @ V[:3, 3]
        for deg in (1, 2, 3):
            r = oracle.render_env(os_, cams.viewmats[e], cams.intrinsics[e], 64, 64, sh_degree=deg)
            for i in range(sc.n):
                if r.proj[i, PROJ_VIS] != 1:
                    continue
                d = sc.means[i].astype(np.float64) - Cc
                d /= np.linalg.norm(d)
                th, ph = math.acos(np.clip(d[2], -1, 1)), math.atan2(d[1], d[0])
                Y = np.array([_real_sh_scipy(l, m, th, ph) for l in range(deg + 1) for m in range(-l, l + 1)])
                ref = np.clip(0.5 + Y @ sc.sh[i, :len(Y)].astype(np.float64), 0, 1)
                assert np.allclose(r.proj[i, PROJ_COL], ref, atol=1e-6)
                n_ok += 1
    assert n_ok > 50


# ---------------------------------------------------------------- O4/O5 ----

def test_empty_scene_background():
    g = GOLD["empty_scene"]
    s = gi.single_gaussian((0, 0, -5), 0.05, 0.8, (0.2, 0.4, 0.6))   # behind the camera
    r = render(s, gi.identity_cameras(1, 32, 32, 32.0), background=(0.1, 0.2, 0.3))
    assert np.all(r.alpha == g["expect_alpha"]) and np.all(r.depth == g["expect_depth"])
    assert np.allclose(r.rgb, [0.1, 0.2, 0.3], atol=0)
    assert len(r.sorted_gid) == 0


def test_single_gaussian_closed_form():
    g = GOLD["single_gaussian_footprint"]
    pk = GOLD["single_gaussian_peak"]
    c = np.array([0.2, 0.4, 0.6])
    bg = np.array([0.3, 0.1, 0.9])
    s = gi.single_gaussian((0, 0, 5), 0.05, pk["opacity"], c)
    cams = gi.identity_cameras(1, 64, 64, 100.0, cx=32, cy=32)
    r = render(s, cams)
    assert (r.alpha > 0).sum() == g["expect_nonbg_pixels"]
    assert r.alpha[32, 32] == pytest.approx(g["expect_alpha_half_offset"], abs=1e-5)
    # full closed form over the rect tiles: alpha = min(.99, o exp(-|p-mu|^2/(2 sig^2)))
    sig2 = float(np.float32(1.3000002))   # a = (f s / z)^2 + 0.3 in f32
    yy, xx = np.mgrid[0:64, 0:64] + 0.5
    a = np.minimum(0.99, 0.8 * np.exp(-((xx - 32) ** 2 + (yy - 32) ** 2) / (2 * sig2)))
    a[a < 1 / 255] = 0
    inrect = (xx >= 16) & (xx < 48) & (yy >= 16) & (yy < 48)
    a[~inrect] = 0
    assert np.allclose(r.alpha, a, atol=1e-6)
    # pixel at the mean (cx = 32.5): alpha = o, C = o c + (1-o) bg, D = z
    cams2 = gi.identity_cameras(1, 64, 64, 100.0, cx=32.5, cy=32.5)
    r2 = render(s, cams2, background=tuple(bg))
    assert r2.alpha[32, 32] == pytest.approx(pk["expect_alpha"], abs=1e-6)
    assert np.allclose(r2.rgb[32, 32], pk["expect_color_weight"] * np.float32(c) + pk["expect_bg_weight"] * bg,
                       atol=1e-6)
    assert r2.depth[32, 32] == 5.0


def test_two_gaussians_expansion():
    c1, c2, bg = np.array([1.0, 0.2, 0.1]), np.array([0.1, 0.9, 0.3]), np.array([0.05, 0.1, 0.2])
    two = gi.concat([gi.single_gaussian((0, 0, 3), 0.5, 0.6, c2),     # back (gid 0)
                     gi.single_gaussian((0, 0, 2), 0.5, 0.7, c1)])    # front (gid 1)
    cams = gi.identity_cameras(1, 32, 32, 16.0, cx=16.5, cy=16.5)
    r = render(two, cams, background=tuple(bg))
    a1, a2 = float(np.float32(0.7)), float(np.float32(0.6))
    C = a1 * c1 + (1 - a1) * a2 * c2 + (1 - a1) * (1 - a2) * bg
    D = (a1 * 2 + (1 - a1) * a2 * 3) / (a1 + (1 - a1) * a2)
    assert np.allclose(r.rgb[16, 16], C, atol=1e-6)
    assert r.depth[16, 16] == pytest.approx(D, rel=1e-7)
    assert r.alpha[16, 16] == pytest.approx(a1 + (1 - a1) * a2, rel=1e-7)


def test_early_out_stack_golden():
    g = GOLD["early_out_stack"]
    parts = [gi.single_gaussian((0, 0, 2 + 0.1 * k), 0.3, g["opacity"], (1.0, 1.0, 1.0)) for k in range(6)]
    cams = gi.identity_cameras(1, 32, 32, 16.0, cx=16.5, cy=16.5)
    r = render(gi.concat(parts), cams)
    op = float(np.float32(g["opacity"]))
    assert r.n_contrib[16, 16] == g["expect_blended"]
    assert r.n_eval[16, 16] == g["expect_blended"] + 1          # the stopping Gaussian is visited
    w = [op, (1 - op) * op, (1 - op) ** 2 * op]
    assert np.allclose(w, g["expect_weights"], rtol=1e-6)
    assert r.alpha[16, 16] == pytest.approx(sum(w), rel=1e-12)
    T_final = 1 - r.alpha[16, 16]
    assert T_final == pytest.approx(g["expect_T_final"], rel=1e-5)
    # no early-out diagnostic: the skipped tail is bounded by the remaining
    # transmittance T_final = 1 - alpha per pixel (colours <= 1, bg = 0)
    r2 = render(gi.concat(parts), cams, flags=oracle.F_NO_EARLY_OUT)
    assert np.all(np.abs(r2.rgb - r.rgb) <= (1 - r.alpha)[..., None] + 1e-12)


# ---------------------------------------------------------------- drivers / invariants

@pytest.mark.parametrize("seed", range(6))
def test_plain_equals_binned_bit_exact(seed):
    sc = gi.random_cloud(100 + seed, 256, sh_degree=seed % 4)
    cams = gi.cloud_cameras(100 + seed, 1, 70 if seed % 2 else 64, 50 if seed % 2 else 64)
    a = render(sc, cams)
    b = render(sc, cams, flags=oracle.F_PLAIN)
    for f in ("rgb", "depth", "alpha", "n_eval", "n_contrib"):
        assert np.array_equal(getattr(a, f), getattr(b, f)), f


def test_invariants_random_scenes():
    """T non-increasing => alpha in [0,1]; alpha == 1 - T_final (bg difference);
    depth within the visible depth range; no-early-out within T_final."""
    for seed in range(5):
        sc = gi.random_cloud(200 + seed, 512)
        cams = gi.cloud_cameras(200 + seed, 1)
        r0 = render(sc, cams)
        r1 = render(sc, cams, background=(1.0, 1.0, 1.0))
        assert np.all(r0.alpha >= 0) and np.all(r0.alpha <= 1 + 1e-12)
        T = r1.rgb[..., 0] - r0.rgb[..., 0]
        assert np.allclose(r0.alpha, 1 - T, atol=1e-12)
        zs = r0.proj[r0.proj[:, 0] == 1, PROJ_Z]
        m = r0.alpha > 0
        assert np.all(r0.depth[m] >= zs.min() - 1e-9) and np.all(r0.depth[m] <= zs.max() + 1e-9)
        assert np.all(r0.depth[~m] == 0)
        r2 = render(sc, cams, flags=oracle.F_NO_EARLY_OUT)
        assert np.all(np.abs(r2.rgb - r0.rgb) <= (1 - r0.alpha)[..., None] + 1e-12)


def test_zero_opacity_insertion_invariance():
    sc = gi.random_cloud(31, 200)
    cams = gi.cloud_cameras(31, 1)
    r0 = render(sc, cams)
    extra = gi.random_cloud(32, 50)
    extra.opacities[:] = 0.0
    both = gi.concat([sc, extra])
    r1 = render(both, cams)
    assert np.array_equal(r0.rgb, r1.rgb) and np.array_equal(r0.depth, r1.depth)
    assert len(r1.sorted_gid) > len(r0.sorted_gid)


def test_permutation_invariance():
    sc = gi.random_cloud(41, 300)
    cams = gi.cloud_cameras(41, 1)
    r0 = render(sc, cams)
    zb = r0.proj[r0.proj[:, 0] == 1, PROJ_Z]
    assert len(np.unique(zb)) == len(zb)
    perm = np.random.default_rng(0).permutation(sc.n)
    sp = gi.Scene(sc.means[perm], sc.scales[perm], sc.quats[perm], sc.opacities[perm], sc.sh[perm], 0)
    r1 = render(sp, cams)
    assert np.array_equal(r0.rgb, r1.rgb) and np.array_equal(r0.depth, r1.depth)
    assert np.array_equal(perm[r1.sorted_gid], r0.sorted_gid)


def test_translation_equivariance_mode_b():
    """SPEC.md:177 shifting scene and camera by the same offset leaves the
    image unchanged (1e-5) — f64 projection (mode B), non-exempt pixels."""
    sc = gi.random_cloud(51, 300)
    cams = gi.cloud_cameras(51, 1)
    r0 = render(sc, cams, mode=oracle.MODE_B)
    d = np.array([0.37, -0.21, 0.13])
    sc2 = gi.Scene(np.float32(sc.means.astype(np.float64) + d), sc.scales, sc.quats, sc.opacities, sc.sh, 0)
    V = cams.viewmats.astype(np.float64).copy()
    V[0, :3, 3] -= V[0, :3, :3] @ d
    cams2 = gi.Cameras(np.float32(V), cams.intrinsics, cams.width, cams.height)
    r1 = render(sc2, cams2, mode=oracle.MODE_B)
    ok = ~(r0.exempt | r1.exempt)
    assert np.max(np.abs(r0.rgb - r1.rgb)[ok]) < 1e-5


def test_round_robin_golden():
    g = GOLD["round_robin"]
    assert list(gi.round_robin(4, 2)) == g["two_four"]
    assert np.all(np.bincount(gi.round_robin(4096, 128)) == g["per_scene_128_4096"])


def test_u8_quantisation_round_half_even():
    # O5: round-half-even(clamp(x)*255); 0.5/255 -> 0, 1.5/255 -> 2
    cams = gi.identity_cameras(1, 16, 16, 16.0)
    s = gi.single_gaussian((0, 0, -1), 0.05, 0.8, (0.2, 0.4, 0.6))   # culled: pure background
    for bgv, want in ((0.5 / 255, 0), (1.5 / 255, 2), (2.5 / 255, 2), (-0.3, 0), (1.7, 255)):
        r = render(s, cams, background=(bgv, bgv, bgv))
        assert np.all(r.rgb8 == want), bgv
