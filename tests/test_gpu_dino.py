"""Render -> DinoV2 input on the GPU vs the oracle (R36), -m gpu.
Tolerance: one bf16 ulp (2^-7 relative): the kernel rounds its f32 value and
the oracle's f64 value may sit on the other side of a bf16 rounding boundary."""
import numpy as np
import pytest

import gg_inputs as gi
import oracle
from test_gpu_parity import dev, load, render

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


def _check(gg, R, rgb_u8, S):
    E, H, W = rgb_u8.shape[:3]
    out = torch.zeros((E, 3, S, S), dtype=torch.bfloat16, device="cuda")
    gg.gg_dino_input(R.ctx, E, W, H, dev(rgb_u8), S, out)
    torch.cuda.synchronize()
    got = out.float().cpu().numpy()
    for e in range(E):
        ref = oracle.dino_input(rgb_u8[e], S)
        err = np.abs(got[e] - ref)
        assert np.all(err <= np.abs(ref) * 2.0 ** -7 + 1e-5), float(err.max())
        # and almost everywhere within half an ulp (round-to-nearest of the same value)
        assert np.mean(err <= np.abs(ref) * 2.0 ** -8 + 1e-6) > 0.999


def test_dino_input_rendered_frames(gg, R):
    sc = gi.config_scene("c1")
    cams = gi.config_cameras("c1", sc, n_envs=3)
    cams.width, cams.height = 640, 480
    cams.intrinsics[:] = gi.pinhole(640, 480)
    sid = load(R, sc)
    rgb, _, _ = render(gg, R, [sid] * 3, cams)
    _check(gg, R, rgb, 224)


def test_dino_input_random_sizes(gg, R):
    g = np.random.default_rng(11)
    for (H, W, S) in ((50, 70, 224), (480, 640, 112), (224, 224, 224)):
        _check(gg, R, g.integers(0, 256, (2, H, W, 3), dtype=np.uint8), S)


def test_dino_input_errors(gg, R):
    with pytest.raises(gg.GGError):
        gg.gg_dino_input(R.ctx, 0, 64, 64, None, 224, None)
