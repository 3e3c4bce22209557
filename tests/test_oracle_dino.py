"""Pins for the oracle's DinoV2-input conversion (reading R36):
closed forms and a library routine that implements the same resampling."""
import numpy as np

import oracle as orc

MEAN = np.array(orc.IMAGENET_MEAN)[:, None, None]
STD = np.array(orc.IMAGENET_STD)[:, None, None]


def test_constant_image():
    img = np.zeros((480, 640, 3), np.uint8)
    img[:] = (17, 128, 250)
    out = orc.dino_input(img)
    expect = (np.array([17, 128, 250])[:, None, None] / 255.0 - MEAN) / STD
    assert out.shape == (3, 224, 224)
    assert np.allclose(out, np.broadcast_to(expect, out.shape), rtol=0, atol=1e-12)


def test_same_size_is_identity():
    g = np.random.default_rng(3)
    img = g.integers(0, 256, (224, 224, 3), dtype=np.uint8)
    out = orc.dino_input(img)
    expect = (img.transpose(2, 0, 1) / 255.0 - MEAN) / STD
    assert np.allclose(out, expect, rtol=0, atol=1e-12)


def test_affine_image_closed_form():
    # v(x) = x on a 256-wide frame: bilinear interpolation of an affine image
    # is exact, so column d of the output is (src(d)/255 - mean)/std with the
    # half-pixel source coordinate src(d) = (d + 0.5) * 256/224 - 0.5 (no clamp
    # is reached: src(0) > 0, src(223) < 255).  A half-pixel or scale error fails.
    W, H = 256, 60
    img = np.zeros((H, W, 3), np.uint8)
    img[:, :, 1] = np.arange(W, dtype=np.uint8)[None, :]
    out = orc.dino_input(img)
    src = (np.arange(224) + 0.5) * (W / 224) - 0.5
    expect = (src / 255.0 - MEAN[1, 0, 0]) / STD[1, 0, 0]
    assert np.allclose(out[1], np.broadcast_to(expect, (224, 224)), rtol=0, atol=1e-12)
    assert np.allclose(out[0], (0.0 - MEAN[0, 0, 0]) / STD[0, 0, 0], rtol=0, atol=1e-12)


def test_matches_torch_bilinear():
    import torch
    g = np.random.default_rng(5)
    for (H, W) in ((480, 640), (50, 70), (240, 320)):
        img = g.integers(0, 256, (H, W, 3), dtype=np.uint8)
        t = torch.from_numpy(img.astype(np.float64) / 255.0).permute(2, 0, 1)[None]
        r = torch.nn.functional.interpolate(t, size=(224, 224), mode="bilinear", align_corners=False,
                                            antialias=False)[0].numpy()
        expect = (r - MEAN) / STD
        assert np.allclose(orc.dino_input(img), expect, rtol=0, atol=1e-9)
