"""Native 3DGS PLY reader (gg_read_ply), CPU only."""
import math
import struct

import numpy as np
import pytest

import gg_inputs as gi


@pytest.fixture(scope="module")
def gg():
    import paper_2510_15352_b200 as m
    m.load_library()
    return m


def _write(path, names, rows, fmt="binary_little_endian"):
    with open(path, "wb") as f:
        f.write(f"ply\nformat {fmt} 1.0\nelement vertex {len(rows)}\n".encode())
        for n in names:
            f.write(f"property float {n}\n".encode())
        f.write(b"end_header\n")
        for r in rows:
            f.write(struct.pack("<%df" % len(r), *r))


BASE = ["x", "y", "z", "f_dc_0", "f_dc_1", "f_dc_2", "opacity", "scale_0", "scale_1", "scale_2",
        "rot_0", "rot_1", "rot_2", "rot_3"]


def test_three_splat_fixture_and_spec_examples(gg, tmp_path):
    # hand-written fixture: logit 0 -> 0.5, log(0.01) -> 0.01
    rows = [[0.0, 1.0, 2.0, 0.1, 0.2, 0.3, 0.0, math.log(0.01), math.log(0.02), math.log(0.03), 1, 0, 0, 0],
            [-1.5, 0.25, 4.0, -0.5, 0.0, 0.5, 2.0, 0.0, -1.0, -2.0, 0.5, 0.5, 0.5, 0.5],
            [3.0, -2.0, 0.5, 1.0, 1.0, 1.0, -3.0, -4.0, -4.0, -4.0, 0, 0, 0, 2]]
    p = tmp_path / "three.ply"
    _write(p, BASE, rows)
    m, s, q, o, sh, d = gg.gg_read_ply(str(p))
    r = np.array(rows, np.float32).astype(np.float64)
    assert d == 0 and m.shape == (3, 3)
    assert np.array_equal(m, np.float32(r[:, 0:3]))
    assert np.array_equal(sh[:, 0, :], np.float32(r[:, 3:6]))
    assert o[0] == 0.5
    assert np.allclose(o, 1 / (1 + np.exp(-r[:, 6])), rtol=1e-7)
    assert s[0, 0] == pytest.approx(0.01, rel=1e-6)
    assert np.allclose(s, np.exp(r[:, 7:10]), rtol=1e-6)
    assert np.array_equal(q, np.float32(r[:, 10:14]))


def test_roundtrip_sh3_channel_major(gg, tmp_path):
    sc = gi.random_cloud(5, 40, sh_degree=3)
    p = tmp_path / "s.ply"
    gi.write_3dgs_ply(str(p), sc)
    m, s, q, o, sh, d = gg.gg_read_ply(str(p))
    assert d == 3
    assert np.array_equal(m, sc.means)
    assert np.allclose(s, sc.scales, rtol=2e-6)
    assert np.allclose(o, np.clip(sc.opacities, 1e-7, 1 - 1e-7), rtol=1e-5, atol=1e-6)
    assert np.array_equal(sh, sc.sh)          # coefficient k of channel c came from f_rest[c*15 + k-1]
    assert np.array_equal(q, sc.quats)


def test_errors(gg, tmp_path):
    p = tmp_path / "bad.ply"
    _write(p, [n for n in BASE if n != "opacity"], [[0.0] * 13])
    with pytest.raises(gg.GGError, match="opacity"):
        gg.gg_read_ply(str(p))
    _write(p, BASE, [])
    with pytest.raises(gg.GGError, match="empty"):
        gg.gg_read_ply(str(p))
    rows = [[0.0] * 14, [0.0, float("nan")] + [0.0] * 12]
    _write(p, BASE, rows)
    with pytest.raises(gg.GGError, match="record 1"):
        gg.gg_read_ply(str(p))
    _write(p, BASE, [[0.0] * 14], fmt="ascii")
    with pytest.raises(gg.GGError, match="unsupported"):
        gg.gg_read_ply(str(p))
