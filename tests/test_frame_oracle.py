"""Pins of the input-frame decode oracle (oracle/frame.py, reading R41) against exact
rational arithmetic and hand-built layouts -- not against itself."""
from fractions import Fraction

import numpy as np

import scenegen
from oracle import frame

F32 = np.float32


def _correctly_rounded(f32, exact: Fraction) -> bool:
    """f32 is a nearest float32 to the exact rational (neighbours are no closer)."""
    f = F32(f32)
    err = abs(Fraction(float(f)) - exact)
    for toward in (np.inf, -np.inf):
        nb = np.nextafter(f, F32(toward), dtype=F32)
        if abs(Fraction(float(nb)) - exact) < err:
            return False
    return True


def test_colour_is_k_over_255_correctly_rounded_for_every_byte():
    rgb = np.zeros((1, 256, 3), np.uint8)
    rgb[0, :, 0] = np.arange(256)
    rgb[0, :, 1] = np.arange(256)[::-1]
    planes, _ = frame.decode_rgbd(rgb, np.zeros((1, 256), np.uint16), 1e-3)
    for k in range(256):
        assert _correctly_rounded(planes[0, 0, k], Fraction(k, 255)), k
        assert _correctly_rounded(planes[1, 0, k], Fraction(255 - k, 255)), k
    assert planes[0, 0, 0] == 0.0 and planes[0, 0, 255] == 1.0
    assert planes[0, 0, 51] == F32(0.2)  # 51 / 255 = 1 / 5 exactly
    assert np.all(planes[2] == 0.0)


def test_depth_is_units_times_scale_correctly_rounded():
    rng = np.random.default_rng(5)
    d = np.concatenate([[0, 1, 1000, 65535], rng.integers(0, 65536, 500)]).astype(np.uint16).reshape(1, -1)
    for scale in (1e-3, 1.0 / 6553.5, 0.25):
        _, depth = frame.decode_rgbd(np.zeros(d.shape + (3,), np.uint8), d, scale)
        s = Fraction(float(F32(scale)))  # the fp32 multiplier the call receives
        for u, v in zip(d[0], depth[0]):
            assert _correctly_rounded(v, int(u) * s), (scale, int(u))
    _, depth = frame.decode_rgbd(np.zeros(d.shape + (3,), np.uint8), d, 1e-3)
    assert depth[0, 0] == 0.0  # invalid stays 0
    assert depth[0, 2] == 1.0  # 1000 mm = 1 m exactly after rounding


def test_interleaved_to_planar_layout():
    H, W = 3, 5
    rgb = np.zeros((H, W, 3), np.uint8)
    for y in range(H):
        for x in range(W):
            for c in range(3):
                rgb[y, x, c] = (7 * y + 3 * x + 100 * c) % 256
    dep = (np.arange(H * W, dtype=np.uint16) * 3).reshape(H, W)
    planes, depth = frame.decode_rgbd(rgb, dep, 0.5)
    assert planes.shape == (3, H, W) and depth.shape == (H, W)
    for y in range(H):
        for x in range(W):
            for c in range(3):
                assert planes[c, y, x] == F32((7 * y + 3 * x + 100 * c) % 256) / F32(255)
            assert depth[y, x] == F32(1.5 * (y * W + x))


def test_quantize_then_decode_round_trip():
    rng = np.random.default_rng(11)
    rgb = rng.uniform(-0.2, 1.2, (3, 9, 13))
    depth = rng.uniform(0.0, 12.0, (9, 13))
    depth[0, 0] = 0.0
    c, d = scenegen.quantize_frame(rgb, depth)
    assert c.dtype == np.uint8 and c.shape == (9, 13, 3) and d.dtype == np.uint16
    planes, dd = frame.decode_rgbd(c, d, scenegen.DEPTH_SCALE)
    assert np.abs(planes - np.clip(rgb, 0, 1)).max() <= 0.5 / 255 + 1e-7
    assert np.abs(dd - depth).max() <= 0.5e-3 + 1e-6
    assert dd[0, 0] == 0.0
