"""Pins of the quadtree / seeding oracle (oracle/seed.py):
closed-form leaf lists, the tiling and contrast invariants, monotonicity in the
threshold (Fig. 3 of the paper), and Eq. 10 initialisation in closed form on a
fronto-parallel plane (mean, isotropic scale, opacity, colour), the weight gate on a
fresh volume and after a second fusion."""
import numpy as np
import pytest

import scenegen
from oracle import seed as Q
from oracle import tsdf as T


def test_single_bright_pixel_closed_form():
    rgb = np.zeros((3, 8, 8), np.float32)
    rgb[:, 0, 0] = 1.0
    assert Q.quadtree(rgb, 0.1, 2) == [(0, 0, 2, 2), (2, 0, 2, 2), (0, 2, 2, 2), (2, 2, 2, 2),
                                       (4, 0, 4, 4), (0, 4, 4, 4), (4, 4, 4, 4)]
    assert Q.quadtree(np.full((3, 37, 23), 0.4, np.float32), 0.1, 2) == [(0, 0, 23, 37)]  # constant: the root


def _check_tiling(leaves, W, H):
    cover = np.zeros((H, W), np.int32)
    for (x, y, w, h) in leaves:
        cover[y:y + h, x:x + w] += 1
    assert np.all(cover == 1)


def test_half_split_image_invariants():
    rgb = np.zeros((3, 64, 64), np.float32)
    rgb[:, :, 32:] = 1.0
    leaves = Q.quadtree(rgb, 0.1, 2)
    _check_tiling(leaves, 64, 64)
    L = Q.luminance(rgb)
    for (x, y, w, h) in leaves:
        c = L[y:y + h, x:x + w]
        assert c.max() - c.min() <= 0.1 or w <= 2 or h <= 2
    assert len(leaves) == 4  # the boundary is at x = 32: every quadrant is constant
    rgb[:, :, 31:] = 1.0     # boundary inside the quadrants: splits down to 2-px cells along x = 31
    leaves = Q.quadtree(rgb, 0.1, 2)
    _check_tiling(leaves, 64, 64)
    assert all(w == 2 for (x, y, w, h) in leaves if x <= 31 < x + w)


def test_threshold_monotone_and_ragged_sizes():
    rng = np.random.default_rng(0)
    rgb = np.clip(rng.normal(0.5, 0.15, size=(3, 45, 71)).cumsum(axis=2) / 20, 0, 1).astype(np.float32)
    counts = [len(Q.quadtree(rgb, t, 2)) for t in (0.3, 0.1, 0.05, 0.01)]
    assert counts == sorted(counts)
    _check_tiling(Q.quadtree(rgb, 0.05, 3), 71, 45)


def test_seed_plane_closed_form_and_gate():
    d0, f = 1.25, 60.0
    cam = scenegen.identity_camera(64, 48, f, 31.5, 23.5)
    depth = scenegen.render_depth(scenegen.plane_faces(d0), cam)
    rng = np.random.default_rng(1)
    rgb = np.repeat(np.repeat(rng.uniform(0, 1, (3, 6, 8)), 8, axis=1), 8, axis=2).astype(np.float32)
    leaves = Q.quadtree(rgb, 0.1, 2)
    p = T.params(0.01, 0.06, 100.0)
    vol = T.Volume(p)
    vol.allocate(cam, depth)
    vol.integrate(cam, depth)
    keys, _, ws = vol.dump()
    G = Q.seed(leaves, cam, depth, rgb, keys, ws, 0.01, p.origin, 0)
    assert G.shape[1] >= 0.95 * len(leaves)  # fresh volume: (almost) every leaf (border voxels aside)
    # closed forms for the accepted leaves (recomputed per leaf in float64)
    got = {(round(float(G[0, k]), 5), round(float(G[1, k]), 5)): k for k in range(G.shape[1])}
    hits = 0
    for (x, y, w, h) in leaves:
        u, v = x + w // 2, y + h // 2
        px, py = d0 * (u - cam.cx) / f, d0 * (v - cam.cy) / f
        k = got.get((round(px, 5), round(py, 5)))
        if k is None:
            continue
        hits += 1
        assert G[2, k] == pytest.approx(d0, abs=1e-6)
        s = d0 * np.hypot(w // 2, h // 2) / f
        assert np.allclose(G[3:6, k], np.log(s), atol=1e-5)
        assert list(G[6:11, k]) == [1.0, 0.0, 0.0, 0.0, 0.0]           # identity rotation, opacity 0.5
        np.testing.assert_allclose(G[11:14, k] * 0.28209479177387814 + 0.5, rgb[:, v, u], atol=1e-6)
    assert hits == G.shape[1]
    vol.integrate(cam, depth)  # a second fusion: every observed voxel now has weight 2
    keys, _, ws = vol.dump()
    assert Q.seed(leaves, cam, depth, rgb, keys, ws, 0.01, p.origin, 0).shape[1] == 0
