"""Pins of the TSDF-fusion oracle (oracle/tsdf_ref.cpp) against
what the paper and geometry fix (-m "not gpu"):
  Morton code values (interleaved coordinate bits), Eq. 7 on a fronto-
  parallel plane in closed form (incl. SPEC.md:136-137's worked values 0.5 and the
  clamp), Eqs. 8-9 worked update (SPEC.md:138-style hand value) and the w_max cap,
  band allocation against an exact float64 segment / box intersection, idempotence
  ("fewer voxel blocks need to be allocated in subsequent frames")."""
import numpy as np
import pytest

import scenegen
from oracle import tsdf as T

VS, EPS = 0.01, 0.06
ORG = 1 << 20


def test_morton_interleaves_bits():
    assert T.morton(1, 0, 0) == 1 and T.morton(0, 1, 0) == 2 and T.morton(0, 0, 1) == 4
    assert T.morton(1, 1, 1) == 7 and T.morton(2, 0, 0) == 8 and T.morton(3, 5, 6) == 0b110101011  # z y x per triple
    rng = np.random.default_rng(0)
    for x, y, z in rng.integers(0, 1 << 21, size=(50, 3)):
        assert T.unmorton(T.morton(x, y, z)) == (x, y, z)


def _plane_frame(z0, w=48, h=36, f=40.0):
    cam = scenegen.identity_camera(w, h, f, (w - 1) / 2, (h - 1) / 2)
    return cam, scenegen.render_depth(scenegen.plane_faces(z0), cam)


def _voxel_centres(keys):
    """World coordinates of every voxel of the blocks (x-fastest inside a block)."""
    out = []
    l = np.arange(512)
    loc = np.stack([l & 7, (l >> 3) & 7, l >> 6], axis=1)
    for k in keys:
        b = np.array(T.unmorton(int(k)))
        v = b * 8 + loc
        out.append((v - ORG + 0.5) * VS)
    return np.stack(out)  # [n][512][3]


def test_plane_closed_form_eq7():
    z0 = 1.0
    cam, depth = _plane_frame(z0)
    vol = T.Volume(T.params(VS, EPS, 100.0))
    assert vol.allocate(cam, depth) > 0
    vol.integrate(cam, depth)
    keys, ts, ws = vol.dump()
    P = _voxel_centres(keys)
    x, y, z = P[..., 0], P[..., 1], P[..., 2]
    u = cam.fx * x / z + cam.cx
    v = cam.fy * y / z + cam.cy
    inside = (z > 0) & (u > -0.5) & (u < cam.width - 0.5) & (v > -0.5) & (v < cam.height - 0.5)
    sdf = z0 - z
    seen = inside & (sdf >= -EPS)
    expect = np.clip(sdf / EPS, -1, 1)
    # away from the image border and the sdf = -eps edge (fp32 rounding of the projection)
    safe = seen & (u > 0) & (u < cam.width - 1) & (v > 0) & (v < cam.height - 1) & (np.abs(sdf + EPS) > 1e-5)
    assert safe.sum() > 1000
    np.testing.assert_allclose(ts[safe], expect[safe], atol=2e-6)
    assert np.all(ws[safe] == 1.0)
    assert np.all(ws[inside & (sdf < -EPS - 1e-5)] == 0.0)
    # SPEC.md:136-137 worked values: sdf = 0.03 -> 0.5; sdf > eps -> 1 (clamped)
    c = np.argmin(np.abs(z - 0.975) + np.abs(x - 0.005) + np.abs(y - 0.005) + ~safe)
    assert np.isclose(sdf.ravel()[c], 0.025) and np.isclose(ts.ravel()[c], 0.025 / EPS, atol=1e-6)
    assert np.all(ts[safe & (sdf > EPS + 1e-5)] == 1.0)


def test_eq8_eq9_update_and_weight_cap():
    cam, d1 = _plane_frame(1.0)
    _, d2 = _plane_frame(1.2)
    vol = T.Volume(T.params(VS, EPS, 100.0))
    vol.allocate(cam, d1)
    vol.integrate(cam, d1)  # voxel at z = 0.975: sdf 0.025 -> tsdf 5/12, w 1
    vol.integrate(cam, d2)  # same voxel: sdf 0.225 -> tsdf 1, w 2 -> (5/12 * 1 + 1 * 2) / 3
    keys, ts, ws = vol.dump()
    P = _voxel_centres(keys)
    c = np.argmin(np.abs(P[..., 2] - 0.975) + np.abs(P[..., 0] - 0.005) + np.abs(P[..., 1] - 0.005))
    assert ws.ravel()[c] == 2.0
    assert ts.ravel()[c] == pytest.approx((0.025 / EPS * 1 + 1.0 * 2) / 3, abs=2e-6)
    vol2 = T.Volume(T.params(VS, EPS, 3.0))  # w_max = 3: weights 1, 2, 3, 3, 3; tsdf fixed point
    vol2.allocate(cam, d1)
    for _ in range(5):
        vol2.integrate(cam, d1)
    _, ts2, ws2 = vol2.dump()
    _, ts1, ws1 = (lambda v: (v.allocate(cam, d1), v.integrate(cam, d1), v.dump())[2])(T.Volume(T.params(VS, EPS, 3.0)))
    seen = ws1 > 0
    assert np.all(ws2[seen] == 3.0) and np.all(ws2[~seen] == 0.0)
    np.testing.assert_allclose(ts2[seen], ts1[seen], atol=1e-6)


def _segment_box_overlap(p0, p1, lo, hi):
    """Length of the segment p0 -> p1 inside the box [lo, hi] (float64 slab test)."""
    d = p1 - p0
    t0, t1 = 0.0, 1.0
    for a in range(3):
        if abs(d[a]) < 1e-15:
            if p0[a] < lo[a] or p0[a] > hi[a]:
                return -1.0
            continue
        ta, tb = (lo[a] - p0[a]) / d[a], (hi[a] - p0[a]) / d[a]
        t0, t1 = max(t0, min(ta, tb)), min(t1, max(ta, tb))
    return (t1 - t0) * np.linalg.norm(d) if t1 >= t0 else -1.0


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_band_allocation_vs_exact_segment_box(seed):
    rng = np.random.default_rng(seed)
    R = scenegen.rot_y(rng.uniform(-0.6, 0.6)) @ np.array([[1, 0, 0], [0, np.cos(0.3), -np.sin(0.3)],
                                                           [0, np.sin(0.3), np.cos(0.3)]])
    cam = scenegen.camera_rt(20, 16, 18.0, 9.5, 7.5, R, rng.uniform(-0.2, 0.2, 3))
    depth = np.zeros((16, 20), np.float32)
    i, j = rng.integers(0, 20), rng.integers(0, 16)
    d = np.float32(rng.uniform(0.7, 2.5))
    depth[j, i] = d
    p = T.params(VS, EPS, 100.0)
    vol = T.Volume(p)
    n = vol.allocate(cam, depth)
    keys, _, _ = vol.dump()
    got = {T.unmorton(int(k)) for k in keys}
    assert n == len(got) > 0
    Rw = np.asarray(cam.R_cw, np.float64)
    tw = np.asarray(cam.t_cw, np.float64)
    ray = np.array([(i - cam.cx) / cam.fx, (j - cam.cy) / cam.fy, 1.0])
    a, b = Rw.T @ (ray * (float(d) - EPS) - tw), Rw.T @ (ray * (float(d) + EPS) - tw)
    lo = np.floor(np.minimum(a, b) / VS / 8).astype(int) - 1 + ORG // 8
    hi = np.floor(np.maximum(a, b) / VS / 8).astype(int) + 2 + ORG // 8
    exact, long_ = set(), set()
    for bx in range(lo[0], hi[0]):
        for by in range(lo[1], hi[1]):
            for bz in range(lo[2], hi[2]):
                blo = (np.array([bx, by, bz]) * 8 - ORG) * VS
                L = _segment_box_overlap(a, b, blo - 1e-6, blo + 8 * VS + 1e-6)
                if L >= 0:
                    exact.add((bx, by, bz))
                if L >= p.step * np.linalg.norm(ray) * 1.01:
                    long_.add((bx, by, bz))
    assert got <= exact           # every allocated block meets the band segment
    assert long_ <= got           # every block the segment crosses for >= one step is allocated


def test_allocation_idempotent_and_empty():
    cam, depth = _plane_frame(1.3)
    vol = T.Volume(T.params(VS, EPS, 100.0))
    assert vol.allocate(cam, np.zeros_like(depth)) == 0
    n = vol.allocate(cam, depth)
    assert n > 0 and vol.allocate(cam, depth) == 0 and vol.num_blocks == n
