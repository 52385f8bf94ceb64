"""Seeded synthetic inputs for the five BASELINE.json configs (input side only).

This module is shared by the CPU oracle (``oracle/``) and the CUDA path
(``paper_2408_12677_b200``).  It holds NONE of the method's arithmetic: it only
draws Gaussian parameters, camera poses, upstream-gradient fields and parameter
perturbations from seeded NumPy PCG64 generators.  Nothing here projects,
sorts, renders or differentiates.

Recipes:

* parameters are stored SoA as float32 ``[F][P_stride]`` with
  ``F = 11 + 3*(deg+1)**2`` and ``P_stride = P`` rounded up to a multiple of 4:
  rows 0-2 mean xyz (m), 3-5 log-scale, 6-9 quaternion (w, x, y, z; not unit),
  10 opacity logit, ``11 + 3k + ch`` SH coefficient ``k`` of channel ``ch``.
  Padding columns are zero and never read.
* colour: RGB ~ U(0,1) is stored as the DC coefficient ``(rgb - 0.5) / Y00``
  with ``Y00 = 0.28209479177387814`` (reading R14), higher SH bands ~ N(0, 0.1).
* seeds: scene = ``seed``, target perturbation = ``seed + 1``, poses = ``seed + 2``.

Replica, ScanNet++ and the paper's large-scale scans are not available in this
container (§IV-A1); the ``replica``/``scannetpp``/``large``
generators stand in for them by taking their *shapes*: resolution, intrinsics,
room extents, surface structure, Gaussian density and scale distribution
(BASELINE.json configs 2-4).
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np

Y00_LITERAL = 0.28209479177387814  # recipe constant: DC coefficient <-> RGB (R14)
TILE = 16

CONFIG_NAMES = ("tiny", "small", "replica", "scannetpp", "large")


def sh_coeffs(deg: int) -> int:
    return (deg + 1) * (deg + 1)


def num_rows(deg: int) -> int:
    return 11 + 3 * sh_coeffs(deg)


def pad4(p: int) -> int:
    return (p + 3) // 4 * 4


@dataclasses.dataclass
class Camera:
    """Pinhole camera, OpenCV axes (x right, y down, z forward).

    ``R_cw``/``t_cw`` map world to camera (the rotation W and translation of
    T_WC^{-1}).  Pixel (i, j) samples continuous (i, j) (R1).
    """

    width: int
    height: int
    fx: float
    fy: float
    cx: float
    cy: float
    R_cw: np.ndarray  # (3,3) float32
    t_cw: np.ndarray  # (3,) float32
    z_near: float = 0.2
    bg: tuple = (0.0, 0.0, 0.0)

    @property
    def tiles_x(self) -> int:
        return (self.width + TILE - 1) // TILE

    @property
    def tiles_y(self) -> int:
        return (self.height + TILE - 1) // TILE

    @property
    def num_tiles(self) -> int:
        return self.tiles_x * self.tiles_y

    @property
    def num_pixels(self) -> int:
        return self.width * self.height


@dataclasses.dataclass
class Scene:
    P: int
    sh_degree: int
    params: np.ndarray  # float32 [F][P_stride]

    @property
    def F(self) -> int:
        return num_rows(self.sh_degree)

    @property
    def P_stride(self) -> int:
        return self.params.shape[1]


@dataclasses.dataclass
class Workload:
    name: str
    scene: Scene
    target_scene: Scene  # perturbed parameters used to render the target images
    cameras: list  # list[Camera]; the views of one batch
    faces: list = None  # surface rectangles the Gaussians were sampled on (depth synthesis)


# ---------------------------------------------------------------------------
# parameter blocks
# ---------------------------------------------------------------------------

def _alloc_params(P: int, deg: int) -> np.ndarray:
    return np.zeros((num_rows(deg), pad4(P)), dtype=np.float32)


def _fill_common(rng, params, P, deg, log_scale_mu, log_scale_sigma, higher_sh_sigma=0.1):
    """Log-scale, quaternion, opacity logit and SH rows (shared by all configs)."""
    params[3:6, :P] = rng.normal(log_scale_mu, log_scale_sigma, size=(3, P))
    params[6:10, :P] = _random_unit_quaternions(rng, P)
    params[10, :P] = rng.normal(0.0, 1.0, size=P)
    rgb = rng.uniform(0.0, 1.0, size=(3, P))
    params[11:14, :P] = (rgb - 0.5) / Y00_LITERAL
    S = sh_coeffs(deg)
    if S > 1:
        params[14:11 + 3 * S, :P] = rng.normal(0.0, higher_sh_sigma, size=(3 * (S - 1), P))


def _random_unit_quaternions(rng, P):
    q = rng.normal(size=(4, P))
    q /= np.linalg.norm(q, axis=0, keepdims=True)
    return q


def perturb(scene: Scene, seed: int, sigma: float = 0.01) -> Scene:
    """Target parameters: every raw row + N(0, sigma) (configs 0-1 recipe)."""
    rng = np.random.default_rng(seed)
    p = scene.params.copy()
    p[:, :scene.P] += rng.normal(0.0, sigma, size=(p.shape[0], scene.P)).astype(np.float32)
    return Scene(scene.P, scene.sh_degree, p)


# ---------------------------------------------------------------------------
# surfaces: area-uniform samples on axis-aligned rectangles
# ---------------------------------------------------------------------------

def _room_faces(x0, x1, y0, y1, z0, z1, with_floor=True, with_ceiling=True):
    """Rectangles as (origin, u-edge, v-edge, normal)."""
    faces = []
    o = np.array
    if with_floor:
        faces.append((o([x0, y0, z0]), o([x1 - x0, 0, 0]), o([0, y1 - y0, 0]), o([0, 0, 1.0])))
    if with_ceiling:
        faces.append((o([x0, y0, z1]), o([x1 - x0, 0, 0]), o([0, y1 - y0, 0]), o([0, 0, -1.0])))
    faces.append((o([x0, y0, z0]), o([x1 - x0, 0, 0]), o([0, 0, z1 - z0]), o([0, 1.0, 0])))
    faces.append((o([x0, y1, z0]), o([x1 - x0, 0, 0]), o([0, 0, z1 - z0]), o([0, -1.0, 0])))
    faces.append((o([x0, y0, z0]), o([0, y1 - y0, 0]), o([0, 0, z1 - z0]), o([1.0, 0, 0])))
    faces.append((o([x1, y0, z0]), o([0, y1 - y0, 0]), o([0, 0, z1 - z0]), o([-1.0, 0, 0])))
    return faces


def _box_faces(cx, cy, sx, sy, sz):
    """Floor-standing box: 4 sides + top (outward normals)."""
    x0, x1, y0, y1 = cx - sx / 2, cx + sx / 2, cy - sy / 2, cy + sy / 2
    o = np.array
    return [
        (o([x0, y0, sz]), o([sx, 0, 0]), o([0, sy, 0]), o([0, 0, 1.0])),
        (o([x0, y0, 0.0]), o([sx, 0, 0]), o([0, 0, sz]), o([0, -1.0, 0])),
        (o([x0, y1, 0.0]), o([sx, 0, 0]), o([0, 0, sz]), o([0, 1.0, 0])),
        (o([x0, y0, 0.0]), o([0, sy, 0]), o([0, 0, sz]), o([-1.0, 0, 0])),
        (o([x1, y0, 0.0]), o([0, sy, 0]), o([0, 0, sz]), o([1.0, 0, 0])),
    ]


def _wall(x, y0, y1, z1):
    """Full-height partition wall in the plane x = const (both sides sampled)."""
    o = np.array
    return [(o([x, y0, 0.0]), o([0, y1 - y0, 0]), o([0, 0, z1]), o([1.0, 0, 0]))]


def _sample_surfaces(rng, faces, n, noise_sigma):
    areas = np.array([np.linalg.norm(np.cross(u, v)) for (_, u, v, _) in faces])
    idx = rng.choice(len(faces), size=n, p=areas / areas.sum())
    a = rng.uniform(0, 1, size=n)
    b = rng.uniform(0, 1, size=n)
    off = rng.normal(0.0, noise_sigma, size=n)
    O = np.stack([faces[i][0] for i in range(len(faces))])
    U = np.stack([faces[i][1] for i in range(len(faces))])
    V = np.stack([faces[i][2] for i in range(len(faces))])
    N = np.stack([faces[i][3] for i in range(len(faces))])
    pts = O[idx] + a[:, None] * U[idx] + b[:, None] * V[idx] + off[:, None] * N[idx]
    return pts.T  # (3, n)


def _random_boxes(rng, n, xlo, xhi, ylo, yhi, side_lo=0.3, side_hi=1.5, max_h=None):
    faces = []
    for _ in range(n):
        sx, sy, sz = rng.uniform(side_lo, side_hi, size=3)
        if max_h is not None:
            sz = min(sz, max_h)
        cx = rng.uniform(xlo + sx / 2, xhi - sx / 2)
        cy = rng.uniform(ylo + sy / 2, yhi - sy / 2)
        faces += _box_faces(cx, cy, sx, sy, sz)
    return faces


# ---------------------------------------------------------------------------
# cameras (world z-up; camera OpenCV axes)
# ---------------------------------------------------------------------------

def camera_from_forward(width, height, f, cx, cy, position, forward, z_near=0.2):
    fwd = np.asarray(forward, dtype=np.float64)
    fwd = fwd / np.linalg.norm(fwd)
    up = np.array([0.0, 0.0, 1.0])
    right = np.cross(fwd, up)
    if np.linalg.norm(right) < 1e-9:
        raise ValueError("forward direction parallel to the world up axis")
    right /= np.linalg.norm(right)
    down = np.cross(fwd, right)
    R_wc = np.stack([right, down, fwd], axis=1)  # columns: camera axes in world
    R_cw = R_wc.T
    t_cw = -R_cw @ np.asarray(position, dtype=np.float64)
    return Camera(width, height, float(f), float(f), float(cx), float(cy),
                  R_cw.astype(np.float32), t_cw.astype(np.float32), z_near)


def camera_rt(width, height, f, cx, cy, R_cw, t_cw, z_near=0.2):
    return Camera(width, height, float(f), float(f), float(cx), float(cy),
                  np.asarray(R_cw, dtype=np.float32).reshape(3, 3), np.asarray(t_cw, dtype=np.float32).reshape(3),
                  z_near)


def rot_y(theta):
    c, s = math.cos(theta), math.sin(theta)
    return np.array([[c, 0.0, s], [0.0, 1.0, 0.0], [-s, 0.0, c]])


def identity_camera(width, height, f, cx, cy, z_near=0.2):
    return Camera(width, height, float(f), float(f), float(cx), float(cy),
                  np.eye(3, dtype=np.float32), np.zeros(3, dtype=np.float32), z_near)


def _yaw_pitch_forward(yaw, pitch):
    return np.array([math.cos(pitch) * math.cos(yaw), math.cos(pitch) * math.sin(yaw), math.sin(pitch)])


# ---------------------------------------------------------------------------
# the five configs (BASELINE.json:7-11)
# ---------------------------------------------------------------------------

def make_tiny(seed: int = 0) -> Workload:
    """Config 0: 64x48, f=60, c=(32,24), 256 Gaussians in a box, SH0, identity pose."""
    rng = np.random.default_rng(seed)
    P, deg = 256, 0
    params = _alloc_params(P, deg)
    params[0, :P] = rng.uniform(-1, 1, P)
    params[1, :P] = rng.uniform(-1, 1, P)
    params[2, :P] = rng.uniform(2, 4, P)
    _fill_common(rng, params, P, deg, math.log(0.05), 0.3)
    scene = Scene(P, deg, params)
    cam = identity_camera(64, 48, 60.0, 32.0, 24.0)
    return Workload("tiny", scene, perturb(scene, seed + 1), [cam])


def make_small(seed: int = 0) -> Workload:
    """Config 1: 320x240, f=300, 20k Gaussians in a 3x3x4 m box 1-5 m ahead, SH1."""
    rng = np.random.default_rng(seed)
    P, deg = 20000, 1
    params = _alloc_params(P, deg)
    params[0, :P] = rng.uniform(-1.5, 1.5, P)
    params[1, :P] = rng.uniform(-1.5, 1.5, P)
    params[2, :P] = rng.uniform(1.0, 5.0, P)
    _fill_common(rng, params, P, deg, math.log(0.05), 0.3)
    scene = Scene(P, deg, params)
    cam = identity_camera(320, 240, 300.0, 160.0, 120.0)
    return Workload("small", scene, perturb(scene, seed + 1), [cam])


def _surface_scene(rng, P, faces, log_mu, log_sigma, deg=3, noise=0.005):
    params = _alloc_params(P, deg)
    params[0:3, :P] = _sample_surfaces(rng, faces, P, noise)
    _fill_common(rng, params, P, deg, log_mu, log_sigma)
    return Scene(P, deg, params)


def make_replica(seed: int = 0, num_views: int = 100, P: int = 300_000) -> Workload:
    """Config 2: 1200x680, f=600, 300k Gaussians on an 8x6x3 m room + 20 boxes, SH3."""
    rng = np.random.default_rng(seed)
    faces = _room_faces(-4, 4, -3, 3, 0, 3) + _random_boxes(rng, 20, -4, 4, -3, 3)
    scene = _surface_scene(rng, P, faces, math.log(0.02), 0.5)
    prng = np.random.default_rng(seed + 2)
    cams = []
    for _ in range(num_views):
        pos = [prng.uniform(-3, 3), prng.uniform(-2, 2), 1.5]
        fwd = _yaw_pitch_forward(prng.uniform(0, 2 * math.pi), math.radians(prng.normal(0, 10)))
        cams.append(camera_from_forward(1200, 680, 600.0, 599.5, 339.5, pos, fwd))
    return Workload("replica", scene, perturb(scene, seed + 1), cams, faces)


def make_scannetpp(seed: int = 0, num_views: int = 8, P: int = 1_000_000) -> Workload:
    """Config 3: 1752x1168, f=1100, 1M Gaussians on a 12x8x3 m room + 60 boxes, SH3,
    a batch of 8 poses on a 1.5 m-radius orbit looking at the room centre."""
    rng = np.random.default_rng(seed)
    faces = _room_faces(-6, 6, -4, 4, 0, 3) + _random_boxes(rng, 60, -6, 6, -4, 4)
    scene = _surface_scene(rng, P, faces, math.log(0.02), 0.5)
    prng = np.random.default_rng(seed + 2)
    cams = []
    for _ in range(num_views):
        ang = prng.uniform(0, 2 * math.pi)
        pos = np.array([1.5 * math.cos(ang), 1.5 * math.sin(ang), 1.5])
        fwd = np.array([0.0, 0.0, 1.0]) - pos
        cams.append(camera_from_forward(1752, 1168, 1100.0, 875.5, 583.5, pos, fwd))
    return Workload("scannetpp", scene, perturb(scene, seed + 1), cams, faces)


def make_large(seed: int = 0, num_views: int = 64, P: int = 4_000_000) -> Workload:
    """Config 4: 1920x1440, f=1200, 4M Gaussians over a 30x20x4 m multi-room set
    (outer shell, 3 partition walls, 120 boxes), log-scale ~ N(log 0.01, 0.7), SH3,
    a batch of 64 views over the floor plan."""
    rng = np.random.default_rng(seed)
    faces = _room_faces(-15, 15, -10, 10, 0, 4)
    for x in (-7.5, 0.0, 7.5):
        faces += _wall(x, -10, 10, 4)
    faces += _random_boxes(rng, 120, -15, 15, -10, 10)
    scene = _surface_scene(rng, P, faces, math.log(0.01), 0.7)
    prng = np.random.default_rng(seed + 2)
    cams = []
    for _ in range(num_views):
        pos = [prng.uniform(-14, 14), prng.uniform(-9, 9), 1.5]
        fwd = _yaw_pitch_forward(prng.uniform(0, 2 * math.pi), math.radians(prng.normal(0, 10)))
        cams.append(camera_from_forward(1920, 1440, 1200.0, 959.5, 719.5, pos, fwd))
    return Workload("large", scene, perturb(scene, seed + 1), cams, faces)


MAKERS = {
    "tiny": make_tiny,
    "small": make_small,
    "replica": make_replica,
    "scannetpp": make_scannetpp,
    "large": make_large,
}


def make(name: str, seed: int = 0, **kw) -> Workload:
    return MAKERS[name](seed, **kw)


# ---------------------------------------------------------------------------
# small hand-built scenes and upstream fields for tests
# ---------------------------------------------------------------------------

def scene_from_gaussians(means, log_scales, quats, logits, sh, deg) -> Scene:
    """Build a Scene from per-Gaussian arrays (means (P,3), log_scales (P,3),
    quats (P,4) w-first, logits (P,), sh (P, S, 3))."""
    means = np.asarray(means, dtype=np.float64).reshape(-1, 3)
    P = means.shape[0]
    params = _alloc_params(P, deg)
    params[0:3, :P] = means.T
    params[3:6, :P] = np.asarray(log_scales, dtype=np.float64).reshape(P, 3).T
    params[6:10, :P] = np.asarray(quats, dtype=np.float64).reshape(P, 4).T
    params[10, :P] = np.asarray(logits, dtype=np.float64).reshape(P)
    S = sh_coeffs(deg)
    shv = np.asarray(sh, dtype=np.float64).reshape(P, S, 3)
    for k in range(S):
        for ch in range(3):
            params[11 + 3 * k + ch, :P] = shv[:, k, ch]
    return Scene(P, deg, params)


def random_small_scene(seed: int, P: int, deg: int, width: int = 32, height: int = 32,
                       f: float = 30.0, log_scale_mu=math.log(0.15), log_scale_sigma=0.3):
    """Few-Gaussian scene in front of an identity camera (FD / brute-force tests)."""
    rng = np.random.default_rng(seed)
    params = _alloc_params(P, deg)
    params[0, :P] = rng.uniform(-0.6, 0.6, P)
    params[1, :P] = rng.uniform(-0.6, 0.6, P)
    params[2, :P] = rng.uniform(1.5, 3.0, P)
    _fill_common(rng, params, P, deg, log_scale_mu, log_scale_sigma, higher_sh_sigma=0.2)
    params[10, :P] = rng.normal(0.5, 1.0, P)
    cam = identity_camera(width, height, f, (width - 1) / 2.0, (height - 1) / 2.0)
    return Scene(P, deg, params), cam


def upstream_fields(seed: int, width: int, height: int, kind: str = "normal"):
    """Seeded dL/dcolour [3][H][W] and dL/ddepth [H][W] fields (float32)."""
    rng = np.random.default_rng(seed)
    if kind == "normal":
        g_rgb = rng.normal(size=(3, height, width))
        g_d = rng.normal(size=(height, width))
    elif kind == "sign":
        g_rgb = rng.choice([-1.0, 1.0], size=(3, height, width))
        g_d = rng.choice([-1.0, 1.0], size=(height, width))
    else:
        raise ValueError(kind)
    return g_rgb.astype(np.float32), g_d.astype(np.float32)


DEPTH_SCALE = 1e-3  # metres per 16-bit depth unit of the synthetic sensor frames (millimetres)


def quantize_frame(rgb, depth, depth_scale: float = DEPTH_SCALE):
    """Sensor form of a float RGB-D frame, as an RGB-D camera / dataset delivers it
    (input generation, R41): uint8 [H][W][3] = round(clip(rgb, 0, 1) x 255) re-laid out
    interleaved, uint16 [H][W] = round(clip(depth / depth_scale, 0, 65535)); rgb
    [3][H][W] and depth [H][W] float arrays."""
    rgb = np.asarray(rgb, np.float64)
    depth = np.asarray(depth, np.float64)
    c = np.rint(np.clip(rgb, 0.0, 1.0) * 255.0).astype(np.uint8)
    d = np.rint(np.clip(depth / depth_scale, 0.0, 65535.0)).astype(np.uint16)
    return np.ascontiguousarray(np.transpose(c, (1, 2, 0))), d


def shard_views(num_views: int, rank: int, world: int):
    """Contiguous view shard of rank ``rank``: [r*B/R, (r+1)*B/R)."""
    lo = (rank * num_views) // world
    hi = ((rank + 1) * num_views) // world
    return list(range(lo, hi))


def new_primitive_counts(num_frames: int, seed: int = 0):
    """Seeded stand-in for the per-frame number of newly initialised Gaussians, the
    keyframe criterion of PAPER.md:149 (its producer, the TSDF-gated quadtree
    seeding of PAPER.md:125-135, is out of scope).  Shape of an online scan: early
    frames see mostly unobserved space (thousands of new primitives, decaying with a
    15-frame time constant and log-normal spread), later frames mostly revisit (a few
    new ones) with occasional turns into unseen areas (probability 0.15, 50-800 new).
    Seed stream: seed + 3.  Returns int64[num_frames]."""
    rng = np.random.default_rng(seed + 3)
    t = np.arange(num_frames)
    base = 4000.0 * np.exp(-t / 15.0) * rng.lognormal(0.0, 0.5, num_frames) + 5.0
    counts = rng.poisson(base)
    turns = rng.random(num_frames) < 0.15
    counts = counts + turns * rng.integers(50, 800, num_frames)
    return counts.astype(np.int64)


def render_depth(faces, cam, noise_sigma: float = 0.0, dropout: float = 0.0, seed: int = 0):
    """Synthetic depth frame (metres of camera z, 0 = invalid) of the surface
    rectangles seen by ``cam``: the input of the TSDF fusion (NEXT-3) in place of a
    sensor's depth map (Replica / ScanNet++ depth is not available).
    Pixel (i, j) looks along p(z) = o + z R^T ((i - cx)/fx, (j - cy)/fy, 1) (R1);
    depth = the smallest z > 0 where the ray meets a rectangle.  Optional Gaussian noise
    (sigma, m) and random invalid pixels (fraction), seed stream seed + 4.  Input
    generation only: none of the fusion arithmetic happens here."""
    R = np.asarray(cam.R_cw, np.float64).reshape(3, 3)
    t = np.asarray(cam.t_cw, np.float64).reshape(3)
    o = -R.T @ t
    jj, ii = np.meshgrid(np.arange(cam.height, dtype=np.float64), np.arange(cam.width, dtype=np.float64),
                         indexing="ij")
    dc = np.stack([(ii - cam.cx) / cam.fx, (jj - cam.cy) / cam.fy, np.ones_like(ii)], axis=-1)
    dw = dc @ R  # rows: R^T dc
    best = np.full(ii.shape, np.inf)
    for (O, U, V, N) in faces:
        O, U, V, N = (np.asarray(x, np.float64) for x in (O, U, V, N))
        # pixel window: the projected corners' bounding box (whole image if the
        # rectangle crosses the camera plane); faces entirely behind are skipped
        corners = np.stack([O, O + U, O + V, O + U + V]) @ R.T + t
        if np.all(corners[:, 2] <= 1e-6):
            continue
        if np.all(corners[:, 2] > 1e-6):
            u = cam.fx * corners[:, 0] / corners[:, 2] + cam.cx
            v = cam.fy * corners[:, 1] / corners[:, 2] + cam.cy
            x0, x1 = max(int(np.floor(u.min())) - 1, 0), min(int(np.ceil(u.max())) + 2, cam.width)
            y0, y1 = max(int(np.floor(v.min())) - 1, 0), min(int(np.ceil(v.max())) + 2, cam.height)
            if x0 >= x1 or y0 >= y1:
                continue
        else:
            x0, x1, y0, y1 = 0, cam.width, 0, cam.height
        dwin = dw[y0:y1, x0:x1]
        n = np.cross(U, V)
        den = dwin @ n
        with np.errstate(divide="ignore", invalid="ignore"):
            z = ((O - o) @ n) / den
        ok = np.isfinite(z) & (z > 1e-6)
        p = o + z[..., None] * dwin - O
        a = (p @ U) / (U @ U)
        b = (p @ V) / (V @ V)
        ok &= (a >= 0) & (a <= 1) & (b >= 0) & (b <= 1)
        win = best[y0:y1, x0:x1]
        best[y0:y1, x0:x1] = np.where(ok & (z < win), z, win)
    depth = np.where(np.isfinite(best), best, 0.0)
    rng = np.random.default_rng(seed + 4)
    if noise_sigma > 0:
        depth = np.where(depth > 0, depth + rng.normal(0.0, noise_sigma, depth.shape), 0.0)
    if dropout > 0:
        depth = np.where(rng.random(depth.shape) < dropout, 0.0, depth)
    return depth.astype(np.float32)


def plane_faces(z0: float, half: float = 50.0):
    """One fronto-parallel rectangle z = z0 (identity camera): TSDF closed-form tests."""
    o = np.array
    return [(o([-half, -half, z0]), o([2 * half, 0.0, 0.0]), o([0.0, 2 * half, 0.0]), o([0.0, 0.0, -1.0]))]
