"""ctypes wrapper of the CPU oracle ``oracle/libgsref.so`` (TEST INFRASTRUCTURE).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this module.  The product path
(``paper_2408_12677_b200``) never does.  See ``oracle/gsref.cpp`` for the
definitions and their PAPER.md citations.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "gsref.cpp")
# GSREF_SANITIZE=1: an ASan + UBSan build (libgsref_san.so; tests/test_oracle_sanitize.py
# runs the pins against it in a subprocess with libasan preloaded)
SANITIZE = os.environ.get("GSREF_SANITIZE") == "1"
SAN_FLAGS = ["-O1", "-g", "-fno-omit-frame-pointer", "-fsanitize=address,undefined", "-fno-sanitize-recover=all"]
LIB = os.path.join(HERE, "libgsref_san.so" if SANITIZE else "libgsref.so")

F32, F64, MIXED, STAGE = 0, 1, 2, 3
FLAG_CULLED = 128


def build(force: bool = False) -> str:
    """Compile the oracle (g++ -O2 -ffp-contract=off, no fast-math)."""
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        cmd = ["g++", *(SAN_FLAGS if SANITIZE else ["-O2"]), "-std=c++17", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-fPIC", "-shared",
               "-o", LIB + ".tmp", SRC]
        subprocess.check_call(cmd)
        os.replace(LIB + ".tmp", LIB)
    return LIB


class RefCamera(C.Structure):
    _fields_ = [("width", C.c_int32), ("height", C.c_int32),
                ("fx", C.c_float), ("fy", C.c_float), ("cx", C.c_float), ("cy", C.c_float),
                ("R_cw", C.c_float * 9), ("t_cw", C.c_float * 3),
                ("z_near", C.c_float), ("bg", C.c_float * 3)]


def ref_camera(cam) -> RefCamera:
    rc = RefCamera()
    rc.width, rc.height = int(cam.width), int(cam.height)
    rc.fx, rc.fy, rc.cx, rc.cy = cam.fx, cam.fy, cam.cx, cam.cy
    R = np.asarray(cam.R_cw, dtype=np.float32).reshape(9)
    t = np.asarray(cam.t_cw, dtype=np.float32).reshape(3)
    for i in range(9):
        rc.R_cw[i] = float(R[i])
    for i in range(3):
        rc.t_cw[i] = float(t[i])
        rc.bg[i] = float(cam.bg[i])
    rc.z_near = cam.z_near
    return rc


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        P = C.c_void_p
        i64 = C.c_int64
        _lib.gsref_sh_basis.argtypes = [C.c_int, i64, P, P, P]
        _lib.gsref_set_threads.argtypes = [C.c_int]
        _lib.gsref_project.argtypes = [P, i64, i64, C.c_int, P, C.c_int, P, P, P, P, P]
        _lib.gsref_bin_tiles.argtypes = [P, i64, i64, C.c_int, P, i64, P, P, P, P]
        _lib.gsref_render_fwd.argtypes = [P, i64, i64, C.c_int, P, C.c_int, P, P, P, P, P, P, P, P]
        _lib.gsref_render_pixels.argtypes = [P, i64, i64, C.c_int, P, C.c_int, i64, P, P, P, P, P, P, P]
        _lib.gsref_render_bwd.argtypes = [P, i64, i64, C.c_int, P, C.c_int, P, P, P, P]
        _lib.gsref_render_bwd_bound.argtypes = [P, i64, i64, C.c_int, P, C.c_int, P, P, P, P, P, P]
        _lib.gsref_margin_bound.argtypes = [P, i64, i64, C.c_int, P, C.c_int, i64, P, P, P]
        _lib.gsref_adam_step.argtypes = [i64, i64, i64, P, P, P, P, P, C.c_double, C.c_double, C.c_double,
                                         i64, P, P, P]
        _lib.gsref_l1_loss_grad.argtypes = [i64, P, P, P, P, C.c_double, P, P, P]
    return _lib


def set_threads(n: int = 0) -> int:
    """OpenMP threads of the oracle (0 = all host cores / OMP_NUM_THREADS); results are
    independent of the count.  Returns the count in effect."""
    return int(lib().gsref_set_threads(int(n)))


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _params(scene):
    return np.ascontiguousarray(scene.params, dtype=np.float32)


def _check(rc, what):
    if rc != 0:
        raise ValueError(f"oracle {what} rejected its arguments (rc={rc})")


def sh_basis(deg: int, dirs: np.ndarray):
    dirs = np.ascontiguousarray(dirs, dtype=np.float64).reshape(-1, 3)
    n, nk = dirs.shape[0], (deg + 1) ** 2
    Y = np.zeros((n, nk))
    dY = np.zeros((n, nk, 3))
    _check(lib().gsref_sh_basis(deg, n, _p(dirs), _p(Y), _p(dY)), "sh_basis")
    return Y, dY


def project(cam, scene, mode=F32):
    """O1-O8.  Returns dict of arrays over the P Gaussians."""
    P = scene.P
    vals = np.zeros((10, P))
    radius = np.zeros(P, np.int32)
    rect = np.zeros((4, P), np.int32)
    tiles = np.zeros(P, np.int32)
    flags = np.zeros(P, np.uint8)
    rc = ref_camera(cam)
    prm = _params(scene)
    _check(lib().gsref_project(C.byref(rc), P, scene.P_stride, scene.sh_degree, _p(prm), mode,
                               _p(vals), _p(radius), _p(rect), _p(tiles), _p(flags)), "project")
    names = ["mu_x", "mu_y", "z", "conic_A", "conic_B", "conic_C", "opacity", "r", "g", "b"]
    out = {n: vals[i] for i, n in enumerate(names)}
    out.update(vals=vals, radius=radius, rect=rect, tiles=tiles, flags=flags)
    return out


def bin_tiles(cam, scene, capacity=None):
    """O9 (fp32 decisions): sorted_ids, sorted_tiles, tile_ranges [NT,2], K."""
    rc = ref_camera(cam)
    prm = _params(scene)
    pr = project(cam, scene, F32)
    K_est = int(pr["tiles"].astype(np.int64).sum())
    cap = K_est if capacity is None else capacity
    ids = np.zeros(max(cap, 1), np.int32)
    tl = np.zeros(max(cap, 1), np.int32)
    ranges = np.zeros((cam.num_tiles, 2), np.int32)
    K = np.zeros(1, np.int64)
    _check(lib().gsref_bin_tiles(C.byref(rc), scene.P, scene.P_stride, scene.sh_degree, _p(prm), cap,
                                 _p(ids), _p(tl), _p(ranges), _p(K)), "bin_tiles")
    K = int(K[0])
    n = min(K, cap)
    return {"sorted_ids": ids[:n], "sorted_tiles": tl[:n], "tile_ranges": ranges, "K": K}


def render_fwd(cam, scene, mode=F32, want_margin=False, want_signature=False):
    H, W = cam.height, cam.width
    rgb = np.zeros((3, H, W))
    depth = np.zeros((H, W))
    T = np.zeros((H, W))
    n = np.zeros((H, W), np.int32)
    nb = np.zeros(1, np.int64)
    ne = np.zeros(1, np.int64)
    margin = np.zeros((H, W)) if want_margin else None
    sig = np.zeros(1, np.uint64) if want_signature else None
    rc = ref_camera(cam)
    prm = _params(scene)
    _check(lib().gsref_render_fwd(C.byref(rc), scene.P, scene.P_stride, scene.sh_degree, _p(prm), mode,
                                  _p(rgb), _p(depth), _p(T), _p(n), _p(nb), _p(ne), _p(margin), _p(sig)),
           "render_fwd")
    out = {"rgb": rgb, "depth": depth, "T_final": T, "n_contrib": n, "blended": int(nb[0]),
           "evaluated": int(ne[0])}
    if want_margin:
        out["margin"] = margin
    if want_signature:
        out["signature"] = int(sig[0])
    return out


def render_pixels(cam, scene, px, py, mode=F32):
    """O10 at selected pixels (sampled parity at full size)."""
    px = np.ascontiguousarray(px, dtype=np.int32)
    py = np.ascontiguousarray(py, dtype=np.int32)
    n = px.size
    rgb = np.zeros((3, n))
    depth = np.zeros(n)
    T = np.zeros(n)
    nc = np.zeros(n, np.int32)
    margin = np.zeros(n)
    rc = ref_camera(cam)
    prm = _params(scene)
    _check(lib().gsref_render_pixels(C.byref(rc), scene.P, scene.P_stride, scene.sh_degree, _p(prm), mode, n,
                                     _p(px), _p(py), _p(rgb), _p(depth), _p(T), _p(nc), _p(margin)), "render_pixels")
    return {"rgb": rgb, "depth": depth, "T_final": T, "n_contrib": nc, "margin": margin}


def render_bwd(cam, scene, g_rgb, g_depth=None, mode=MIXED):
    """Parameter gradients [F][P] (double) and screen-space grads [10][P]."""
    F, P = scene.F, scene.P
    grad = np.zeros((F, P))
    screen = np.zeros((10, P))
    g_rgb = np.ascontiguousarray(g_rgb, dtype=np.float32)
    g_d = None if g_depth is None else np.ascontiguousarray(g_depth, dtype=np.float32)
    rc = ref_camera(cam)
    prm = _params(scene)
    _check(lib().gsref_render_bwd(C.byref(rc), P, scene.P_stride, scene.sh_degree, _p(prm), mode,
                                  _p(g_rgb), _p(g_d), _p(grad), _p(screen)), "render_bwd")
    return grad, screen


U32 = 2.0 ** -24  # fp32 unit roundoff


def render_bwd_bound(cam, scene, g_rgb, g_depth=None, stage=True):
    """MIXED-mode gradients [F][P] (bit-identical to render_bwd(mode=MIXED)) with their
    first-order running error bounds M [F][P] in units of U32 (see gsref.cpp, struct
    Rn): an fp32 evaluation of the same maths is expected within c * U32 * M.  Also the
    screen-space gradients [10][P] and their bounds."""
    F, P = scene.F, scene.P
    grad = np.zeros((F, P))
    bound = np.zeros((F, P))
    screen = np.zeros((10, P))
    sbound = np.zeros((10, P))
    g_rgb = np.ascontiguousarray(g_rgb, dtype=np.float32)
    g_d = None if g_depth is None else np.ascontiguousarray(g_depth, dtype=np.float32)
    rc = ref_camera(cam)
    prm = _params(scene)
    _check(lib().gsref_render_bwd_bound(C.byref(rc), P, scene.P_stride, scene.sh_degree, _p(prm), int(stage),
                                        _p(g_rgb), _p(g_d),
                                        _p(grad), _p(bound), _p(screen), _p(sbound)), "render_bwd_bound")
    return {"grad": grad, "bound": bound, "screen": screen, "screen_bound": sbound}


def margin_bound(cam, scene, px=None, py=None, stage=True):
    """Per-pixel decision margin in units of the running error bound (min over the
    pixel's skip / cap / stop decisions of |q - threshold| / (U32 m_q)).  px, py: pixel
    coordinates (default: every pixel, returned as [H][W])."""
    full = px is None
    if full:
        yy, xx = np.mgrid[0:cam.height, 0:cam.width]
        px, py = xx.ravel(), yy.ravel()
    px = np.ascontiguousarray(px, dtype=np.int32)
    py = np.ascontiguousarray(py, dtype=np.int32)
    out = np.zeros(px.size)
    rc = ref_camera(cam)
    prm = _params(scene)
    _check(lib().gsref_margin_bound(C.byref(rc), scene.P, scene.P_stride, scene.sh_degree, _p(prm), int(stage), px.size,
                                    _p(px),
                                    _p(py), _p(out)), "margin_bound")
    return out.reshape(cam.height, cam.width) if full else out


def adam_step(params, grad, m, v, lr_per_row, step, beta1=0.9, beta2=0.999, eps=1e-15, P=None):
    F, P_stride = params.shape
    P = P_stride if P is None else P
    out_p = np.zeros((F, P))
    out_m = np.zeros((F, P))
    out_v = np.zeros((F, P))
    args = [np.ascontiguousarray(a, dtype=np.float32) for a in (params, grad, m, v)]
    lr = np.ascontiguousarray(lr_per_row, dtype=np.float32)
    _check(lib().gsref_adam_step(F, P, P_stride, *[_p(a) for a in args], _p(lr), beta1, beta2, eps, step,
                                 _p(out_p), _p(out_m), _p(out_v)), "adam_step")
    return out_p, out_m, out_v


def l1_loss_grad(rgb, depth, t_rgb, t_depth, w_depth=1.0):
    npix = depth.size
    g_rgb = np.zeros(rgb.shape)
    g_d = np.zeros(depth.shape)
    loss = np.zeros(1)
    args = [np.ascontiguousarray(rgb, np.float64), np.ascontiguousarray(depth, np.float64),
            np.ascontiguousarray(t_rgb, np.float32), np.ascontiguousarray(t_depth, np.float32)]
    _check(lib().gsref_l1_loss_grad(npix, *[_p(a) for a in args], w_depth, _p(g_rgb), _p(g_d), _p(loss)),
           "l1_loss_grad")
    return float(loss[0]), g_rgb, g_d
