"""ctypes wrapper of the TSDF-fusion CPU oracle ``oracle/libtsdfref.so`` (TEST
INFRASTRUCTURE).  Only tests/ and bench.py's CPU legs may
import it.  Definitions and citations: ``oracle/tsdf_ref.cpp``."""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "tsdf_ref.cpp")
SANITIZE = os.environ.get("GSREF_SANITIZE") == "1"  # see oracle/gsref.py
SAN_FLAGS = ["-O1", "-g", "-fno-omit-frame-pointer", "-fsanitize=address,undefined", "-fno-sanitize-recover=all"]
LIB = os.path.join(HERE, "libtsdfref_san.so" if SANITIZE else "libtsdfref.so")


def build(force: bool = False) -> str:
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        subprocess.check_call(["g++", *(SAN_FLAGS if SANITIZE else ["-O2"]), "-std=c++17", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared",
                               "-o", LIB + ".tmp", SRC])
        os.replace(LIB + ".tmp", LIB)
    return LIB


class Params(C.Structure):
    _fields_ = [("voxel_size", C.c_float), ("trunc", C.c_float), ("w_max", C.c_float), ("step", C.c_float),
                ("origin", C.c_int32 * 3)]


class Camera(C.Structure):
    _fields_ = [("width", C.c_int32), ("height", C.c_int32),
                ("fx", C.c_float), ("fy", C.c_float), ("cx", C.c_float), ("cy", C.c_float),
                ("R_cw", C.c_float * 9), ("t_cw", C.c_float * 3),
                ("z_near", C.c_float), ("bg", C.c_float * 3)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(LIB)
        L.ref_morton.restype = C.c_uint64
        L.ref_morton.argtypes = [C.c_uint32] * 3
        L.ref_unmorton.argtypes = [C.c_uint64, C.c_void_p]
        L.ref_tsdf_new.restype = C.c_void_p
        L.ref_tsdf_new.argtypes = [C.c_void_p]
        L.ref_tsdf_free.argtypes = [C.c_void_p]
        L.ref_tsdf_num_blocks.restype = C.c_int64
        L.ref_tsdf_num_blocks.argtypes = [C.c_void_p]
        for fn in ("ref_tsdf_allocate", "ref_tsdf_integrate"):
            getattr(L, fn).restype = C.c_int64
            getattr(L, fn).argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
        L.ref_tsdf_dump.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        _lib = L
    return _lib


def params(voxel_size=0.01, trunc=None, w_max=100.0, step=None, origin=(1 << 20,) * 3) -> Params:
    p = Params()
    p.voxel_size = voxel_size
    p.trunc = trunc if trunc is not None else 6 * voxel_size
    p.w_max = w_max
    p.step = step if step is not None else voxel_size / 2
    for a in range(3):
        p.origin[a] = int(origin[a])
    return p


def camera(cam) -> Camera:
    c = Camera()
    c.width, c.height = int(cam.width), int(cam.height)
    c.fx, c.fy, c.cx, c.cy = float(cam.fx), float(cam.fy), float(cam.cx), float(cam.cy)
    R = np.asarray(cam.R_cw, np.float32).reshape(9)
    for i in range(9):
        c.R_cw[i] = float(R[i])
    for i in range(3):
        c.t_cw[i] = float(np.asarray(cam.t_cw, np.float32)[i])
        c.bg[i] = 0.0
    c.z_near = float(cam.z_near)
    return c


def morton(x, y, z) -> int:
    return int(lib().ref_morton(int(x), int(y), int(z)))


def unmorton(m):
    out = (C.c_uint32 * 3)()
    lib().ref_unmorton(int(m), out)
    return tuple(out)


class Volume:
    """The oracle's TSDF volume (std::map of Morton key -> 8^3 block)."""

    def __init__(self, p: Params):
        self.p = p
        self.h = lib().ref_tsdf_new(C.byref(p))

    def __del__(self):
        if getattr(self, "h", None):
            lib().ref_tsdf_free(self.h)
            self.h = None

    def allocate(self, cam, depth) -> int:
        d = np.ascontiguousarray(depth, np.float32)
        return int(lib().ref_tsdf_allocate(self.h, C.byref(camera(cam)), d.ctypes.data_as(C.c_void_p)))

    def integrate(self, cam, depth) -> int:
        d = np.ascontiguousarray(depth, np.float32)
        return int(lib().ref_tsdf_integrate(self.h, C.byref(camera(cam)), d.ctypes.data_as(C.c_void_p)))

    @property
    def num_blocks(self) -> int:
        return int(lib().ref_tsdf_num_blocks(self.h))

    def dump(self):
        """(keys uint64[n] ascending, tsdf float32[n][512], weight float32[n][512])."""
        n = self.num_blocks
        keys = np.zeros(max(n, 1), np.uint64)
        ts = np.zeros((max(n, 1), 512), np.float32)
        ws = np.zeros((max(n, 1), 512), np.float32)
        lib().ref_tsdf_dump(self.h, keys.ctypes.data_as(C.c_void_p), ts.ctypes.data_as(C.c_void_p),
                            ws.ctypes.data_as(C.c_void_p))
        return keys[:n], ts[:n], ws[:n]
