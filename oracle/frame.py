"""Oracle of the input-frame decode -- TEST INFRASTRUCTURE.

Only tests/, __graft_entry__.smoke() and bench.py's reference legs may import this
module.  Plain definition, independent of the CUDA path (paper_2408_12677_b200/csrc/
frame.cu):

PAPER.md:58 (Fig. 2): "At each time step, it takes a pair of RGB-D images as input."
SPEC.md:463: a frame holds "rgb: H x W x 3 8-bit image; depth: H x W depth image (16-bit
units x depth_scale -> meters, 0 = invalid)"; "depth_scale: multiplier
converting stored depth units to meters"; SPEC.md:265 uses colour as rgb / 255.
Reading R41: colour = value / 255 and depth = units x depth_scale, each
one IEEE float32 operation (correctly rounded), rgb re-laid out as planes [3][H][W].
"""
from __future__ import annotations

import numpy as np

F32 = np.float32


def decode_rgbd(rgb_u8, depth_u16, depth_scale):
    """rgb_u8 uint8 [H][W][3], depth_u16 uint16 [H][W] -> (float32 [3][H][W], float32 [H][W])."""
    rgb = np.asarray(rgb_u8, np.uint8)
    dep = np.asarray(depth_u16, np.uint16)
    planes = np.transpose(rgb, (2, 0, 1)).astype(F32) / F32(255.0)
    depth = dep.astype(F32) * F32(depth_scale)
    return np.ascontiguousarray(planes, F32), depth.astype(F32)
