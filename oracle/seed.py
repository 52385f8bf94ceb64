"""Oracle of GSFusion's quadtree seeding and weight-gated Gaussian initialisation --
TEST INFRASTRUCTURE.  Only tests/ may import it.

Plain definitions written from the paper, independent of the CUDA path
(paper_2408_12677_b200/csrc/seed.cu):

PAPER.md:127 (§III-B2): "we divide the image based on contrast so that each leaf node
contains a specific subregion with its contrast lower than a pre-defined threshold";
"each node in the tree having either exactly four children or none at all".
Readings: R37 contrast = max - min of luminance L = 0.299 R + 0.587 G +
0.114 B over the cell, cells split at integer halves (NW, NE, SW, SE)
while both sides exceed min_cell; leaves listed depth first.

PAPER.md:129-133, Eq. 10: p_q = T_WC pi^-1(u_q, D_k[u_q]); "we simply query the nearest
voxel to p_q.  If the voxel weight is equal to 1 [...] initialize a new 3D Gaussian":
R_q = I, S_q = diag(d, d, d) with d "the back-projected length from the quadrant center
to its corners", alpha_q = 0.5, colour = I_k[u_q] (SH DC).  Readings R38 (centre pixel
(x + w/2, y + h/2), corner (x, y)), R39 (the voxel containing p_q), R40 (fuse first).
Arithmetic in float32 with one rounded operation per step, as the GPU (R9).
"""
from __future__ import annotations

import math

import numpy as np

F32 = np.float32
Y00 = F32(0.28209479177387814)


def luminance(rgb):
    """L = (0.299 R + 0.587 G) + 0.114 B in float32; rgb [3][H][W]."""
    r, g, b = (np.asarray(rgb[c], F32) for c in range(3))
    return (F32(0.299) * r + F32(0.587) * g) + F32(0.114) * b


def quadtree(rgb, threshold, min_cell):
    """Depth-first (NW, NE, SW, SE) list of leaves (x, y, w, h)."""
    L = luminance(rgb)
    H, W = L.shape
    leaves = []

    def visit(x, y, w, h):
        cell = L[y:y + h, x:x + w]
        contrast = F32(cell.max()) - F32(cell.min())
        if w > min_cell and h > min_cell and contrast > F32(threshold):
            hw, hh = w // 2, h // 2
            visit(x, y, hw, hh)
            visit(x + hw, y, w - hw, hh)
            visit(x, y + hh, hw, h - hh)
            visit(x + hw, y + hh, w - hw, h - hh)
        else:
            leaves.append((x, y, w, h))

    visit(0, 0, W, H)
    return leaves


def seed(leaves, cam, depth, rgb, vol_keys, vol_weight, voxel_size, origin, sh_degree):
    """Gaussians initialised from the leaves, in leaf order.  vol_keys / vol_weight: the
    oracle TSDF volume's dump (Morton keys ascending, weights [n][512]) AFTER fusing the
    frame.  Returns a float32 parameter block [F][n_new]."""
    from oracle import tsdf as T
    index = {int(k): i for i, k in enumerate(vol_keys)}
    R = np.asarray(cam.R_cw, F32).reshape(3, 3)
    t = np.asarray(cam.t_cw, F32).reshape(3)
    inv_vs = F32(1.0) / F32(voxel_size)
    F = 11 + 3 * (sh_degree + 1) ** 2
    cols = []
    for (x, y, w, h) in leaves:
        u, v = x + w // 2, y + h // 2
        d = F32(depth[v, u])
        if not d > 0:
            continue
        rx = (F32(u) - F32(cam.cx)) / F32(cam.fx)
        ry = (F32(v) - F32(cam.cy)) / F32(cam.fy)
        pc = np.array([rx * d, ry * d, d], F32)
        q = pc - t
        p = np.zeros(3, F32)
        for a in range(3):  # p = R^T (p_c - t)
            p[a] = (R[0, a] * q[0] + R[1, a] * q[1]) + R[2, a] * q[2]
        vox = [int(np.floor(p[a] * inv_vs)) + int(origin[a]) for a in range(3)]
        if any(c < 0 or c >= (1 << 21) for c in vox):
            continue
        key = T.morton(vox[0] >> 3, vox[1] >> 3, vox[2] >> 3)
        if key not in index:
            continue
        loc = (vox[0] & 7) + 8 * (vox[1] & 7) + 64 * (vox[2] & 7)
        if vol_weight[index[key], loc] != F32(1.0):
            continue
        cx0 = ((F32(x) - F32(cam.cx)) / F32(cam.fx)) * d
        cy0 = ((F32(y) - F32(cam.cy)) / F32(cam.fy)) * d
        dx, dy = pc[0] - cx0, pc[1] - cy0
        s = np.sqrt(dx * dx + dy * dy, dtype=F32)
        if not s > 0:
            continue
        col = np.zeros(F, F32)
        col[0:3] = p
        col[3:6] = F32(math.log(float(s)))
        col[6] = 1.0
        for c in range(3):
            col[11 + c] = (F32(rgb[c][v, u]) - F32(0.5)) / Y00
        cols.append(col)
    return np.stack(cols, axis=1) if cols else np.zeros((F, 0), F32)
