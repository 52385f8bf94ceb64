"""Scenes built to put decisions on their thresholds (test infrastructure).

near_skip_scene: isolated isotropic Gaussians, each centred on a pixel, whose opacity
is tuned (with the oracle's fp32 projection, the records every fp32 implementation
composites, R9) so that alpha = o exp(power) at the pixel two columns to the right
equals 1/255 up to a relative offset of a few 1e-7: any two fp32 evaluations (the
oracle's, a GPU's) may take different skip decisions (R15) there, and the fp64
decision (on the unrounded records) differs from the fp32 one on some of them.  Used to show that every mismatch the margins must explain is
actually flagged by them (tests/test_oracle_bound.py, tests/test_gpu_parity.py).
"""
from __future__ import annotations

import math

import numpy as np

import scenegen
from oracle import gsref


def near_skip_scene(seed: int, n: int = 12, width: int = 96, height: int = 64, f: float = 60.0):
    rng = np.random.default_rng(seed)
    cam = scenegen.identity_camera(width, height, f, width / 2.0, height / 2.0)
    z = 3.0
    means, pix = [], []
    tx, ty = width // 16, height // 16
    cells = rng.choice(tx * ty, n, replace=False)
    for c in cells:
        cy_t, cx_t = divmod(int(c), tx)
        u, v = cx_t * 16 + 5, cy_t * 16 + 8
        means.append([(u - cam.cx) * z / f, (v - cam.cy) * z / f, z])
        pix.append((u + 2, v))
    sh = np.zeros((n, 1, 3))
    sh[:, 0] = (np.array([0.6, 0.4, 0.8]) - 0.5) / 0.28209479177387814
    logs = np.full((n, 3), math.log(0.04))
    scene = scenegen.scene_from_gaussians(means, logs, [[1, 0, 0, 0]] * n, np.zeros(n), sh, 0)
    pr = gsref.project(cam, scene, gsref.F32)
    logits = []
    for i, (px, py) in enumerate(pix):
        dx, dy = pr["mu_x"][i] - px, pr["mu_y"][i] - py
        pw = -0.5 * (pr["conic_A"][i] * dx * dx + pr["conic_C"][i] * dy * dy) - pr["conic_B"][i] * dx * dy
        o = (1.0 / 255.0) * math.exp(-pw) * (1.0 + rng.uniform(-4e-7, 4e-7))
        logits.append(math.log(o / (1.0 - o)))
    scene = scenegen.scene_from_gaussians(means, logs, [[1, 0, 0, 0]] * n, logits, sh, 0)
    return scene, cam, pix
