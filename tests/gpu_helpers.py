"""Shared helpers of the -m gpu parity tests (marshalling oracle outputs into the
GPU layouts and back).  Test infrastructure only."""
from __future__ import annotations

import numpy as np
import torch

import scenegen
from oracle import gsref
from paper_2408_12677_b200 import gsr

DEV = torch.device("cuda:0") if torch.cuda.is_available() else None
REC_NAMES = ["mu_x", "mu_y", "z", "opacity", "conic_A", "conic_B", "conic_C", "r", "g", "b"]


def oracle_rec(pr) -> np.ndarray:
    """Oracle fp32 projection -> the GPU's [P][12] record layout (gsr.h)."""
    P = pr["radius"].shape[0]
    rec = np.zeros((max(P, 1), 12), np.float32)
    for k, name in enumerate(REC_NAMES):
        rec[:P, k] = pr[name].astype(np.float32)
    rx = (pr["rect"][0].astype(np.uint32) | (pr["rect"][1].astype(np.uint32) << 16))
    ry = (pr["rect"][2].astype(np.uint32) | (pr["rect"][3].astype(np.uint32) << 16))
    rec[:P, 10] = rx.view(np.float32)
    rec[:P, 11] = ry.view(np.float32)
    return rec


def proj_from_oracle(pr):
    """Device projection buffers filled with the oracle's fp32 projection."""
    P = pr["radius"].shape[0]
    proj, t = gsr.make_proj(P, DEV)
    t["rec"].copy_(torch.from_numpy(oracle_rec(pr)))
    if P:
        t["radius"][:P].copy_(torch.from_numpy(pr["radius"]))
        t["tiles"][:P].copy_(torch.from_numpy(pr["tiles"]))
        t["flags"][:P].copy_(torch.from_numpy(pr["flags"]))
    return proj, t


def gpu_project(lib, cam, scene):
    P = scene.P
    proj, t = gsr.make_proj(P, DEV)
    params = torch.from_numpy(scene.params).to(DEV)
    lib.project(gsr.camera(cam), gsr.scene_desc(P, scene.P_stride, scene.sh_degree), params, proj)
    torch.cuda.synchronize()
    return proj, t, params


def gpu_bin(lib, cam, scene, proj, capacity=None, sync=True):
    K_cap = capacity if capacity is not None else 1 << 16
    while True:
        ws = torch.empty(lib.bin_tiles_workspace(gsr.camera(cam), scene.P, K_cap) // 4 + 4, dtype=torch.int32,
                         device=DEV)
        ids = torch.full((max(K_cap, 1),), -7, dtype=torch.int32, device=DEV)
        ranges = torch.full((cam.num_tiles, 2), -7, dtype=torch.int32, device=DEV)
        kdev = torch.full((1,), -1, dtype=torch.int64, device=DEV)
        K, st = lib.bin_tiles(gsr.camera(cam), gsr.scene_desc(scene.P, scene.P_stride, scene.sh_degree), proj, ws,
                              K_cap, ids, ranges, num_keys_dev=kdev, sync=sync, allow_capacity=True)
        torch.cuda.synchronize()
        if capacity is not None or st == gsr.GS_OK:
            return {"K": K, "status": st, "sorted_ids": ids, "ranges": ranges, "K_dev": int(kdev.item())}
        K_cap = int(K * 1.2) + 64


def gpu_render(lib, cam, scene, proj, ids, ranges, blended=True):
    H, W = cam.height, cam.width
    rgb = torch.full((3, H, W), np.nan, dtype=torch.float32, device=DEV)
    depth = torch.full((H, W), np.nan, dtype=torch.float32, device=DEV)
    T = torch.full((H, W), np.nan, dtype=torch.float32, device=DEV)
    n = torch.full((H, W), -1, dtype=torch.int32, device=DEV)
    b = torch.zeros(1, dtype=torch.int64, device=DEV) if blended else None
    lib.render_fwd(gsr.camera(cam), gsr.scene_desc(scene.P, scene.P_stride, scene.sh_degree), proj, ids, ranges, rgb,
                   depth, T, n, blended=b)
    torch.cuda.synchronize()
    return {"rgb": rgb, "depth": depth, "T_final": T, "n_contrib": n, "blended": int(b.item()) if blended else None}


def gpu_bwd(lib, cam, scene, params, proj, ids, ranges, T, n, g_rgb, g_d):
    P = scene.P
    sc = gsr.scene_desc(P, scene.P_stride, scene.sh_degree)
    ws = torch.full((max(lib.render_bwd_workspace(sc) // 4, 4),), 3.0, dtype=torch.float32, device=DEV)
    grad = torch.zeros((scene.F, scene.P_stride), dtype=torch.float32, device=DEV)
    lib.render_bwd(gsr.camera(cam), sc, params, proj, ids, ranges, T, n,
                   torch.as_tensor(g_rgb, device=DEV), None if g_d is None else torch.as_tensor(g_d, device=DEV), ws,
                   grad)
    torch.cuda.synchronize()
    return grad[:, :P].cpu().numpy().astype(np.float64), ws.view(-1)[:12 * P].view(P, 12).cpu().numpy()




# --------------------------------------------------------------------------- parity tolerance
# Element-wise gradient parity (R42): against the stage-wise reference
# (oracle STAGE mode: fp32 decisions and records, fp64 values) every element must
# satisfy |g - ref| <= max(ATOL * scale, RTOL |ref|, C_TOL * U * M), M the oracle's
# running error bound (oracle/gsref.cpp, struct Rn; pinned against the oracle's own
# fp32 evaluation in tests/test_oracle_bound.py).  Threshold flips: a pixel whose
# decision margin, in units of the bound, is below C_FLIP may legitimately take a
# different decision on the GPU; its upstream gradient is zeroed on both sides and
# its forward values are excused (and counted).
U = 2.0 ** -24
RTOL, ATOL = 1e-3, 1e-6  # north_star
C_TOL = 8.0
C_FLIP = 8.0


def grad_check(g, ref, bound, scale=1.0, c=C_TOL):
    """(bad mask, max ratio |g - ref| / allowed) for the element-wise tolerance."""
    d = np.abs(np.asarray(g, np.float64) - ref)
    allowed = np.maximum(np.maximum(ATOL * scale, RTOL * np.abs(ref)), c * U * bound)
    return d > allowed, float((d / allowed).max()) if d.size else 0.0


def _log_parity(what, g, ref, bound, scale, exclude):
    """GSR_PARITY_LOG=path: append one JSON line per check (worst ratio, how many
    elements the bound term relaxed) -- the evidence behind profiles/*/parity_*.txt."""
    import json
    import os
    path = os.environ.get("GSR_PARITY_LOG")
    if not path:
        return
    g = np.asarray(g, np.float64)
    d = np.abs(g - ref)
    base = np.maximum(ATOL * scale, RTOL * np.abs(ref))
    allowed = np.maximum(base, C_TOL * U * bound)
    keep = np.ones_like(d, bool) if exclude is None else ~exclude
    rec = {"test": os.environ.get("PYTEST_CURRENT_TEST", "?").split(" ")[0], "what": what,
           "elements": int(keep.sum()), "nonzero_ref": int(np.count_nonzero(ref[keep])),
           "worst_ratio": float((d / allowed)[keep].max()) if keep.any() else 0.0,
           "worst_ratio_vs_u_M": float((d / np.maximum(U * bound, 1e-300))[keep & (d > 0)].max())
           if (keep & (d > 0)).any() else 0.0,
           "outside_north_star_tol": int(((d > base) & keep).sum()),
           "relaxed_by_bound": int(((C_TOL * U * bound > base) & keep).sum()),
           "excluded": int((~keep).sum())}
    with open(path, "a") as f:
        f.write(json.dumps(rec) + "\n")


def assert_grad_parity(g, ref, bound, scale=1.0, what="gradient", exclude=None):
    _log_parity(what, g, ref, bound, scale, exclude)
    bad, worst = grad_check(g, ref, bound, scale)
    if exclude is not None:
        bad &= ~exclude
    if bad.any():
        k = np.argwhere(bad)[:5]
        det = [(tuple(int(x) for x in kk), float(np.asarray(g)[tuple(kk)]), float(ref[tuple(kk)]),
                float(U * bound[tuple(kk)])) for kk in k]
        raise AssertionError(f"{what}: {int(bad.sum())}/{bad.size} elements outside max(atol, rtol|ref|, "
                             f"{C_TOL} u M); (index, gpu, ref, u M): {det}")
    return worst


def flip_pixels(cam, scene, px=None, py=None):
    """Pixels whose decisions are within C_FLIP error bounds of a threshold."""
    return gsref.margin_bound(cam, scene, px, py) < C_FLIP
