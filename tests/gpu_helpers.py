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


def grad_mismatch(g, ref, rtol=1e-3, atol=1e-6):
    """Elements failing 'rel < rtol OR abs < atol' (north_star tolerance)."""
    d = np.abs(g - ref)
    return ~((d <= atol) | (d <= rtol * np.abs(ref)))
