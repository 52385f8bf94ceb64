"""Parity report (run on the GPU box): GPU vs CPU oracle on the same seeded inputs for
every BASELINE config, with the numbers the tests only assert on -- written to
profiles/<round>/parity_report.txt.  Test infrastructure (imports oracle/).

Per config (view 0):
  projection: radius / tiles / rect / mu / z / conic / opacity mismatches (must be 0),
              max |colour - oracle|;
  binning:    K, sorted-id and tile-range mismatches (must be 0);
  forward:    stage-wise on 3000 sampled pixels (all pixels for tiny / small): max abs
              rgb / depth error, n_contrib mismatches, threshold flips (oracle decision
              margin < 1e-5) and unexplained mismatches (must be 0);
  backward:   upstream N(0,1) on 64 sampled tiles (all pixels for tiny / small):
              fraction of gradient elements outside rel 1e-3 / abs 1e-6, worst rel err.
"""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import scenegen  # noqa: E402
from oracle import gsref  # noqa: E402
from paper_2408_12677_b200 import gsr  # noqa: E402
from gpu_helpers import DEV, gpu_bin, gpu_bwd, gpu_project, gpu_render, grad_mismatch, proj_from_oracle  # noqa: E402

FLIP = 1e-5


def report(name, out):
    lib = gsr.load()
    kw = {"num_views": 1} if name in ("replica", "scannetpp", "large") else {}
    w = scenegen.make(name, **kw)
    cam, scene = w.cameras[0], w.scene
    t0 = time.time()
    ref = gsref.project(cam, scene, gsref.F32)
    proj, t, params = gpu_project(lib, cam, scene)
    P = scene.P
    vis = ref["radius"] > 0
    rec = t["rec"][:P].cpu().numpy()
    mism = int((t["radius"][:P].cpu().numpy() != ref["radius"]).sum() + (t["tiles"][:P].cpu().numpy() != ref["tiles"]).sum())
    for k, nm in enumerate(["mu_x", "mu_y", "z", "opacity", "conic_A", "conic_B", "conic_C"]):
        mism += int((rec[vis, k] != ref[nm][vis].astype(np.float32)).sum())
    col = max(float(np.abs(rec[vis, 7 + c] - ref[nm][vis]).max()) for c, nm in enumerate("rgb"))
    out.append(f"[{name}] P={P} visible={int(vis.sum())}")
    out.append(f"  projection: integer/geometry mismatches {mism}, max |colour err| {col:.2e}")
    rb = gsref.bin_tiles(cam, scene)
    b = gpu_bin(lib, cam, scene, proj_from_oracle(ref)[0])
    K = b["K"]
    id_mm = int((b["sorted_ids"][:K].cpu().numpy() != rb["sorted_ids"]).sum()) if K == rb["K"] else -1
    rg_mm = int((b["ranges"].cpu().numpy() != rb["tile_ranges"]).sum())
    out.append(f"  binning: K gpu {K} oracle {rb['K']}, sorted-id mismatches {id_mm}, range mismatches {rg_mm}")
    # forward, stage-wise (oracle projection and lists)
    pr_proj, _ = proj_from_oracle(ref)
    ids = torch.from_numpy(np.ascontiguousarray(rb["sorted_ids"])).to(DEV)
    ranges = torch.from_numpy(rb["tile_ranges"]).to(DEV)
    f = gpu_render(lib, cam, scene, pr_proj, ids, ranges)
    small = name in ("tiny", "small")
    if small:
        rf = gsref.render_fwd(cam, scene, gsref.F32, want_margin=True)
        rgb, dep, n = f["rgb"].cpu().numpy(), f["depth"].cpu().numpy(), f["n_contrib"].cpu().numpy()
        e_rgb = np.abs(rgb - rf["rgb"]).max(0)
        e_dep = np.abs(dep - rf["depth"])
        nmm = n != rf["n_contrib"]
        margin = rf["margin"]
        npx = rgb.shape[1] * rgb.shape[2]
    else:
        rng = np.random.default_rng(0)
        px, py = rng.integers(0, cam.width, 3000), rng.integers(0, cam.height, 3000)
        rf = gsref.render_pixels(cam, scene, px, py, gsref.F32)
        e_rgb = np.abs(f["rgb"].cpu().numpy()[:, py, px] - rf["rgb"]).max(0)
        e_dep = np.abs(f["depth"].cpu().numpy()[py, px] - rf["depth"])
        nmm = f["n_contrib"].cpu().numpy()[py, px] != rf["n_contrib"]
        margin = rf["margin"]
        npx = cam.width * cam.height
    bad = (e_rgb > 1e-5) | (e_dep > 1e-5 * np.maximum(1.0, np.abs(rf["depth"]))) | nmm
    flips = bad & (margin < FLIP)
    out.append(f"  forward ({'all' if small else '3000 sampled'} of {npx} px): max |rgb err| {e_rgb.max():.2e}, "
               f"max |depth err| {e_dep.max():.2e}, n_contrib mismatches {int(nmm.sum())}, "
               f"threshold flips {int(flips.sum())}, unexplained {int((bad & ~flips).sum())}")
    # backward, stage-wise, on sampled tiles (MIXED oracle)
    rfw = gsref.render_fwd(cam, scene, gsref.F32, want_margin=True) if small else None
    g_rgb, g_d = scenegen.upstream_fields(1, cam.width, cam.height)
    if small:
        keep = ~(rfw["margin"] < FLIP)
        T = torch.from_numpy(rfw["T_final"].astype(np.float32)).to(DEV)
        nc = torch.from_numpy(rfw["n_contrib"]).to(DEV)
    else:
        rng = np.random.default_rng(3)
        keep = np.zeros((cam.height, cam.width), bool)
        for tt in rng.choice(cam.num_tiles, 64, replace=False):
            ty, tx = divmod(int(tt), cam.tiles_x)
            keep[ty * 16:(ty + 1) * 16, tx * 16:(tx + 1) * 16] = True
        T, nc = f["T_final"], f["n_contrib"]
        # flip pixels of the sampled tiles (oracle decision margin) carry no upstream
        ys, xs = np.nonzero(keep)
        mr = gsref.render_pixels(cam, scene, xs, ys, gsref.F32)["margin"]
        keep[ys[mr < FLIP], xs[mr < FLIP]] = False
    g_rgb = (g_rgb * keep[None]).astype(np.float32)
    g_d = (g_d * keep).astype(np.float32)
    g, _ = gpu_bwd(lib, cam, scene, params, pr_proj, ids, ranges, T, nc, g_rgb, g_d)
    gref, _ = gsref.render_bwd(cam, scene, g_rgb, g_d, mode=gsref.MIXED)
    bm = grad_mismatch(g, gref)
    rel = np.abs(g - gref) / np.maximum(np.abs(gref), 1e-6)
    out.append(f"  backward ({'all pixels' if small else '64 sampled tiles'}): {bm.size} gradient elements, "
               f"outside rel 1e-3 / abs 1e-6: {int(bm.sum())} ({bm.mean():.1e}), median rel err {np.median(rel[np.abs(gref) > 1e-6]):.1e}")
    out.append(f"  ({time.time() - t0:.0f} s)")


def main():
    names = sys.argv[1:] or ["tiny", "small", "replica", "scannetpp", "large"]
    out = [f"# parity report ({torch.cuda.get_device_name(0)}), GPU vs CPU oracle, view 0 of each config"]
    for nm in names:
        report(nm, out)
        print("\n".join(out[-6:]), flush=True)
    path = os.path.join(ROOT, "gpurun_out", "parity_report.txt")
    os.makedirs(os.path.dirname(path), exist_ok=True)
    open(path, "w").write("\n".join(out) + "\n")


if __name__ == "__main__":
    main()
