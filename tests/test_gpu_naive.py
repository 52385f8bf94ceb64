"""Parity of the K13 comparison baseline (gs_naive_render_fwd / gs_naive_render_bwd_screen,
the per-pixel port the north_star's >= 10x target is measured against) with the CPU
oracle, stage-wise, same tolerances and flip accounting as the product calls
(tests/test_gpu_parity.py).  The ratio bench.py reports is only meaningful if both
arms compute the same thing."""
import numpy as np
import pytest
import torch

import scenegen
from oracle import gsref

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_2408_12677_b200 import gsr
    from gpu_helpers import DEV, assert_grad_parity, flip_pixels, proj_from_oracle



@pytest.fixture(scope="module")
def lib():
    return gsr.load()


def _inputs(name):
    w = scenegen.make(name)
    cam, scene = w.cameras[0], w.scene
    pr = gsref.project(cam, scene, gsref.F32)
    b = gsref.bin_tiles(cam, scene)
    proj, _ = proj_from_oracle(pr)
    ids = torch.from_numpy(np.ascontiguousarray(b["sorted_ids"])).to(DEV)
    ranges = torch.from_numpy(b["tile_ranges"]).to(DEV)
    return cam, scene, proj, ids, ranges


@pytest.mark.parametrize("name", ["tiny", "small"])
def test_naive_fwd_parity(lib, name):
    cam, scene, proj, ids, ranges = _inputs(name)
    H, W = cam.height, cam.width
    rgb = torch.full((3, H, W), np.nan, device=DEV)
    dep = torch.full((H, W), np.nan, device=DEV)
    T = torch.full((H, W), np.nan, device=DEV)
    n = torch.full((H, W), -1, dtype=torch.int32, device=DEV)
    bl = torch.zeros(1, dtype=torch.int64, device=DEV)
    lib.naive_render_fwd(gsr.camera(cam), gsr.scene_desc(scene.P, scene.P_stride, scene.sh_degree), proj, ids, ranges,
                         rgb, dep, T, n, blended=bl)
    torch.cuda.synchronize()
    ref = gsref.render_fwd(cam, scene, gsref.F32)
    bad = ((np.abs(rgb.cpu().numpy() - ref["rgb"]).max(0) > 1e-5) | (np.abs(dep.cpu().numpy() - ref["depth"]) > 1e-5)
           | (n.cpu().numpy() != ref["n_contrib"]))
    flips = flip_pixels(cam, scene)
    assert (bad & ~flips).sum() == 0
    assert abs(int(bl.item()) - ref["blended"]) <= 4 * int(flips.sum())


@pytest.mark.parametrize("name", ["tiny", "small"])
def test_naive_bwd_parity(lib, name):
    cam, scene, proj, ids, ranges = _inputs(name)
    f = gsref.render_fwd(cam, scene, gsref.F32)
    g_rgb, g_d = scenegen.upstream_fields(1, cam.width, cam.height)
    keep = ~flip_pixels(cam, scene)
    g_rgb = (g_rgb * keep[None]).astype(np.float32)
    g_d = (g_d * keep).astype(np.float32)
    P = scene.P
    sc = gsr.scene_desc(P, scene.P_stride, scene.sh_degree)
    T = torch.from_numpy(f["T_final"].astype(np.float32)).to(DEV)
    n = torch.from_numpy(f["n_contrib"]).to(DEV)
    sgrad = torch.zeros((P, gsr.SGRAD_FLOATS), device=DEV)
    lib.naive_render_bwd_screen(gsr.camera(cam), sc, proj, ids, ranges, T, n, torch.from_numpy(g_rgb).to(DEV),
                                torch.from_numpy(g_d).to(DEV), sgrad)
    grad = torch.zeros((scene.F, scene.P_stride), device=DEV)
    params = torch.from_numpy(scene.params).to(DEV)
    lib.project_bwd_views([gsr.camera(cam)], sc, params, [proj._tensors["flags"]], [sgrad], grad, accumulate=True)
    torch.cuda.synchronize()
    ref = gsref.render_bwd_bound(cam, scene, g_rgb, g_d)
    assert_grad_parity(grad[:, :P].cpu().numpy().astype(np.float64), ref["grad"], ref["bound"])
    assert torch.count_nonzero(sgrad) == 0  # consumed and cleared by the projection backward
