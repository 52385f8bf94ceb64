"""GPU-vs-oracle parity through the C ABI (-m gpu).

Stage-wise parity is binding (SURVEY.md §8(c) parity policy): each GPU call is
fed the ORACLE's outputs of the previous stage on identical seeded inputs.
  gs_project    bit-exact radius, tiles, rect, mu, z, conic, opacity; colour 1e-6
  gs_bin_tiles  bit-exact sorted ids, tile ranges, K
  gs_render_fwd 1e-5 absolute rgb/depth, exact n_contrib, except proven threshold
                flips (the pixel's decision margin is below C_FLIP running error
                bounds, gpu_helpers.flip_pixels); the GSR_EXACT_EXP build is
                bit-identical
  gs_render_bwd EVERY gradient element within max(1e-6, 1e-3 |ref|, C_TOL u M)
                of the stage-wise oracle (STAGE: fp32 decisions and records, fp64
                values; M its running error bound), no fraction allowance; pixels
                with a proven flip have their upstream gradient zeroed on both sides
  gs_adam_step  1e-6 relative
Full-size configs are checked on sampled pixels / sampled upstream gradients.
"""
import numpy as np
import pytest
import torch

import scenegen
from oracle import gsref

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_2408_12677_b200 import gsr, pipeline
    from gpu_helpers import (DEV, assert_grad_parity, flip_pixels, gpu_bin, gpu_bwd, gpu_project, gpu_render,
                             proj_from_oracle)
    from threshold_scenes import near_skip_scene


@pytest.fixture(scope="module")
def lib():
    return gsr.load()


@pytest.fixture(scope="module")
def lib_exact():
    return gsr.load(exact=True)


_WL = {}


def workload(name):
    if name not in _WL:
        kw = {}
        if name == "replica":
            kw = {"num_views": 2}
        if name == "large":
            kw = {"num_views": 2}
        _WL[name] = scenegen.make(name, **kw)
    return _WL[name]


def test_libraries_load(lib, lib_exact):
    assert not lib.exact and lib_exact.exact
    assert lib.lib.gs_version() == 2


# ----------------------------------------------------------------------------- gs_project
@pytest.mark.parametrize("name", ["tiny", "small", "replica", "scannetpp", "large"])
def test_project_bitexact(lib, name):
    w = workload(name)
    cam, scene = w.cameras[0], w.scene
    ref = gsref.project(cam, scene, gsref.F32)
    proj, t, _ = gpu_project(lib, cam, scene)
    P = scene.P
    radius = t["radius"][:P].cpu().numpy()
    tiles = t["tiles"][:P].cpu().numpy()
    flags = t["flags"][:P].cpu().numpy()
    np.testing.assert_array_equal(radius, ref["radius"])
    np.testing.assert_array_equal(tiles, ref["tiles"])
    vis = ref["radius"] > 0
    assert vis.sum() > 0
    np.testing.assert_array_equal(flags & 0xF8, ref["flags"] & 0xF8)  # cull + J clamps exact
    rec = t["rec"][:P].cpu().numpy()
    for k, nm in enumerate(["mu_x", "mu_y", "z", "opacity", "conic_A", "conic_B", "conic_C"]):
        np.testing.assert_array_equal(rec[vis, k], ref[nm][vis].astype(np.float32), err_msg=nm)
    rx = rec[vis, 10].view(np.uint32)
    ry = rec[vis, 11].view(np.uint32)
    np.testing.assert_array_equal(rx & 0xFFFF, ref["rect"][0][vis])
    np.testing.assert_array_equal(rx >> 16, ref["rect"][1][vis])
    np.testing.assert_array_equal(ry & 0xFFFF, ref["rect"][2][vis])
    np.testing.assert_array_equal(ry >> 16, ref["rect"][3][vis])
    for k, nm in zip((7, 8, 9), "rgb"):
        np.testing.assert_allclose(rec[vis, k], ref[nm][vis], atol=1e-6, rtol=0, err_msg=nm)
    # colour clamp flags exact except where the unclamped value is within 1e-6 of 0
    diff = (flags ^ ref["flags"]) & 0x7
    assert np.all(diff[~vis] == 0)
    for ch, nm in enumerate("rgb"):
        d = ((diff >> ch) & 1).astype(bool) & vis
        assert np.all(np.abs(ref[nm][d]) <= 1e-6)


# ----------------------------------------------------------------------------- gs_bin_tiles
@pytest.mark.parametrize("name", ["tiny", "small", "replica", "scannetpp", "large"])
def test_bin_bitexact_stagewise(lib, name):
    w = workload(name)
    cam, scene = w.cameras[0], w.scene
    pr = gsref.project(cam, scene, gsref.F32)
    ref = gsref.bin_tiles(cam, scene)
    proj, _ = proj_from_oracle(pr)
    out = gpu_bin(lib, cam, scene, proj)
    K = out["K"]
    assert K == ref["K"] == out["K_dev"]
    np.testing.assert_array_equal(out["sorted_ids"][:K].cpu().numpy(), ref["sorted_ids"])
    np.testing.assert_array_equal(out["ranges"].cpu().numpy(), ref["tile_ranges"])


def test_bin_depth_ties_and_one_pass_tile_sort(lib):
    """Equal depths fall back to the index (R12); <= 256 tiles use one radix pass."""
    scene, cam = scenegen.random_small_scene(4, 300, 1, width=96, height=80, f=80.0)
    scene.params[2, :150] = scene.params[2, 0]  # 150 exactly-equal depths
    proj, _, _ = gpu_project(lib, cam, scene)
    out = gpu_bin(lib, cam, scene, proj)
    ref = gsref.bin_tiles(cam, scene)
    assert out["K"] == ref["K"]
    np.testing.assert_array_equal(out["sorted_ids"][:out["K"]].cpu().numpy(), ref["sorted_ids"])


def test_bin_capacity_overflow(lib):
    w = workload("small")
    cam, scene = w.cameras[0], w.scene
    proj, _, _ = gpu_project(lib, cam, scene)
    K_true = int(gsref.project(cam, scene)["tiles"].sum())
    out = gpu_bin(lib, cam, scene, proj, capacity=K_true - 1, sync=True)
    assert out["status"] == gsr.GS_ERR_CAPACITY and out["K"] == K_true
    r = out["ranges"].cpu().numpy()
    assert np.all(r[:, 1] - r[:, 0] == 0)  # every tile empty -> background only
    out = gpu_bin(lib, cam, scene, proj, capacity=K_true - 1, sync=False)  # async mode reports K on device
    assert out["K_dev"] == K_true and out["status"] == gsr.GS_OK
    out = gpu_bin(lib, cam, scene, proj, capacity=K_true, sync=True)
    assert out["status"] == gsr.GS_OK and out["K"] == K_true


# ----------------------------------------------------------------------------- gs_render_fwd
def _fwd_stagewise(lib, cam, scene):
    pr = gsref.project(cam, scene, gsref.F32)
    b = gsref.bin_tiles(cam, scene)
    proj, _ = proj_from_oracle(pr)
    ids = torch.from_numpy(np.ascontiguousarray(b["sorted_ids"])).to(DEV) if b["K"] else torch.zeros(1, dtype=torch.int32, device=DEV)
    ranges = torch.from_numpy(b["tile_ranges"]).to(DEV)
    return proj, ids, ranges, gpu_render(lib, cam, scene, proj, ids, ranges)


@pytest.mark.parametrize("name", ["tiny", "small"])
def test_render_fwd_exact_build_bitexact(lib_exact, name):
    w = workload(name)
    cam, scene = w.cameras[0], w.scene
    ref = gsref.render_fwd(cam, scene, gsref.F32)
    _, _, _, out = _fwd_stagewise(lib_exact, cam, scene)
    np.testing.assert_array_equal(out["rgb"].cpu().numpy(), ref["rgb"].astype(np.float32))
    np.testing.assert_array_equal(out["depth"].cpu().numpy(), ref["depth"].astype(np.float32))
    np.testing.assert_array_equal(out["T_final"].cpu().numpy(), ref["T_final"].astype(np.float32))
    np.testing.assert_array_equal(out["n_contrib"].cpu().numpy(), ref["n_contrib"])
    assert out["blended"] == ref["blended"]


@pytest.mark.parametrize("name", ["tiny", "small"])
def test_render_fwd_parity_with_flip_accounting(lib, name):
    w = workload(name)
    cam, scene = w.cameras[0], w.scene
    ref = gsref.render_fwd(cam, scene, gsref.F32)
    _, _, _, out = _fwd_stagewise(lib, cam, scene)
    rgb = out["rgb"].cpu().numpy()
    dep = out["depth"].cpu().numpy()
    n = out["n_contrib"].cpu().numpy()
    bad = (np.abs(rgb - ref["rgb"]).max(0) > 1e-5) | (np.abs(dep - ref["depth"]) > 1e-5) | (n != ref["n_contrib"])
    flagged = flip_pixels(cam, scene)
    unexplained = bad & ~flagged
    assert unexplained.sum() == 0, f"{int(unexplained.sum())} pixels off without a threshold flip"
    assert flagged.sum() <= max(2, 1e-3 * bad.size)
    T = out["T_final"].cpu().numpy()
    assert T.min() >= 1e-4 and T.max() <= 1.0  # R16 invariant on the GPU path


@pytest.mark.parametrize("name", ["replica", "scannetpp", "large"])
def test_render_fwd_sampled_full_size(lib, name):
    """Full-size config, GPU chain project -> bin -> fwd (the bench launch), checked
    on 3000 sampled pixels (random + two complete tiles + the ragged last row/col)."""
    w = workload(name)
    cam, scene = w.cameras[0], w.scene
    proj, _, _ = gpu_project(lib, cam, scene)
    b = gpu_bin(lib, cam, scene, proj)
    out = gpu_render(lib, cam, scene, proj, b["sorted_ids"], b["ranges"])
    rng = np.random.default_rng(0)
    px = list(rng.integers(0, cam.width, 2000))
    py = list(rng.integers(0, cam.height, 2000))
    for tx, ty in ((cam.tiles_x // 2, cam.tiles_y // 2), (cam.tiles_x - 1, cam.tiles_y - 1)):
        for j in range(16):
            for i in range(16):
                x, y = tx * 16 + i, ty * 16 + j
                if x < cam.width and y < cam.height:
                    px.append(x)
                    py.append(y)
    px, py = np.array(px), np.array(py)
    ref = gsref.render_pixels(cam, scene, px, py, gsref.F32)
    rgb = out["rgb"].cpu().numpy()[:, py, px]
    dep = out["depth"].cpu().numpy()[py, px]
    n = out["n_contrib"].cpu().numpy()[py, px]
    # depth is unnormalised (z * alpha * T sums up to ~10 m): 1e-5 absolute on rgb, 1e-5 relative on depth
    bad = (np.abs(rgb - ref["rgb"]).max(0) > 1e-5) | (np.abs(dep - ref["depth"]) > 1e-5 * np.maximum(1.0, np.abs(ref["depth"]))) | (n != ref["n_contrib"])
    unexplained = bad & ~flip_pixels(cam, scene, px, py)
    assert unexplained.sum() == 0, f"{int(unexplained.sum())} sampled pixels off without a flip"


# ----------------------------------------------------------------------------- gs_render_bwd
def _bwd_stagewise(lib, cam, scene, seed=1, sample_mask=None, screen=False):
    """gs_render_bwd fed the oracle's fp32 projection, lists, T_final and n_contrib;
    reference: the STAGE oracle with running error bounds.  Flip pixels (and pixels
    outside sample_mask) get zero upstream on both sides."""
    pr = gsref.project(cam, scene, gsref.F32)
    b = gsref.bin_tiles(cam, scene)
    f = gsref.render_fwd(cam, scene, gsref.F32)
    g_rgb, g_d = scenegen.upstream_fields(seed, cam.width, cam.height)
    keep = np.ones((cam.height, cam.width), bool) if sample_mask is None else sample_mask.copy()
    ys, xs = np.nonzero(keep)
    flips = np.zeros_like(keep)
    flips[ys, xs] = flip_pixels(cam, scene, xs, ys)
    keep &= ~flips
    g_rgb = (g_rgb * keep[None]).astype(np.float32)
    g_d = (g_d * keep).astype(np.float32)
    proj, _ = proj_from_oracle(pr)
    ids = torch.from_numpy(np.ascontiguousarray(b["sorted_ids"])).to(DEV)
    ranges = torch.from_numpy(b["tile_ranges"]).to(DEV)
    T = torch.from_numpy(f["T_final"].astype(np.float32)).to(DEV)
    n = torch.from_numpy(f["n_contrib"]).to(DEV)
    params = torch.from_numpy(scene.params).to(DEV)
    g, ws = gpu_bwd(lib, cam, scene, params, proj, ids, ranges, T, n, g_rgb, g_d)
    if screen:
        sg = torch.zeros((scene.P, 12), dtype=torch.float32, device=DEV)
        lib.render_bwd_screen(gsr.camera(cam), gsr.scene_desc(scene.P, scene.P_stride, scene.sh_degree), proj, ids,
                              ranges, T, n, torch.from_numpy(g_rgb).to(DEV), torch.from_numpy(g_d).to(DEV), sg)
        torch.cuda.synchronize()
        ws = sg.cpu().numpy().astype(np.float64)
    ref = gsref.render_bwd_bound(cam, scene, g_rgb, g_d)
    return g, ref, ws, int(flips.sum())


@pytest.mark.parametrize("name", ["tiny", "small"])
def test_render_bwd_parity_stagewise(lib, name):
    """Every gradient element (all F rows of all P Gaussians) within tolerance."""
    w = workload(name)
    g, ref, ws, _ = _bwd_stagewise(lib, w.cameras[0], w.scene, screen=True)
    assert_grad_parity(g, ref["grad"], ref["bound"])
    # the raster half alone (gs_render_bwd_screen), element by element: sgrad [P][12]
    # = (dmu_x, dmu_y, dA, dB, dC, dopacity, dr, dg, db, dz, pad, pad), the oracle's order
    assert_grad_parity(ws[:, :10].T, ref["screen"], ref["screen_bound"], what="screen-space gradient")


@pytest.mark.parametrize("name", ["replica", "scannetpp", "large"])
def test_render_bwd_sampled_full_size(lib, name):
    """Full-size view with upstream gradient on a sampled set of 64 tiles: every
    gradient element of every Gaussian within tolerance."""
    w = workload(name)
    cam, scene = w.cameras[0], w.scene
    rng = np.random.default_rng(3)
    mask = np.zeros((cam.height, cam.width), bool)
    for t in rng.choice(cam.num_tiles, 64, replace=False):
        ty, tx = divmod(int(t), cam.tiles_x)
        mask[ty * 16:(ty + 1) * 16, tx * 16:(tx + 1) * 16] = True
    g, ref, _, _ = _bwd_stagewise(lib, cam, scene, sample_mask=mask)
    assert np.count_nonzero(ref["grad"]) > 1000
    assert_grad_parity(g, ref["grad"], ref["bound"])


@pytest.mark.parametrize("seed", range(3))
def test_threshold_scene_flips_explained(lib, seed):
    """Decisions placed ON the 1/255 threshold (tests/threshold_scenes.py): the GPU's
    forward may differ from the oracle only at flagged pixels, and with those pixels'
    upstream zeroed every gradient element matches."""
    scene, cam, pix = near_skip_scene(seed)
    ref = gsref.render_fwd(cam, scene, gsref.F32)
    _, _, _, out = _fwd_stagewise(lib, cam, scene)
    bad = (np.abs(out["rgb"].cpu().numpy() - ref["rgb"]).max(0) > 1e-5) | \
          (out["n_contrib"].cpu().numpy() != ref["n_contrib"])
    flagged = flip_pixels(cam, scene)
    assert (bad & ~flagged).sum() == 0
    assert all(flagged[py, px] for px, py in pix)
    g, refb, _, nflip = _bwd_stagewise(lib, cam, scene)
    assert nflip >= len(pix)
    assert_grad_parity(g, refb["grad"], refb["bound"])


# ----------------------------------------------------------------------------- end-to-end chain
@pytest.mark.parametrize("name", ["tiny", "small"])
def test_chain_end_to_end(lib, name):
    w = workload(name)
    cam, scene = w.cameras[0], w.scene
    proj, t, params = gpu_project(lib, cam, scene)
    b = gpu_bin(lib, cam, scene, proj)
    out = gpu_render(lib, cam, scene, proj, b["sorted_ids"], b["ranges"])
    ref = gsref.render_fwd(cam, scene, gsref.F32)
    flagged = flip_pixels(cam, scene)
    rgb = out["rgb"].cpu().numpy()
    bad = np.abs(rgb - ref["rgb"]).max(0) > 1e-5
    assert (bad & ~flagged).sum() == 0
    assert abs(out["blended"] - ref["blended"]) <= 4 * flagged.sum()
    g_rgb, g_d = scenegen.upstream_fields(2, cam.width, cam.height)
    keep = ~flagged
    g_rgb = (g_rgb * keep[None]).astype(np.float32)
    g_d = (g_d * keep).astype(np.float32)
    g, _ = gpu_bwd(lib, cam, scene, params, proj, b["sorted_ids"], b["ranges"], out["T_final"], out["n_contrib"],
                   g_rgb, g_d)
    r = gsref.render_bwd_bound(cam, scene, g_rgb, g_d)
    assert_grad_parity(g, r["grad"], r["bound"])


# ----------------------------------------------------------------------------- Adam / L1
@pytest.mark.parametrize("n_views,side", [(3, True), (3, False), (11, True)])
def test_project_bwd_views_adam_dev_matches_separate(lib, n_views, side):
    """gs_project_bwd_views_adam_dev (the Trainer's graph-path tail: the SH rows' Adam on
    a side stream under the chain's geometry half) == gs_project_bwd_views +
    gs_adam_step_dev, bit for bit (gradient, parameters, moments, step counter), and the
    screen-gradient buffers are left zero; n = 11 takes the wide chain."""
    w = workload("small")
    scene = w.scene
    cams = [scenegen.camera_rt(320, 240, 300.0, 160.0, 120.0, scenegen.rot_y(0.05 * (k - 1)),
                               [0.1 * (k % 4), -0.05 * (k % 3), 0.02 * k]) for k in range(n_views)]
    sc = gsr.scene_desc(scene.P, scene.P_stride, scene.sh_degree)
    params0 = torch.from_numpy(scene.params).to(DEV)
    flags, sgrads, gcams = [], [], []
    for k, cam in enumerate(cams):
        proj, t, _ = gpu_project(lib, cam, scene)
        b = gpu_bin(lib, cam, scene, proj)
        out = gpu_render(lib, cam, scene, proj, b["sorted_ids"], b["ranges"])
        ur, ud = scenegen.upstream_fields(20 + k, 320, 240)
        sg = torch.zeros((scene.P, 12), dtype=torch.float32, device=DEV)
        lib.render_bwd_screen(gsr.camera(cam), sc, proj, b["sorted_ids"], b["ranges"], out["T_final"],
                              out["n_contrib"], torch.from_numpy(ur).to(DEV), torch.from_numpy(ud).to(DEV), sg)
        flags.append(t["flags"])
        sgrads.append(sg)
        gcams.append(gsr.camera(cam))
    torch.cuda.synchronize()
    lr = pipeline.lr_per_row(scene.sh_degree)
    rng = np.random.default_rng(3)
    m0 = torch.from_numpy((rng.normal(size=params0.shape) * 1e-3).astype(np.float32)).to(DEV)
    v0 = torch.from_numpy(rng.uniform(0, 1e-4, size=params0.shape).astype(np.float32)).to(DEV)
    res = {}
    for mode in ("separate", "fused"):
        p, m, v = params0.clone(), m0.clone(), v0.clone()
        g = torch.full_like(p, 7.0)  # overwritten (accumulate = 0)
        sgs = [x.clone() for x in sgrads]
        t = torch.full((1,), 4, dtype=torch.int64, device=DEV)
        if mode == "separate":
            lib.project_bwd_views(gcams, sc, p, flags, sgs, g, accumulate=False)
            lib.adam_step_dev(sc, p, g, m, v, lr, t, zero_grad=False)
        else:
            lib.project_bwd_views_adam_dev(gcams, sc, p, flags, sgs, g, m, v, lr, t, accumulate=False,
                                           side_stream=torch.cuda.Stream(device=DEV) if side else None)
        torch.cuda.synchronize()
        assert all(int(torch.count_nonzero(x)) == 0 for x in sgs)
        res[mode] = [x.cpu().numpy() for x in (g, p, m, v, t)]
    assert np.abs(res["separate"][0]).max() > 0
    for a, c, nm in zip(res["separate"], res["fused"], ("grad", "params", "m", "v", "step")):
        assert np.array_equal(a, c), nm


def test_adam_parity(lib):
    rng = np.random.default_rng(0)
    P, deg = 1000, 3
    F = 11 + 3 * 16
    S = scenegen.pad4(P)
    sc = gsr.scene_desc(P, S, deg)
    p = rng.normal(size=(F, S)).astype(np.float32)
    m = (rng.normal(size=(F, S)) * 1e-2).astype(np.float32)
    v = (rng.uniform(0, 1e-3, size=(F, S))).astype(np.float32)
    g = rng.normal(size=(F, S)).astype(np.float32)
    lr = pipeline.lr_per_row(deg)
    tp, tm, tv, tg = (torch.from_numpy(a).to(DEV) for a in (p, m, v, g))
    lib.adam_step(sc, tp, tg, tm, tv, lr, 7, zero_grad=True)
    torch.cuda.synchronize()
    # the ABI takes fp32 hyper-parameters: give the oracle the same fp32-rounded betas
    rp, rm, rv = gsref.adam_step(p, g, m, v, np.array(lr, np.float32), 7, P=S, beta1=float(np.float32(0.9)),
                                 beta2=float(np.float32(0.999)), eps=float(np.float32(1e-15)))
    # 1e-6 relative to the magnitude of the terms each fp32 update combines (m and v
    # are differences of two products and can cancel; p moves by ~lr per step)
    b1, b2 = float(np.float32(0.9)), float(np.float32(0.999))
    sm = b1 * np.abs(m) + (1 - b1) * np.abs(g)
    sv = b2 * np.abs(v) + (1 - b2) * g * g
    lr_col = np.array(lr, np.float64)[:, None]
    assert np.all(np.abs(tm.cpu().numpy() - rm) <= 1e-6 * sm + 1e-12)
    assert np.all(np.abs(tv.cpu().numpy() - rv) <= 1e-6 * sv + 1e-15)
    assert np.all(np.abs(tp.cpu().numpy() - rp) <= 1e-6 * (np.abs(p) + lr_col))
    assert torch.count_nonzero(tg) == 0


def test_l1_parity(lib):
    rng = np.random.default_rng(1)
    H, W = 37, 29
    rgb, trgb = rng.uniform(size=(2, 3, H, W)).astype(np.float32)
    d, td = rng.uniform(1, 5, size=(2, H, W)).astype(np.float32)
    trgb[0, 0, 0] = rgb[0, 0, 0]
    # targets that are not measurements (R43): no loss, zero gradient
    trgb[1, 3, 4], trgb[2, 5, 6], trgb[0, 7, 8] = np.nan, np.inf, -np.inf
    td[2, 2], td[4, 4], td[6, 6], td[8, 8] = 0.0, -1.0, np.nan, np.inf
    t = [torch.from_numpy(a).to(DEV) for a in (rgb, d, trgb, td)]
    g1 = torch.empty_like(t[0])
    g2 = torch.empty_like(t[1])
    loss = torch.zeros(1, device=DEV)
    lib.l1_loss_grad(t[0], t[1], t[2], t[3], 0.5, g1, g2, loss)
    L, r1, r2 = gsref.l1_loss_grad(rgb.astype(np.float64), d.astype(np.float64), trgb, td, 0.5)
    assert loss.item() == pytest.approx(L, rel=1e-5)
    np.testing.assert_allclose(g1.cpu().numpy(), r1, rtol=1e-6)
    np.testing.assert_allclose(g2.cpu().numpy(), r2, rtol=1e-6)
    assert g1[1, 3, 4] == 0 and g1[2, 5, 6] == 0 and g1[0, 7, 8] == 0
    assert g2[2, 2] == 0 and g2[4, 4] == 0 and g2[6, 6] == 0 and g2[8, 8] == 0
    assert np.isfinite(loss.item())


@pytest.mark.parametrize("name,rows", [("replica", 0), ("scannetpp", 0), ("large", 0), ("large", 1)])
def test_product_chain_full_size_sampled(lib, name, rows):
    """The product backward at full size, element by element: the GPU chain project ->
    bin -> render_fwd with key masks -> gs_render_bwd_screen_l1 (fused Eq. 12, the
    Trainer's kernel) -> gs_project_bwd_views, against the STAGE oracle with running
    error bounds.  The loss is restricted to 64 sampled tiles by the R43 masking: every
    other target sample (and every flagged flip pixel) is NaN, so it has no loss and
    no gradient.  In the sampled tiles the targets are the ORACLE's fp32 render offset by
    +-0.02 (colour) and +-(0.01 + 1%) (depth) with random signs, so the residual signs
    -- hence the upstream gradient -- are fixed by oracle-side data alone (the GPU
    render is within 1e-5 of the oracle's).  rows=1: with the render kernels' block-row
    walk (gs_set_render_rows), the form the bench's autotune picks for config 4."""
    was = lib.render_rows()
    lib.set_render_rows(rows)
    try:
        _product_chain_full_size_sampled(lib, name)
    finally:
        lib.set_render_rows(was)


def _product_chain_full_size_sampled(lib, name):
    w = workload(name)
    cam, scene = w.cameras[0], w.scene
    H, W, npix = cam.height, cam.width, cam.height * cam.width
    sc = gsr.scene_desc(scene.P, scene.P_stride, scene.sh_degree)
    gcam = gsr.camera(cam)
    proj, t, params = gpu_project(lib, cam, scene)
    b = gpu_bin(lib, cam, scene, proj)
    K = b["K"]
    rgb = torch.empty((3, H, W), device=DEV)
    dep = torch.empty((H, W), device=DEV)
    T = torch.empty((H, W), device=DEV)
    n = torch.empty((H, W), dtype=torch.int32, device=DEV)
    kb = torch.zeros(K + 16, dtype=torch.uint8, device=DEV)
    lib.render_fwd(gcam, sc, proj, b["sorted_ids"], b["ranges"], rgb, dep, T, n, key_blocks=kb)
    # sampled tiles -> target images
    rng = np.random.default_rng(21)
    ys, xs = [], []
    for tt in rng.choice(cam.num_tiles, 64, replace=False):
        ty, tx = divmod(int(tt), cam.tiles_x)
        yy, xx = np.mgrid[ty * 16:min(ty * 16 + 16, H), tx * 16:min(tx * 16 + 16, W)]
        ys.append(yy.ravel())
        xs.append(xx.ravel())
    ys, xs = np.concatenate(ys), np.concatenate(xs)
    ok = ~flip_pixels(cam, scene, xs, ys)
    ys, xs = ys[ok], xs[ok]
    ref_px = gsref.render_pixels(cam, scene, xs, ys, gsref.F32)
    sgn = rng.choice([-1.0, 1.0], size=(4, xs.size))
    t_rgb = np.full((3, H, W), np.nan, np.float32)
    t_dep = np.full((H, W), np.nan, np.float32)
    t_rgb[:, ys, xs] = (ref_px["rgb"] + 0.02 * sgn[:3]).astype(np.float32)
    t_dep[ys, xs] = (ref_px["depth"] + sgn[3] * (0.01 + 0.01 * np.abs(ref_px["depth"]))).astype(np.float32)
    # oracle upstream: sign(oracle render - target) x the fp32 scales the GPU uses, R43 mask
    s_c = np.float32(1.0 / (3.0 * npix))
    s_d = np.float32(1.0 / npix)
    g_rgb = np.zeros((3, H, W), np.float32)
    g_d = np.zeros((H, W), np.float32)
    g_rgb[:, ys, xs] = (np.sign(ref_px["rgb"] - t_rgb[:, ys, xs]) * s_c).astype(np.float32)
    dv = t_dep[ys, xs] > 0
    g_d[ys[dv], xs[dv]] = (np.sign(ref_px["depth"][dv] - t_dep[ys[dv], xs[dv]]) * s_d).astype(np.float32)
    # the GPU render agrees with the oracle well inside the offsets (signs are shared)
    assert np.abs(rgb.cpu().numpy()[:, ys, xs] - ref_px["rgb"]).max() < 1e-4
    sg = torch.zeros((scene.P, 12), device=DEV)
    loss = torch.zeros(1, device=DEV)
    lib.render_bwd_screen_l1(gcam, sc, proj, b["sorted_ids"], b["ranges"], T, n, rgb, dep,
                             torch.from_numpy(t_rgb).to(DEV), torch.from_numpy(t_dep).to(DEV), 1.0, sg, loss=loss,
                             key_blocks=kb)
    grad = torch.full((scene.F, scene.P_stride), np.nan, device=DEV)
    lib.project_bwd_views([gcam], sc, params, [t["flags"]], [sg], grad, accumulate=False)
    torch.cuda.synchronize()
    L_ref = (np.abs(ref_px["rgb"] - t_rgb[:, ys, xs]).sum() * float(s_c) +
             np.abs(ref_px["depth"][dv] - t_dep[ys[dv], xs[dv]]).sum() * float(s_d))
    assert loss.item() == pytest.approx(L_ref, rel=1e-4)
    ref = gsref.render_bwd_bound(cam, scene, g_rgb, g_d)
    g = grad[:, :scene.P].cpu().numpy().astype(np.float64)
    # colour-clamp decisions (R13) are the only projection decisions not bit-exact (the
    # GPU colour is within 1e-6, not bit-identical): a differing flag must be a proven
    # flip (both colours within 1e-6 of 0); such a Gaussian's SH and mean rows are excused
    pr = gsref.project(cam, scene, gsref.F32)
    fl_gpu = t["flags"][:scene.P].cpu().numpy()
    excl = np.zeros_like(g, bool)
    for ch in range(3):
        differ = ((fl_gpu >> ch) & 1) != ((pr["flags"] >> ch) & 1)
        if differ.any():
            col = t["rec"][:scene.P, 7 + ch].cpu().numpy()[differ]
            assert np.all(np.abs(col) <= 1e-6) and np.all(np.abs(pr[("r", "g", "b")[ch]][differ]) <= 1e-6)
            excl[:, differ] = True
    assert np.count_nonzero(ref["grad"]) > 1000
    assert_grad_parity(g, ref["grad"], ref["bound"], scale=float(s_c), exclude=excl)


# ----------------------------------------------------------------------------- edge cases
def test_empty_scene(lib):
    cam = scenegen.identity_camera(40, 24, 30.0, 19.5, 11.5)
    cam.bg = (0.25, 0.5, 0.75)
    scene = scenegen.Scene(0, 0, np.zeros((14, 0), np.float32))
    proj, t = gsr.make_proj(0, DEV)
    sc = gsr.scene_desc(0, 0, 0)
    params = torch.zeros(4, device=DEV)
    lib.project(gsr.camera(cam), sc, params, proj)
    out = gpu_bin(lib, cam, scene, proj, capacity=16)
    assert out["K"] == 0
    r = gpu_render(lib, cam, scene, proj, out["sorted_ids"], out["ranges"])
    assert torch.all(r["rgb"][0] == 0.25) and torch.all(r["rgb"][2] == 0.75) and torch.all(r["T_final"] == 1)
    with pytest.raises(gsr.GsError) as e:
        lib.adam_step(sc, params, params, params, params, [1e-3] * 14, 1)
    assert e.value.status == gsr.GS_ERR_EMPTY


def test_all_culled(lib):
    w = scenegen.make("tiny")
    scene = scenegen.Scene(w.scene.P, 0, w.scene.params.copy())
    scene.params[2, :scene.P] = -3.0  # everything behind the camera
    proj, t, params = gpu_project(lib, w.cameras[0], scene)
    assert int(t["radius"][:scene.P].abs().sum()) == 0
    out = gpu_bin(lib, w.cameras[0], scene, proj, capacity=64)
    assert out["K"] == 0
    g, _ = gpu_bwd(lib, w.cameras[0], scene, params, proj, out["sorted_ids"], out["ranges"],
                   torch.ones((48, 64), device=DEV), torch.zeros((48, 64), dtype=torch.int32, device=DEV),
                   np.ones((3, 48, 64), np.float32), np.ones((48, 64), np.float32))
    assert np.all(g == 0)


@pytest.mark.parametrize("wh", [(37, 29), (16, 16), (17, 1), (1000, 8)])
def test_ragged_images(lib, wh):
    W, H = wh
    scene, cam = scenegen.random_small_scene(7, 60, 1, width=W, height=H, f=0.8 * max(W, H))
    ref = gsref.render_fwd(cam, scene, gsref.F32)
    proj, _, params = gpu_project(lib, cam, scene)
    b = gpu_bin(lib, cam, scene, proj)
    out = gpu_render(lib, cam, scene, proj, b["sorted_ids"], b["ranges"])
    bad = np.abs(out["rgb"].cpu().numpy() - ref["rgb"]).max(0) > 1e-5
    assert (bad & ~flip_pixels(cam, scene)).sum() == 0


def test_single_gaussian_peak_closed_form(lib):
    """Isotropic on-axis Gaussian: C(cx, cy) = c a0 + (1 - a0) bg, D = z a0, T = 1 - a0."""
    cam = scenegen.identity_camera(64, 48, 60.0, 32.0, 24.0)
    cam.bg = (0.1, 0.2, 0.3)
    c = np.array([0.9, 0.4, 0.05])
    sh = np.zeros((1, 1, 3))
    sh[0, 0] = (c - 0.5) / 0.28209479177387814
    sc = scenegen.scene_from_gaussians([[0, 0, 3.0]], np.log([[0.05] * 3]), [[1, 0, 0, 0]], [0.0], sh, 0)
    proj, t, _ = gpu_project(lib, cam, sc)
    assert int(t["radius"][0]) == 4 and int(t["tiles"][0]) == 2
    b = gpu_bin(lib, cam, sc, proj)
    out = gpu_render(lib, cam, sc, proj, b["sorted_ids"], b["ranges"])
    np.testing.assert_allclose(out["rgb"][:, 24, 32].cpu().numpy(), c * 0.5 + 0.5 * np.array(cam.bg), atol=1e-6)
    assert out["depth"][24, 32].item() == pytest.approx(1.5, abs=1e-6)
    assert out["T_final"][24, 32].item() == pytest.approx(0.5, abs=1e-6)
    assert out["blended"] == 37  # footprint closed form (tests/golden/closed_forms.json)


def test_huge_footprint(lib):
    """A near-camera Gaussian whose footprint covers every tile (> 256 tiles: 2-pass tile sort)."""
    cam = scenegen.identity_camera(320, 240, 300.0, 160.0, 120.0)
    sh = np.zeros((2, 1, 3))
    sh[0, 0] = (np.array([0.9, 0.4, 0.05]) - 0.5) / 0.28209479177387814
    sh[1, 0] = (np.array([0.2, 0.2, 0.2]) - 0.5) / 0.28209479177387814
    sc = scenegen.scene_from_gaussians([[0, 0, 3.0], [0.0, 0.0, 0.5]], np.log([[0.02] * 3, [2.0] * 3]),
                                       [[1, 0, 0, 0]] * 2, [0.0, -4.0], sh, 0)
    proj, t, params = gpu_project(lib, cam, sc)
    assert int(t["tiles"][1]) == cam.num_tiles
    b = gpu_bin(lib, cam, sc, proj)
    ref_b = gsref.bin_tiles(cam, sc)
    np.testing.assert_array_equal(b["sorted_ids"][:b["K"]].cpu().numpy(), ref_b["sorted_ids"])
    out = gpu_render(lib, cam, sc, proj, b["sorted_ids"], b["ranges"])
    ref = gsref.render_fwd(cam, sc, gsref.F32)
    np.testing.assert_allclose(out["rgb"].cpu().numpy(), ref["rgb"], atol=1e-5)


def test_trainer_step_runs_and_decreases_loss(lib):
    w = workload("small")
    model = pipeline.GaussianModel(w.scene, DEV)
    tgt_model = pipeline.GaussianModel(w.target_scene, DEV)
    K = pipeline.measure_keys(lib, model, w.cameras, DEV)
    cap = pipeline.default_capacity(K)
    targets = pipeline.render_targets(lib, tgt_model, w.cameras, DEV, cap)
    tr = pipeline.Trainer(lib, model, w.cameras, targets, DEV, cap)
    losses = []
    for _ in range(20):
        tr.loss.zero_()
        tr.step([0])
        losses.append(tr.loss.item())
    tr.check_capacity()
    assert losses[-1] < losses[0]


def test_trainer_step_host_matches_step(lib):
    """Targets streamed from pinned host memory on the copy stream (Trainer.step_host,
    the bench's e2e path) give the same iteration as device-resident targets."""
    w = workload("small")
    models = [pipeline.GaussianModel(w.scene, DEV) for _ in range(2)]
    tgt_model = pipeline.GaussianModel(w.target_scene, DEV)
    K = pipeline.measure_keys(lib, models[0], w.cameras, DEV)
    cap = pipeline.default_capacity(K)
    cams = [w.cameras[0]] * 5  # 5 views through 2 slots: slot reuse within one step
    targets = pipeline.render_targets(lib, tgt_model, cams, DEV, cap)
    host = {v: (targets[v][0].cpu().pin_memory(), targets[v][1].cpu().pin_memory()) for v in range(len(cams))}
    trs = [pipeline.Trainer(lib, m, cams, targets, DEV, cap, deterministic=True) for m in models]
    for it in range(3):
        trs[0].loss.zero_()
        trs[1].loss.zero_()
        trs[0].step(list(range(len(cams))))
        trs[1].step_host(list(range(len(cams))), host)
        torch.cuda.synchronize()
        assert trs[1].loss.item() == pytest.approx(trs[0].loss.item(), rel=1e-5)
    # deterministic reduction mode: the two iterations are bit-identical
    assert torch.equal(models[0].params, models[1].params)
    assert torch.equal(models[0].m, models[1].m) and torch.equal(models[0].v, models[1].v)


@pytest.mark.parametrize("n_views", [3, 11])
def test_batched_views_backward_matches_per_view(lib, n_views):
    """gs_render_bwd_screen x n + gs_project_bwd_views == sum of per-view gs_render_bwd
    (and the sgrad buffers are left zero); n = 11 > 8 takes the wide kernels (views in
    the inner loop, one pass for all views)."""
    w = workload("small")
    scene = w.scene
    cams = []
    for k in range(n_views):
        c = scenegen.camera_rt(320, 240, 300.0, 160.0, 120.0, scenegen.rot_y(0.05 * (k - 1)),
                               [0.1 * (k % 4), -0.05 * (k % 3), 0.02 * k])
        cams.append(c)
    params = torch.from_numpy(scene.params).to(DEV)
    sc = gsr.scene_desc(scene.P, scene.P_stride, scene.sh_degree)
    grad_sum = torch.zeros_like(params)
    grad_b = torch.zeros_like(params)
    flags, sgrads, gcams, keep, upstream = [], [], [], [], []
    for k, cam in enumerate(cams):
        proj, t, _ = gpu_project(lib, cam, scene)
        b = gpu_bin(lib, cam, scene, proj)
        out = gpu_render(lib, cam, scene, proj, b["sorted_ids"], b["ranges"])
        keep_px = ~flip_pixels(cam, scene)
        ur, ud = scenegen.upstream_fields(10 + k, 320, 240)
        ur, ud = (ur * keep_px[None]).astype(np.float32), (ud * keep_px).astype(np.float32)
        upstream.append((ur, ud))
        g_rgb, g_d = torch.from_numpy(ur).to(DEV), torch.from_numpy(ud).to(DEV)
        ws = torch.zeros(scene.P * 12, dtype=torch.float32, device=DEV)  # gs_render_bwd clears it
        lib.render_bwd(gsr.camera(cam), sc, params, proj, b["sorted_ids"], b["ranges"], out["T_final"],
                       out["n_contrib"], g_rgb, g_d, ws, grad_sum)
        sg = torch.zeros((scene.P, 12), dtype=torch.float32, device=DEV)
        lib.render_bwd_screen(gsr.camera(cam), sc, proj, b["sorted_ids"], b["ranges"], out["T_final"],
                              out["n_contrib"], g_rgb, g_d, sg)
        flags.append(t["flags"])
        sgrads.append(sg)
        gcams.append(gsr.camera(cam))
        keep.append((proj, t, b, out))
    lib.project_bwd_views(gcams, sc, params, flags, sgrads, grad_b)
    torch.cuda.synchronize()
    a, bb = grad_sum.cpu().numpy(), grad_b.cpu().numpy()
    assert np.abs(a).max() > 0
    # both against the oracle's sum over the views (R21), element by element; the
    # per-view bounds add (the view sum is one more accumulation)
    ref = np.zeros((scene.F, scene.P))
    bound = np.zeros((scene.F, scene.P))
    for k, cam in enumerate(cams):
        g_rgb, g_d = upstream[k]
        r = gsref.render_bwd_bound(cam, scene, g_rgb, g_d)
        ref += r["grad"]
        bound += r["bound"] + np.abs(r["grad"])
    assert_grad_parity(a[:, :scene.P], ref, bound, what="per-view gs_render_bwd sum")
    assert_grad_parity(bb[:, :scene.P], ref, bound, what="batched screen + gs_project_bwd_views")
    for sg in sgrads:
        assert int(torch.count_nonzero(sg)) == 0


@pytest.mark.parametrize("host,bins", [(False, None), (True, None), (False, "0"), (False, "2")])
def test_trainer_streams_match_single_stream(lib, host, bins, monkeypatch):
    """Views in flight on 3 streams (own buffers each) give the same iteration as one
    stream: 11 distinct views, chunks of 4, so sgrad / flag slots are reused across
    projection-backward chains within a step; host=True also streams the targets.
    bins: GSR_BIN_STREAMS (None = the default bin-ahead streams; "0" = each view's whole
    chain on its render stream; "2" = a ring of 5 view buffers, reused within a step)."""
    if bins is not None:
        monkeypatch.setenv("GSR_BIN_STREAMS", bins)
    w = workload("small")
    cams = [scenegen.camera_rt(320, 240, 300.0, 160.0, 120.0, scenegen.rot_y(0.03 * (k - 5)),
                               [0.05 * (k - 5), 0.02 * k, 0.0]) for k in range(11)]
    models = [pipeline.GaussianModel(w.scene, DEV) for _ in range(2)]
    tgt_model = pipeline.GaussianModel(w.target_scene, DEV)
    cap = pipeline.default_capacity(pipeline.measure_keys(lib, models[0], cams, DEV))
    targets = pipeline.render_targets(lib, tgt_model, cams, DEV, cap)
    trs = [pipeline.Trainer(lib, m, cams, targets, DEV, cap, chunk=4, streams=s, deterministic=True)
           for m, s in zip(models, (1, 3))]
    host_t = {v: (targets[v][0].cpu().pin_memory(), targets[v][1].cpu().pin_memory()) for v in range(len(cams))}
    for it in range(3):
        for tr in trs:
            tr.loss.zero_()
            tr.blended.zero_()
            if host:
                tr.step_host(list(range(len(cams))), host_t)
            else:
                tr.step(list(range(len(cams))))
        torch.cuda.synchronize()
        assert trs[1].loss.item() == pytest.approx(trs[0].loss.item(), rel=1e-5)
        assert trs[1].blended.item() == trs[0].blended.item()  # identical parameters every step
    # deterministic reduction: the iterations are bit-identical whatever the streams
    assert torch.equal(models[0].params, models[1].params)
    for sg in trs[1].sgrad:
        assert int(torch.count_nonzero(sg)) == 0


def test_tile_order_permutation_and_invariance(lib):
    """gs_tile_order is a permutation of the tiles by non-increasing key count
    (bucketed by count / 4); rendering in that order gives bit-identical forward
    outputs and, in the deterministic reduction mode, bit-identical gradients."""
    w = workload("replica")
    cam, scene = w.cameras[0], w.scene
    proj, t, params = gpu_project(lib, cam, scene)
    b = gpu_bin(lib, cam, scene, proj)
    gcam = gsr.camera(cam)
    order = torch.full((cam.num_tiles,), -1, dtype=torch.int32, device=DEV)
    lib.tile_order(gcam, b["ranges"], order)
    torch.cuda.synchronize()
    o = order.cpu().numpy()
    assert np.array_equal(np.sort(o), np.arange(cam.num_tiles))
    r = b["ranges"].cpu().numpy()
    lens = np.minimum(r[:, 1] - r[:, 0], 4095) // 4
    assert np.all(np.diff(lens[o]) <= 0)
    sc = gsr.scene_desc(scene.P, scene.P_stride, scene.sh_degree)
    outs = []
    for tord in (None, order):
        H, W = cam.height, cam.width
        rgb, dep, T = (torch.zeros(s, device=DEV) for s in ((3, H, W), (H, W), (H, W)))
        n = torch.zeros((H, W), dtype=torch.int32, device=DEV)
        lib.render_fwd(gcam, sc, proj, b["sorted_ids"], b["ranges"], rgb, dep, T, n, tile_order=tord)
        g_rgb, g_d = (torch.from_numpy(a).to(DEV) for a in scenegen.upstream_fields(5, W, H))
        sg = torch.zeros((scene.P, 12), device=DEV)
        det = torch.empty((b["K"] + 16, 12), device=DEV)
        lib.render_bwd_screen(gcam, sc, proj, b["sorted_ids"], b["ranges"], T, n, g_rgb, g_d, sg, tile_order=tord,
                              det=det)
        torch.cuda.synchronize()
        outs.append((rgb.cpu().numpy(), dep.cpu().numpy(), n.cpu().numpy(), sg.cpu().numpy().astype(np.float64)))
    for a, c in zip(outs[0][:3], outs[1][:3]):
        assert np.array_equal(a, c)
    assert np.array_equal(outs[1][3], outs[0][3]) and np.abs(outs[0][3]).max() > 0


def test_keyframe_optimizer_runs_plan(lib):
    """NEXT-1: the keyframe-scheduled plan drives the GPU path view by view; every
    planned iteration is one step (Adam step counter), the loss on the keyframes drops."""
    w = scenegen.make("small")
    cams = [scenegen.camera_rt(320, 240, 300.0, 160.0, 120.0, scenegen.rot_y(0.02 * (k - 6)), [0.04 * (k - 6), 0.0, 0.0])
            for k in range(12)]
    model = pipeline.GaussianModel(w.scene, DEV)
    tgt = pipeline.GaussianModel(w.target_scene, DEV)
    cap = pipeline.default_capacity(pipeline.measure_keys(lib, model, cams, DEV))
    targets = pipeline.render_targets(lib, tgt, cams, DEV, cap)
    tr = pipeline.Trainer(lib, model, cams, targets, DEV, cap)
    new = scenegen.new_primitive_counts(len(cams), seed=0)
    ko = pipeline.KeyframeOptimizer(lib, tr, new, threshold=50, m=5, n=3, global_iters=2, seed=0)

    def kf_loss():
        tot = 0.0
        for v in np.flatnonzero(ko.is_keyframe):
            b = tr.buf
            pipeline.render(lib, model, cams[v], b)
            tot += float((b.rgb - targets[v][0]).abs().mean() + (b.depth - targets[v][1]).abs().mean())
        return tot
    before = kf_loss()
    ko.run()
    torch.cuda.synchronize()
    assert model.step_count == len(ko.views)
    assert kf_loss() < before


def test_adam_step_range_matches_full_step(lib):
    """gs_adam_step_range on [b, e) == gs_adam_step restricted to [b, e); untouched
    outside; misaligned bounds rejected."""
    rng = np.random.default_rng(4)
    P, deg = 999, 1
    F, S = 11 + 3 * 4, scenegen.pad4(999)
    sc = gsr.scene_desc(P, S, deg)
    arrs = [rng.normal(size=(F, S)).astype(np.float32) for _ in range(2)] + \
           [(rng.uniform(0, 1e-3, size=(F, S))).astype(np.float32), rng.normal(size=(F, S)).astype(np.float32)]
    lr = pipeline.lr_per_row(deg)
    full = [torch.from_numpy(a.copy()).to(DEV) for a in arrs]  # p, m, v, g
    part = [torch.from_numpy(a.copy()).to(DEV) for a in arrs]
    lib.adam_step(sc, full[0], full[3], full[1], full[2], lr, 3, zero_grad=False)
    b, e = 4 * 1001, 4 * 3777
    gr = part[3].view(-1)[b:e].clone()
    lib.adam_step_range(sc, part[0], gr, part[1], part[2], lr, 3, b, e)
    torch.cuda.synchronize()
    for x, y, a in zip(full[:3], part[:3], arrs[:3]):
        xf, yf = x.view(-1).cpu().numpy(), y.view(-1).cpu().numpy()
        np.testing.assert_array_equal(yf[b:e], xf[b:e])
        np.testing.assert_array_equal(np.delete(yf, np.s_[b:e]), np.delete(a.reshape(-1), np.s_[b:e]))
    with pytest.raises(gsr.GsError):
        lib.adam_step_range(sc, part[0], gr, part[1], part[2], lr, 3, b + 1, e)


def test_sharded_adam_single_rank_nccl(lib):
    """pipeline.ShardedAdam through a real NCCL process group (world size 1 on this
    GPU: reduce_scatter_tensor / all_gather_into_tensor + gs_adam_step_range) gives
    the same parameters as the replicated gs_adam_step."""
    import os
    import socket
    import torch.distributed as dist
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=DEV)
    try:
        w = workload("small")
        rng = np.random.default_rng(8)
        g = torch.from_numpy(rng.normal(size=w.scene.params.shape).astype(np.float32)).to(DEV)
        ma, mb = pipeline.GaussianModel(w.scene, DEV), pipeline.GaussianModel(w.scene, DEV)
        opt = pipeline.ShardedAdam(lib, mb)
        for it in range(3):
            ma.grad.copy_(g * (it + 1))
            mb.grad.copy_(g * (it + 1))
            ma.step_count += 1
            lib.adam_step(ma.desc, ma.params, ma.grad, ma.m, ma.v, ma.lr, ma.step_count, zero_grad=False)
            mb.step_count += 1
            opt.step()
        torch.cuda.synchronize()
        assert torch.equal(ma.params, mb.params)
    finally:
        dist.destroy_process_group()


def test_peer_sharded_adam_single_rank(lib):
    """PeerShardedAdam (gs_adam_step_peers over torch symmetric memory, world size 1 on
    this GPU): the fused kernel's pull / Adam / push path equals gs_adam_step."""
    import os
    import socket
    import torch.distributed as dist
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=DEV)
    try:
        w = workload("small")
        rng = np.random.default_rng(9)
        g = torch.from_numpy(rng.normal(size=w.scene.params.shape).astype(np.float32)).to(DEV)
        ma, mb = pipeline.GaussianModel(w.scene, DEV), pipeline.GaussianModel(w.scene, DEV)
        opt = pipeline.PeerShardedAdam(lib, mb)
        for it in range(3):
            ma.grad.copy_(g * (it + 1))
            mb.grad.copy_(g * (it + 1))
            ma.step_count += 1
            lib.adam_step(ma.desc, ma.params, ma.grad, ma.m, ma.v, ma.lr, ma.step_count, zero_grad=False)
            mb.step_count += 1
            opt.step()
        torch.cuda.synchronize()
        assert torch.equal(ma.params, mb.params)
        assert torch.equal(ma.m, mb.m) and torch.equal(ma.v, mb.v)
        assert pipeline.params_agree_across_ranks(mb)
    finally:
        dist.destroy_process_group()


def test_exchange_self_test_catches_a_wrong_sum(lib):
    """PeerShardedAdam's construction-time self-test (a known gradient exchanged with zero
    learning rates) rejects a path that sums the wrong terms -- here the kernel pointed
    at a zero gradient buffer -- and leaves the model's state as it was."""
    import os
    import socket
    import torch.distributed as dist
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=DEV)
    try:
        w = workload("small")
        zero = torch.zeros(w.scene.params.size + 64, device=DEV)

        class Broken(pipeline.PeerShardedAdam):
            def _launch(self, lr, step):
                m = self.model
                self.lib.adam_step_peers(m.desc, self.world, self.rank, [zero.data_ptr()], self.pptrs, m.m, m.v, lr,
                                         step, self.begin, self.end)
        mb = pipeline.GaussianModel(w.scene, DEV)
        mb.m.fill_(0.25)
        p0 = mb.params.clone()
        with pytest.raises(RuntimeError, match="self-test"):
            Broken(lib, mb)
        torch.cuda.synchronize()
        assert torch.equal(mb.params, p0) and bool(torch.all(mb.m == 0.25))
        pipeline.PeerShardedAdam(lib, pipeline.GaussianModel(w.scene, DEV))  # the real path passes
    finally:
        dist.destroy_process_group()


def test_nvls_sharded_adam_single_rank(lib):
    """NvlsShardedAdam (gs_adam_step_multimem: multimem.ld_reduce of the gradient shard
    through the NVSwitch, Adam, multimem.st of the parameters; world size 1 on this GPU,
    so the in-switch sum has one term) equals gs_adam_step bit for bit, with the host and
    the device step counter.  Where the box has no multicast the optimizer must refuse
    cleanly (RuntimeError) and the test says so by skipping."""
    import os
    import socket
    import torch.distributed as dist
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=DEV)
    try:
        w = workload("small")
        rng = np.random.default_rng(10)
        g = torch.from_numpy(rng.normal(size=w.scene.params.shape).astype(np.float32)).to(DEV)
        ma, mb = pipeline.GaussianModel(w.scene, DEV), pipeline.GaussianModel(w.scene, DEV)
        try:
            opt = pipeline.NvlsShardedAdam(lib, mb)
        except RuntimeError as ex:
            assert "multicast" in str(ex)
            pytest.skip("torch symmetric memory has no multicast address on this box (the kernel itself is "
                        "covered by test_adam_multimem_one_device_multicast)")
        for it in range(4):
            ma.grad.copy_(g * (it + 1))
            mb.grad.copy_(g * (it + 1))
            ma.step_count += 1
            lib.adam_step(ma.desc, ma.params, ma.grad, ma.m, ma.v, ma.lr, ma.step_count, zero_grad=False)
            opt.device_step = it >= 2
            mb.step_count += 1
            if it == 2:
                mb.step_dev.fill_(mb.step_count - 1)
            opt.step()
        torch.cuda.synchronize()
        assert int(mb.step_dev.item()) == 4
        assert torch.equal(ma.params, mb.params)
        assert torch.equal(ma.m, mb.m) and torch.equal(ma.v, mb.v)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("device_step", [False, True])
def test_adam_multimem_one_device_multicast(lib, device_step):
    """gs_adam_step_multimem on a real NVLS multicast object of this one device
    (tests/mc_helpers.py): multimem.ld_reduce of the gradient, Adam, multimem.st of the
    parameters through the multicast address, over a sharded range with a ragged end;
    equals gs_adam_step (unicast) bit for bit inside the range and leaves the rest alone."""
    import mc_helpers
    w = workload("small")
    rng = np.random.default_rng(12)
    F, S = w.scene.params.shape
    n = F * S
    try:
        gb, pb = mc_helpers.MulticastBuffer(n), mc_helpers.MulticastBuffer(n)
    except RuntimeError as ex:
        pytest.skip(f"no multicast object on this box: {ex}")
    try:
        ma = pipeline.GaussianModel(w.scene, DEV)
        g = torch.from_numpy(rng.normal(size=(F, S)).astype(np.float32)).to(DEV)
        pb.tensor.copy_(ma.params.reshape(-1))
        m2, v2 = torch.zeros_like(ma.m), torch.zeros_like(ma.v)
        begin, end = 4 * 37, n - 4 * 5  # a sharded range: neither end at the array's
        ref_p = ma.params.clone()
        ref_m, ref_v = ma.m.clone(), ma.v.clone()
        step_dev = torch.zeros(1, dtype=torch.int64, device=DEV)
        for it in range(1, 4):
            gb.tensor.copy_((g * it).reshape(-1))
            ma.grad.copy_(g * it)
            lib.adam_step(ma.desc, ma.params, ma.grad, ma.m, ma.v, ma.lr, it, zero_grad=False)
            lib.adam_step_multimem(ma.desc, gb.mc, pb.mc, pb.tensor, m2, v2, ma.lr, step_dev if device_step else it,
                                   begin, end)
        torch.cuda.synchronize()
        if device_step:
            assert int(step_dev.item()) == 3
        got = pb.tensor.reshape(F, S)
        inside = torch.zeros(n, dtype=torch.bool, device=DEV)
        inside[begin:end] = True
        inside = inside.reshape(F, S)
        assert torch.equal(got[inside], ma.params[inside])
        assert torch.equal(m2[inside], ma.m[inside]) and torch.equal(v2[inside], ma.v[inside])
        assert torch.equal(got[~inside], ref_p[~inside])  # outside the shard: untouched
        assert torch.count_nonzero(m2[~inside]) == 0
        assert not torch.equal(got, ref_p)
    finally:
        gb.close()
        pb.close()


@pytest.mark.parametrize("streams", [1, 3])
def test_graph_replay_matches_eager(lib, streams):
    """Trainer.capture: a whole iteration (project/bin/fwd/L1/bwd per view on its
    stream, projection backward, Adam with the device step counter) replayed as a CUDA
    graph gives the same iterations as eager steps."""
    w = workload("small")
    cams = [scenegen.camera_rt(320, 240, 300.0, 160.0, 120.0, scenegen.rot_y(0.03 * (k - 2)), [0.05 * k, 0.0, 0.0])
            for k in range(5)]
    models = [pipeline.GaussianModel(w.scene, DEV) for _ in range(2)]
    tgt = pipeline.GaussianModel(w.target_scene, DEV)
    cap = pipeline.default_capacity(pipeline.measure_keys(lib, models[0], cams, DEV))
    targets = pipeline.render_targets(lib, tgt, cams, DEV, cap)
    trs = [pipeline.Trainer(lib, m, cams, targets, DEV, cap, streams=streams, deterministic=True) for m in models]
    views = list(range(len(cams)))
    trs[0].step(views)  # both start from one eager step
    trs[1].step(views)
    g = trs[1].capture(views)  # runs one more eager step while capturing
    trs[0].step(views)
    losses = []
    for it in range(3):
        for tr in trs:
            tr.loss.zero_()
        trs[0].step(views)
        trs[1].replay(g)
        torch.cuda.synchronize()
        losses.append((trs[0].loss.item(), trs[1].loss.item()))
    assert models[0].step_count == models[1].step_count == int(models[1].step_dev.item()) == 5
    for a, b in losses:
        assert b == pytest.approx(a, rel=1e-4)
    # deterministic reduction: graph replays are bit-identical to eager steps
    assert torch.equal(models[0].params, models[1].params)
    assert torch.equal(models[0].m, models[1].m) and torch.equal(models[0].v, models[1].v)


def test_adam_touches_live_columns_only(lib):
    """A map growing into its capacity (P < P_stride): gs_adam_step / gs_adam_step_dev
    update columns [0, P) as the full step would and leave the spare columns alone."""
    rng = np.random.default_rng(5)
    P, S, deg = 999, 1200, 0
    F = 14
    arrs = [rng.normal(size=(F, S)).astype(np.float32), (rng.normal(size=(F, S)) * 1e-2).astype(np.float32),
            rng.uniform(0, 1e-3, size=(F, S)).astype(np.float32), rng.normal(size=(F, S)).astype(np.float32)]
    lr = pipeline.lr_per_row(deg)
    full = [torch.from_numpy(a.copy()).to(DEV) for a in arrs]
    lib.adam_step(gsr.scene_desc(S, S, deg), full[0], full[3], full[1], full[2], lr, 2, zero_grad=False)
    for dev_step in (False, True):
        part = [torch.from_numpy(a.copy()).to(DEV) for a in arrs]
        sc = gsr.scene_desc(P, S, deg)
        if dev_step:
            t = torch.ones(1, dtype=torch.int64, device=DEV)
            lib.adam_step_dev(sc, part[0], part[3], part[1], part[2], lr, t)
        else:
            lib.adam_step(sc, part[0], part[3], part[1], part[2], lr, 2, zero_grad=False)
        torch.cuda.synchronize()
        for x, y, a in zip(full[:3], part[:3], arrs[:3]):
            np.testing.assert_allclose(y.cpu().numpy()[:, :P], x.cpu().numpy()[:, :P], rtol=1e-6, atol=1e-7)
            np.testing.assert_array_equal(y.cpu().numpy()[:, 1000:], a[:, 1000:])


def test_bench_launch_configuration_full_size_sampled(lib):
    """The bench's launch configuration at full size: scannetpp (1M Gaussians, 8 views of
    1752x1168), Morton layout, 4 views in flight, the whole iteration replayed as a CUDA
    graph.  After one replay, the view buffers hold the renders of the last views that
    used them, made with the pre-step parameters: sampled pixels against the oracle
    (1e-5, flips explained by the decision margin), and the per-view key counts against
    the oracle's."""
    w = workload("scannetpp")
    model = pipeline.GaussianModel(w.scene, DEV)
    pipeline.spatially_order(lib, model)
    tgt = pipeline.GaussianModel(w.target_scene, DEV)
    pipeline.spatially_order(lib, tgt)
    cams = w.cameras
    cap = pipeline.default_capacity(max(pipeline.measure_keys(lib, model, cams, DEV),
                                        pipeline.measure_keys(lib, tgt, cams, DEV)))
    targets = pipeline.render_targets(lib, tgt, cams, DEV, cap)
    tr = pipeline.Trainer(lib, model, cams, targets, DEV, cap, streams=4)
    views = list(range(len(cams)))
    g = tr.capture(views)
    snap = model.params.detach().cpu().numpy().copy()
    tr.num_keys.zero_()
    tr.replay(g)
    torch.cuda.synchronize()
    scene = scenegen.Scene(w.scene.P, w.scene.sh_degree, snap)
    rng = np.random.default_rng(11)
    nb = len(tr.bufs)
    for v in (len(cams) - 4, len(cams) - 1):  # buffer v % nb last held view v
        assert v + nb >= len(cams)
        cam = cams[v]
        px, py = rng.integers(0, cam.width, 1500), rng.integers(0, cam.height, 1500)
        ref = gsref.render_pixels(cam, scene, px, py, gsref.F32)
        rgb = tr.bufs[v % nb].rgb.cpu().numpy()[:, py, px]
        bad = np.abs(rgb - ref["rgb"]).max(0) > 1e-5
        assert (bad & ~flip_pixels(cam, scene, px, py)).sum() == 0
        K_ref = int(gsref.project(cam, scene, gsref.F32)["tiles"].sum())
        assert int(tr.num_keys[v].item()) == K_ref


def test_fused_l1_backward_matches_separate(lib):
    """gs_render_bwd_screen_l1 (Eq. 12 upstream inside the backward) gives the same
    screen-space gradients and loss as gs_l1_loss_grad + gs_render_bwd_screen."""
    w = workload("small")
    cam, scene = w.cameras[0], w.scene
    proj, t, params = gpu_project(lib, cam, scene)
    b = gpu_bin(lib, cam, scene, proj)
    out = gpu_render(lib, cam, scene, proj, b["sorted_ids"], b["ranges"])
    tw = scenegen.make("small").target_scene
    tproj, _, _ = gpu_project(lib, cam, tw)
    tb = gpu_bin(lib, cam, tw, tproj)
    tgt = gpu_render(lib, cam, tw, tproj, tb["sorted_ids"], tb["ranges"])
    sc = gsr.scene_desc(scene.P, scene.P_stride, scene.sh_degree)
    gcam = gsr.camera(cam)
    g_rgb, g_d = torch.empty_like(out["rgb"]), torch.empty_like(out["depth"])
    loss_a, loss_b = torch.zeros(1, device=DEV), torch.zeros(1, device=DEV)
    lib.l1_loss_grad(out["rgb"], out["depth"], tgt["rgb"], tgt["depth"], 0.7, g_rgb, g_d, loss_a)
    det = torch.empty((b["K"] + 16, 12), device=DEV)
    sa = torch.zeros((scene.P, 12), device=DEV)
    lib.render_bwd_screen(gcam, sc, proj, b["sorted_ids"], b["ranges"], out["T_final"], out["n_contrib"], g_rgb, g_d, sa,
                          det=det)
    sb = torch.zeros((scene.P, 12), device=DEV)
    lib.render_bwd_screen_l1(gcam, sc, proj, b["sorted_ids"], b["ranges"], out["T_final"], out["n_contrib"],
                             out["rgb"], out["depth"], tgt["rgb"], tgt["depth"], 0.7, sb, loss=loss_b, det=det)
    torch.cuda.synchronize()
    assert loss_b.item() == pytest.approx(loss_a.item(), rel=1e-5)
    a, c = sa.cpu().numpy(), sb.cpu().numpy()
    assert np.abs(a).max() > 0
    assert np.array_equal(c, a)  # same upstream values, deterministic reduction: bit-identical


def test_project_views_bitexact_vs_project(lib):
    """gs_project_views (one pass over the parameters for a batch of views) writes, for
    every view, exactly gs_project's outputs: records of visible Gaussians, radius,
    tiles, flags -- 11 views (two batches of <= 8), the Morton-ordered scannetpp scene."""
    w = workload("scannetpp")
    scene = w.scene
    params = torch.from_numpy(scene.params).to(DEV)
    sc = gsr.scene_desc(scene.P, scene.P_stride, scene.sh_degree)
    cams = [w.cameras[k % len(w.cameras)] for k in range(11)]
    cams[9] = scenegen.camera_rt(320, 240, 300.0, 160.0, 120.0, scenegen.rot_y(2.0), [0.0, 0.0, 0.0])  # other size
    outs, refs = [], []
    for cam in cams:
        pa, ta = gsr.make_proj(scene.P, DEV)
        pb, tb = gsr.make_proj(scene.P, DEV)
        lib.project(gsr.camera(cam), sc, params, pb)
        outs.append((pa, ta))
        refs.append(tb)
    lib.project_views([gsr.camera(c) for c in cams], sc, params, [o[0] for o in outs])
    torch.cuda.synchronize()
    for (pa, ta), tb in zip(outs, refs):
        P = scene.P
        for key in ("radius", "tiles", "flags"):
            assert torch.equal(ta[key][:P], tb[key][:P]), key
        vis = tb["radius"][:P] > 0
        assert int(vis.sum()) > 0
        ra = ta["rec"][:P][vis].view(torch.int32)
        rb = tb["rec"][:P][vis].view(torch.int32)
        assert torch.equal(ra[:, :10], rb[:, :10]) and torch.equal(ra[:, 10:12], rb[:, 10:12])


@pytest.mark.parametrize("kind", ["sharded", "peer", "allreduce"])
def test_graph_capture_with_exchange(lib, kind):
    """The N > 1 iteration as one CUDA graph (bench.py at N > 1): the exchange (NCCL
    reduce-scatter / all-gather, the peer-memory kernel and its symmetric-memory
    barriers, or an NCCL all-reduce) and Adam with the device step counter captured with
    the views; replays are bit-identical to eager steps (deterministic mode; world size 1
    on this GPU, so the collectives run with one rank)."""
    import os
    import socket
    import torch.distributed as dist
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=DEV)
    try:
        w = workload("small")
        cams = [scenegen.camera_rt(320, 240, 300.0, 160.0, 120.0, scenegen.rot_y(0.03 * (k - 2)),
                                   [0.05 * k, 0.0, 0.0]) for k in range(4)]
        models = [pipeline.GaussianModel(w.scene, DEV) for _ in range(2)]
        tgt = pipeline.GaussianModel(w.target_scene, DEV)
        cap = pipeline.default_capacity(pipeline.measure_keys(lib, models[0], cams, DEV))
        targets = pipeline.render_targets(lib, tgt, cams, DEV, cap)
        trs = []
        for m in models:
            opt, ar = None, None
            if kind == "sharded":
                opt = pipeline.ShardedAdam(lib, m)
            elif kind == "peer":
                opt = pipeline.PeerShardedAdam(lib, m)
            else:
                ar = lambda g: dist.all_reduce(g, op=dist.ReduceOp.SUM)  # noqa: E731
            trs.append(pipeline.Trainer(lib, m, cams, targets, DEV, cap, streams=2, optimizer=opt, allreduce=ar,
                                        deterministic=True))
        views = list(range(len(cams)))
        trs[0].step(views)
        trs[1].step(views)
        g = trs[1].capture(views)  # one more eager step while capturing
        trs[0].step(views)
        for it in range(3):
            trs[0].step(views)
            trs[1].replay(g)
        torch.cuda.synchronize()
        assert models[0].step_count == models[1].step_count == int(models[1].step_dev.item()) == 5
        assert torch.equal(models[0].params, models[1].params)
        assert torch.equal(models[0].m, models[1].m) and torch.equal(models[0].v, models[1].v)
    finally:
        dist.destroy_process_group()
