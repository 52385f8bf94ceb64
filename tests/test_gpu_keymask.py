"""The forward's per-key block masks (gs_render_fwd key_blocks) used by the backward
give the same gradients as the geometric block masks, and both match the oracle
(-m gpu).  Also checks the mask semantics directly: a key's bit b is set iff the
Gaussian was composited into >= 1 pixel of 8x4 block b of its tile."""
import numpy as np
import pytest
import torch

import scenegen
from oracle import gsref

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_2408_12677_b200 import gsr
    from gpu_helpers import DEV, assert_grad_parity, flip_pixels, gpu_bin, gpu_project


def _run(name, seed=3):
    lib = gsr.load()
    kw = {"num_views": 1} if name in ("replica", "scannetpp") else {}
    w = scenegen.make(name, **kw)
    cam, scene = w.cameras[0], w.scene
    proj, t, params = gpu_project(lib, cam, scene)
    b = gpu_bin(lib, cam, scene, proj)
    K = b["K"]
    H, W = cam.height, cam.width
    sc = gsr.scene_desc(scene.P, scene.P_stride, scene.sh_degree)
    rgb = torch.empty((3, H, W), device=DEV)
    dep = torch.empty((H, W), device=DEV)
    T = torch.empty((H, W), device=DEV)
    n = torch.empty((H, W), dtype=torch.int32, device=DEV)
    kb = torch.full((max(K, 1) + 16,), 0xAB, dtype=torch.uint8, device=DEV)
    lib.render_fwd(gsr.camera(cam), sc, proj, b["sorted_ids"], b["ranges"], rgb, dep, T, n, key_blocks=kb)
    keep = ~flip_pixels(cam, scene)  # proven threshold flips: zero upstream on both sides
    g_rgb, g_d = (torch.from_numpy(np.ascontiguousarray(a * (keep[None] if a.ndim == 3 else keep)).astype(np.float32)).to(DEV)
                  for a in scenegen.upstream_fields(seed, W, H))
    out = {}
    for mode in ("geometric", "keymask"):
        ws = torch.zeros(scene.P * 12, device=DEV)
        grad = torch.zeros((scene.F, scene.P_stride), device=DEV)
        lib.render_bwd(gsr.camera(cam), sc, params, proj, b["sorted_ids"], b["ranges"], T, n, g_rgb, g_d, ws, grad,
                       key_blocks=kb if mode == "keymask" else None)
        torch.cuda.synchronize()
        out[mode] = grad[:, :scene.P].cpu().numpy().astype(np.float64)
    return w, cam, scene, b, n, kb, out, g_rgb, g_d


@pytest.mark.parametrize("name", ["tiny", "small"])
def test_keymask_backward_equals_geometric_and_oracle(name):
    w, cam, scene, b, n, kb, out, g_rgb, g_d = _run(name)
    # the full GPU chain (its own projection, lists, forward, key masks), every element
    ref = gsref.render_bwd_bound(cam, scene, g_rgb.cpu().numpy(), g_d.cpu().numpy())
    for mode in ("keymask", "geometric"):
        assert_grad_parity(out[mode], ref["grad"], ref["bound"], what=mode)


def test_keymask_semantics_small():
    """Bit b of a key set  <=>  the oracle composites that Gaussian into >= 1 pixel of
    block b of that tile (checked on every visited key of the small config)."""
    w, cam, scene, b, n, kb, out, _, _ = _run("small")
    ids = b["sorted_ids"].cpu().numpy()
    ranges = b["ranges"].cpu().numpy()
    kbn = kb.cpu().numpy()
    ref = gsref.render_fwd(cam, scene, gsref.F32, want_margin=True)
    pr = gsref.project(cam, scene, gsref.F32)
    nref = ref["n_contrib"]
    checked = 0
    for t in range(0, cam.num_tiles, 7):
        s, e = ranges[t]
        ty, tx = divmod(t, cam.tiles_x)
        tile_n = nref[ty * 16:(ty + 1) * 16, tx * 16:(tx + 1) * 16]
        maxn = int(tile_n.max())
        for pos in range(maxn):
            i = ids[s + pos]
            want = 0
            for blk in range(8):
                x0, y0 = tx * 16 + 8 * (blk & 1), ty * 16 + 4 * (blk >> 1)
                for yy in range(y0, min(y0 + 4, cam.height)):
                    for xx in range(x0, min(x0 + 8, cam.width)):
                        if pos >= nref[yy, xx]:
                            continue
                        dx, dy = pr["mu_x"][i] - xx, pr["mu_y"][i] - yy
                        pw = -0.5 * (pr["conic_A"][i] * dx * dx + pr["conic_C"][i] * dy * dy) - pr["conic_B"][i] * dx * dy
                        a = min(0.99, pr["opacity"][i] * np.exp(pw))
                        if pw <= 0 and a >= 1 / 255:
                            want |= 1 << blk
                            break
                    if want >> blk & 1:
                        break
            assert kbn[s + pos] == want, (t, pos, kbn[s + pos], want)
            checked += 1
    assert checked > 1000


def test_packed_gaussian_ids_match_unpacked():
    """The product backward packs each staged record's Gaussian id into its flag word
    when P < 2^22 (render.cu kPack) and reads it from shared memory otherwise.  The
    small scene alone (packed) and the same scene followed by 2^22 culled Gaussians
    (P >= 2^22: unpacked) have identical key lists, so their screen gradients agree
    (up to the atomics' summation order) and every culled Gaussian's stays zero."""
    lib = gsr.load()
    w = scenegen.make("small")
    cam, small = w.cameras[0], w.scene
    P_big = (1 << 22) + 64
    S_big = (P_big + 3) // 4 * 4
    pb = np.zeros((small.F, S_big), np.float32)
    pb[:, :small.P] = small.params[:, :small.P]
    pb[:, small.P:P_big] = small.params[:, :1]  # copies of Gaussian 0 ...
    pb[2, small.P:P_big] = -5.0  # ... behind the camera: culled, no keys
    big = scenegen.Scene(P_big, small.sh_degree, pb)
    sg = {}
    for nm, scene in (("packed", small), ("unpacked", big)):
        proj, t, params = gpu_project(lib, cam, scene)
        b = gpu_bin(lib, cam, scene, proj)
        H, W = cam.height, cam.width
        sc = gsr.scene_desc(scene.P, scene.P_stride, scene.sh_degree)
        rgb, dep, T = (torch.empty((3, H, W), device=DEV), torch.empty((H, W), device=DEV),
                       torch.empty((H, W), device=DEV))
        n = torch.empty((H, W), dtype=torch.int32, device=DEV)
        kb = torch.zeros((max(b["K"], 1) + 16,), dtype=torch.uint8, device=DEV)
        lib.render_fwd(gsr.camera(cam), sc, proj, b["sorted_ids"], b["ranges"], rgb, dep, T, n, key_blocks=kb)
        g_rgb, g_d = (torch.from_numpy(np.ascontiguousarray(a).astype(np.float32)).to(DEV)
                      for a in scenegen.upstream_fields(5, W, H))
        s = torch.zeros((scene.P, 12), device=DEV)
        lib.render_bwd_screen(gsr.camera(cam), sc, proj, b["sorted_ids"], b["ranges"], T, n, g_rgb, g_d, s,
                              key_blocks=kb)
        torch.cuda.synchronize()
        sg[nm] = s.cpu().numpy()
    a, c = sg["packed"], sg["unpacked"]
    assert np.abs(a).max() > 0
    assert not np.any(c[small.P:])
    # north_star's gradient tolerance (float atomics reorder the sums)
    np.testing.assert_allclose(c[:small.P], a, rtol=1e-3, atol=1e-6)


@pytest.mark.parametrize("name", ["small", "large"])
def test_render_rows_walk_identical(name):
    """gs_set_render_rows is a performance switch only: the forward (images, T, n_contrib,
    key masks) and, in deterministic-reduction mode, the backward's screen gradients are
    bit-identical with and without the block-row walk (large: config 4's small
    Gaussians, first view at full size)."""
    lib = gsr.load()
    kw = {"num_views": 1} if name == "large" else {}
    w = scenegen.make(name, **kw)
    cam, scene = w.cameras[0], w.scene
    proj, t, params = gpu_project(lib, cam, scene)
    b = gpu_bin(lib, cam, scene, proj)
    H, W = cam.height, cam.width
    sc = gsr.scene_desc(scene.P, scene.P_stride, scene.sh_degree)
    g_rgb, g_d = (torch.from_numpy(np.ascontiguousarray(a).astype(np.float32)).to(DEV)
                  for a in scenegen.upstream_fields(9, W, H))
    out = {}
    was = lib.render_rows()
    try:
        for mode in (0, 1):
            lib.set_render_rows(mode)
            assert lib.render_rows() == bool(mode)
            rgb, dep, T = (torch.empty((3, H, W), device=DEV), torch.empty((H, W), device=DEV),
                           torch.empty((H, W), device=DEV))
            n = torch.empty((H, W), dtype=torch.int32, device=DEV)
            kb = torch.zeros((max(b["K"], 1) + 16,), dtype=torch.uint8, device=DEV)
            lib.render_fwd(gsr.camera(cam), sc, proj, b["sorted_ids"], b["ranges"], rgb, dep, T, n, key_blocks=kb)
            s = torch.zeros((scene.P, 12), device=DEV)
            det = torch.empty((b["K"] + 16, 12), device=DEV)
            lib.render_bwd_screen(gsr.camera(cam), sc, proj, b["sorted_ids"], b["ranges"], T, n, g_rgb, g_d, s,
                                  key_blocks=kb, det=det)
            torch.cuda.synchronize()
            out[mode] = [x.cpu().numpy() for x in (rgb, dep, T, n, kb, s)]
    finally:
        lib.set_render_rows(was)
    for k, nm in enumerate(["rgb", "depth", "T", "n_contrib", "key_blocks", "sgrad (deterministic)"]):
        assert np.array_equal(out[0][k], out[1][k]), nm
    assert np.abs(out[0][5]).max() > 0
    # (the atomic form differs from run to run by summation order alone; its parity
    # with the oracle is test_gpu_parity's, whichever form the bench's autotune picks)
