"""gs_fwd_state / GS_ERR_STATE (SPEC.md:345-353 StateMismatch) and the deterministic
reduction mode through the C ABI (-m gpu)."""
import numpy as np
import pytest
import torch

import scenegen
from oracle import gsref

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_2408_12677_b200 import gsr, pipeline
    from gpu_helpers import DEV, assert_grad_parity, flip_pixels, gpu_bin, gpu_project


def _view(lib, cam, scene, proj, b, key_blocks=True):
    H, W = cam.height, cam.width
    out = {"rgb": torch.empty((3, H, W), device=DEV), "depth": torch.empty((H, W), device=DEV),
           "T": torch.empty((H, W), device=DEV), "n": torch.empty((H, W), dtype=torch.int32, device=DEV),
           "kb": torch.zeros(b["K"] + 16, dtype=torch.uint8, device=DEV) if key_blocks else None,
           "state": gsr.GsFwdState()}
    lib.render_fwd(gsr.camera(cam), gsr.scene_desc(scene.P, scene.P_stride, scene.sh_degree), proj, b["sorted_ids"],
                   b["ranges"], out["rgb"], out["depth"], out["T"], out["n"], key_blocks=out["kb"],
                   fwd_state=out["state"])
    return out


def test_state_checks_through_the_abi():
    lib = gsr.load()
    w = scenegen.make("small")
    scene = w.scene
    sc = gsr.scene_desc(scene.P, scene.P_stride, scene.sh_degree)
    cams = [w.cameras[0], scenegen.camera_rt(320, 240, 300.0, 160.0, 120.0, scenegen.rot_y(0.1), [0.1, 0.0, 0.0])]
    views = []
    for cam in cams:
        proj, t, _ = gpu_project(lib, cam, scene)
        b = gpu_bin(lib, cam, scene, proj)
        views.append((cam, proj, b, _view(lib, cam, scene, proj, b)))
    (cam0, proj0, b0, v0), (cam1, proj1, b1, v1) = views
    assert v0["state"].id != 0 and v1["state"].id > v0["state"].id
    assert v0["state"].width == 320 and v0["state"].height == 240
    g_rgb, g_d = (torch.from_numpy(a).to(DEV) for a in scenegen.upstream_fields(1, 320, 240))
    sg = torch.zeros((scene.P, 12), device=DEV)
    gc0 = gsr.camera(cam0)

    def bwd(state, kb=v0["kb"], n=v0["n"], T=v0["T"], proj=proj0, ids=b0["sorted_ids"], cam=gc0):
        return lib.lib.gs_render_bwd_screen(
            gsr._ref(cam), gsr._ref(sc), proj, gsr._ptr(ids), gsr._ptr(b0["ranges"]), None, gsr._ptr(T),
            gsr._ptr(n), gsr._ptr(g_rgb), gsr._ptr(g_d), gsr._ptr(kb), gsr._ptr(sg),
            gsr._ref(gsr.bwd_opts(fwd=state)), gsr._stream())
    assert bwd(v0["state"]) == gsr.GS_OK
    # key masks / n_contrib / T_final / records / lists of ANOTHER forward -> GS_ERR_STATE
    assert bwd(v0["state"], kb=v1["kb"]) == gsr.GS_ERR_STATE and "key_blocks" in lib.last_error()
    assert bwd(v0["state"], n=v1["n"]) == gsr.GS_ERR_STATE
    assert bwd(v0["state"], T=v1["T"]) == gsr.GS_ERR_STATE
    assert bwd(v0["state"], proj=proj1) == gsr.GS_ERR_STATE and "proj.rec" in lib.last_error()
    assert bwd(v0["state"], ids=b1["sorted_ids"]) == gsr.GS_ERR_STATE
    small = gsr.camera(scenegen.identity_camera(160, 120, 150.0, 80.0, 60.0))
    assert bwd(v0["state"], cam=small) == gsr.GS_ERR_STATE and "size" in lib.last_error()
    # the fused-loss backward also checks the rendered images it reads
    t_img = torch.zeros_like(v0["rgb"])
    st = lib.lib.gs_render_bwd_screen_l1(
        gsr._ref(gc0), gsr._ref(sc), proj0, gsr._ptr(b0["sorted_ids"]), gsr._ptr(b0["ranges"]), None,
        gsr._ptr(v0["T"]), gsr._ptr(v0["n"]), gsr._ptr(v1["rgb"]), gsr._ptr(v0["depth"]), gsr._ptr(t_img),
        gsr._ptr(v0["depth"]), 1.0, None, gsr._ptr(v0["kb"]), gsr._ptr(sg), gsr._ref(gsr.bwd_opts(fwd=v0["state"])),
        gsr._stream())
    assert st == gsr.GS_ERR_STATE and "rgb" in lib.last_error()
    # a later forward into view 0's buffers makes the old state stale
    old = gsr.GsFwdState.from_buffer_copy(v0["state"])
    lib.render_fwd(gc0, sc, proj0, b0["sorted_ids"], b0["ranges"], v0["rgb"], v0["depth"], v0["T"], v0["n"],
                   key_blocks=v0["kb"], fwd_state=v0["state"])
    assert bwd(old) == gsr.GS_ERR_STATE and "rewritten" in lib.last_error()
    assert bwd(v0["state"]) == gsr.GS_OK
    with pytest.raises(gsr.GsError) as e:  # the binding raises with the status
        lib.render_bwd_screen(gc0, sc, proj0, b0["sorted_ids"], b0["ranges"], v0["T"], v0["n"], g_rgb, g_d, sg,
                              key_blocks=v1["kb"], fwd=v0["state"])
    assert e.value.status == gsr.GS_ERR_STATE
    torch.cuda.synchronize()


@pytest.mark.parametrize("name", ["small", "replica"])
def test_deterministic_mode_reproducible_and_oracle_exact(name):
    """gs_bwd_opts.det_ws: repeated backward passes (and a different tile schedule) give
    bit-identical screen gradients, which match the stage-wise oracle element by element
    like the atomic path does."""
    lib = gsr.load()
    kw = {"num_views": 1} if name == "replica" else {}
    w = scenegen.make(name, **kw)
    cam, scene = w.cameras[0], w.scene
    sc = gsr.scene_desc(scene.P, scene.P_stride, scene.sh_degree)
    gcam = gsr.camera(cam)
    proj, t, params = gpu_project(lib, cam, scene)
    b = gpu_bin(lib, cam, scene, proj)
    v = _view(lib, cam, scene, proj, b)
    keep = ~flip_pixels(cam, scene) if name == "small" else np.ones((cam.height, cam.width), bool)
    ur, ud = scenegen.upstream_fields(3, cam.width, cam.height)
    ur, ud = (ur * keep[None]).astype(np.float32), (ud * keep).astype(np.float32)
    g_rgb, g_d = torch.from_numpy(ur).to(DEV), torch.from_numpy(ud).to(DEV)
    det = torch.empty((b["K"] + 64, 12), device=DEV)
    order = torch.empty(cam.num_tiles, dtype=torch.int32, device=DEV)
    lib.tile_order(gcam, b["ranges"], order)
    outs = []
    for rep in range(3):
        sg = torch.zeros((scene.P, 12), device=DEV)
        lib.render_bwd_screen(gcam, sc, proj, b["sorted_ids"], b["ranges"], v["T"], v["n"], g_rgb, g_d, sg,
                              key_blocks=v["kb"], fwd=v["state"], det=det, tile_order=order if rep == 2 else None)
        torch.cuda.synchronize()
        outs.append(sg.cpu().numpy())
    assert np.array_equal(outs[0], outs[1]) and np.array_equal(outs[0], outs[2])
    assert np.abs(outs[0]).max() > 0
    if name == "small":  # full oracle comparison of the deterministic path
        grad = torch.zeros((scene.F, scene.P_stride), device=DEV)
        sg = torch.from_numpy(outs[0]).to(DEV)
        lib.project_bwd_views([gcam], sc, params, [t["flags"]], [sg], grad, accumulate=False)
        torch.cuda.synchronize()
        ref = gsref.render_bwd_bound(cam, scene, ur, ud)
        assert_grad_parity(outs[0][:, :10].T.astype(np.float64), ref["screen"], ref["screen_bound"],
                           what="deterministic screen-space gradient")
        assert_grad_parity(grad[:, :scene.P].cpu().numpy().astype(np.float64), ref["grad"], ref["bound"],
                           what="deterministic gradient")


def test_trainer_deterministic_runs_are_identical():
    """Two Trainers (deterministic mode, 3 streams with bin-ahead) from the same start give
    bit-identical parameters after several steps; the atomic path differs only within the
    element-wise tolerance of the first step's gradient."""
    lib = gsr.load()
    w = scenegen.make("small")
    cams = [scenegen.camera_rt(320, 240, 300.0, 160.0, 120.0, scenegen.rot_y(0.03 * (k - 2)), [0.05 * k, 0.0, 0.0])
            for k in range(5)]
    tgt = pipeline.GaussianModel(w.target_scene, DEV)
    models = [pipeline.GaussianModel(w.scene, DEV) for _ in range(2)]
    cap = pipeline.default_capacity(pipeline.measure_keys(lib, models[0], cams, DEV))
    targets = pipeline.render_targets(lib, tgt, cams, DEV, cap)
    trs = [pipeline.Trainer(lib, m, cams, targets, DEV, cap, streams=3, deterministic=True) for m in models]
    for _ in range(4):
        for tr in trs:
            tr.step(list(range(len(cams))))
    torch.cuda.synchronize()
    assert torch.equal(models[0].params, models[1].params)
    assert not torch.equal(models[0].params, torch.from_numpy(w.scene.params).to(DEV))
