"""gs_decode_rgbd (input frames, R41) against the oracle (bit-exact), its error
behaviour, and the sensor-frame path of Trainer.step_host (the bench's e2e leg)."""
import numpy as np
import pytest
import torch

import scenegen
from gpu_helpers import DEV
from oracle import frame
from paper_2408_12677_b200 import gsr, pipeline

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def lib():
    return gsr.load()


def _frame(seed, H, W):
    rng = np.random.default_rng(seed)
    c = rng.integers(0, 256, (H, W, 3)).astype(np.uint8)
    d = rng.integers(0, 65536, (H, W)).astype(np.uint16)
    k = min(3, H * W)
    c.reshape(-1)[:3] = (0, 255, 51)
    d.reshape(-1)[:k] = (0, 65535, 1000)[:k]
    return c, d


def _gpu_decode(lib, c, d, scale, offset=0):
    """Decode on the GPU; offset > 0 shifts every buffer off its 16-B alignment."""
    H, W = d.shape
    n = H * W
    c_t = torch.zeros(n * 3 + 16, dtype=torch.uint8, device=DEV)
    d_t = torch.zeros(n + 8, dtype=torch.int16, device=DEV)
    o_rgb = torch.full((3 * n + 8,), -1.0, dtype=torch.float32, device=DEV)
    o_d = torch.full((n + 8,), -1.0, dtype=torch.float32, device=DEV)
    cv = c_t[offset:offset + 3 * n].view(H, W, 3)
    dv = d_t[offset:offset + n].view(H, W)
    cv.copy_(torch.from_numpy(c))
    dv.copy_(torch.from_numpy(d.view(np.int16)))
    rv, ov = o_rgb[offset:offset + 3 * n].view(3, H, W), o_d[offset:offset + n].view(H, W)
    lib.decode_rgbd(cv, dv, scale, rv, ov)
    torch.cuda.synchronize()
    # nothing written outside the outputs
    assert bool((o_rgb[:offset] == -1).all()) and bool((o_rgb[offset + 3 * n:] == -1).all())
    assert bool((o_d[:offset] == -1).all()) and bool((o_d[offset + n:] == -1).all())
    return rv.cpu().numpy(), ov.cpu().numpy()


@pytest.mark.parametrize("hw", [(1, 1), (3, 5), (16, 16), (37, 29), (584, 876), (1168, 1752)])
@pytest.mark.parametrize("offset", [0, 1])
def test_decode_bitexact(lib, hw, offset):
    """Vectorised (W*H % 4 == 0, aligned) and per-pixel paths; odd sizes; misaligned buffers."""
    H, W = hw
    c, d = _frame(H * 7 + W, H, W)
    for scale in (1e-3, 1.0 / 6553.5):
        rgb, dep = _gpu_decode(lib, c, d, scale, offset)
        r_rgb, r_dep = frame.decode_rgbd(c, d, scale)
        assert np.array_equal(rgb.view(np.uint32), r_rgb.view(np.uint32))
        assert np.array_equal(dep.view(np.uint32), r_dep.view(np.uint32))


def test_decode_argument_errors(lib):
    c = torch.zeros((4, 4, 3), dtype=torch.uint8, device=DEV)
    d = torch.zeros((4, 4), dtype=torch.int16, device=DEV)
    o_rgb = torch.empty((3, 4, 4), device=DEV)
    o_d = torch.empty((4, 4), device=DEV)
    for scale in (0.0, -1.0, float("inf"), float("nan")):
        with pytest.raises(gsr.GsError):
            lib.decode_rgbd(c, d, scale, o_rgb, o_d)
    st = lib.lib.gs_decode_rgbd(0, 4, c.data_ptr(), d.data_ptr(), 1e-3, o_rgb.data_ptr(), o_d.data_ptr(), None)
    assert st == gsr.GS_ERR_ARG
    st = lib.lib.gs_decode_rgbd(4, 4, None, d.data_ptr(), 1e-3, o_rgb.data_ptr(), o_d.data_ptr(), None)
    assert st == gsr.GS_ERR_ARG
    with pytest.raises(ValueError):
        lib.decode_rgbd(c.view(4, 12), d, 1e-3, o_rgb, o_d)


@pytest.mark.parametrize("streams", [1, 3])
def test_step_host_sensor_frames_match_decoded_targets(lib, streams):
    """Trainer.step_host with uint8 / 16-bit sensor frames (copied + decoded on the copy
    stream) gives the iteration of Trainer.step on the oracle-decoded float targets."""
    w = scenegen.make("small")
    models = [pipeline.GaussianModel(w.scene, DEV) for _ in range(2)]
    tgt_model = pipeline.GaussianModel(w.target_scene, DEV)
    cap = pipeline.default_capacity(pipeline.measure_keys(lib, models[0], w.cameras, DEV))
    cams = [w.cameras[0]] * 5  # 5 views through the slots: slot reuse within one step
    rendered = pipeline.render_targets(lib, tgt_model, cams, DEV, cap)
    host, targets = {}, []
    for v, (r, d) in enumerate(rendered):
        c8, d16 = scenegen.quantize_frame(r.cpu().numpy(), d.cpu().numpy())
        host[v] = (torch.from_numpy(c8).pin_memory(), torch.from_numpy(d16.view(np.int16)).pin_memory())
        o_rgb, o_d = frame.decode_rgbd(c8, d16, scenegen.DEPTH_SCALE)
        targets.append((torch.from_numpy(o_rgb).to(DEV), torch.from_numpy(o_d).to(DEV)))
    trs = [pipeline.Trainer(lib, m, cams, targets, DEV, cap, streams=streams, deterministic=True) for m in models]
    for it in range(3):
        for tr in trs:
            tr.loss.zero_()
            tr.blended.zero_()
        trs[0].step(list(range(len(cams))))
        trs[1].step_host(list(range(len(cams))), host, scenegen.DEPTH_SCALE)
        torch.cuda.synchronize()
        assert trs[1].loss.item() == pytest.approx(trs[0].loss.item(), rel=1e-5)
        if it == 0:
            assert trs[1].blended.item() == trs[0].blended.item()
    assert torch.equal(models[0].params, models[1].params)  # deterministic reduction: bit-identical
    with pytest.raises(ValueError):
        trs[1].step_host([0], host)  # sensor frames need depth_scale


@pytest.mark.parametrize("graph_copies", [False, True])
def test_host_streamed_graphs_match_step_host(lib, graph_copies):
    """pipeline.HostStreamedGraphs (bench.py's e2e path for the batched configs: per step
    parity a frame copy + decode on a copy stream and a captured iteration reading those
    slots, the loss read back on a side stream) gives the iterations of Trainer.step on
    the oracle-decoded targets bit for bit (deterministic reduction)."""
    w = scenegen.make("small")
    models = [pipeline.GaussianModel(w.scene, DEV) for _ in range(2)]
    tgt_model = pipeline.GaussianModel(w.target_scene, DEV)
    cams = [scenegen.camera_rt(320, 240, 300.0, 160.0, 120.0, scenegen.rot_y(0.03 * (k - 2)), [0.05 * k, 0.0, 0.0])
            for k in range(4)]
    cap = pipeline.default_capacity(pipeline.measure_keys(lib, models[0], cams, DEV))
    rendered = pipeline.render_targets(lib, tgt_model, cams, DEV, cap)
    host, targets = {}, []
    for v, (r, d) in enumerate(rendered):
        c8, d16 = scenegen.quantize_frame(r.cpu().numpy(), d.cpu().numpy())
        host[v] = (torch.from_numpy(c8).pin_memory(), torch.from_numpy(d16.view(np.int16)).pin_memory())
        o_rgb, o_d = frame.decode_rgbd(c8, d16, scenegen.DEPTH_SCALE)
        targets.append((torch.from_numpy(o_rgb).to(DEV), torch.from_numpy(o_d).to(DEV)))
    trs = [pipeline.Trainer(lib, m, cams, targets, DEV, cap, streams=2, deterministic=True) for m in models]
    views = list(range(len(cams)))
    hs = pipeline.HostStreamedGraphs(trs[1], views, [host, host], scenegen.DEPTH_SCALE, graph_copies=graph_copies)
    trs[0].step(views)  # HostStreamedGraphs' two captures ran one eager iteration each
    trs[0].step(views)
    for it in range(4):
        trs[0].loss.zero_()
        trs[0].step(views)
        p = hs.step(prefetch=it + 2 < 4)
        torch.cuda.synchronize()
        # (the loss sums warp partials by atomics in any order: equal to fp32 rounding)
        assert hs.loss_host[p].item() == pytest.approx(trs[0].loss.item(), rel=1e-5)
    assert models[0].step_count == models[1].step_count == 6
    assert torch.equal(models[0].params, models[1].params)
    assert torch.equal(models[0].m, models[1].m) and torch.equal(models[0].v, models[1].v)
