"""The data-parallel exchange with MORE THAN ONE TERM, on one GPU (-m gpu).

Only one GPU exists in this run, so the ranks' sums are formed the two ways that do
not need a second device (and never make one rank's kernels wait on another's):

* gs_adam_step_peers / _dev with world = 2 pointer tables whose "peer" buffers are two
  gradient / parameter buffer sets on the same GPU, each rank's launch updating its own
  shard: the result is the oracle's Adam of the SUM of both gradients, bit-identical in
  both parameter copies, and the device-step variant equals the host-step one.
* Trainer.step in two processes (gloo group, both on cuda:0), each rendering its shard of
  the views and all-reducing the gradient through the host: the summed gradient against
  the oracle's sum over ALL views (element by element with the running error bound),
  Adam against the oracle's Adam of that gradient, and both ranks' parameters identical.
"""
import os
import socket
import tempfile

import numpy as np
import pytest
import torch

import scenegen
from oracle import gsref

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_2408_12677_b200 import gsr, pipeline
    from gpu_helpers import DEV, assert_grad_parity, flip_pixels


def _adam_ref(p, g, m, v, lr, step):
    b1, b2, eps = (float(np.float32(x)) for x in (0.9, 0.999, 1e-15))
    return gsref.adam_step(p, g, m, v, np.array(lr, np.float32), step, beta1=b1, beta2=b2, eps=eps, P=p.shape[1])


@pytest.mark.parametrize("device_step", [False, True])
def test_adam_peers_world2_sums_two_ranks(device_step):
    lib = gsr.load()
    rng = np.random.default_rng(7)
    deg, P = 1, 1000
    F = 11 + 3 * 4
    S = scenegen.pad4(P)
    sc = gsr.scene_desc(P, S, deg)
    lr = pipeline.lr_per_row(deg)
    p0 = rng.normal(size=(F, S)).astype(np.float32)
    g = [rng.normal(size=(F, S)).astype(np.float32) for _ in range(2)]
    m0 = (rng.normal(size=(F, S)) * 1e-2).astype(np.float32)
    v0 = rng.uniform(0, 1e-3, size=(F, S)).astype(np.float32)
    grads = [torch.from_numpy(x).to(DEV) for x in g]
    params = [torch.from_numpy(p0).to(DEV) for _ in range(2)]
    ms = [torch.from_numpy(m0).to(DEV) for _ in range(2)]
    vs = [torch.from_numpy(v0).to(DEV) for _ in range(2)]
    gptr = [t.data_ptr() for t in grads]
    pptr = [t.data_ptr() for t in params]
    n = F * S
    shard = ((n + 1) // 2 + 3) // 4 * 4
    steps = [torch.full((1,), 2, dtype=torch.int64, device=DEV) for _ in range(2)]
    for r in range(2):
        b, e = min(r * shard, n), min((r + 1) * shard, n)
        lib.adam_step_peers(sc, 2, r, gptr, pptr, ms[r], vs[r], lr, steps[r] if device_step else 3, b, e)
    torch.cuda.synchronize()
    if device_step:
        assert all(int(t.item()) == 3 for t in steps)
    assert torch.equal(params[0], params[1])  # every rank's copy receives every shard
    rp, rm, rv = _adam_ref(p0, g[0].astype(np.float64) + g[1], m0, v0, lr, 3)
    got = params[0].cpu().numpy()
    b1, b2 = float(np.float32(0.9)), float(np.float32(0.999))
    gs = np.abs(g[0].astype(np.float64)) + np.abs(g[1])
    lr_col = np.array(lr, np.float64)[:, None]
    assert np.all(np.abs(got - rp) <= 1e-6 * (np.abs(p0) + lr_col) + 4e-7 * lr_col * gs / (np.abs(g[0] + g[1]) + 1e-30))
    # each rank's moments were updated on its own shard only, with the summed gradient
    mm = np.concatenate([ms[0].cpu().numpy().reshape(-1)[:shard], ms[1].cpu().numpy().reshape(-1)[shard:]]).reshape(F, S)
    sm = b1 * np.abs(m0) + (1 - b1) * gs
    assert np.all(np.abs(mm - rm) <= 1e-6 * sm + 1e-12)
    vv = np.concatenate([vs[0].cpu().numpy().reshape(-1)[:shard], vs[1].cpu().numpy().reshape(-1)[shard:]]).reshape(F, S)
    assert np.all(np.abs(vv - rv) <= 1e-6 * (b2 * np.abs(v0) + (1 - b2) * gs * gs) + 1e-15)


def test_adam_peers_dev_equals_host_step():
    """gs_adam_step_peers_dev (graph-capturable) == gs_adam_step_peers bit for bit."""
    lib = gsr.load()
    rng = np.random.default_rng(8)
    P, deg = 512, 0
    F, S = 14, 512
    sc = gsr.scene_desc(P, S, deg)
    lr = pipeline.lr_per_row(deg)
    arrs = [rng.normal(size=(F, S)).astype(np.float32) for _ in range(4)]
    outs = []
    for dev_step in (False, True):
        p, g, m = (torch.from_numpy(a.copy()).to(DEV) for a in arrs[:3])
        v = torch.from_numpy(np.abs(arrs[3])).to(DEV)
        for t in range(1, 4):
            step = torch.full((1,), t - 1, dtype=torch.int64, device=DEV) if dev_step else t
            lib.adam_step_peers(sc, 1, 0, [g.data_ptr()], [p.data_ptr()], m, v, lr, step, 0, F * S)
        torch.cuda.synchronize()
        outs.append((p.cpu(), m.cpu(), v.cpu()))
    for a, b in zip(*outs):
        assert torch.equal(a, b)


# ----------------------------------------------------------------------------- two processes
def _views():
    w = scenegen.make("small")
    cams = [scenegen.camera_rt(320, 240, 300.0, 160.0, 120.0, scenegen.rot_y(0.04 * (k - 1.5)),
                               [0.06 * (k - 1.5), 0.03 * k, 0.0]) for k in range(4)]
    return w, cams


def _targets(w, cams):
    """Oracle-side targets: the oracle's fp32 render +- offsets (signs fixed by oracle
    data alone), NaN at possible threshold-flip pixels (no loss, R43)."""
    rng = np.random.default_rng(31)
    out, fields = [], []
    npix = cams[0].width * cams[0].height
    s_c, s_d = np.float32(1.0 / (3.0 * npix)), np.float32(1.0 / npix)
    for cam in cams:
        f = gsref.render_fwd(cam, w.scene, gsref.F32)
        sg = rng.choice([-1.0, 1.0], size=(4, cam.height, cam.width))
        tr = (f["rgb"] + 0.02 * sg[:3]).astype(np.float32)
        td = (f["depth"] + sg[3] * (0.01 + 0.01 * np.abs(f["depth"]))).astype(np.float32)
        flip = flip_pixels(cam, w.scene)
        tr[:, flip] = np.nan
        td[flip] = np.nan
        gr = np.where(np.isfinite(tr), np.sign(f["rgb"] - tr) * s_c, 0).astype(np.float32)
        gd = np.where(np.isfinite(td) & (td > 0), np.sign(f["depth"] - td) * s_d, 0).astype(np.float32)
        out.append((tr, td))
        fields.append((gr, gd))
    return out, fields, float(s_c)


def _rank_main(rank, world, port, outdir):
    import torch.distributed as dist
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        lib = gsr.load()
        w, cams = _views()
        tgt, _, _ = _targets(w, cams)
        mine = scenegen.shard_views(len(cams), rank, world)
        model = pipeline.GaussianModel(w.scene, DEV)
        cap = pipeline.default_capacity(pipeline.measure_keys(lib, model, cams, DEV))
        targets = [(torch.from_numpy(a).to(DEV), torch.from_numpy(b).to(DEV)) for a, b in tgt]
        grads = {}

        def allreduce(g):  # the exchange through the host (gloo): g := sum over ranks
            c = g.cpu()
            grads["local"] = c.clone()
            dist.all_reduce(c, op=dist.ReduceOp.SUM)
            g.copy_(c)
            grads["sum"] = c.clone()
        tr = pipeline.Trainer(lib, model, cams, targets, DEV, cap, allreduce=allreduce, streams=2)
        tr.step(mine)
        torch.cuda.synchronize()
        np.savez(os.path.join(outdir, f"r{rank}.npz"), params=model.params.cpu().numpy(),
                 grad_sum=grads["sum"].numpy(), grad_local=grads["local"].numpy(), views=np.array(mine))
    finally:
        dist.destroy_process_group()


def test_trainer_step_world2_gloo_one_gpu():
    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    with tempfile.TemporaryDirectory() as d:
        mp.start_processes(_rank_main, args=(2, port, d), nprocs=2, join=True, start_method="spawn")
        r = [np.load(os.path.join(d, f"r{k}.npz")) for k in range(2)]
    w, cams = _views()
    _, fields, s_c = _targets(w, cams)
    assert sorted(np.concatenate([x["views"] for x in r]).tolist()) == [0, 1, 2, 3]
    assert np.array_equal(r[0]["params"], r[1]["params"])  # replicated Adam on the same sum
    assert np.array_equal(r[0]["grad_sum"], r[1]["grad_sum"])
    P, F = w.scene.P, w.scene.F
    # the summed gradient: the oracle's sum over all four views (R21)
    ref = np.zeros((F, P))
    bound = np.zeros((F, P))
    for cam, (gr, gd) in zip(cams, fields):
        b = gsref.render_bwd_bound(cam, w.scene, gr, gd)
        ref += b["grad"]
        bound += b["bound"] + np.abs(b["grad"])  # the view / rank sums are accumulations too
    g = r[0]["grad_sum"][:, :P].astype(np.float64)
    assert np.count_nonzero(r[0]["grad_local"]) and np.count_nonzero(r[1]["grad_local"])
    assert not np.array_equal(r[0]["grad_local"], r[0]["grad_sum"])  # a real two-term sum
    assert_grad_parity(g, ref, bound, scale=s_c, what="all-reduced gradient (2 ranks)")
    # Adam of that gradient (step 1 from zero moments), against the oracle's Adam
    lr = pipeline.lr_per_row(w.scene.sh_degree)
    S = w.scene.params.shape[1]
    zero = np.zeros((F, S), np.float32)
    rp, _, _ = _adam_ref(w.scene.params, r[0]["grad_sum"], zero, zero, lr, 1)
    lr_col = np.array(lr, np.float64)[:, None]
    assert np.all(np.abs(r[0]["params"] - rp) <= 1e-6 * (np.abs(w.scene.params) + lr_col))
