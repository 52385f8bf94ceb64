"""World-size-2 gloo test of the data-parallel path's host logic (-m "not gpu").

The path shards a batch of views contiguously over ranks (scenegen.shard_views,
the function bench.py uses), sums per-view gradients locally, all-reduces (SUM)
once, then runs a replicated Adam step (reading R21).  Here the
per-rank compute is the CPU oracle; the test checks that the all-reduced gradient
equals the single-process sum over all views and that parameters stay
bit-identical across ranks after Adam.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import scenegen

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _views():
    w = scenegen.make("tiny")
    cams = []
    for k in range(5):  # 5 views over 2 ranks: uneven shards (3 + 2)
        R = scenegen.rot_y(0.06 * (k - 2))
        cams.append(scenegen.camera_rt(64, 48, 60.0, 32.0, 24.0, R, [0.1 * np.cos(k), 0.1 * np.sin(k), 0.2]))
    return w, cams


def _view_grad(w, cam):
    from oracle import gsref
    tgt = gsref.render_fwd(cam, w.target_scene, gsref.F32)
    f = gsref.render_fwd(cam, w.scene, gsref.F32)
    _, g_rgb, g_d = gsref.l1_loss_grad(f["rgb"], f["depth"], tgt["rgb"].astype(np.float32),
                                       tgt["depth"].astype(np.float32), 1.0)
    grad, _ = gsref.render_bwd(cam, w.scene, g_rgb.astype(np.float32), g_d.astype(np.float32), mode=gsref.MIXED)
    return grad


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import gsref
    w, cams = _views()
    g = np.zeros((w.scene.F, w.scene.P))
    mine = scenegen.shard_views(len(cams), rank, world)
    for v in mine:
        g += _view_grad(w, cams[v])
    t = torch.from_numpy(g)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    grad = np.zeros_like(w.scene.params)
    grad[:, :w.scene.P] = t.numpy()
    z = np.zeros_like(w.scene.params)
    from paper_2408_12677_b200.pipeline import lr_per_row
    p1, _, _ = gsref.adam_step(w.scene.params, grad, z, z, np.array(lr_per_row(0), np.float32), 1)
    gathered = [torch.zeros(p1.size, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(gathered, torch.from_numpy(p1.ravel().copy()))
    if rank == 0:
        out["grad"] = t.numpy().copy()
        out["params"] = [x.numpy().copy() for x in gathered]
        out["shards"] = [scenegen.shard_views(len(cams), r, world) for r in range(world)]
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_shard_views_partition():
    for B in (1, 5, 8, 64):
        for R in (1, 2, 3, 4, 8):
            shards = [scenegen.shard_views(B, r, R) for r in range(R)]
            flat = [v for s in shards for v in s]
            assert flat == list(range(B))
            assert max(map(len, shards)) - min(map(len, shards)) <= 1


def test_gloo_two_ranks_allreduce_matches_sum():
    from oracle import gsref
    gsref.build()
    mgr = mp.get_context("spawn").Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    w, cams = _views()
    ref = sum(_view_grad(w, c) for c in cams)
    assert all(np.abs(_view_grad(w, c)).sum() > 0 for c in cams)  # every view contributes
    np.testing.assert_allclose(out["grad"], ref, rtol=1e-12, atol=1e-15)
    assert out["shards"] == [[0, 1], [2, 3, 4]]
    np.testing.assert_array_equal(out["params"][0], out["params"][1])


def _sharded_worker(rank, world, port, out):
    """pipeline.ShardedAdam on gloo: reduce-scatter (emulated) -> Adam on the rank's
    shard (here the CPU oracle's Adam restricted to the range) -> all-gather."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import gsref
    from paper_2408_12677_b200 import pipeline
    w, _ = _views()
    model = pipeline.GaussianModel(w.scene, torch.device("cpu"))
    rng = np.random.default_rng(100 + rank)
    model.grad.copy_(torch.from_numpy(rng.normal(size=model.grad.shape).astype(np.float32)))
    lr = np.array(model.lr, np.float32)

    def adam_range(b, e, g):
        S = model.P_stride
        p = model.params.numpy().astype(np.float64).reshape(-1).copy()
        full_g = np.zeros_like(p)
        full_g[b:e] = g[:e - b].numpy()
        mm = model.m.numpy().reshape(-1).astype(np.float64)
        vv = model.v.numpy().reshape(-1).astype(np.float64)
        p1, m1, v1 = gsref.adam_step(p.reshape(model.F, S), full_g.reshape(model.F, S), mm.reshape(model.F, S),
                                     vv.reshape(model.F, S), lr, model.step_count, P=S)
        model.params.view(-1)[b:e] = torch.from_numpy(p1.reshape(-1)[b:e].astype(np.float32))
        model.m.view(-1)[b:e] = torch.from_numpy(m1.reshape(-1)[b:e].astype(np.float32))
        model.v.view(-1)[b:e] = torch.from_numpy(v1.reshape(-1)[b:e].astype(np.float32))

    opt = pipeline.ShardedAdam(None, model, adam_range=adam_range)
    g_local = model.grad.clone()
    model.step_count += 1
    opt.step()
    gathered = [torch.zeros(model.params.numel()) for _ in range(world)]
    dist.all_gather(gathered, model.params.reshape(-1).contiguous())
    glist = [torch.zeros(g_local.numel()) for _ in range(world)]
    dist.all_gather(glist, g_local.reshape(-1).contiguous())
    if rank == 0:
        out["params"] = [x.numpy().copy() for x in gathered]
        out["grads"] = [x.numpy().copy() for x in glist]
        out["shard"], out["n"] = opt.shard, opt.n
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_two_ranks_sharded_adam_matches_replicated():
    from oracle import gsref
    from paper_2408_12677_b200 import pipeline
    mgr = mp.get_context("spawn").Manager()
    out = mgr.dict()
    mp.spawn(_sharded_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    w, _ = _views()
    F, S = w.scene.params.shape
    assert out["n"] == F * S and out["shard"] % 4 == 0 and 2 * out["shard"] >= F * S
    gsum = (out["grads"][0].astype(np.float32) + out["grads"][1].astype(np.float32)).astype(np.float64)
    z = np.zeros((F, S))
    ref, _, _ = gsref.adam_step(w.scene.params.astype(np.float64), gsum.reshape(F, S), z, z,
                                np.array(pipeline.lr_per_row(0), np.float32), 1, P=S)
    np.testing.assert_array_equal(out["params"][0], out["params"][1])  # bit-identical across ranks
    np.testing.assert_allclose(out["params"][0].reshape(F, S), ref, rtol=1e-6, atol=1e-7)


def _torch_sparse_ops(model):
    """CPU stand-ins with the device calls' signatures (test only)."""
    from oracle import gsref

    def union(flags, P, vis, acc):
        u = torch.zeros(P, dtype=torch.bool)
        for f in flags:
            u |= (f[:P] & 128) == 0
        vis[:P] = (vis[:P].bool() | u).to(torch.uint8) if acc else u.to(torch.uint8)

    def compact(vis, P, ws, idx, cnt):
        nz = torch.nonzero(vis[:P]).flatten().to(torch.int32)
        idx[:len(nz)] = nz
        cnt[0] = len(nz)

    def gather(full, F, S, idx, M, packed):
        packed.copy_(full[:, idx[:M].long()])

    def scatter(packed, F, S, idx, M, full):
        full[:, idx[:M].long()] = packed

    def adam():
        S = model.P_stride
        p1, m1, v1 = gsref.adam_step(model.params.numpy().astype(np.float64), model.grad.numpy().astype(np.float64),
                                     model.m.numpy().astype(np.float64), model.v.numpy().astype(np.float64),
                                     np.array(model.lr, np.float32), model.step_count, P=S)
        model.params.copy_(torch.from_numpy(p1.astype(np.float32)))
        model.m.copy_(torch.from_numpy(m1.astype(np.float32)))
        model.v.copy_(torch.from_numpy(v1.astype(np.float32)))

    return {"union": union, "compact_workspace": lambda P: 16, "compact": compact, "gather": gather,
            "scatter": scatter, "adam": adam}


def _sparse_worker(rank, world, port, out):
    """pipeline.SparseExchangeAdam on gloo: each rank's gradient is zero outside the
    columns its views see; only the union's columns are all-reduced."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2408_12677_b200 import pipeline
    w, _ = _views()
    model = pipeline.GaussianModel(w.scene, torch.device("cpu"))
    P = model.P
    rng = np.random.default_rng(200 + rank)
    flags = [torch.from_numpy(np.where(rng.random(P + 16) < 0.3, 0, 128).astype(np.uint8)) for _ in range(2)]
    seen = np.zeros(model.P_stride, bool)
    for f in flags:
        seen[:P] |= (f.numpy()[:P] & 128) == 0
    g = rng.normal(size=model.grad.shape).astype(np.float32) * seen[None, :]
    model.grad.copy_(torch.from_numpy(g))
    opt = pipeline.SparseExchangeAdam(None, model, ops=_torch_sparse_ops(model))
    opt.note_views(flags[:1])
    opt.note_views(flags[1:])
    g_local = model.grad.clone()
    model.step_count += 1
    opt.step()
    gathered = [torch.zeros(model.params.numel()) for _ in range(world)]
    dist.all_gather(gathered, model.params.reshape(-1).contiguous())
    glist = [torch.zeros(g_local.numel()) for _ in range(world)]
    dist.all_gather(glist, g_local.reshape(-1).contiguous())
    seen_all = [torch.zeros(model.P_stride, dtype=torch.uint8) for _ in range(world)]
    dist.all_gather(seen_all, torch.from_numpy(seen.astype(np.uint8)))
    if rank == 0:
        out["params"] = [x.numpy().copy() for x in gathered]
        out["grads"] = [x.numpy().copy() for x in glist]
        out["seen"] = [x.numpy().copy() for x in seen_all]
        out["M"] = opt.last_M
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_two_ranks_sparse_exchange_matches_dense():
    from oracle import gsref
    from paper_2408_12677_b200 import pipeline
    mgr = mp.get_context("spawn").Manager()
    out = mgr.dict()
    mp.spawn(_sparse_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    w, _ = _views()
    F, S = w.scene.params.shape
    union = (out["seen"][0] | out["seen"][1]).astype(bool)
    assert out["M"] == int(union.sum()) and 0 < out["M"] < w.scene.P
    gsum = (out["grads"][0].astype(np.float32) + out["grads"][1].astype(np.float32)).astype(np.float64)
    z = np.zeros((F, S))
    ref, _, _ = gsref.adam_step(w.scene.params.astype(np.float64), gsum.reshape(F, S), z, z,
                                np.array(pipeline.lr_per_row(0), np.float32), 1, P=S)
    np.testing.assert_array_equal(out["params"][0], out["params"][1])  # bit-identical across ranks
    np.testing.assert_array_equal(out["params"][0].reshape(F, S), ref.astype(np.float32))
