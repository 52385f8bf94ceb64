"""Visibility-sparse gradient exchange: the union / ordered
compaction / gather / scatter kernels against numpy (bit-exact), and
pipeline.SparseExchangeAdam through a real NCCL group (world size 1) against the
replicated step."""
import numpy as np
import pytest
import torch

import scenegen
from gpu_helpers import DEV
from paper_2408_12677_b200 import gsr, pipeline

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def lib():
    return gsr.load()


def _flags(rng, n, P, p_vis):
    return [np.where(rng.random(P) < p_vis, rng.integers(0, 32, P), 128 | rng.integers(0, 32, P)).astype(np.uint8)
            for _ in range(n)]


@pytest.mark.parametrize("P", [0, 1, 4095, 4096, 70001])
@pytest.mark.parametrize("p_vis", [0.0, 0.3, 1.0])
def test_union_and_compaction(lib, P, p_vis):
    rng = np.random.default_rng(P + int(10 * p_vis))
    fa, fb = _flags(rng, 3, P, p_vis), _flags(rng, 2, P, p_vis / 2)
    vis = torch.full((P + 8,), 7, dtype=torch.uint8, device=DEV)
    lib.visibility_union([torch.from_numpy(f).to(DEV) for f in fa], P, vis)
    lib.visibility_union([torch.from_numpy(f).to(DEV) for f in fb], P, vis, accumulate=True)
    ref = np.zeros(P, np.uint8)
    for f in fa + fb:
        ref |= (f & 128) == 0
    got = vis.cpu().numpy()
    assert np.array_equal(got[:P], ref) and np.all(got[P:] == 7)
    ws = torch.empty(max(1, lib.compact_workspace(P)), dtype=torch.uint8, device=DEV)
    idx = torch.full((P + 8,), -5, dtype=torch.int32, device=DEV)
    cnt = torch.zeros(1, dtype=torch.int64, device=DEV)
    lib.compact_index(vis, P, ws, idx, cnt)
    M = int(cnt.item())
    nz = np.nonzero(ref)[0]
    assert M == len(nz)
    assert np.array_equal(idx.cpu().numpy()[:M], nz)
    assert np.all(idx.cpu().numpy()[M:] == -5)


def test_gather_scatter_columns(lib):
    rng = np.random.default_rng(3)
    F, P, S = 59, 5000, 5004
    full = rng.normal(size=(F, S)).astype(np.float32)
    idx = np.sort(rng.choice(P, 1234, replace=False)).astype(np.int32)
    M = len(idx)
    t_full = torch.from_numpy(full).to(DEV)
    t_idx = torch.from_numpy(idx).to(DEV)
    packed = torch.empty((F, M), dtype=torch.float32, device=DEV)
    lib.gather_columns(t_full, F, S, t_idx, M, packed)
    assert np.array_equal(packed.cpu().numpy(), full[:, idx])
    new = rng.normal(size=(F, M)).astype(np.float32)
    lib.scatter_columns(torch.from_numpy(new).to(DEV), F, S, t_idx, M, t_full)
    exp = full.copy()
    exp[:, idx] = new
    assert np.array_equal(t_full.cpu().numpy(), exp)
    lib.gather_columns(t_full, F, S, t_idx, 0, packed)  # M = 0: nothing to do
    with pytest.raises(gsr.GsError):
        lib.gather_columns(t_full, F, S, t_idx, S + 1, packed)


def test_sparse_exchange_adam_single_rank_nccl(lib):
    """World size 1 through a real NCCL group: the visibility-sparse step (union,
    compaction, gather, all-reduce, scatter, replicated Adam) inside Trainer.step equals
    the replicated step, and it exchanges exactly the columns visible in some view."""
    import os
    import torch.distributed as dist
    from oracle import gsref
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29547")
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=DEV)
    try:
        w = scenegen.make("small")
        cams = [scenegen.camera_rt(320, 240, 300.0, 160.0, 120.0, scenegen.rot_y(0.3 * (k - 1)),
                                   [0.6 * (k - 1), 0.0, 0.0]) for k in range(3)]
        models = [pipeline.GaussianModel(w.scene, DEV) for _ in range(2)]
        tgt = pipeline.GaussianModel(w.target_scene, DEV)
        cap = pipeline.default_capacity(pipeline.measure_keys(lib, models[0], cams, DEV))
        targets = pipeline.render_targets(lib, tgt, cams, DEV, cap)
        opt = pipeline.SparseExchangeAdam(lib, models[1])
        trs = [pipeline.Trainer(lib, models[0], cams, targets, DEV, cap, streams=2, deterministic=True),
               pipeline.Trainer(lib, models[1], cams, targets, DEV, cap, streams=2, optimizer=opt, deterministic=True)]
        for it in range(3):
            snap = models[1].params.cpu().numpy().copy()
            for tr in trs:
                tr.loss.zero_()
                tr.step([0, 1, 2])
            torch.cuda.synchronize()
            assert trs[1].loss.item() == pytest.approx(trs[0].loss.item(), rel=1e-5)
            if it == 0:
                scene = scenegen.Scene(w.scene.P, w.scene.sh_degree, snap)
                vis = np.zeros(w.scene.P, bool)
                for c in cams:
                    vis |= (gsref.project(c, scene, gsref.F32)["flags"] & 128) == 0
                assert opt.last_M == int(vis.sum()) and 0 < opt.last_M < w.scene.P
        # deterministic reduction: the sparse exchange updates exactly what the dense step does
        assert torch.equal(models[0].params, models[1].params)
    finally:
        dist.destroy_process_group()
