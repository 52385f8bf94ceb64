"""Small run of every kernel family (a quick integration smoke; compute-sanitizer is
closed on this GPU pool: tests/test_gpu_bounds.py runs this script against the
bounds-checked build, GSR_LIB=libgsr_check.so with CUDA_LAUNCH_BLOCKING=1):
projection,
binning (both tile placements via env), render fwd/bwd (+ fused L1, key masks, tile
order), the K13 port, the projection backward, Adam (host / device step / range),
the sparse-exchange kernels, TSDF allocate + integrate, quadtree + seeding.  Exits 0 if everything ran."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import scenegen  # noqa: E402
from paper_2408_12677_b200 import gsr, pipeline  # noqa: E402

dev = torch.device("cuda:0")
lib = gsr.load()
print("library", lib.path)
w = scenegen.make("small")
cams = [scenegen.camera_rt(320, 240, 300.0, 160.0, 120.0, scenegen.rot_y(0.03 * (k - 2)), [0.05 * k, 0.0, 0.0])
        for k in range(5)]
cams.append(scenegen.camera_rt(37, 29, 40.0, 18.0, 14.0, np.eye(3), [0.0, 0.0, 0.0]))  # ragged tiny view
model = pipeline.GaussianModel(w.scene, dev)
tgt = pipeline.GaussianModel(w.target_scene, dev)
cap = pipeline.default_capacity(pipeline.measure_keys(lib, model, cams[:5], dev))
targets = pipeline.render_targets(lib, tgt, cams[:5], dev, cap)
tr = pipeline.Trainer(lib, model, cams[:5], targets, dev, cap, chunk=2, streams=2)
tr.step(list(range(5)))
tr.fuse_l1 = False
tr.step(list(range(5)))
tr.naive = True
tr.step([0, 1])
tr.naive = False
g = tr.capture([0, 1, 2])
tr.replay(g)
# single-stream path with tile order, ragged view
tr1 = pipeline.Trainer(lib, model, [cams[5]], [pipeline.render_targets(lib, tgt, [cams[5]], dev, cap)[0]], dev, cap)
tr1.step([0])
# Adam range
sc = model.desc
gr = model.grad.view(-1)[4:4 + 4 * 1000].clone()
lib.adam_step_range(sc, model.params, gr, model.m, model.v, model.lr, 3, 4, 4 + 4 * 1000)
# visibility-sparse exchange kernels (union, compaction, gather, scatter)
vis = torch.zeros(model.P_stride, dtype=torch.uint8, device=dev)
proj_flags = [torch.randint(0, 2, (model.P,), dtype=torch.uint8, device=dev) for _ in range(2)]
lib.visibility_union(proj_flags, model.P, vis, accumulate=False)
idx = torch.zeros(model.P_stride, dtype=torch.int32, device=dev)
cnt = torch.zeros(1, dtype=torch.int64, device=dev)
ws = torch.empty(max(1, lib.compact_workspace(model.P_stride)), dtype=torch.uint8, device=dev)
lib.compact_index(vis, model.P, ws, idx, cnt)
M = int(cnt.item())
packed = torch.empty(model.F * max(M, 1), device=dev)
lib.gather_columns(model.grad, model.F, model.P_stride, idx, M, packed)
lib.scatter_columns(packed, model.F, model.P_stride, idx, M, model.grad)
# TSDF + seeding
wr = scenegen.make("replica", num_views=3)
vcams = [scenegen.camera_from_forward(97, 61, 50.0, 48.0, 30.0, -c.R_cw.T @ c.t_cw, c.R_cw[2]) for c in wr.cameras]
vol = pipeline.TsdfVolume(lib, dev, 1 << 14, voxel_size=0.02)
m2 = pipeline.empty_model(5000, 1, dev)
sd = pipeline.Seeder(lib, 97, 61, dev, min_cell=2)
for k, c in enumerate(vcams):
    d = torch.from_numpy(scenegen.render_depth(wr.faces, c, noise_sigma=0.002, dropout=0.05, seed=k)).to(dev)
    rgb = torch.rand((3, 61, 97), device=dev)
    vol.integrate_frame(c, d)
    sd.seed_frame(c, d, rgb, vol, m2)
torch.cuda.synchronize()
print("kernel smoke ok", model.step_count, m2.P, int(vol.num_blocks.item()))
