"""Diagnostic for a split-warp render design (each half-warp walks the keys of one
16x8 half of the tile): from the forward's key masks of one view, the number of key
iterations of the current warp-per-tile loop vs the split loop (per 32-key batch,
max over the halves of the keys touching each half) and the block-evaluation counts.
python tools/split_probe.py [config]"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import scenegen  # noqa: E402
from paper_2408_12677_b200 import gsr, pipeline  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "large"
w = scenegen.make(name, num_views=2) if name in ("replica", "scannetpp", "large") else scenegen.make(name)
dev = torch.device("cuda:0")
lib = gsr.load()
model = pipeline.GaussianModel(w.scene, dev)
pipeline.spatially_order(lib, model)
cam = w.cameras[0]
K = pipeline.measure_keys(lib, model, [cam], dev)
buf = pipeline.ViewBuffers(lib, cam, model.P, pipeline.default_capacity(K), dev)
K = pipeline.render(lib, model, cam, buf, sync_keys=True)
lib.render_fwd(gsr.camera(cam), model.desc, buf.proj, buf.sorted_ids, buf.ranges, buf.rgb, buf.depth, buf.T, buf.n,
               key_blocks=buf.key_blocks)
torch.cuda.synchronize()
kb = buf.key_blocks[:K].cpu().numpy().astype(np.int64)
rg = buf.ranges.cpu().numpy().reshape(-1, 2)
top = (kb & 0x0F) != 0
bot = (kb & 0xF0) != 0
pc = np.unpackbits(kb.astype(np.uint8)[:, None], axis=1).sum(1)
print(name, "K", K, "visited(nonzero)", int((kb != 0).sum()), "top only", int((top & ~bot).sum()),
      "bottom only", int((bot & ~top).sum()), "both", int((top & bot).sum()))
print("popc hist", np.bincount(pc, minlength=9).tolist())
cur_it = 0
split_it = 0
split_blocks = 0
cur_blocks = int(pc.sum())
for t in range(rg.shape[0]):
    a, b = rg[t]
    for s in range(a, b, 32):
        e = min(b, s + 32)
        k = kb[s:e]
        cur_it += int((k != 0).sum())
        ta = np.nonzero(k & 0x0F)[0]
        tb = np.nonzero(k & 0xF0)[0]
        n = max(len(ta), len(tb))
        split_it += n
        for i in range(n):
            ma = (k[ta[i]] & 0x0F) if i < len(ta) else 0
            mb = ((k[tb[i]] >> 4) & 0x0F) if i < len(tb) else 0
            split_blocks += bin(int(ma | mb)).count("1")
print("iterations: current", cur_it, "split", split_it, f"ratio {split_it / max(cur_it, 1):.3f}")
print("block evaluations (warp): current", cur_blocks, "(1 px/lane each); split", split_blocks,
      f"(2 px/lane each) ratio {2 * split_blocks / max(cur_blocks, 1):.3f}")
# Gaussians that composited anything (a nonzero key mask) vs the projected-visible set
ids = buf.sorted_ids[:K].long()
hit = torch.zeros(model.P, dtype=torch.bool, device=dev)
hit[ids[buf.key_blocks[:K] != 0]] = True
nvis = int((buf.proj_t["radius"][:model.P] > 0).sum())
print("gaussians visible", nvis, "hit (composited >= 1 pixel)", int(hit.sum()), "of P", model.P)
# tile list lengths (for per-tile sorting designs)
lens = (rg[:, 1] - rg[:, 0]).astype(np.int64)
q = np.percentile(lens, [50, 90, 99, 99.9, 100])
print("tile list lengths: tiles", len(lens), "mean", lens.mean(), "p50/p90/p99/p99.9/max", q.tolist(),
      "keys in tiles > 2048:", int(lens[lens > 2048].sum()), "> 4096:", int(lens[lens > 4096].sum()))
