"""Diagnostic: lane utilisation of the render kernels on one view of a config.
bwd work = sum over keys of popc(key_blocks) x 32 lane-pixel slots; useful = blended
pairs.  Also the distribution of popc(key_blocks) and of blended pixels per block."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import scenegen  # noqa: E402
from paper_2408_12677_b200 import gsr, pipeline  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "scannetpp"
w = scenegen.make(name, num_views=2) if name in ("replica", "scannetpp", "large") else scenegen.make(name)
dev = torch.device("cuda:0")
lib = gsr.load()
model = pipeline.GaussianModel(w.scene, dev)
pipeline.spatially_order(lib, model)
cam = w.cameras[0]
K = pipeline.measure_keys(lib, model, [cam], dev)
buf = pipeline.ViewBuffers(lib, cam, model.P, pipeline.default_capacity(K), dev)
bl = torch.zeros(1, dtype=torch.int64, device=dev)
K = pipeline.render(lib, model, cam, buf, sync_keys=True)
lib.render_fwd(gsr.camera(cam), model.desc, buf.proj, buf.sorted_ids, buf.ranges, buf.rgb, buf.depth, buf.T, buf.n,
               blended=bl, key_blocks=buf.key_blocks)
torch.cuda.synchronize()
kb = buf.key_blocks[:K].cpu().numpy()
pc = np.unpackbits(kb[:, None], axis=1).sum(1)
blended = int(bl.item())
print(f"{name}: K={K} blended={blended} ({blended / (cam.width * cam.height):.1f}/px)")
print(f"keys with mask: {np.count_nonzero(pc)} ({np.count_nonzero(pc) / K:.3f} of K)")
print(f"bwd (key, block) pairs: {pc.sum()}  lane slots {32 * pc.sum()}  utilisation {blended / (32 * pc.sum()):.3f}")
print("popc histogram:", np.bincount(pc, minlength=9))
n = buf.n.cpu().numpy()
print(f"evaluated (sum n_contrib): {int(n.sum())}  ({n.sum() / (cam.width * cam.height):.1f}/px)")
r = buf.ranges.cpu().numpy()
L = r[:, 1] - r[:, 0]
print(f"tile lists: mean {L.mean():.0f} p50 {np.median(L):.0f} p99 {np.percentile(L, 99):.0f} max {L.max()}")
