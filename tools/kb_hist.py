import torch, numpy as np, sys
sys.path.insert(0, '.')
import scenegen
from paper_2408_12677_b200 import gsr, pipeline
lib = gsr.load()
w = scenegen.make("scannetpp", num_views=1)
dev = torch.device("cuda:0")
model = pipeline.GaussianModel(w.scene, dev)
pipeline.spatially_order(lib, model)
K = pipeline.measure_keys(lib, model, w.cameras, dev)
buf = pipeline.ViewBuffers(lib, w.cameras[0], model.P, pipeline.default_capacity(K), dev)
cam = w.cameras[0]
K = pipeline.render(lib, model, cam, buf, sync_keys=True)
gcam = gsr.camera(cam)
lib.render_fwd(gcam, model.desc, buf.proj, buf.sorted_ids, buf.ranges, buf.rgb, buf.depth, buf.T, buf.n, key_blocks=buf.key_blocks)
torch.cuda.synchronize()
kb = buf.key_blocks[:K].cpu().numpy()
pc = np.unpackbits(kb[:, None], axis=1).sum(1)
print("K", K, "nonzero", (kb != 0).sum(), "hist popc", np.bincount(pc, minlength=9).tolist())
n = buf.n.cpu().numpy(); print("sum n", n.sum(), "mean n", n.mean())
r = buf.ranges.cpu().numpy(); L = r[:,1]-r[:,0]; print("tile len mean/p50/p99/max", L.mean(), np.percentile(L,50), np.percentile(L,99), L.max())
