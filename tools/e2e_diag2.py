import sys
sys.path.insert(0, "/root/repo")
import torch
import scenegen
from paper_2408_12677_b200 import gsr, pipeline
cfg = sys.argv[1]
lib = gsr.load(); dev = torch.device("cuda:0")
w = scenegen.make(cfg)
model = pipeline.GaussianModel(w.scene, dev); pipeline.spatially_order(lib, model)
tgt = pipeline.GaussianModel(w.target_scene, dev); pipeline.spatially_order(lib, tgt)
cams = w.cameras
cap = pipeline.default_capacity(pipeline.measure_keys(lib, model, cams, dev))
targets = pipeline.render_targets(lib, tgt, cams, dev, cap)
tr = pipeline.Trainer(lib, model, cams, targets, dev, cap, streams=8, chunk=min(64, len(cams)))
views = list(range(len(cams)))
H, W = cams[0].height, cams[0].width
frames = {v: (torch.randint(0, 255, (H, W, 3), dtype=torch.uint8).pin_memory(),
              torch.randint(500, 4000, (H, W), dtype=torch.int16).pin_memory()) for v in views}
for _ in range(2): tr.step(views)
g = tr.capture(views)
def timeit(fn, n=8):
    for _ in range(2): fn()
    torch.cuda.synchronize()
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s0.record()
    for _ in range(n): fn()
    s1.record(); torch.cuda.synchronize()
    return s0.elapsed_time(s1) / n
print("plain graph", timeit(lambda: tr.replay(g)))
for prio, gc in ((None, False), (0, False), (None, True)):
    hs = pipeline.HostStreamedGraphs(tr, views, [frames, frames], 0.001, copy_priority=prio, graph_copies=gc)
    print("hs prio", prio, "graph copies", gc, timeit(hs.step))
    print("plain graph", timeit(lambda: tr.replay(g)))
    del hs
print("eager step_host", timeit(lambda: tr.step_host(views, frames, 0.001)))
print("plain graph", timeit(lambda: tr.replay(g)))
