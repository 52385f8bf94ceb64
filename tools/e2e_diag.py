import sys, os, time
sys.path.insert(0, "/root/repo")
import torch, numpy as np
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
hs = pipeline.HostStreamedGraphs(tr, views, [frames, frames], 0.001)
torch.cuda.synchronize()
def timeit(fn, n=4):
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn(); torch.cuda.synchronize()
    s0.record()
    for _ in range(n): fn()
    s1.record(); torch.cuda.synchronize()
    return s0.elapsed_time(s1) / n
print("plain graph", timeit(lambda: tr.replay(g)))
print("hs compute only", timeit(lambda: tr.replay(hs.compute_graphs[0])))
print("hs step (copies)", timeit(hs.step))
def copies_only():
    with torch.cuda.stream(hs.copy_stream):
        hs.copy_graphs[0].replay()
    torch.cuda.current_stream().wait_stream(hs.copy_stream)
print("copies only", timeit(copies_only))
print("eager step_host", timeit(lambda: tr.step_host(views, frames, 0.001)))
loss_host = torch.zeros(1, dtype=torch.float32).pin_memory()
def hs_loss():
    tr.loss.zero_()
    hs.step()
    loss_host.copy_(tr.loss, non_blocking=True)
print("hs step + loss zero/readback", timeit(hs_loss))
# variants of the step for diagnosis
def variant(readback, zero, waitread):
    def fn():
        p = hs.i % 2
        main = torch.cuda.current_stream()
        main.wait_event(hs.copied[p])
        if waitread:
            main.wait_event(hs.read[p])
        if zero:
            hs.losses[p].zero_()
        hs.trainer.replay(hs.compute_graphs[p])
        hs.computed[p].record(main)
        if readback:
            rb = hs.readback_stream
            rb.wait_event(hs.computed[p])
            with torch.cuda.stream(rb):
                hs.loss_host[p].copy_(hs.losses[p], non_blocking=True)
            hs.read[p].record(rb)
        hs.i += 1
        hs._copy(p)
    return fn
for rb_, z_, w_ in [(0, 0, 0), (0, 1, 0), (1, 0, 0), (1, 1, 1), (1, 1, 0)]:
    print("variant readback", rb_, "zero", z_, "waitread", w_, timeit(variant(rb_, z_, w_)))
