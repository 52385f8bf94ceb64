"""Text timeline of one (pre-enqueued) eager scannetpp-shaped step with views in flight: CUDA events
around every stage on the stream it is launched on (Trainer hooks), relative to the
step start -- shows where the streams idle.  python tools/timeline.py [config]"""
import sys

import torch

sys.path.insert(0, ".")
import scenegen  # noqa: E402
from paper_2408_12677_b200 import gsr, pipeline  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "scannetpp"
lib = gsr.load()
dev = torch.device("cuda:0")
w = scenegen.make(cfg)
model = pipeline.GaussianModel(w.scene, dev)
pipeline.spatially_order(lib, model)
tgt = pipeline.GaussianModel(w.target_scene, dev)
pipeline.spatially_order(lib, tgt)
cams = w.cameras
cap = pipeline.default_capacity(pipeline.measure_keys(lib, model, cams, dev))
targets = pipeline.render_targets(lib, tgt, cams, dev, cap)
tr = pipeline.Trainer(lib, model, cams, targets, dev, cap, streams=8, chunk=min(64, len(cams)))
views = list(range(len(cams)))
for _ in range(3):
    tr.step(views)
torch.cuda.synchronize()
rec = []
open_ev = {}
count = {}


def hook(stage, what):
    ev = torch.cuda.Event(enable_timing=True)
    ev.record(torch.cuda.current_stream())
    key = (stage, count.get(stage, 0))
    if what == "begin":
        open_ev[stage] = (ev, torch.cuda.current_stream().stream_id)
    else:
        b, sid = open_ev.pop(stage)
        rec.append((stage, count.get(stage, 0), sid, b, ev))
        count[stage] = count.get(stage, 0) + 1


t0 = torch.cuda.Event(enable_timing=True)
t1 = torch.cuda.Event(enable_timing=True)
tr.hooks = hook
# a long spin first, so that the host has enqueued the whole step before the device
# starts it: the timeline shows device scheduling, not the host's launch rate
torch.cuda._sleep(100_000_000)
t0.record()
tr.step(views)
t1.record()
torch.cuda.synchronize()
total = t0.elapsed_time(t1)
print(f"step {total:.3f} ms")
for stage, k, sid, b, e in sorted(rec, key=lambda r: t0.elapsed_time(r[3])):
    s0, s1 = t0.elapsed_time(b), t0.elapsed_time(e)
    bar = [" "] * 80
    for x in range(int(s0 / total * 80), max(int(s0 / total * 80) + 1, int(s1 / total * 80))):
        if 0 <= x < 80:
            bar[x] = "#"
    print(f"{stage:12s}{k:3d} stream {sid:>4d} {s0:7.3f}-{s1:7.3f} |{''.join(bar)}|")
