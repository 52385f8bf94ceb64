"""Which part of the host-streamed frame traffic slows a graph-replayed config-4 step:
the H2D copies, the decode kernels, or both (tools/e2e_diag2.py found 91-93 vs 80 ms)."""
import sys
sys.path.insert(0, "/root/repo")
import torch
import scenegen
from paper_2408_12677_b200 import gsr, pipeline
cfg = sys.argv[1] if len(sys.argv) > 1 else "large"
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
host = {v: (torch.randint(0, 255, (H, W, 3), dtype=torch.uint8).pin_memory(),
            torch.randint(500, 4000, (H, W), dtype=torch.int16).pin_memory()) for v in views}
for _ in range(2):
    tr.step(views)
g = tr.capture(views)
raw = {v: (torch.empty((H, W, 3), dtype=torch.uint8, device=dev), torch.empty((H, W), dtype=torch.int16, device=dev))
       for v in views}
slots = {v: (torch.empty((3, H, W), device=dev), torch.empty((H, W), device=dev)) for v in views}
cs = torch.cuda.Stream(device=dev)
done = torch.cuda.Event()


def side(copy, decode, grouped=False):
    cs.wait_event(done)
    with torch.cuda.stream(cs):
        if grouped:  # every copy first, then every decode
            for v in views:
                raw[v][0].copy_(host[v][0], non_blocking=True)
                raw[v][1].copy_(host[v][1], non_blocking=True)
            for v in views:
                lib.decode_rgbd(raw[v][0], raw[v][1], 0.001, slots[v][0], slots[v][1])
            return
        for v in views:
            if copy:
                raw[v][0].copy_(host[v][0], non_blocking=True)
                raw[v][1].copy_(host[v][1], non_blocking=True)
            if decode:
                lib.decode_rgbd(raw[v][0], raw[v][1], 0.001, slots[v][0], slots[v][1])


def run(copy, decode, n=6, grouped=False):
    def once():
        tr.replay(g)
        done.record(torch.cuda.current_stream())
        if copy or decode:
            side(copy, decode, grouped)
    for _ in range(2):
        once()
    torch.cuda.synchronize()
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s0.record()
    for _ in range(n):
        once()
    s1.record()
    torch.cuda.synchronize()
    return s0.elapsed_time(s1) / n


for c, d in [(False, False), (True, True)]:
    print(f"copy {c} decode {d}: {run(c, d):.2f} ms/step")
print(f"grouped copies then decodes: {run(True, True, grouped=True):.2f} ms/step")
lo = torch.cuda.Stream.priority_range()
cs = torch.cuda.Stream(device=dev, priority=lo[1])
print(f"high-priority copy stream, grouped: {run(True, True, grouped=True):.2f} ms/step")
print(f"high-priority copy stream, interleaved: {run(True, True):.2f} ms/step")
