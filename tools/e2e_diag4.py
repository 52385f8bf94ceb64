"""Config 4 (every variant from the same restored training state -- the step time
drifts 81 -> 72 ms as training moves the Gaussians): is the host-streamed slowdown (93 vs 81 ms, tools/e2e_diag2.py) in the
copies or in the compute graphs that read the slot sets (Trainer.capture with
targets_override)?"""
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
frames = {v: (torch.randint(0, 255, (H, W, 3), dtype=torch.uint8).pin_memory(),
              torch.randint(500, 4000, (H, W), dtype=torch.int16).pin_memory()) for v in views}
for _ in range(2): tr.step(views)
g = tr.capture(views)


snap = [t.clone() for t in (model.params, model.m, model.v, model.step_dev)]


def timeit(fn, n=6):
    for t, s in zip((model.params, model.m, model.v, model.step_dev), snap):
        t.copy_(s)
    for _ in range(2): fn()
    torch.cuda.synchronize()
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s0.record()
    for _ in range(n): fn()
    s1.record(); torch.cuda.synchronize()
    return s0.elapsed_time(s1) / n


hs = pipeline.HostStreamedGraphs(tr, views, [frames, frames], 0.001)
raw = {v: (torch.empty((H, W, 3), dtype=torch.uint8, device=dev), torch.empty((H, W), dtype=torch.int16, device=dev))
       for v in views}
slots = {v: (torch.empty((3, H, W), device=dev), torch.empty((H, W), device=dev)) for v in views}
cs = torch.cuda.Stream(device=dev, priority=torch.cuda.Stream.priority_range()[1])
done = torch.cuda.Event()


side_ms = []


def side_after_plain(copy=True, decode=True, plain=True):
    if plain:
        tr.replay(g)
    done.record(torch.cuda.current_stream())
    cs.wait_event(done)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    side_ms.append((a, b))
    a.record(cs)
    with torch.cuda.stream(cs):
        for v in views:
            if copy:
                raw[v][0].copy_(frames[v][0], non_blocking=True)
                raw[v][1].copy_(frames[v][1], non_blocking=True)
            if decode:
                lib.decode_rgbd(raw[v][0], raw[v][1], 0.001, slots[v][0], slots[v][1])
    b.record(cs)


def side_report(tag):
    torch.cuda.synchronize()
    print(tag, "side work ms per step:", [round(a.elapsed_time(b), 1) for a, b in side_ms[-6:]])
    side_ms.clear()




def hs_step_instr(wait_copied=True, log=None):
    """HostStreamedGraphs.step with timing events (and optionally without the wait)."""
    p = hs.i % 2
    main = torch.cuda.current_stream()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
    e[0].record(main)
    if wait_copied:
        main.wait_event(hs.copied[p])
    main.wait_event(hs.read[p])
    e[1].record(main)
    hs.losses[p].zero_()
    tr.replay(hs.compute_graphs[p])
    hs.computed[p].record(main)
    e[2].record(main)
    rb = hs.readback_stream
    rb.wait_event(hs.computed[p])
    with torch.cuda.stream(rb):
        hs.loss_host[p].copy_(hs.losses[p], non_blocking=True)
    hs.read[p].record(rb)
    hs.i += 1
    cs = hs.copy_stream
    cs.wait_event(hs.computed[p])
    e[3].record(cs)
    with torch.cuda.stream(cs):
        hs._copies(p)
    hs.copied[p].record(cs)
    e[4].record(cs)
    if log is not None:
        log.append(e)


print("hs step, prefetch", timeit(hs.step))
print("hs instrumented", timeit(lambda: hs_step_instr(True)))
orig = pipeline.HostStreamedGraphs._copy


def copy_with_marker(self, p, timing):
    cs = self.copy_stream
    cs.wait_event(self.computed[p])
    torch.cuda.Event(enable_timing=timing).record(cs)
    with torch.cuda.stream(cs):
        self._copies(p)
    self.copied[p].record(cs)


hs._copy = lambda p: copy_with_marker(hs, p, True)
print("hs step, timing marker after the wait", timeit(hs.step))
hs._copy = lambda p: copy_with_marker(hs, p, False)
print("hs step, plain marker after the wait", timeit(hs.step))


def step_with_marker(self, prefetch=True):
    p = self.i % 2
    main = torch.cuda.current_stream()
    torch.cuda.Event(enable_timing=True).record(main)
    return pipeline.HostStreamedGraphs.step(self, prefetch)


hs._copy = lambda p: orig(hs, p)
print("hs step, original", timeit(hs.step))
print("hs step, timing marker on main first", timeit(lambda: step_with_marker(hs)))
