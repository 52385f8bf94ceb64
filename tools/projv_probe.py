"""Event-timed gs_project_views over a config's first 8 views (Morton layout), median of
reps; checks the outputs are bit-identical across the libraries named on the command
line (A/B of build variants: python tools/projv_probe.py scannetpp libgsr.so libgsr_x.so)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import scenegen  # noqa: E402
from paper_2408_12677_b200 import gsr, pipeline  # noqa: E402

cfg, libs = sys.argv[1], sys.argv[2:]
single = os.environ.get("PROBE_SINGLE", "0") == "1"  # gs_project of view 0 instead
dev = torch.device("cuda:0")
w = scenegen.make(cfg, 0)
outs = {}
for name in libs * 2:
    os.environ["GSR_LIB"] = name
    lib = gsr.load()
    model = pipeline.GaussianModel(w.scene, dev)
    pipeline.spatially_order(lib, model)
    cams8 = w.cameras[:8]
    projs_t = [gsr.make_proj(model.P_stride, dev) for _ in cams8]
    projs = [p for p, _ in projs_t]
    gcams = [gsr.camera(c) for c in cams8]
    ts = []
    for r in range(30):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        if single:
            lib.project(gcams[0], model.desc, model.params, projs[0])
        else:
            lib.project_views(gcams, model.desc, model.params, projs)
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts = sorted(ts[5:])
    sig = [(t["radius"][:model.P].clone(), t["tiles"][:model.P].clone(), t["flags"][:model.P].clone())
           for _, t in projs_t[:1 if single else len(projs_t)]]
    if "ref" in outs:
        same = all(torch.equal(a, b) for x, y in zip(outs["ref"], sig) for a, b in zip(x, y))
    else:
        outs["ref"], same = sig, True
    print(cfg, name, "median_us", round(1e3 * ts[len(ts) // 2], 1), "min_us", round(1e3 * ts[0], 1), "identical", same)
