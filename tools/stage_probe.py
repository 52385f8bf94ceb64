"""Run single stages of one scannetpp-shaped view (or a batch) a few times, for ncu
captures of one kernel: python tools/stage_probe.py [--config scannetpp] [--reps 3]
(project, project_views of 8 views, bin, render fwd/bwd, project_bwd_views, adam)."""
from __future__ import annotations

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import scenegen  # noqa: E402
from paper_2408_12677_b200 import gsr, pipeline  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="scannetpp")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--views", type=int, default=8)
    ap.add_argument("--chunk", type=int, default=8)
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    lib = gsr.load()
    w = scenegen.make(a.config)
    model = pipeline.GaussianModel(w.scene, dev)
    pipeline.spatially_order(lib, model)
    tgt = pipeline.GaussianModel(w.target_scene, dev)
    pipeline.spatially_order(lib, tgt)
    cams = w.cameras[:a.views]
    cap = pipeline.default_capacity(pipeline.measure_keys(lib, model, cams, dev))
    targets = pipeline.render_targets(lib, tgt, cams, dev, cap)
    tr = pipeline.Trainer(lib, model, cams, targets, dev, cap, streams=1, chunk=a.chunk)
    tr.tile_order = False
    views = list(range(len(cams)))
    for _ in range(a.reps):
        tr.step(views)
    # isolated projections of a batch (gs_project_views) for the capture
    projs = [gsr.make_proj(model.P, dev) for _ in cams[:8]]
    for _ in range(a.reps):
        lib.project_views([gsr.camera(c) for c in cams[:8]], model.desc, model.params, [p[0] for p in projs])
    torch.cuda.synchronize()
    print("ok", model.P, len(cams))


if __name__ == "__main__":
    main()
