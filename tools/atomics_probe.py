"""One view through the product backward (key masks + fused L1, k_render_bwd<1,1>) and
through the K13 per-pixel port's backward, for an ncu capture of their L2 reduction
traffic (reds per blended pair against the naive port's 10).

  python tools/atomics_probe.py [--config scannetpp] [--view 0]
prints the blended pair count of the view (the denominator) as JSON.
"""
from __future__ import annotations

import argparse
import json
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
    ap.add_argument("--view", type=int, default=0)
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    lib = gsr.load()
    w = scenegen.make(a.config)
    model = pipeline.GaussianModel(w.scene, dev)
    pipeline.spatially_order(lib, model)
    tgt = pipeline.GaussianModel(w.target_scene, dev)
    pipeline.spatially_order(lib, tgt)
    cam = w.cameras[a.view]
    cap = pipeline.default_capacity(pipeline.measure_keys(lib, model, [cam], dev))
    tb = pipeline.ViewBuffers(lib, cam, tgt.P, cap, dev)
    pipeline.render(lib, tgt, cam, tb)
    b = pipeline.ViewBuffers(lib, cam, model.P, cap, dev)
    gcam = gsr.camera(cam)
    blended = torch.zeros(1, dtype=torch.int64, device=dev)
    lib.project(gcam, model.desc, model.params, b.proj)
    lib.bin_tiles(gcam, model.desc, b.proj, b.bin_ws, b.key_capacity, b.sorted_ids, b.ranges)
    lib.render_fwd(gcam, model.desc, b.proj, b.sorted_ids, b.ranges, b.rgb, b.depth, b.T, b.n, blended=blended,
                   key_blocks=b.key_blocks)
    sg = torch.zeros((model.P, 12), device=dev)
    for _ in range(2):  # product backward: forward key masks + fused Eq. 12 upstream
        lib.render_bwd_screen_l1(gcam, model.desc, b.proj, b.sorted_ids, b.ranges, b.T, b.n, b.rgb, b.depth, tb.rgb,
                                 tb.depth, 1.0, sg, key_blocks=b.key_blocks)
    lib.l1_loss_grad(b.rgb, b.depth, tb.rgb, tb.depth, 1.0, b.g_rgb, b.g_depth)
    for _ in range(2):  # K13 port: one thread per pixel, 10 atomicAdd per composited pair
        lib.naive_render_bwd_screen(gcam, model.desc, b.proj, b.sorted_ids, b.ranges, b.T, b.n, b.g_rgb, b.g_depth,
                                    sg)
    torch.cuda.synchronize()
    print(json.dumps({"config": a.config, "view": a.view, "blended_pairs": int(blended.item()),
                      "tiles": cam.num_tiles, "P": model.P}))


if __name__ == "__main__":
    main()
