#!/usr/bin/env python
"""Benchmark: fwd + bwd + Adam iterations of the GSFusion rasterizer hot path.

python bench.py [--gpus N --steps K --warmup W --config scannetpp]
N > 1: launched with torch.distributed.run, one rank per GPU (NCCL); the views of
the batch are sharded contiguously over ranks and the gradient is all-reduced
(SUM) over NVLink before a replicated Adam step.

Prints ONE JSON line on rank 0 (see DESIGN.md §Measurement for every key).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
# before the CUDA context exists: 32 hardware work queues for the ~18 streams of a step
# (see paper_2408_12677_b200/__init__.py)
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

METRIC = "fwd+bwd+Adam iters/s and blended Gaussian-pixels/s, 1/2/4/8 B200"
UNIT = "blended Gaussian-pixels/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="scannetpp", choices=["tiny", "small", "replica", "scannetpp", "large"])
    ap.add_argument("--impl", default="gsr", choices=["gsr", "reference"])
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-morton", action="store_true", help="keep the generated Gaussian order")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--streams", type=int, default=int(os.environ.get("GSR_STREAMS", "8")),
                    help="views in flight (one CUDA stream + buffer set each)")
    ap.add_argument("--graph", type=int, default=1, help="1: time CUDA-graph replays of whole iterations (N = 1)")
    ap.add_argument("--chunk", type=int, default=int(os.environ.get("GSR_CHUNK", "0")),
                    help="views chained per projection-backward pass (<= 64; 0 = all views of a step)")
    ap.add_argument("--optim", default="nvls", choices=["nvls", "peer", "sharded", "replicated", "sparse"],
                    help="N > 1: 'nvls' in-switch reduce (multimem) + Adam + multicast store kernel (falls back to "
                         "'peer' without multicast), fused peer-memory reduce-scatter+Adam+all-gather kernel (falls back to 'sharded' if "
                         "symmetric memory is unavailable), NCCL reduce-scatter + sharded Adam + all-gather, "
                         "NCCL all-reduce + replicated Adam, or the visibility-sparse exchange (all-reduce of the "
                         "union-visible gradient columns only) + replicated Adam")
    ap.add_argument("--no-naive", action="store_true", help="skip the K13 per-pixel-port comparison arm")
    ap.add_argument("--schedule", action="store_true",
                    help="keyframe-scheduled online + global optimisation run (PAPER.md:149; SURVEY §8(f) NEXT-1)")
    ap.add_argument("--tsdf", action="store_true",
                    help="TSDF band allocation + integration over a pose sequence (PAPER.md:105-115; SURVEY §8(f) NEXT-3)")
    ap.add_argument("--online", action="store_true",
                    help="the incremental mapping loop: TSDF fusion + quadtree seeding + keyframe-scheduled steps per "
                         "frame, then global passes (PAPER.md:101-149; NEXT-1/3/4); --steps = frames")
    ap.add_argument("--profile", action="store_true", help="minimal run for ncu (no e2e / cpu / clocks)")
    return ap.parse_args()


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """SM clock + throttle reasons sampled DURING the timed region: NVML (the library
    nvidia-smi reads) polled every 10 ms from a thread, so that even a ~100 ms timed
    region gets ~10 samples; nvidia-smi -lms 200 is the fallback when NVML is absent."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, index: int):
        self.index, self.samples, self.proc, self.nvml = index, [], None, None
        self.stop_flag = threading.Event()

    def _nvml_handle(self):
        import pynvml
        pynvml.nvmlInit()
        vis = os.environ.get("CUDA_VISIBLE_DEVICES")
        ent = vis.split(",")[self.index].strip() if vis else str(self.index)
        if ent.isdigit():
            return pynvml, pynvml.nvmlDeviceGetHandleByIndex(int(ent))
        return pynvml, pynvml.nvmlDeviceGetHandleByUUID(ent)

    def start(self):
        try:
            nv, h = self._nvml_handle()
            self.nvml = (nv, h)
            bits = [nv.nvmlClocksThrottleReasonHwSlowdown, nv.nvmlClocksThrottleReasonHwThermalSlowdown,
                    nv.nvmlClocksThrottleReasonSwThermalSlowdown, nv.nvmlClocksThrottleReasonSwPowerCap]
            self.max_mhz = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)

            def poll():
                while not self.stop_flag.is_set():
                    sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                    r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                    self.samples.append([str(sm), str(self.max_mhz), "", ""] +
                                        ["Active" if r & b else "Not Active" for b in bits])
                    time.sleep(0.01)
            self.thread = threading.Thread(target=poll, daemon=True)
            self.thread.start()
            return
        except Exception:  # noqa: BLE001  (no NVML: fall back to nvidia-smi)
            self.nvml = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except (OSError, FileNotFoundError):
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 8:
                self.samples.append(parts)

    def stop(self):
        if self.nvml is not None:
            self.stop_flag.set()
            self.thread.join(timeout=1)
            src = "nvml (10 ms poll)"
        elif self.proc is not None:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()
            src = "nvidia-smi -lms 200"
        else:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["clock sampling unavailable"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        reasons = sorted({self.NAMES[k] for s in self.samples for k in range(4) if s[4 + k].lower() == "active"})
        sm.sort()
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "sm_min_mhz": sm[0] if sm else None, "reasons": reasons, "samples": len(self.samples),
                "source": src}


# ----------------------------------------------------------------------------- CPU oracle legs
def cpu_window_camera(cam, size=584):
    """Central size x size window of a view (tile-aligned origin), same intrinsics:
    a bounded sample of the same workload for the CPU oracle."""
    import copy
    c = copy.copy(cam)
    x0 = max(0, (cam.width - size) // 2 // 16 * 16)
    y0 = max(0, (cam.height - size) // 2 // 16 * 16)
    c.width, c.height = min(size, cam.width), min(size, cam.height)
    c.cx, c.cy = cam.cx - x0, cam.cy - y0
    return c


def oracle_step_sample(w, view=0, size=584, tgt=None, views=None):
    """fwd (F32) + L1 + bwd (MIXED) per view, the views' gradients summed (R21), then one
    Adam step, on the oracle: views (default [view]) on a size x size central window (or
    the full image when size covers it).  The target images (setup, untimed) are rendered
    once and can be passed back in (a list, one per view)."""
    import numpy as np
    from oracle import gsref
    from paper_2408_12677_b200.pipeline import lr_per_row
    views = [view] if views is None else list(views)
    cams = [cpu_window_camera(w.cameras[v], size) for v in views]
    t0 = time.perf_counter()
    if tgt is None:  # the target scene's render as a sensor frame (R41), decoded
        import scenegen
        from oracle import frame
        tgt = []
        for cam in cams:
            t = gsref.render_fwd(cam, w.target_scene, gsref.F32)
            c8, d16 = scenegen.quantize_frame(t["rgb"], t["depth"])
            t["rgb"], t["depth"] = frame.decode_rgbd(c8, d16, scenegen.DEPTH_SCALE)
            tgt.append(t)
    t1 = time.perf_counter()
    gfull = np.zeros(w.scene.params.shape, np.float64)
    blended = 0
    for cam, t in zip(cams, tgt):
        f = gsref.render_fwd(cam, w.scene, gsref.F32)
        L, g_rgb, g_d = gsref.l1_loss_grad(f["rgb"], f["depth"], t["rgb"].astype(np.float32),
                                           t["depth"].astype(np.float32), 1.0)
        grad, _ = gsref.render_bwd(cam, w.scene, g_rgb.astype(np.float32), g_d.astype(np.float32), mode=gsref.MIXED)
        gfull[:, :w.scene.P] += grad
        blended += f["blended"]
    S = w.scene.params.shape[1]
    z = np.zeros_like(w.scene.params)
    gsref.adam_step(w.scene.params, gfull.astype(np.float32), z, z,
                    np.array(lr_per_row(w.scene.sh_degree), np.float32), 1, P=S)
    t2 = time.perf_counter()
    return {"seconds": t2 - t1, "blended": blended, "window": f"{cams[0].width}x{cams[0].height}",
            "views": len(cams), "target_seconds": t1 - t0, "target": tgt}


def host_cpu():
    """nproc and the CPU model of this host (recorded with every CPU number)."""
    model = "unknown"
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"nproc": os.cpu_count(), "cpu_model": model}


def pilot_cost(w):
    """Two windows (128^2, 256^2) of view 0 through oracle_step_sample: the per-view
    fixed cost a (projection of all P Gaussians, list building, Adam) and the cost b per
    pixel, so that a workload can be sized to a time budget on this host."""
    cam0 = w.cameras[0]
    t = []
    for size in (128, 256):
        r = oracle_step_sample(w, 0, size)
        t.append((min(size, cam0.width) * min(size, cam0.height), r["seconds"]))
    (p1, t1), (p2, t2) = t
    b = max((t2 - t1) / max(p2 - p1, 1), 1e-12)
    return max(t1 - b * p1, 0.0), b


def cpu_oracle_legs(w, config, budget_s=60.0):
    """The CPU oracle as it stands (never tuned), timed on this host:
    (a) on ALL host cores (OpenMP over tiles; results independent of the thread count)
        on the §8(d) workload -- scannetpp one full iteration of its 8 views, large one
        full view (the rate is per blended pixel, so x64 views is the same rate), the
        single-view configs one full view -- or, if a pilot predicts more than budget_s,
        the same views on a central window sized to fit the budget;
    (b) on ONE core, a bounded sample (one view, 584x584 central window).
    Returns the cpu_baseline object: value = (a)'s rate, with (b) under single_core."""
    from oracle import gsref
    gsref.build()
    n_all = gsref.set_threads(0)
    batched = config in ("scannetpp", "large")
    views = list(range(len(w.cameras))) if config == "scannetpp" else [0]
    cam0 = w.cameras[0]
    full_px = cam0.width * cam0.height
    a, b = pilot_cost(w)  # all cores: seconds per view = a + b * pixels on this host
    est = len(views) * (a + b * full_px)
    if est <= budget_s:
        size = max(cam0.width, cam0.height)
    else:  # a central window with about budget_s of work
        side = int(max(budget_s / len(views) - a, 0.0) / b) ** 0.5 // 16 * 16
        size = int(max(64, min(side, max(cam0.width, cam0.height))))
    r = oracle_step_sample(w, 0, size, views=views)
    full = size >= max(cam0.width, cam0.height)
    what = (f"{'one full iteration of ' if batched and len(views) > 1 else ''}{len(views)} view(s) of "
            f"'{config}' at {r['window']}" + ("" if full else " (central window: the full workload was predicted "
                                                              f"at {est:.0f} s)") +
            (" (large: 1 of its 64 views; per-pixel rate, so the 64-view iteration has the same rate)"
             if config == "large" else ""))
    gsref.set_threads(1)
    one = oracle_step_sample(w, 0, 584)
    gsref.set_threads(n_all)
    return {"value": r["blended"] / r["seconds"], "unit": UNIT, "cores": n_all, "kind": "oracle",
            "sample": f"{what}: fwd(F32)+L1+bwd(MIXED) per view, summed gradient, Adam; {r['seconds']:.1f} s",
            "iters_per_s": (1.0 / r["seconds"]) if full and (len(views) == len(w.cameras) or not batched) else None,
            "single_core": {"value": one["blended"] / one["seconds"], "unit": UNIT, "cores": 1,
                            "sample": f"1 view, {one['window']} central window of '{config}' view 0, "
                                      f"{one['seconds']:.1f} s"},
            **host_cpu()}


def run_reference(args, rank, world):
    """--impl reference: the CPU oracle as it stands, timed on this box's host cores (all
    of them, OpenMP over tiles), on the same config, metric and unit.  Each step is a
    bounded sample of the workload (one view on a central window sized from a pilot so
    that warm-up + steps take about two minutes); under torchrun only rank 0 runs."""
    if rank != 0:
        return
    import scenegen
    from oracle import gsref
    gsref.build()
    n_all = gsref.set_threads(0)
    kw = {"num_views": 1} if args.config in ("replica", "scannetpp", "large") else {}
    w = scenegen.make(args.config, args.seed, **kw)
    cam0 = w.cameras[0]
    a, b = pilot_cost(w)
    per_step = min(10.0, 120.0 / max(1, args.steps + min(args.warmup, 1)))
    size = int(max(64, min(int(max(per_step - a, 0.0) / b) ** 0.5 // 16 * 16, max(cam0.width, cam0.height))))
    tgt = None
    for _ in range(min(args.warmup, 1)):
        tgt = oracle_step_sample(w, 0, size)["target"]
    tot_s, tot_b = 0.0, 0
    for _ in range(args.steps):
        r = oracle_step_sample(w, 0, size, tgt)
        tgt = r["target"]
        tot_s += r["seconds"]
        tot_b += r["blended"]
    value = tot_b / tot_s
    sample = (f"1 view, {r['window']} " + ("full image" if size >= max(cam0.width, cam0.height) else "central window")
              + f" of config '{args.config}', fwd(F32)+L1+bwd(MIXED)+Adam per step, {n_all} threads")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * tot_s / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic", "config": {"workload": args.config, "seed": args.seed},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": n_all, "kind": "oracle", "sample": sample,
                             **host_cpu()},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- NEXT-1
def run_schedule(args):
    """The keyframe-scheduled online mapping loop of PAPER.md:149 over a config's pose
    sequence (replica: 100 poses, m = 5, n = 3, 2 random keyframes; scannetpp setting:
    m = 10, n = 1, every frame in the list; threshold 50, 10 global passes,
    PAPER.md:174), each planned iteration one fwd + bwd + Adam step on one view.
    Device time (CUDA events) of the online phase and of the global passes."""
    import torch

    import scenegen
    from paper_2408_12677_b200 import gsr, pipeline
    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0)))
    torch.cuda.set_device(dev)
    lib = gsr.load()
    w = scenegen.make(args.config, args.seed)
    cams = w.cameras
    model = pipeline.GaussianModel(w.scene, dev)
    tgt = pipeline.GaussianModel(w.target_scene, dev)
    pipeline.spatially_order(lib, model)
    pipeline.spatially_order(lib, tgt)
    cap = pipeline.default_capacity(max(pipeline.measure_keys(lib, model, cams, dev),
                                        pipeline.measure_keys(lib, tgt, cams, dev)))
    targets = pipeline.render_targets(lib, tgt, cams, dev, cap)
    del tgt
    scannet = args.config in ("scannetpp", "large")
    setting = dict(m=10, n=1, store_all_frames=True) if scannet else dict(m=5, n=3, store_all_frames=False)
    new = scenegen.new_primitive_counts(len(cams), args.seed)
    tr = pipeline.Trainer(lib, model, cams, targets, dev, cap)
    ko = pipeline.KeyframeOptimizer(lib, tr, new, threshold=50, global_iters=10, seed=args.seed, **setting)
    for v in range(min(args.warmup, len(cams))):
        tr.step([v])
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    ev = {}

    def mark(i, v, f):
        if i == 0:
            ev["start"] = torch.cuda.Event(enable_timing=True)
            ev["start"].record(stream)
        if f < 0 and "glob" not in ev:
            ev["glob"] = torch.cuda.Event(enable_timing=True)
            ev["glob"].record(stream)
    tr.blended.zero_()
    ko.run(mark)
    end = torch.cuda.Event(enable_timing=True)
    end.record(stream)
    torch.cuda.synchronize()
    n_on = ko.n_online
    n_gl = len(ko.views) - n_on
    t_on = ev["start"].elapsed_time(ev.get("glob", end))
    t_gl = ev["glob"].elapsed_time(end) if "glob" in ev else 0.0
    tr.check_capacity()
    line = {"metric": "keyframe-scheduled online mapping: frames/s and ms per iteration (PAPER.md:149)",
            "value": len(cams) / (t_on / 1e3), "unit": "frames/s (online phase)", "n_gpus": 1,
            "higher_is_better": True, "dtype": "f32", "data": "synthetic",
            "config": {"workload": args.config, "frames": len(cams), "keyframes": int(ko.is_keyframe.sum()),
                       "threshold": 50, **setting, "global_iters": 10,
                       "new_primitives": "scenegen.new_primitive_counts (stand-in for the out-of-scope seeding)"},
            "online": {"iterations": n_on, "ms": t_on, "ms_per_iteration": t_on / max(n_on, 1)},
            "global": {"iterations": n_gl, "ms": t_gl, "ms_per_iteration": t_gl / max(n_gl, 1)},
            "blended_per_s": int(tr.blended.item()) / ((t_on + t_gl) / 1e3),
            "paper_context": "RTX 3060 global optimisation (derived, SURVEY.md §6b): Replica 25.5 ms/iteration (PAPER.md:354-356), ScanNet++ 876x584 17.7 ms/iteration (PAPER.md:314-316)"}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- NEXT-3
def run_tsdf(args):
    """TSDF fusion (gs_tsdf_allocate + gs_tsdf_integrate, Eqs. 6-9) of a config's pose
    sequence at 1 cm voxels, eps = 6 cm, w_max 100: `--warmup` frames,
    then `--steps` timed frames (CUDA events).  Depth frames are synthetic (scenegen.
    render_depth of the config's surfaces, 2 mm noise, 1% invalid), on the device before
    the timed region.  Roofline of k_tsdf_integrate: 16 B of voxel state (tsdf + weight,
    read + write) per allocated voxel per frame, against the HBM peak."""
    import torch

    import scenegen
    from paper_2408_12677_b200 import gsr, pipeline
    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0)))
    torch.cuda.set_device(dev)
    lib = gsr.load()
    n = args.warmup + args.steps
    cfg = args.config if args.config in ("replica", "scannetpp", "large") else "replica"
    w = scenegen.make(cfg, args.seed, num_views=n)
    cams = w.cameras[:n]
    depths = [torch.from_numpy(scenegen.render_depth(w.faces, c, noise_sigma=0.002, dropout=0.01, seed=k)).to(dev)
              for k, c in enumerate(cams)]
    vol = pipeline.TsdfVolume(lib, dev, 1 << 20, voxel_size=0.01, w_max=100.0)
    for k in range(args.warmup):
        vol.integrate_frame(cams[k], depths[k])
    torch.cuda.synchronize()
    nb0 = int(vol.num_blocks.item())
    vol.new_blocks.zero_()
    vol.updated.zero_()
    stream = torch.cuda.current_stream()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3 * args.steps + 1)]
    ev[0].record(stream)
    gcams = [gsr.camera(c) for c in cams]
    for i in range(args.steps):
        k = args.warmup + i
        lib.tsdf_allocate(vol.prm, vol.vol, gcams[k], depths[k], vol.new_blocks)
        ev[3 * i + 1].record(stream)
        lib.tsdf_integrate(vol.prm, vol.vol, gcams[k], depths[k], vol.updated)
        ev[3 * i + 2].record(stream)
        ev[3 * i + 3] = ev[3 * i + 2]
    torch.cuda.synchronize()
    ms = ev[0].elapsed_time(ev[-1])
    alloc_ms = sum(ev[3 * i].elapsed_time(ev[3 * i + 1]) for i in range(args.steps)) / args.steps
    int_ms = sum(ev[3 * i + 1].elapsed_time(ev[3 * i + 2]) for i in range(args.steps)) / args.steps
    nb1 = int(vol.num_blocks.item())
    if nb1 > vol.block_cap:
        raise RuntimeError("TSDF block pool overflow")
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except OSError:
        pass
    peak = peaks.get("hbm_gbs") or 6556.2
    vox_bytes = (nb0 + nb1) / 2 * 512 * 16  # mean allocated voxels x (tsdf, weight) read + write
    gbs = vox_bytes / (int_ms / 1e3) / 1e9
    upd = int(vol.updated.item())
    line = {"metric": "TSDF fusion (band allocation + Eqs. 6-9 integration): frames/s and voxel updates/s",
            "value": args.steps / (ms / 1e3), "unit": "frames/s", "n_gpus": 1, "steps": args.steps,
            "warmup": args.warmup, "ms_per_frame": ms / args.steps, "higher_is_better": True, "dtype": "f32",
            "data": "synthetic", "config": {"workload": cfg, "resolution": f"{cams[0].width}x{cams[0].height}",
                                            "voxel_size_m": 0.01, "trunc_m": 0.06, "w_max": 100, "step_m": 0.005,
                                            "depth": "scenegen.render_depth: 2 mm noise, 1% invalid"},
            "voxel_updates_per_s": upd / (ms / 1e3), "blocks": {"before": nb0, "after": nb1,
                                                                 "new_in_timed": int(vol.new_blocks.item())},
            "stage_ms": {"allocate": alloc_ms, "integrate": int_ms},
            "roofline": {"kernel": "k_tsdf_integrate", "bound": "hbm", "achieved": gbs, "peak": peak, "unit": "GB/s",
                         "frac": gbs / peak, "algorithmic_bytes_per_launch": vox_bytes,
                         "note": "16 B per allocated voxel (tsdf + weight read and written); depth reads not counted"}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- online loop
def run_online(args):
    """GSFusion's incremental mapping over `--steps` frames of a config's pose sequence
    (replica: 1200x680, the paper's Replica settings PAPER.md:174: 1 cm voxels,
    quadtree threshold 0.1, keyframe threshold 50, m = 5, n = 3, 10 global passes;
    scannetpp / large: m = 10, n = 1, every frame a list member).  Per frame: TSDF fusion,
    seeding, the frame's iterations; then the global passes.  Colour frames are renders
    of the config's ground-truth Gaussians (stand-in for the sensor), depth frames
    scenegen.render_depth (2 mm noise).  Device time (CUDA events); the per-frame seed
    count read-back is a host sync inside the loop, as in the paper's system."""
    import torch

    import scenegen
    from paper_2408_12677_b200 import gsr, pipeline
    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0)))
    torch.cuda.set_device(dev)
    lib = gsr.load()
    cfg = args.config if args.config in ("replica", "scannetpp", "large") else "replica"
    n_frames = args.steps
    w = scenegen.make(cfg, args.seed, num_views=max(n_frames, 1))
    cams = w.cameras[:n_frames]
    gt = pipeline.GaussianModel(w.scene, dev)
    pipeline.spatially_order(lib, gt)
    cap = pipeline.default_capacity(pipeline.measure_keys(lib, gt, cams, dev))
    rgbs = [t[0].contiguous() for t in pipeline.render_targets(lib, gt, cams, dev, cap)]
    del gt
    depths = [torch.from_numpy(scenegen.render_depth(w.faces, c, noise_sigma=0.002, seed=k)).to(dev)
              for k, c in enumerate(cams)]
    scannet = cfg != "replica"
    kf = dict(m=10, n=1, store_all_frames=True) if scannet else dict(m=5, n=3, store_all_frames=False)
    om = pipeline.OnlineMapper(lib, cams, dev, capacity=2_000_000, sh_degree=3, key_capacity=12 << 20,
                               voxel_size=0.01, block_cap=1 << 20, threshold=0.1, min_cell=4, kf_threshold=50,
                               global_iters=10, seed=args.seed, **kf)
    stream = torch.cuda.current_stream()
    torch.cuda.synchronize()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    e[0].record(stream)
    for t in range(n_frames):
        om.add_frame(t, rgbs[t], depths[t])
    e[1].record(stream)
    it_online = om.iterations
    P_online = om.model.P
    is_kf = om.finish()
    e[2].record(stream)
    torch.cuda.synchronize()
    om.trainer.check_capacity()
    t_on, t_gl = e[0].elapsed_time(e[1]), e[1].elapsed_time(e[2])
    it_gl = om.iterations - it_online
    line = {"metric": "online mapping (TSDF fusion + quadtree seeding + keyframe-scheduled optimisation)",
            "value": n_frames / (t_on / 1e3), "unit": "frames/s (online phase)", "n_gpus": 1, "steps": n_frames,
            "higher_is_better": True, "dtype": "f32", "data": "synthetic",
            "config": {"workload": cfg, "resolution": f"{cams[0].width}x{cams[0].height}", "frames": n_frames,
                       "voxel_size_m": 0.01, "quadtree_threshold": 0.1, "min_cell": 4, "keyframe_threshold": 50, **kf,
                       "global_iters": 10, "sh_degree": 3,
                       "inputs": "colour = render of the config's ground-truth Gaussians, depth = render_depth 2 mm"},
            "online": {"ms": t_on, "ms_per_frame": t_on / n_frames, "iterations": it_online,
                       "gaussians": P_online, "keyframes": int(is_kf.sum()), "new_per_frame": om.counts},
            "global": {"ms": t_gl, "iterations": it_gl, "ms_per_iteration": t_gl / max(it_gl, 1)},
            "tsdf_blocks": int(om.tsdf.num_blocks.item()),
            "paper_context": "RTX 3060 + i7-13700, whole system: Replica 9.73 FPS, ScanNet++ (876x584) 6.14 FPS "
                             "(PAPER.md:236-239); global optimisation 25.5 / 17.7 ms per iteration (derived)"}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- launcher
def self_launch(args) -> int:
    """`bench.py --gpus N` (N > 1) run without torchrun: re-launch this command under
    torch.distributed.run with N ranks, one per GPU (the contract's launch line).  Fails
    loudly when fewer than N GPUs are visible (no silent 1-GPU number)."""
    import socket
    if args.impl != "reference":
        import torch
        n_vis = torch.cuda.device_count() if torch.cuda.is_available() else 0
        if n_vis < args.gpus:
            print(f"bench.py: --gpus {args.gpus} but only {n_vis} GPU(s) visible; refusing to report a "
                  f"{n_vis}-GPU number as {args.gpus}", file=sys.stderr, flush=True)
            return 2
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


# ----------------------------------------------------------------------------- GPU arm
def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(self_launch(args))
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    if world != max(args.gpus, 1) and "WORLD_SIZE" in os.environ and os.environ.get("GSR_FORCE_DIST") != "1":
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr, flush=True)
        sys.exit(2)
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if args.schedule:
        run_schedule(args)
        return
    if args.tsdf:
        run_tsdf(args)
        return
    if args.online:
        run_online(args)
        return

    import numpy as np
    import torch
    import torch.distributed as dist

    import scenegen
    from paper_2408_12677_b200 import gsr, pipeline

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    # GSR_FORCE_DIST=1: run the N > 1 exchange + optimiser path even at world size 1 (a
    # functional check of that path on a single GPU; the sums then have one term)
    dist_on = world > 1 or os.environ.get("GSR_FORCE_DIST") == "1"
    if dist_on:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29531")
        dist.init_process_group("nccl", device_id=dev, rank=rank, world_size=world)
    lib = gsr.load()

    w = scenegen.make(args.config, args.seed)
    cams = w.cameras
    B = len(cams)
    my_views = scenegen.shard_views(B, rank, world)
    model = pipeline.GaussianModel(w.scene, dev)
    tgt_model = pipeline.GaussianModel(w.target_scene, dev)
    if not args.no_morton:  # setup-time layout: Gaussians in Morton order of their means
        pipeline.spatially_order(lib, model)
        pipeline.spatially_order(lib, tgt_model)
    my_cams = [cams[v] for v in my_views]
    K0 = max(pipeline.measure_keys(lib, model, my_cams, dev), pipeline.measure_keys(lib, tgt_model, my_cams, dev))
    cap = pipeline.default_capacity(K0)
    tg = pipeline.render_targets(lib, tgt_model, my_cams, dev, cap)
    # the targets as an RGB-D sensor delivers them (R41): 8-bit colour and
    # 16-bit depth in mm.  The host frames feed the e2e leg; the device-resident float
    # targets of the timed region are decoded from the same frames (gs_decode_rgbd).
    targets = [None] * B
    frames = {}
    for v, t in zip(my_views, tg):
        c8, d16 = scenegen.quantize_frame(t[0].cpu().numpy(), t[1].cpu().numpy())
        frames[v] = (torch.from_numpy(c8), torch.from_numpy(d16.view(np.int16)))
        lib.decode_rgbd(frames[v][0].to(dev), frames[v][1].to(dev), scenegen.DEPTH_SCALE, t[0], t[1])
        targets[v] = t
    del tgt_model, tg
    torch.cuda.empty_cache()

    # scannetpp / large: a batch of views per iteration, sharded over ranks, gradient
    # all-reduced (strong scaling).  tiny / small / replica: one view per iteration
    # (PAPER.md:149), cycling through the poses; N > 1 runs independent replicas.
    batched = args.config in ("scannetpp", "large")
    allreduce = None
    if dist_on and batched:
        allreduce = lambda g: dist.all_reduce(g, op=dist.ReduceOp.SUM)  # noqa: E731

    def step_views(i):
        return my_views if batched else [my_views[i % len(my_views)]]
    optimizer, optim_used = None, ("replicated" if dist_on and batched else "local")
    if dist_on and batched and args.optim in ("nvls", "peer"):
        if args.optim == "nvls":
            try:
                optimizer, optim_used = pipeline.NvlsShardedAdam(lib, model), "nvls"
            except Exception as ex:  # noqa: BLE001  (no multicast: the P2P kernel)
                model.params, model.grad = model.params.clone(), model.grad.clone()
                optim_used = f"peer (nvls unavailable: {ex})"
        if optimizer is None:
            try:
                optimizer = pipeline.PeerShardedAdam(lib, model)
                optim_used = optim_used if optim_used.startswith("peer") else "peer"
            except Exception as ex:  # noqa: BLE001  (no symmetric memory / P2P: NCCL path)
                optim_used = f"sharded (peer unavailable: {type(ex).__name__})"
        ok = torch.tensor([1 if optimizer is not None else 0], dtype=torch.int32, device=dev)
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)  # every rank takes the same path
        if int(ok.item()) == 0 and optimizer is not None:
            # another rank could not set up the peer path: undo ours (copy the state out of
            # the symmetric buffers) and use the NCCL path everywhere
            model.params = model.params.clone()
            model.grad = model.grad.clone()
            optimizer, optim_used = None, "sharded (peer unavailable on another rank)"
    if dist_on and batched and args.optim == "sparse":
        optimizer, optim_used = pipeline.SparseExchangeAdam(lib, model), "visibility-sparse exchange, replicated"
    if dist_on and batched and optimizer is None and args.optim in ("nvls", "peer", "sharded"):
        optimizer = pipeline.ShardedAdam(lib, model)
        optim_used = optim_used if optim_used.startswith("sharded") else "sharded"
    if optimizer is not None:
        allreduce = None
    chunk = args.chunk if args.chunk > 0 else min(64, max(1, len(my_views) if batched else 1))
    tr = pipeline.Trainer(lib, model, cams, targets, dev, cap, allreduce=allreduce,
                          streams=args.streams if batched else 1, optimizer=optimizer, chunk=chunk)
    stream = torch.cuda.current_stream()

    # --- warm-up (and the render kernels' block-row walk chosen for this scene by timing
    # both forms of a few views' render passes: gs_set_render_rows, same results)
    render_tune = None
    if not args.profile and os.environ.get("GSR_RENDER_ROWS") is None:
        tr.autotune_render(step_views(0))
        render_tune = tr.render_tune
    elif os.environ.get("GSR_RENDER_ROWS") is not None:
        lib.set_render_rows(os.environ["GSR_RENDER_ROWS"] != "0")
    for i in range(args.warmup):
        tr.step(step_views(i))
    torch.cuda.synchronize()
    if dist_on and not pipeline.params_agree_across_ranks(model):
        if not optim_used.startswith(("peer", "nvls")):
            raise RuntimeError(f"parameters differ across ranks after warm-up (optimiser: {optim_used})")
        # the peer-memory path misbehaved on this machine: resynchronise from rank 0
        # and continue on the NCCL reduce-scatter path (m, v shards keep their owners)
        dist.broadcast(model.params, src=0)
        tr.optimizer = pipeline.ShardedAdam(lib, model)
        optim_used = "sharded (peer failed the cross-rank check)"
        for i in range(args.warmup):
            tr.step(step_views(i))
        torch.cuda.synchronize()
        if not pipeline.params_agree_across_ranks(model):
            raise RuntimeError("parameters differ across ranks after warm-up (sharded)")

    # --- timed region (device time, CUDA events, max over ranks)
    clocks = ClockSampler(local)
    if not args.profile:
        clocks.start()
    tr.blended.zero_()
    tr.num_keys.zero_()
    stage_ev = {"project": [], "bin": [], "render_fwd": [], "render_bwd": [], "project_bwd": []}
    open_ev = {}

    def hooks(stage, what):
        ev = torch.cuda.Event(enable_timing=True)
        ev.record(torch.cuda.current_stream())  # the stream the stage is launched on
        if what == "begin":
            open_ev[stage] = ev
        else:
            stage_ev[stage].append((open_ev.pop(stage), ev))

    # CUDA-graph mode: each distinct view set of the timed steps is captured once as a
    # whole iteration -- at N > 1 including the exchange (NCCL collectives, or the
    # peer-memory kernel and its barriers) and Adam with the device step counter -- and
    # replayed, so N = 1 and N = 8 are timed alike; launches per step are counted while
    # capturing (a replay does not pass through the library's counter).  The
    # visibility-sparse exchange reads its size on the host and stays eager.
    use_graph = (args.graph and not args.profile and
                 (tr.optimizer is None or hasattr(tr.optimizer, "device_step")))
    graphs, graph_launches = {}, {}
    if use_graph:
        for i in range(args.steps):
            key = tuple(step_views(args.warmup + i))
            if key not in graphs:
                c0 = lib.launch_count()
                graphs[key] = tr.capture(list(key))
                graph_launches[key] = (lib.launch_count() - c0) // 2  # eager warm-up + captured step
        torch.cuda.synchronize()
        tr.blended.zero_()
        tr.num_keys.zero_()

    def timed_loop(graph_mode):
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        tr.hooks = None if graph_mode else hooks
        a.record(stream)
        if args.profile:
            torch.cuda.nvtx.range_push("timed")
        done, nl = 0, 0
        for i in range(args.steps):
            sv = step_views(args.warmup + i)
            if graph_mode:
                tr.replay(graphs[tuple(sv)])
                nl += graph_launches[tuple(sv)]
            else:
                tr.step(sv)
            done += len(sv)
        b.record(stream)
        if args.profile:
            torch.cuda.nvtx.range_pop()
        tr.hooks = None
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        return a.elapsed_time(b), done, nl

    # the training state the timed steps start from: the K13 arm below re-runs the same
    # steps from it, so both arms composite identical scenes
    state0 = ([t.clone() for t in (model.params, model.m, model.v, model.step_dev)], model.step_count)

    def restore_state():
        for t, c in zip((model.params, model.m, model.v, model.step_dev), state0[0]):
            t.copy_(c)
        model.step_count = state0[1]

    l0 = lib.launch_count()
    ms, views_done, nl = timed_loop(use_graph)
    launches = nl if use_graph else lib.launch_count() - l0
    clk = clocks.stop() if not args.profile else None
    stage_ms = {k: sum(a.elapsed_time(b) for a, b in v) / max(len(v), 1) for k, v in stage_ev.items()}
    # Per-kernel rooflines need each stage's own duration: with views in flight on
    # several streams the stages overlap, so an extra serialised pass (streams = 1,
    # same steps, CUDA events on the launching stream) times them in isolation.
    blended_timed = int(tr.blended.item())
    stage_ms_overlapped = None
    eager = None
    if use_graph:  # the same steps eager (no graph), for comparison
        tr.blended.zero_()
        e_ms, _, _ = timed_loop(False)
        eager = {"ms_per_step": e_ms / args.steps, "value": int(tr.blended.item()) / (e_ms / 1e3), "unit": UNIT,
                 "note": "same steps launched eagerly from Python (no CUDA graph)"}
        stage_ms = {k: sum(a.elapsed_time(b) for a, b in v) / max(len(v), 1) for k, v in stage_ev.items()}
    if (tr._streams is not None or use_graph) and not args.profile:
        stage_ms_overlapped = stage_ms if tr._streams is not None else None
        tr.serial = True
        tr.step(step_views(0))
        for v in stage_ev.values():
            v.clear()
        tr.hooks = hooks
        for i in range(min(args.steps, 5)):
            tr.step(step_views(args.warmup + i))
        tr.hooks = None
        torch.cuda.synchronize()
        tr.serial = False
        stage_ms = {k: sum(a.elapsed_time(b) for a, b in v) / max(len(v), 1) for k, v in stage_ev.items()}
    kmax = int(tr.num_keys.max().item())
    if kmax > cap:
        raise RuntimeError(f"key capacity overflow during the timed region: K={kmax} > {cap}")
    blended = blended_timed
    fwd_ms, bwd_ms = stage_ms["render_fwd"], stage_ms["render_bwd"]
    stats = torch.tensor([ms, float(blended), fwd_ms, bwd_ms], dtype=torch.float64, device=dev)
    if world > 1:
        mx = stats.clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        sm = stats.clone()
        dist.all_reduce(sm, op=dist.ReduceOp.SUM)
        ms, blended = float(mx[0]), int(sm[1])
    ms_step = ms / args.steps
    value = blended / (ms / 1000.0)
    iters = args.steps / (ms / 1000.0)

    # --- end to end: targets from pinned host memory every step, loss read back
    e2e = None
    if not args.no_e2e and not args.profile:
        # sensor frames (uint8 rgb, 16-bit depth) from pinned host memory, decoded on the GPU
        host_t = {v: (frames[v][0].pin_memory(), frames[v][1].pin_memory()) for v in my_views}
        h2d = sum(host_t[v][0].numel() * host_t[v][0].element_size() +
                  host_t[v][1].numel() * host_t[v][1].element_size() for v in step_views(0))
        loss_host = torch.zeros(1, dtype=torch.float32).pin_memory()
        tr.step_host(step_views(0), host_t, scenegen.DEPTH_SCALE)  # allocate the slots + copy stream (untimed)
        torch.cuda.synchronize()
        tr.blended.zero_()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        hs = None
        # the graph-replayed iteration fed from the host (pipeline.HostStreamedGraphs):
        # scannetpp 82 MB of frames per step (e2e 5.87 vs 6.18 ms eager), config 4 885 MB
        # (80.4 ms vs 82-84 eager, once CUDA_DEVICE_MAX_CONNECTIONS lifts the false
        # serialisation of the copy stream with the render streams, tools/e2e_diag4.py)
        if use_graph and batched:
            hs = pipeline.HostStreamedGraphs(tr, step_views(0), [host_t, host_t], scenegen.DEPTH_SCALE)
            for _ in range(2):  # first replay of each parity's graphs (upload) outside the timing
                hs.step()
            torch.cuda.synchronize()
            tr.blended.zero_()
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize()
        s0.record(stream)
        for i in range(args.steps):
            sv = step_views(i)
            if hs is not None:
                # frames copied + decoded under the previous step; loss read back on a side stream
                hs.step(prefetch=i + 2 < args.steps)
            else:
                tr.loss.zero_()
                tr.step_host(sv, host_t, scenegen.DEPTH_SCALE)  # every view's frame: host -> device + decode
                loss_host.copy_(tr.loss, non_blocking=True)
        s1.record(stream)
        if hs is not None:
            stream.wait_stream(hs.readback_stream)  # the last loss has reached the host
            s1.record(stream)
        torch.cuda.synchronize()
        ems = s0.elapsed_time(s1)
        eb = int(tr.blended.item())
        st = torch.tensor([ems, float(eb)], dtype=torch.float64, device=dev)
        if world > 1:
            mx = st.clone()
            dist.all_reduce(mx, op=dist.ReduceOp.MAX)
            sm = st.clone()
            dist.all_reduce(sm, op=dist.ReduceOp.SUM)
            ems, eb = float(mx[0]), int(sm[1])
        e2e = {"value": eb / (ems / 1000.0), "unit": UNIT, "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": 4,
               "iters_per_s": args.steps / (ems / 1000.0),
               "inputs": "per view an RGB-D sensor frame (uint8 [H][W][3] + uint16 mm [H][W]) from pinned host "
                         "memory, copied and decoded (gs_decode_rgbd) inside the step; loss read back",
               "mode": ("per step the frames copied + decoded on a high-priority copy stream under the "
                        "previous step, then the iteration graph (pipeline.HostStreamedGraphs)" if hs is not None else "eager (Trainer.step_host)")}

    # --- K13: the straightforward per-pixel GPU port (north_star's >= 10x target), same
    # steps with gs_naive_render_fwd / gs_naive_render_bwd_screen, device-timed the same way
    naive = None
    if not args.no_naive and not args.profile:
        tr.naive = True
        tr.step(step_views(0))
        restore_state()
        tr.blended.zero_()
        nsteps = min(args.steps, 3)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        n0, n1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n0.record(stream)
        for i in range(nsteps):
            tr.step(step_views(args.warmup + i))
        n1.record(stream)
        torch.cuda.synchronize()
        tr.naive = False
        nms = n0.elapsed_time(n1)
        nb = int(tr.blended.item())
        st = torch.tensor([nms, float(nb)], dtype=torch.float64, device=dev)
        if world > 1:
            mx = st.clone()
            dist.all_reduce(mx, op=dist.ReduceOp.MAX)
            sm = st.clone()
            dist.all_reduce(sm, op=dist.ReduceOp.SUM)
            nms, nb = float(mx[0]), int(sm[1])
        nval = nb / (nms / 1000.0)
        naive = {"value": nval, "unit": UNIT, "ms_per_step": nms / nsteps, "steps": nsteps,
                 "speedup": value / nval, "start": "the timed region's first steps from its starting state",
                 "what": "K13: same project/bin/project-bwd/Adam; render fwd and bwd one thread per pixel, "
                         "records read from global memory, 10 atomicAdd per composited pair"}

    if rank != 0:
        if dist_on:
            dist.destroy_process_group()
        return

    # --- roofline of the dominant kernel
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except OSError:
        pass
    n_views = views_done
    # evaluated pairs of the backward = sum of n_contrib over the views (untimed re-render)
    evaluated, vis, keys = 0, 0, 0
    eval_views = my_views[:8]
    for v in eval_views:
        keys += pipeline.render(lib, model, cams[v], tr.buf, sync_keys=True)
        evaluated += int(tr.buf.n.sum().item())
        vis += int((tr.buf.proj_t["tiles"][:model.P] > 0).sum().item())
    nv = len(eval_views)
    hbm = stage_hbm(peaks, stage_ms, model.P, w.scene.sh_degree, vis / nv, keys / nv, cams[0].num_tiles)
    traffic = None
    try:
        traffic = json.load(open(os.path.join(ROOT, "profiles", "traffic.json"))).get(args.config, {}).get("k_render_bwd")
    except (OSError, ValueError):
        pass
    roof = roofline(dev, peaks, clk, stage_ms, blended / max(world, 1) / n_views, evaluated / len(eval_views), traffic)
    roof["timing"] = ("CUDA events around each launch on its stream, serialised pass (streams=1) of the same steps "
                      "right after the timed region" if (stage_ms_overlapped is not None or use_graph) else
                      "CUDA events around each launch on its stream, inside the timed region")
    if stage_ms_overlapped is not None:
        roof["launch_ms_overlapped"] = stage_ms_overlapped["render_bwd"]

    cpu = None
    if world == 1 and not args.no_cpu_baseline and not args.profile:
        try:
            cpu = cpu_oracle_legs(w, args.config)
        except Exception as ex:  # noqa: BLE001
            cpu = {"value": None, "unit": UNIT, "cores": None, "kind": "oracle", "sample": f"failed: {ex}"}

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "iters_per_s": iters, "higher_is_better": True,
        "scaling": "strong" if batched else "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": args.config, "views_per_step": B if batched else 1, "views": B, "P": w.scene.P, "sh_degree": w.scene.sh_degree,
                   "resolution": f"{cams[0].width}x{cams[0].height}", "parallelism": (f"views/dp{world}" + (f" ({optim_used} Adam)" if dist_on else "")) if batched else f"replicas x{world}",
                   "key_capacity": cap, "streams": args.streams if batched else 1, "chunk": chunk, "max_keys_per_view": kmax,
                   "gaussian_order": "generated" if args.no_morton else "morton",
                   "render_rows": lib.render_rows(), "render_tune": render_tune,
                   "targets": "renders of the target scene quantised to RGB-D sensor frames (8-bit colour, 16-bit mm "
                              "depth) and decoded on the GPU",
                   "launch": "CUDA graph per iteration" if use_graph else "eager",
                   "l2": "inputs larger than L2 (params+grad+m+v %.0f MB, targets %.0f MB per rank)" % (
                       4 * model.nbytes / 1e6, sum(t[0].numel() * 4 + t[1].numel() * 4 for t in targets if t) / 1e6)},
        "gpu_launches": int(launches),
        "stage_ms": stage_ms, "stage_ms_overlapped": stage_ms_overlapped, "stage_hbm": hbm,
        "work": {"blended_per_view": blended / max(world, 1) / n_views, "evaluated_per_view": evaluated / nv,
                 "keys_per_view": keys / nv, "views_per_s": views_done * world / (ms / 1e3),
                 "evaluated_per_s": evaluated / nv * views_done * world / (ms / 1e3),
                 "keys_per_s": keys / nv * views_done * world / (ms / 1e3),
                 "note": "evaluated = sum of n_contrib (list entries visited up to each pixel's stop, R24), "
                         "measured on up to 8 of this rank's views after the timed region"},
        "roofline": roof, "clocks": clk, "e2e": e2e, "cpu_baseline": cpu, "naive_port": naive, "eager": eager,
    }
    if getattr(tr.optimizer, "last_M", None) is not None:  # visibility-sparse exchange: columns on the wire
        line["exchange"] = {"union_visible_columns": tr.optimizer.last_M, "P": model.P,
                            "bytes_per_rank": 4 * model.F * tr.optimizer.last_M,
                            "dense_bytes_per_rank": 4 * model.F * model.P}
    print(json.dumps(line), flush=True)
    if dist_on:
        dist.destroy_process_group()


def stage_hbm(peaks, stage_ms, P, deg, V, K, NT):
    """HBM roofline of the projection and binning stages (north_star: >= 50% of HBM
    peak on project/bin), each against its COMPULSORY bytes: inputs
    read once and outputs written once, no intermediate traffic counted.
      project: P (12 B mean + 9 B radius/tiles/flags) + V (32 B scale/quat/logit +
               12 (deg+1)^2 B SH + 48 B record)
      bin:     P 4 B tiles + V 12 B (depth, rect) + K 4 B sorted ids + NT 8 B ranges
    V = visible Gaussians, K = keys, per view (means over the measured views)."""
    peak = peaks.get("hbm_gbs") or 6556.2
    S = (deg + 1) ** 2
    out = {}
    for st, by in (("project", P * 21 + V * (32 + 12 * S + 48)), ("bin", P * 4 + V * 12 + K * 4 + NT * 8)):
        ms = stage_ms.get(st)
        if ms:
            gbs = by / (ms / 1e3) / 1e9
            out[st] = {"ms": ms, "compulsory_bytes": int(by), "achieved": gbs, "peak": peak, "unit": "GB/s",
                       "frac": gbs / peak}
    out["V_per_view"], out["K_per_view"] = int(V), int(K)
    return out


def roofline(dev, peaks, clk, stage_ms, blended_per_view, evaluated_per_view, traffic):
    """Issue-bound roofline of the dominant kernel, k_render_bwd, on
    SURVEY.md §8(d) row a5's algorithmic count: 70 lane-instructions per blended pair
    (the row's 60-80 range, bounds reported as frac_range) + 15 per evaluated-but-skipped
    pair, against the FP32-lane issue peak SMs x 128 lanes x SM clock measured during the
    run.  The builder's narrower count (8 FP32 ops per evaluated + 21 per blended pair:
    the arithmetic alone) is reported alongside as "arith"."""
    import torch
    props = torch.cuda.get_device_properties(dev)
    sms = props.multi_processor_count
    mhz = (clk or {}).get("sm_mhz") or peaks.get("sm_max_mhz") or 1965.0
    peak = sms * 128 * mhz * 1e6 / 1e12
    skipped = max(0.0, evaluated_per_view - blended_per_view)
    ms = stage_ms["render_bwd"]

    def rate(per_blended):
        return (per_blended * blended_per_view + 15.0 * skipped) / (ms / 1e3) / 1e12
    ops = 70.0 * blended_per_view + 15.0 * skipped
    achieved = rate(70.0)
    arith_ops = 8.0 * evaluated_per_view + 21.0 * blended_per_view
    arith = arith_ops / (ms / 1e3) / 1e12
    return {"kernel": "k_render_bwd (gs_render_bwd_screen_l1)", "bound": "alu", "achieved": achieved, "peak": peak,
            "unit": "T lane-instr/s", "frac": achieved / peak, "frac_range": [rate(60.0) / peak, rate(80.0) / peak],
            "count": "SURVEY 8(d) a5: 70 (60-80) lane-instr per blended pair + 15 per skipped pair",
            "traffic": traffic, "algorithmic_ops_per_launch": ops, "launch_ms": ms,
            "arith": {"ops_per_launch": arith_ops, "achieved": arith, "frac": arith / peak,
                      "count": "8 FP32 ops per evaluated pair + 21 per blended pair"},
            "peak_source": f"derived: {sms} SMs x 128 FP32 lanes x {mhz:.0f} MHz (SM clock sampled during the run)"}


if __name__ == "__main__":
    main()
