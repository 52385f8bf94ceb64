"""Host orchestration of one optimisation iteration through the C ABI.

This is the user-facing API: it owns the device buffers (torch tensors) and
issues the ABI calls in the order of SURVEY.md CS2/CS3 -- per view
gs_project -> gs_bin_tiles -> gs_render_fwd -> gs_l1_loss_grad -> gs_render_bwd,
then (optionally) a gradient all-reduce across ranks and gs_adam_step.  No
arithmetic of the method happens here.
"""
from __future__ import annotations

import math
import os

import torch

from . import gsr

# Per-row learning rates (reading R20; SPEC.md:436 defaults)
LR_MEAN, LR_LOGSCALE, LR_QUAT, LR_OPACITY, LR_SH = 2e-4, 5e-3, 1e-3, 5e-2, 2.5e-3


def lr_per_row(sh_degree: int):
    F = 11 + 3 * (sh_degree + 1) ** 2
    return [LR_MEAN] * 3 + [LR_LOGSCALE] * 3 + [LR_QUAT] * 4 + [LR_OPACITY] + [LR_SH] * (F - 11)


class GaussianModel:
    """Parameters, gradient and Adam moments, each float32 [F][P_stride] on one device."""

    def __init__(self, scene, device, params=None):
        self.P, self.sh_degree = int(scene.P), int(scene.sh_degree)
        self.F, self.P_stride = int(scene.params.shape[0]), int(scene.params.shape[1])
        self.params = params if params is not None else torch.from_numpy(scene.params).to(device)
        self.grad = torch.zeros_like(self.params)
        self.m = torch.zeros_like(self.params)
        self.v = torch.zeros_like(self.params)
        self.step_count = 0
        # device copy of the step counter for graph-captured iterations (gs_adam_step_dev)
        self.step_dev = torch.zeros(1, dtype=torch.int64, device=device)
        self.lr = lr_per_row(self.sh_degree)
        self.desc = gsr.scene_desc(self.P, self.P_stride, self.sh_degree)

    @property
    def nbytes(self):
        return 4 * self.params.numel()


def spatially_order(lib, model: GaussianModel):
    """Permute the model's Gaussians into Morton order of their means (gs_spatial_order):
    a setup-time layout transform; returns the permutation (new index -> old index)."""
    out = torch.empty_like(model.params)
    perm = torch.empty(max(model.P, 1), dtype=torch.int32, device=model.params.device)
    lib.spatial_order(model.desc, model.params, out, perm)
    model.params = out
    return perm[:model.P]


class ViewBuffers:
    """Device buffers for one view in flight (reused across views of equal size)."""

    def __init__(self, lib: gsr.Library, cam, P: int, key_capacity: int, device, deterministic: bool = False):
        self.lib = lib
        self.W, self.H = int(cam.width), int(cam.height)
        self.NT = ((self.W + 15) // 16) * ((self.H + 15) // 16)
        self.key_capacity = int(key_capacity)
        self.proj, self.proj_t = gsr.make_proj(P, device)
        gcam = gsr.camera(cam)
        self.bin_ws = torch.empty(lib.bin_tiles_workspace(gcam, P, key_capacity) // 4 + 4, dtype=torch.int32,
                                  device=device)
        self.sorted_ids = torch.empty(max(key_capacity, 1), dtype=torch.int32, device=device)
        self.key_blocks = torch.empty(max(key_capacity, 1) + 16, dtype=torch.uint8, device=device)
        self.ranges = torch.empty((self.NT, 2), dtype=torch.int32, device=device)
        self.tile_order = torch.empty(self.NT, dtype=torch.int32, device=device)
        npx = self.W * self.H
        self.rgb = torch.empty((3, self.H, self.W), dtype=torch.float32, device=device)
        self.depth = torch.empty((self.H, self.W), dtype=torch.float32, device=device)
        self.T = torch.empty((self.H, self.W), dtype=torch.float32, device=device)
        self.n = torch.empty((self.H, self.W), dtype=torch.int32, device=device)
        self.g_rgb = torch.empty((3, self.H, self.W), dtype=torch.float32, device=device)
        self.g_depth = torch.empty((self.H, self.W), dtype=torch.float32, device=device)
        sgrad_bytes = lib.render_bwd_workspace(gsr.scene_desc(P, P, 0))
        self.bwd_ws = torch.empty(max(sgrad_bytes // 4, 4), dtype=torch.float32, device=device)
        # the forward's state (gs_fwd_state), filled by gs_render_fwd and checked by the
        # backward (GS_ERR_STATE on buffers of another forward)
        self.fwd_state = gsr.GsFwdState()
        # deterministic reduction workspace (gs_bwd_opts.det_ws): float[key_capacity][12]
        self.det = (torch.empty((max(key_capacity, 1), gsr.SGRAD_FLOATS), dtype=torch.float32, device=device)
                    if deterministic else None)
        assert npx > 0


def render(lib, model: GaussianModel, cam, buf: ViewBuffers, num_keys_dev=None, blended=None, sync_keys=False):
    """gs_project -> gs_bin_tiles -> gs_render_fwd for one view.  Returns K if sync_keys."""
    gcam = gsr.camera(cam)
    lib.project(gcam, model.desc, model.params, buf.proj)
    K, _ = lib.bin_tiles(gcam, model.desc, buf.proj, buf.bin_ws, buf.key_capacity, buf.sorted_ids, buf.ranges,
                         num_keys_dev=num_keys_dev, sync=sync_keys, allow_capacity=sync_keys)
    lib.render_fwd(gcam, model.desc, buf.proj, buf.sorted_ids, buf.ranges, buf.rgb, buf.depth, buf.T, buf.n,
                   blended=blended)
    return K


def measure_keys(lib, model: GaussianModel, cameras, device) -> int:
    """Exact max K over the views (synchronous, setup only)."""
    best = 0
    P = model.P
    cap = 1 << 20
    buf = None
    for cam in cameras:
        while True:
            if buf is None or buf.key_capacity < cap or (buf.W, buf.H) != (cam.width, cam.height):
                buf = ViewBuffers(lib, cam, P, cap, device)
            K = render(lib, model, cam, buf, sync_keys=True)
            if K <= cap:
                break
            cap = int(K * 1.25) + 1024
        best = max(best, K)
    return best


class Trainer:
    """fwd + bwd + Adam over a batch of views.

    Per view: gs_project -> gs_bin_tiles -> gs_render_fwd -> gs_l1_loss_grad ->
    gs_render_bwd_screen (screen-space gradients of that view); after every
    ``chunk`` views (<= 8) one gs_project_bwd_views chains them all to the parameter
    gradient in a single pass.  ``allreduce`` (optional) is called on the gradient
    between the last view and the Adam step -- the one exchange of the data-parallel
    path (NCCL all-reduce over NVLink in bench.py).  ``hooks`` (optional) is called
    as hooks(stage, "begin"/"end") around the render_fwd and render_bwd stages (used
    by bench.py to time them with CUDA events on the launching stream)."""

    def __init__(self, lib, model: GaussianModel, cameras, targets, device, key_capacity: int,
                 w_depth: float = 1.0, allreduce=None, chunk: int = 8, streams: int = 1, optimizer=None,
                 capacity: int = None, deterministic: bool = False):
        # capacity: the most Gaussians the per-view buffers must hold (a growing online
        # map passes its P_stride; default the model's current P)
        cap_p = int(capacity) if capacity is not None else model.P
        self.lib, self.model, self.cameras, self.targets = lib, model, cameras, targets
        self.device, self.w_depth, self.allreduce = device, w_depth, allreduce
        # optimizer: None = (allreduce +) replicated gs_adam_step; else an object whose
        # step() combines the gradient across ranks and updates the parameters
        # (ShardedAdam); it is called after the step counter is incremented
        self.optimizer = optimizer
        # views chained per gs_project_bwd_views pass: up to 64 (above 8 the wide kernels
        # chain them all in one pass: every parameter / gradient row touched once)
        self.chunk = max(1, min(64, int(chunk)))
        # views in flight: view k of a step runs on stream k % streams with its own
        # buffers, so that one view's latency-bound projection / binning kernels overlap
        # another view's rendering (the views of a batch are independent until the
        # projection backward sums them, R21)
        n_streams = max(1, int(streams))
        # bin-ahead (views in flight only): every view's projection + binning runs on
        # one of n = GSR_BIN_STREAMS (default 8) streams of the highest priority into its
        # own view buffer (a ring of streams + n buffers), ahead of the render streams,
        # which only wait for their view's lists; the binning kernels' CTAs are then
        # dispatched before pending render CTAs.  scannetpp: 6.30 -> 6.245 ms/step vs
        # each view's whole chain on its render stream (GSR_BIN_STREAMS=0); with 1-3
        # bin streams of normal priority it was 1-10% slower (their kernels wait behind
        # the render CTAs that fill the GPU).
        nb = os.environ.get("GSR_BIN_STREAMS")
        self.n_bin = (int(nb) if nb is not None else 8) if n_streams > 1 else 0
        n_bufs = n_streams + self.n_bin
        # deterministic: the backward's reduction in a fixed order (gs_bwd_opts.det_ws), so
        # an iteration's parameters are bit-reproducible whatever the streams / graphs
        self.deterministic = bool(deterministic)
        self.bufs = [ViewBuffers(lib, cameras[0], cap_p, key_capacity, device, deterministic=self.deterministic)
                     for _ in range(n_bufs)]
        self.buf = self.bufs[0]
        # (equal priorities: staggering the streams' priorities measured 4% slower)
        self._streams = [torch.cuda.Stream(device=device) for _ in range(n_streams)] if n_streams > 1 else None
        self._bin_streams = []
        if self.n_bin:
            bp = os.environ.get("GSR_BIN_PRIO")
            bp = int(bp) if bp is not None else torch.cuda.Stream.priority_range()[1]  # highest
            self._bin_streams = [torch.cuda.Stream(device=device, priority=bp) for _ in range(self.n_bin)]
        P = max(cap_p, 1)
        # per in-flight view: projection flags and screen-space gradients (zeroed once;
        # gs_project_bwd_views leaves them zero again).  Two slot sets when a step has
        # more views than one chain takes, so that chunk c + 1's views render while
        # chunk c's projection backward runs (they only wait for chunk c - 1's chain).
        n_sets = 2 if len(cameras) > self.chunk and n_streams > 1 else 1
        self.flags = [torch.empty(P + 16, dtype=torch.uint8, device=device) for _ in range(n_sets * self.chunk)]
        self.sgrad = [torch.zeros((P, gsr.SGRAD_FLOATS), dtype=torch.float32, device=device)
                      for _ in range(n_sets * self.chunk)]
        self._n_sets = n_sets
        self.num_keys = torch.zeros(len(cameras), dtype=torch.int64, device=device)
        self._adam_side = None  # side stream of gs_project_bwd_views_adam_dev (created on first use)
        self.blended = torch.zeros(1, dtype=torch.int64, device=device)
        self.loss = torch.zeros(1, dtype=torch.float32, device=device)
        self.hooks = None
        # K13 comparison baseline (bench.py only): per-pixel render kernels, no
        # block masks; projection, binning, projection backward and Adam unchanged
        self.naive = False
        # serial = True runs the views on the caller's stream only (bench.py's isolated
        # kernel-timing pass)
        self.serial = False
        # device_step = True: Adam reads / advances model.step_dev (graph capture)
        self.device_step = False
        # fuse_l1: the L1 upstream (Eq. 12) computed inside the backward kernel
        # (gs_render_bwd_screen_l1) instead of a gs_l1_loss_grad pass; GSR_FUSE_L1=0 for A/B
        self.fuse_l1 = os.environ.get("GSR_FUSE_L1", "1") != "0"
        # render tiles longest-list-first (gs_tile_order): 7% faster render kernels when
        # one view is in flight; with several views in flight the other streams already
        # fill each kernel's tail and the extra launch cost 2% (B200, scannetpp), so the
        # default is on for streams == 1 only.  GSR_TILE_ORDER=0/1 overrides.
        env = os.environ.get("GSR_TILE_ORDER")
        self.tile_order = (env != "0") if env is not None else n_streams == 1

    def _hook(self, stage, what):
        if self.hooks is not None:
            self.hooks(stage, what)

    def _view(self, v: int, slot: int, t_rgb, t_depth, targets_ready=None, targets_consumed=None, buf=None):
        b = buf if buf is not None else self.buf
        gcam, proj, order = self._bin_view(v, slot, b)
        self._render_view(v, slot, b, gcam, proj, order, t_rgb, t_depth, targets_ready, targets_consumed)
        return gcam

    def _bin_view(self, v: int, slot: int, b, projected=False):
        """gs_project (unless ``projected``: done by a batched gs_project_views) ->
        gs_bin_tiles (-> gs_tile_order) of view v into buffer b."""
        lib, m, cam = self.lib, self.model, self.cameras[v]
        gcam = gsr.camera(cam)
        proj = gsr.GsProj(b.proj.rec, b.proj.radius, b.proj.tiles, self.flags[slot].data_ptr())
        if not projected:
            self._hook("project", "begin")
            lib.project(gcam, m.desc, m.params, proj)
            self._hook("project", "end")
        self._hook("bin", "begin")
        lib.bin_tiles(gcam, m.desc, proj, b.bin_ws, b.key_capacity, b.sorted_ids, b.ranges,
                      num_keys_dev=self.num_keys[v:v + 1])
        order = None
        if self.tile_order and not self.naive:
            lib.tile_order(gcam, b.ranges, b.tile_order)
            order = b.tile_order
        self._hook("bin", "end")
        return gcam, proj, order

    def _project_chunk(self, views, k0, base, buf_ev, chain_ev):
        """Bin-ahead mode, at the first view of a chunk: gs_project_views of the chunk's
        views (the parameters read once instead of once per view) on the first bin
        stream, when none of their buffers or slots is still in use this step (else
        None: each view projects itself).  Returns the event the bins wait for."""
        n = min(self.chunk, len(views) - k0)
        bis = [(k0 + j) % len(self.bufs) for j in range(n)]
        if (os.environ.get("GSR_PROJECT_VIEWS", "1") == "0" or chain_ev is not None or len(set(bis)) < n
                or any(buf_ev[bi] is not None for bi in bis)):
            return None
        m = self.model
        cams = [gsr.camera(self.cameras[views[k0 + j]]) for j in range(n)]
        projs = [gsr.GsProj(self.bufs[bi].proj.rec, self.bufs[bi].proj.radius, self.bufs[bi].proj.tiles,
                            self.flags[base + j].data_ptr()) for j, bi in enumerate(bis)]
        bs = self._bin_streams[0]
        with torch.cuda.stream(bs):
            self._hook("project", "begin")
            self.lib.project_views(cams, m.desc, m.params, projs)
            self._hook("project", "end")
            ev = torch.cuda.Event()
            ev.record(bs)
        return ev

    def _render_view(self, v, slot, b, gcam, proj, order, t_rgb, t_depth, targets_ready, targets_consumed):
        """gs_render_fwd -> (L1) -> gs_render_bwd_screen of view v from buffer b."""
        lib, m = self.lib, self.model
        self._hook("render_fwd", "begin")
        if self.naive:
            lib.naive_render_fwd(gcam, m.desc, proj, b.sorted_ids, b.ranges, b.rgb, b.depth, b.T, b.n,
                                 blended=self.blended, fwd_state=b.fwd_state)
        else:
            lib.render_fwd(gcam, m.desc, proj, b.sorted_ids, b.ranges, b.rgb, b.depth, b.T, b.n,
                           blended=self.blended, key_blocks=b.key_blocks, tile_order=order, fwd_state=b.fwd_state)
        self._hook("render_fwd", "end")
        if targets_ready is not None:
            torch.cuda.current_stream().wait_event(targets_ready)
        if self.naive or not self.fuse_l1:
            lib.l1_loss_grad(b.rgb, b.depth, t_rgb, t_depth, self.w_depth, b.g_rgb, b.g_depth, loss=self.loss)
            if targets_consumed is not None:
                targets_consumed.record()
        self._hook("render_bwd", "begin")
        if self.naive:
            lib.naive_render_bwd_screen(gcam, m.desc, proj, b.sorted_ids, b.ranges, b.T, b.n, b.g_rgb, b.g_depth,
                                        self.sgrad[slot], fwd=b.fwd_state)
        elif self.fuse_l1:  # Eq. 12's upstream computed inside the backward (one kernel)
            lib.render_bwd_screen_l1(gcam, m.desc, proj, b.sorted_ids, b.ranges, b.T, b.n, b.rgb, b.depth, t_rgb,
                                     t_depth, self.w_depth, self.sgrad[slot], loss=self.loss, key_blocks=b.key_blocks,
                                     tile_order=order, fwd=b.fwd_state, det=b.det)
            if targets_consumed is not None:
                targets_consumed.record()
        else:
            lib.render_bwd_screen(gcam, m.desc, proj, b.sorted_ids, b.ranges, b.T, b.n, b.g_rgb, b.g_depth,
                                  self.sgrad[slot], key_blocks=b.key_blocks, tile_order=order, fwd=b.fwd_state,
                                  det=b.det)
        self._hook("render_bwd", "end")

    def autotune_render(self, views=None, reps=3):
        """Choose the render kernels' block-row walk (gs_set_render_rows; results are
        identical either way) for this scene: times gs_render_fwd + the backward of up
        to 4 views with each setting (best of ``reps``, CUDA events on the current
        stream) and keeps the faster (the row walk only if >= 1% faster: config 4
        measures ~5% faster, scannetpp ~3% slower).  Nothing is updated: the screen gradients, loss
        and blended counter the timing runs write are cleared.  Returns the setting."""
        lib, b = self.lib, self.buf
        views = list(views if views is not None else range(len(self.cameras)))[:4]
        stream = torch.cuda.current_stream()
        best = {}
        for mode in (0, 1):
            lib.set_render_rows(mode)
            t = []
            for _ in range(reps + 1):  # the first pass warms up
                ms = 0.0
                for v in views:
                    gcam, proj, order = self._bin_view(v, 0, b)
                    tr = (self.targets[v] if self.targets is not None and self.targets[v] is not None
                          else (b.rgb, b.depth))
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record(stream)
                    self._render_view(v, 0, b, gcam, proj, order, tr[0], tr[1], None, None)
                    e1.record(stream)
                    e1.synchronize()
                    ms += e0.elapsed_time(e1)
                t.append(ms)
            best[mode] = min(t[1:])
        self.sgrad[0].zero_()
        self.loss.zero_()
        self.blended.zero_()
        mode = 1 if best[1] < 0.99 * best[0] else 0  # the row walk only when clearly faster
        lib.set_render_rows(mode)
        self.render_tune = {"rows": mode, "ms_dense": best[0], "ms_rows": best[1], "views": views}
        torch.cuda.synchronize()
        return mode

    def step(self, views, targets_override=None):
        """One iteration over ``views``; targets_override: {v: (rgb, depth)} device tensors."""
        def targets(k, v):
            t = targets_override[v] if targets_override is not None else self.targets[v]
            return t[0], t[1], None, None
        self._run(views, targets, None)

    def step_host(self, views, host_targets, depth_scale=None):
        """One iteration with the targets streamed from (pinned) host memory:
        host_targets {v: (rgb, depth)} CPU tensors, either float32 rgb [3][H][W] + depth
        [H][W], or a sensor frame (R41): uint8 rgb [H][W][3] + 16-bit
        depth [H][W] in units of ``depth_scale`` metres, shipped as is (5 B/px instead
        of 16) and decoded on the device (gs_decode_rgbd) right after its copy.  View
        k's targets are copied on a side stream into device slot k % n (n = 2 x the
        views in flight, so every in-flight view has its slot and the next ones are
        already loading); the loss of view k waits for its copy only, and the copy into
        a slot waits until the loss that last read it has run.  The host enqueues ahead
        of the GPU, so the next iteration's first copies overlap this one's tail."""
        dev = self.device
        n_slots = max(2, 2 * (len(self._streams) if self._streams else 1))
        r0, d0 = host_targets[views[0]]
        sensor = r0.dtype == torch.uint8
        if sensor and depth_scale is None:
            raise ValueError("step_host: sensor frames (uint8 rgb) need depth_scale")
        if getattr(self, "_slots", None) is None or self._sensor != sensor:
            H, W = int(d0.shape[0]), int(d0.shape[1])
            self._slots = [(torch.empty((3, H, W), dtype=torch.float32, device=dev),
                            torch.empty((H, W), dtype=torch.float32, device=dev)) for _ in range(n_slots)]
            # sensor frames land in raw slots first (uint8 [H][W][3], 16-bit [H][W])
            self._raw = ([(torch.empty((H, W, 3), dtype=torch.uint8, device=dev),
                           torch.empty((H, W), dtype=d0.dtype, device=dev)) for _ in range(n_slots)]
                         if sensor else None)
            self._sensor = sensor
            n_cs = int(os.environ.get("GSR_COPY_STREAMS", "1"))  # 2-3 measured no faster
            self._copy_streams = [torch.cuda.Stream(device=dev) for _ in range(max(1, n_cs))]
            self._ready = [torch.cuda.Event() for _ in range(n_slots)]
            self._free = [torch.cuda.Event() for _ in range(n_slots)]
        n_slots = len(self._slots)

        def issue(k):
            s = k % n_slots
            cs = self._copy_streams[k % len(self._copy_streams)]  # copies alternate DMA queues
            with torch.cuda.stream(cs):
                cs.wait_event(self._free[s])
                r, d = host_targets[views[k]]
                if sensor:
                    self._raw[s][0].copy_(r, non_blocking=True)
                    self._raw[s][1].copy_(d, non_blocking=True)
                    self.lib.decode_rgbd(self._raw[s][0], self._raw[s][1], depth_scale, self._slots[s][0],
                                         self._slots[s][1])
                else:
                    self._slots[s][0].copy_(r, non_blocking=True)
                    self._slots[s][1].copy_(d, non_blocking=True)
                self._ready[s].record(cs)

        def targets(k, v):
            s = k % n_slots
            return self._slots[s][0], self._slots[s][1], self._ready[s], self._free[s]

        def after_view(k):
            if k + n_slots < len(views):
                issue(k + n_slots)

        for k in range(min(n_slots, len(views))):
            issue(k)
        self._run(views, targets, after_view)

    def _run(self, views, targets, after_view):
        m = self.model
        main = torch.cuda.current_stream()
        S = 1 if self.serial or self._streams is None else len(self._streams)
        if S > 1:  # side streams start after the previous step's Adam / chains
            start = torch.cuda.Event()
            start.record(main)
            for s in self._streams + self._bin_streams:
                s.wait_event(start)
        pending, done = [], []
        buf_ev = [None] * len(self.bufs)  # per view buffer: the render that last read it (this step)
        proj_ev = None  # bin-ahead: the batched projection of the current chunk (or None)
        n_sets = self._n_sets if S > 1 else 1
        chain_ev = [None] * n_sets  # per slot set: the chain that last consumed it
        first = True  # the first chain of an iteration overwrites grad (no zeroing pass needed)
        n_chain = 0
        # the last chain and Adam in one library call with the SH rows' update on a side
        # stream under the chain's geometry half (gs_project_bwd_views_adam_dev): the
        # single-GPU device-step (graph) path; GSR_ADAM_OVERLAP=0 for A/B
        fuse_tail = (self.optimizer is None and self.allreduce is None and self.device_step and S > 1
                     and os.environ.get("GSR_ADAM_OVERLAP", "1") != "0")
        # A/B: view k's binning waits for view k - lag's (0: all views bin concurrently)
        # and views >= 1 for view 0's when head is set (the first render starts sooner)
        bin_lag = int(os.environ.get("GSR_BIN_LAG", "0"))
        bin_head = os.environ.get("GSR_BIN_HEAD", "0") != "0"
        binned_evs = []
        for k, v in enumerate(views):
            t_rgb, t_depth, ready, consumed = targets(k, v)
            base = (n_chain % n_sets) * self.chunk  # slot set of the chunk being filled
            if S == 1:
                pending.append(self._view(v, base + len(pending), t_rgb, t_depth, ready, consumed))
            elif self.n_bin:  # bin-ahead: project + bin on a bin stream, render on a render stream
                slot, bi = base + len(pending), k % len(self.bufs)
                b, bs, s = self.bufs[bi], self._bin_streams[k % self.n_bin], self._streams[k % S]
                if not pending:  # a new chunk: project its views in one pass if nothing waits
                    proj_ev = self._project_chunk(views, k, base, buf_ev, chain_ev[n_chain % n_sets])
                if chain_ev[n_chain % n_sets] is not None:  # this slot was consumed by that chain
                    bs.wait_event(chain_ev[n_chain % n_sets])
                if buf_ev[bi] is not None:  # the buffer's previous view has been rendered
                    bs.wait_event(buf_ev[bi])
                if proj_ev is not None:
                    bs.wait_event(proj_ev)
                if bin_lag and k >= bin_lag:
                    bs.wait_event(binned_evs[k - bin_lag])
                if bin_head and k >= 1:
                    bs.wait_event(binned_evs[0])
                with torch.cuda.stream(bs):
                    gcam, proj, order = self._bin_view(v, slot, b, projected=proj_ev is not None)
                    binned = torch.cuda.Event()
                    binned.record(bs)
                binned_evs.append(binned)
                s.wait_event(binned)
                with torch.cuda.stream(s):
                    self._render_view(v, slot, b, gcam, proj, order, t_rgb, t_depth, ready, consumed)
                    ev = torch.cuda.Event()
                    ev.record(s)
                    done.append(ev)
                    buf_ev[bi] = ev
                pending.append(gcam)
            else:
                s = self._streams[k % S]
                if chain_ev[n_chain % n_sets] is not None:  # this slot was consumed by that chain
                    s.wait_event(chain_ev[n_chain % n_sets])
                with torch.cuda.stream(s):
                    pending.append(self._view(v, base + len(pending), t_rgb, t_depth, ready, consumed,
                                              self.bufs[k % S]))
                    ev = torch.cuda.Event()
                    ev.record(s)
                    done.append(ev)
            if after_view is not None:
                after_view(k)
            if len(pending) == self.chunk and not (fuse_tail and k == len(views) - 1):
                for ev in done:
                    main.wait_event(ev)
                done = []
                self._chain(pending, accumulate=not first, base=base)
                pending, first = [], False
                if S > 1:
                    ev = torch.cuda.Event()
                    ev.record(main)
                    chain_ev[n_chain % n_sets] = ev
                n_chain += 1
        for ev in done:
            main.wait_event(ev)
        if fuse_tail and pending:
            if self._adam_side is None:
                self._adam_side = torch.cuda.Stream(device=self.device)
            base, n = (n_chain % n_sets) * self.chunk, len(pending)
            self._hook("project_bwd", "begin")
            self.lib.project_bwd_views_adam_dev(pending, m.desc, m.params, self.flags[base:base + n],
                                                self.sgrad[base:base + n], m.grad, m.m, m.v, m.lr, m.step_dev,
                                                accumulate=not first, side_stream=self._adam_side)
            self._hook("project_bwd", "end")
            m.step_count += 1
            return
        if pending or first:
            self._chain(pending, accumulate=not first, base=(n_chain % n_sets) * self.chunk)
        m.step_count += 1
        if self.optimizer is not None:
            self.optimizer.step()
            return
        if self.allreduce is not None:
            self.allreduce(m.grad)
        if self.device_step:
            self.lib.adam_step_dev(m.desc, m.params, m.grad, m.m, m.v, m.lr, m.step_dev, zero_grad=False)
        else:
            self.lib.adam_step(m.desc, m.params, m.grad, m.m, m.v, m.lr, m.step_count, zero_grad=False)

    def capture(self, views, targets_override=None):
        """One whole iteration over ``views`` (every view's project -> bin -> fwd -> L1 ->
        bwd on its stream, the projection backward, Adam) captured in a CUDA graph
        (the launch-bound configs run as one graph per iteration).
        Binning runs in capacity mode (K stays on the device), Adam takes the step
        counter from the device.  Returns the graph; replay it with replay()."""
        if self.optimizer is not None and not hasattr(self.optimizer, "device_step"):
            raise ValueError("this optimiser cannot be graph-captured (its exchange size is read on the host)")
        m = self.model
        m.step_dev.fill_(m.step_count)
        self.device_step = True
        if self.optimizer is not None:
            self.optimizer.device_step = True
        hooks, self.hooks = self.hooks, None
        side = torch.cuda.Stream(device=self.device)
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            self.step(views, targets_override)  # one eager iteration on a side stream (lazy allocations)
        torch.cuda.current_stream().wait_stream(side)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            self.step(views, targets_override)
        m.step_count -= 1  # the captured iteration has not run yet
        self.hooks = hooks
        return g

    def replay(self, g):
        g.replay()
        self.model.step_count += 1

    def _chain(self, gcams, accumulate, base=0):
        n = len(gcams)
        self._hook("project_bwd", "begin")
        self.lib.project_bwd_views(gcams, self.model.desc, self.model.params, self.flags[base:base + n],
                                   self.sgrad[base:base + n], self.model.grad, accumulate=accumulate)
        if n and hasattr(self.optimizer, "note_views"):  # visibility-sparse exchange: this chunk's views
            self.optimizer.note_views(self.flags[base:base + n])
        self._hook("project_bwd", "end")

    def check_capacity(self) -> int:
        """Max K seen since construction (host sync); raises if any view overflowed."""
        k = int(self.num_keys.max().item())
        if k > self.buf.key_capacity:  # every view buffer has the same capacity
            raise gsr.GsError("gs_bin_tiles", gsr.GS_ERR_CAPACITY, f"K={k} > capacity {self.buf.key_capacity}")
        return k


def render_targets(lib, target_model: GaussianModel, cameras, device, key_capacity: int):
    """Target images per view, rendered through the same kernels (setup, untimed)."""
    buf = ViewBuffers(lib, cameras[0], target_model.P, key_capacity, device)
    out = []
    for cam in cameras:
        K = render(lib, target_model, cam, buf, sync_keys=True)
        if K > key_capacity:
            buf = ViewBuffers(lib, cam, target_model.P, int(K * 1.25), device)
            render(lib, target_model, cam, buf, sync_keys=True)
        out.append((buf.rgb.clone(), buf.depth.clone()))
    return out


def default_capacity(K: int) -> int:
    return int(math.ceil(K * 1.3)) + 4096



class HostStreamedGraphs:
    """Graph-replayed iterations over a fixed view set, fed sensor frames from pinned
    host memory (the end-to-end path of bench.py for the batched configs).  Two slot
    sets alternate by step parity; per parity one CUDA graph copies every view's frame
    (uint8 rgb [H][W][3] + 16-bit depth [H][W], R41) host -> device and
    decodes it (gs_decode_rgbd) on a copy stream, and one graph runs the whole
    iteration (Trainer.capture) reading that slot set.  Step i's compute waits only for
    its own copies; the copies of step i + 2 start as soon as step i has consumed its
    slots, so the frames' DMA runs under the previous step's rendering instead of ahead
    of it.  host_frames[p] = {view: (rgb_u8, depth_u16)} pinned CPU tensors for parity p."""

    def __init__(self, trainer, views, host_frames, depth_scale, copy_priority=None, graph_copies=False):
        lib, dev = trainer.lib, trainer.device
        self.trainer, self.views = trainer, list(views)
        r0, d0 = host_frames[0][self.views[0]]
        H, W = int(d0.shape[0]), int(d0.shape[1])
        # highest priority: the decode kernels between the copies must not queue behind the
        # render CTAs of the step they run under
        self.copy_stream = torch.cuda.Stream(device=dev, priority=(torch.cuda.Stream.priority_range()[1]
                                                                   if copy_priority is None else copy_priority))
        self.slots = [{v: (torch.empty((3, H, W), dtype=torch.float32, device=dev),
                           torch.empty((H, W), dtype=torch.float32, device=dev)) for v in self.views}
                      for _ in range(2)]
        self.raw = [{v: (torch.empty((H, W, 3), dtype=torch.uint8, device=dev),
                         torch.empty((H, W), dtype=d0.dtype, device=dev)) for v in self.views} for _ in range(2)]
        self.h2d_bytes = sum(host_frames[0][v][0].numel() * host_frames[0][v][0].element_size() +
                             host_frames[0][v][1].numel() * host_frames[0][v][1].element_size() for v in self.views)

        def copies(p):
            for v in self.views:
                r, d = host_frames[p][v]
                self.raw[p][v][0].copy_(r, non_blocking=True)
                self.raw[p][v][1].copy_(d, non_blocking=True)
                lib.decode_rgbd(self.raw[p][v][0], self.raw[p][v][1], depth_scale, self.slots[p][v][0],
                                self.slots[p][v][1])
        # the copies are issued eagerly by default (copy-engine DMA); graph_copies=True
        # captures them (measured slower for large frame volumes: config 4 moves 885 MB
        # per step)
        self._copies = copies
        self.copy_graphs = []
        cs = self.copy_stream
        cs.wait_stream(torch.cuda.current_stream())
        for p in range(2):
            with torch.cuda.stream(cs):
                copies(p)  # eager once: the slots hold valid targets for the capture below
            if graph_copies:
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=cs):
                    copies(p)
                self.copy_graphs.append(g)
        torch.cuda.current_stream().wait_stream(cs)
        # per parity its own loss accumulator (baked into that parity's graph) and pinned
        # host copy: the loss readback runs on its own stream and never holds the
        # compute stream behind the copy engine's frame transfers
        self.losses = [torch.zeros(1, dtype=torch.float32, device=dev) for _ in range(2)]
        self.loss_host = [torch.zeros(1, dtype=torch.float32).pin_memory() for _ in range(2)]
        self.readback_stream = torch.cuda.Stream(device=dev)
        saved_loss = trainer.loss
        self.compute_graphs = []
        for p in range(2):
            trainer.loss = self.losses[p]
            self.compute_graphs.append(trainer.capture(self.views, targets_override=self.slots[p]))
        trainer.loss = saved_loss
        self.copied = [torch.cuda.Event() for _ in range(2)]
        self.computed = [torch.cuda.Event() for _ in range(2)]
        self.read = [torch.cuda.Event() for _ in range(2)]
        self.i = 0
        for p in range(2):
            self._copy(p)

    def _copy(self, p):
        cs = self.copy_stream
        cs.wait_event(self.computed[p])  # the compute that last read slot set p
        with torch.cuda.stream(cs):
            if self.copy_graphs:
                self.copy_graphs[p].replay()
            else:
                self._copies(p)
        self.copied[p].record(cs)

    def step(self, prefetch=True):
        """One iteration: waits for its frames, replays the iteration, reads its loss back
        to the host (self.loss_host[parity], a separate stream), then (prefetch) launches
        the frame copies of the iteration after next into the slots it has just consumed.
        Returns the parity whose loss_host entry this step fills."""
        p = self.i % 2
        main = torch.cuda.current_stream()
        main.wait_event(self.copied[p])
        main.wait_event(self.read[p])  # the readback of two steps ago has taken this loss
        self.losses[p].zero_()
        self.trainer.replay(self.compute_graphs[p])
        self.computed[p].record(main)
        rb = self.readback_stream
        rb.wait_event(self.computed[p])
        with torch.cuda.stream(rb):
            self.loss_host[p].copy_(self.losses[p], non_blocking=True)
        self.read[p].record(rb)
        self.i += 1
        if prefetch:
            self._copy(p)
        return p


class KeyframeOptimizer:
    """GSFusion's keyframe-scheduled online optimisation (settings
    PAPER.md:174) on top of the built path: the plan comes from
    the library's host scheduler (gs_keyframe_schedule: keyframe if more than
    ``threshold`` new primitives, m / n iterations, (m - n) shuffled keyframes for
    non-keyframes, ``global_iters`` passes over the keyframe list after scanning) and
    every planned iteration is one fwd + bwd + Adam step of ``trainer`` on one view.
    ``new_prims`` is the per-frame count of newly initialised Gaussians (the output of
    the out-of-scope seeding stage; scenegen.new_primitive_counts stands in for it)."""

    def __init__(self, lib, trainer: Trainer, new_prims, threshold=50, m=5, n=3, global_iters=10,
                 store_all_frames=False, seed=0):
        self.trainer = trainer
        self.views, self.frames, self.is_keyframe = lib.keyframe_schedule(
            new_prims, threshold, m, n, global_iters, store_all_frames, seed)

    @property
    def n_online(self) -> int:
        return int((self.frames >= 0).sum())

    def run(self, on_iteration=None):
        """Executes the whole plan (asynchronously on the current stream).
        on_iteration(i, view, frame) is called before each iteration."""
        for i, (v, f) in enumerate(zip(self.views.tolist(), self.frames.tolist())):
            if on_iteration is not None:
                on_iteration(i, v, f)
            self.trainer.step([v])


class ShardedAdam:
    """The gradient exchange + optimiser step of the data-parallel path as
    reduce-scatter -> Adam on this rank's shard -> all-gather of the parameters
    (SURVEY.md §8(e) "equivalent alternative", §8(f) NEXT-2): the same wire bytes as
    the all-reduce, 1/world of the optimiser's HBM traffic per rank, parameters
    bit-identical on every rank (each scalar is updated by exactly one rank).

    The flattened [F][P_stride] arrays are cut into `world` shards of `shard` scalars
    (a multiple of 4); model.grad and model.params become views of zero-padded flat
    buffers of world x shard scalars so the collectives need no copies.
    adam_range(begin, end, grad_shard) applies the optimiser to scalars [begin, end)
    (default: the library's gs_adam_step_range on the model's device buffers)."""

    def __init__(self, lib, model: GaussianModel, group=None, adam_range=None):
        import torch.distributed as dist
        self.dist, self.group = dist, group
        self.world, self.rank = dist.get_world_size(group), dist.get_rank(group)
        self.model = model
        F, S = model.F, model.P_stride
        self.n = F * S
        self.shard = ((self.n + self.world - 1) // self.world + 3) // 4 * 4
        dev = model.params.device
        self.gpad = torch.zeros(self.world * self.shard, dtype=torch.float32, device=dev)
        self.ppad = torch.zeros(self.world * self.shard, dtype=torch.float32, device=dev)
        self.gpad[:self.n].copy_(model.grad.reshape(-1))
        self.ppad[:self.n].copy_(model.params.reshape(-1))
        model.grad = self.gpad[:self.n].view(F, S)
        model.params = self.ppad[:self.n].view(F, S)
        self.gshard = torch.empty(self.shard, dtype=torch.float32, device=dev)
        self.pshard = torch.empty(self.shard, dtype=torch.float32, device=dev)
        self.begin = min(self.rank * self.shard, self.n)
        self.end = min(self.begin + self.shard, self.n)
        self.nccl = dist.get_backend(group) == "nccl"
        # device_step: Adam reads / advances model.step_dev (CUDA-graph capture, Trainer.capture)
        self.device_step = False
        if adam_range is None:
            def adam_range(b, e, g):
                step = model.step_dev if self.device_step else model.step_count
                lib.adam_step_range(model.desc, model.params, g, model.m, model.v, model.lr, step, b, e)
        self.adam_range = adam_range

    def step(self):
        d = self.dist
        if self.nccl:
            d.reduce_scatter_tensor(self.gshard, self.gpad, op=d.ReduceOp.SUM, group=self.group)
        else:  # gloo (CPU tests): no reduce-scatter; all-reduce and keep this rank's shard
            d.all_reduce(self.gpad, op=d.ReduceOp.SUM, group=self.group)
            self.gshard.copy_(self.gpad[self.rank * self.shard:(self.rank + 1) * self.shard])
        if self.end > self.begin or self.device_step:  # (an empty range still advances step_dev)
            self.adam_range(self.begin, self.end, self.gshard)
        self.pshard.copy_(self.ppad[self.rank * self.shard:(self.rank + 1) * self.shard])
        if self.nccl:
            d.all_gather_into_tensor(self.ppad, self.pshard, group=self.group)
        else:
            parts = list(self.ppad.view(self.world, self.shard).unbind(0))
            d.all_gather(parts, self.pshard, group=self.group)


class SparseExchangeAdam:
    """Visibility-sparse gradient exchange + replicated Adam (SURVEY.md §8(f) NEXT-2,
    "union of visible masks, then compaction").  A Gaussian culled in
    every view of every rank has an exactly zero gradient on every rank (the first
    projection-backward chain of a step writes those columns as zeros), so only the
    columns of the union of the ranks' visible sets are summed across ranks:

      note_views(flags): visible |= the views' visible sets (gs_visibility_union; the
                         Trainer calls it after each projection-backward chain)
      step():            all-reduce MAX of the P-byte mask -> ordered compaction
                         (gs_compact_index; M = the union's size, read by the host) ->
                         gather the M gradient columns (gs_gather_columns) -> all-reduce
                         SUM of F x M floats -> scatter them back (gs_scatter_columns)
                         -> replicated Adam over every column (gs_adam_step; the
                         moments of unseen Gaussians decay as in the dense step).

    Every rank reduces the same packed array and runs the same Adam, so the parameters
    stay bit-identical across ranks.  ``ops`` replaces the device calls with the same
    signatures (the CPU gloo tests pass torch implementations).  Reading M costs one host
    sync per step (an NCCL collective's size is a host argument), so this optimiser runs
    eagerly and is never graph-captured; the default N > 1 exchanges (nvls, peer) are
    fixed-size and captured."""

    def __init__(self, lib, model: GaussianModel, group=None, ops=None):
        import torch.distributed as dist
        self.dist, self.group, self.lib, self.model = dist, group, lib, model
        dev = model.params.device
        S = model.P_stride
        self.visible = torch.zeros(S, dtype=torch.uint8, device=dev)
        self.idx = torch.zeros(S, dtype=torch.int32, device=dev)
        self.count = torch.zeros(1, dtype=torch.int64, device=dev)
        self.packed = torch.empty(model.F * S, dtype=torch.float32, device=dev)
        self.ops = ops if ops is not None else self._device_ops(lib)
        self.ws = torch.empty(max(1, self.ops["compact_workspace"](S)), dtype=torch.uint8, device=dev)
        self.last_M = None
        self._fresh = True  # the next note_views starts a new step's union

    def _device_ops(self, lib):
        m = self.model
        return {
            "union": lambda flags, P, vis, acc: lib.visibility_union(flags, P, vis, accumulate=acc),
            "compact_workspace": lib.compact_workspace,
            "compact": lambda vis, P, ws, idx, cnt: lib.compact_index(vis, P, ws, idx, cnt),
            "gather": lambda full, F, S, idx, M, packed: lib.gather_columns(full, F, S, idx, M, packed),
            "scatter": lambda packed, F, S, idx, M, full: lib.scatter_columns(packed, F, S, idx, M, full),
            "adam": lambda: lib.adam_step(m.desc, m.params, m.grad, m.m, m.v, m.lr, m.step_count, zero_grad=False),
        }

    def note_views(self, flags):
        self.ops["union"](list(flags), self.model.P, self.visible, not self._fresh)
        self._fresh = False

    def step(self):
        d, m, o = self.dist, self.model, self.ops
        P, F, S = m.P, m.F, m.P_stride
        if self._fresh:  # no view this step: nothing is visible
            self.visible.zero_()
        d.all_reduce(self.visible[:P], op=d.ReduceOp.MAX, group=self.group)
        o["compact"](self.visible, P, self.ws, self.idx, self.count)
        M = int(self.count.item())  # the collective's size
        packed = self.packed[:F * M].view(F, M)
        o["gather"](m.grad, F, S, self.idx, M, packed)
        d.all_reduce(packed, op=d.ReduceOp.SUM, group=self.group)
        o["scatter"](packed, F, S, self.idx, M, m.grad)
        o["adam"]()
        self.last_M = M
        self._fresh = True


class PeerShardedAdam:
    """ShardedAdam's reduce-scatter + Adam + all-gather fused into ONE kernel over peer
    memory (gs_adam_step_peers): the gradient and parameter
    buffers live in torch symmetric memory, so every rank maps every other rank's
    buffers; rank r pulls its shard of all gradients over NVLink, applies Adam and
    pushes the new parameters into every rank's buffer.  Two device-side barriers on
    the stream order it: gradients final before, parameters delivered after.  No
    NCCL call and no intermediate shard buffers on the step's path."""

    def __init__(self, lib, model: GaussianModel, group=None):
        import torch.distributed as dist
        import torch.distributed._symmetric_memory as symm
        self.lib, self.model = lib, model
        group = group if group is not None else dist.group.WORLD
        self.world, self.rank = dist.get_world_size(group), dist.get_rank(group)
        F, S = model.F, model.P_stride
        self.n = F * S
        self.shard = ((self.n + self.world - 1) // self.world + 3) // 4 * 4
        dev = model.params.device
        self.gbuf = symm.empty(self.world * self.shard, dtype=torch.float32, device=dev)
        self.pbuf = symm.empty(self.world * self.shard, dtype=torch.float32, device=dev)
        self.gbuf.zero_()
        self.pbuf.zero_()
        self.gbuf[:self.n].copy_(model.grad.reshape(-1))
        self.pbuf[:self.n].copy_(model.params.reshape(-1))
        self.hg = symm.rendezvous(self.gbuf, group)
        self.hp = symm.rendezvous(self.pbuf, group)
        self.gptrs = [int(p) for p in self.hg.buffer_ptrs]
        self.pptrs = [int(p) for p in self.hp.buffer_ptrs]
        model.grad = self.gbuf[:self.n].view(F, S)
        model.params = self.pbuf[:self.n].view(F, S)
        self.begin = min(self.rank * self.shard, self.n)
        self.end = min(self.begin + self.shard, self.n)
        torch.cuda.synchronize(dev)
        self.hg.barrier(channel=0)
        self.device_step = False  # True: the step counter is model.step_dev (graph capture)
        self._self_test()

    def _launch(self, lr, step):
        m = self.model
        self.lib.adam_step_peers(m.desc, self.world, self.rank, self.gptrs, self.pptrs, m.m, m.v, lr, step,
                                 self.begin, self.end)

    def step(self):
        m = self.model
        self.hg.barrier(channel=0)  # every rank's gradient is final
        self._launch(m.lr, m.step_dev if self.device_step else m.step_count)
        self.hp.barrier(channel=1)  # every rank's parameter stores have landed

    def _self_test(self):
        """One exchange of a known gradient before the first real step: rank r's whole
        gradient buffer holds r + 1, every learning rate is 0 (parameters unchanged), m
        starts at 0, so after the kernel m on this rank's shard must equal
        fp32(1 - beta1) x world (world + 1) / 2 exactly.  Catches a path that sums the
        wrong terms on a machine where it has never run (the cross-rank parameter check
        cannot: the owner of a shard writes it to every rank).  Raises RuntimeError on
        any rank's mismatch; state is restored either way."""
        import torch.distributed as dist
        m = self.model
        saved = (self.gbuf.clone(), m.m.clone(), m.v.clone())
        try:
            self.gbuf.fill_(float(self.rank + 1))
            m.m.zero_()
            m.v.zero_()
            torch.cuda.synchronize()
            self.hg.barrier(channel=0)
            self._launch([0.0] * len(m.lr), 1)
            self.hp.barrier(channel=1)
            torch.cuda.synchronize()
            f32 = torch.float32  # the kernel's fp32 ops: (1 - beta1) x g, g an exact small integer
            expect = ((torch.tensor(1.0, dtype=f32) - torch.tensor(0.9, dtype=f32)) *
                      torch.tensor(float(self.world * (self.world + 1) // 2), dtype=f32)).to(m.m.device)
            got = m.m.reshape(-1)[self.begin:self.end]
            ok = torch.tensor([1 if bool(torch.all(got == expect)) else 0], dtype=torch.int32, device=got.device)
            dist.all_reduce(ok, op=dist.ReduceOp.MIN)
        finally:
            self.gbuf.copy_(saved[0])
            m.m.copy_(saved[1])
            m.v.copy_(saved[2])
            torch.cuda.synchronize()
            self.hg.barrier(channel=0)
        if int(ok.item()) != 1:
            raise RuntimeError(f"{type(self).__name__}: exchange self-test failed (the summed gradient is wrong)")


class NvlsShardedAdam(PeerShardedAdam):
    """PeerShardedAdam with the NVSwitch doing the reduction and the broadcast
    (gs_adam_step_multimem): the gradient and parameter
    buffers' MULTICAST addresses come from torch symmetric memory; rank r's kernel
    load-reduces its shard of the summed gradient in the switch (one multimem.ld_reduce
    per 16 B instead of world P2P loads), updates it, and multicast-stores the new
    parameters to every rank (one multimem.st instead of world P2P stores).  Raises
    RuntimeError where multicast is unavailable (no NVSwitch multicast support, e.g.
    a single-GPU box) so that callers fall back to the peer / NCCL paths."""

    def __init__(self, lib, model: GaussianModel, group=None):
        super().__init__(lib, model, group)
        mcg, mcp = int(self.hg.multicast_ptr), int(self.hp.multicast_ptr)
        if not mcg or not mcp:
            raise RuntimeError("symmetric memory has no multicast address (NVLS unavailable)")
        self.mc_grad, self.mc_param = mcg, mcp
        self._self_test()  # again, now through the multicast kernel

    def _launch(self, lr, step):
        m = self.model
        if not hasattr(self, "mc_grad"):  # during the base class's construction: the P2P kernel
            return super()._launch(lr, step)
        self.lib.adam_step_multimem(m.desc, self.mc_grad, self.mc_param, self.pbuf, m.m, m.v, lr, step,
                                    self.begin, self.end)


def params_agree_across_ranks(model: GaussianModel, group=None) -> bool:
    """Runtime check of the data-parallel invariant: parameters bit-identical on every
    rank (a float64 checksum and a sampled-bits hash compared across ranks)."""
    import torch.distributed as dist
    p = model.params.reshape(-1)
    bits = p.view(torch.int32)[:: max(1, p.numel() // 65536)].to(torch.int64)
    sig = torch.stack([p.double().sum(), (bits * torch.arange(1, bits.numel() + 1, device=p.device)).sum().double()])
    allv = [torch.zeros_like(sig) for _ in range(dist.get_world_size(group))]
    dist.all_gather(allv, sig, group=group)
    return all(torch.equal(allv[0], x) for x in allv[1:])


class TsdfVolume:
    """Device buffers of the TSDF grid (NEXT-3, gs_tsdf_* calls): hash table of block
    Morton keys, block pool of 8^3 (tsdf, weight) voxels.  integrate_frame() is one
    frame of GSFusion's TSDF fusion: band allocation, then Eqs. 6-9."""

    def __init__(self, lib, device, block_cap: int, voxel_size=0.01, trunc=None, w_max=100.0, step=None,
                 origin=(1 << 20,) * 3):
        self.lib = lib
        self.block_cap = int(block_cap)
        table_cap = 1
        while table_cap < 2 * self.block_cap:
            table_cap *= 2
        self.keys = torch.empty(table_cap, dtype=torch.int64, device=device)
        self.slots = torch.empty(table_cap, dtype=torch.int32, device=device)
        self.pool_keys = torch.zeros(self.block_cap, dtype=torch.int64, device=device)
        self.tsdf = torch.empty((self.block_cap, 512), dtype=torch.float32, device=device)
        self.weight = torch.empty((self.block_cap, 512), dtype=torch.float32, device=device)
        self.num_blocks = torch.zeros(1, dtype=torch.int64, device=device)
        self.new_blocks = torch.zeros(1, dtype=torch.int64, device=device)
        self.updated = torch.zeros(1, dtype=torch.int64, device=device)
        self.vol = gsr.GsTsdfVolume(self.keys.data_ptr(), self.slots.data_ptr(), self.pool_keys.data_ptr(),
                                    self.tsdf.data_ptr(), self.weight.data_ptr(), table_cap, self.block_cap,
                                    self.num_blocks.data_ptr())
        self.prm = gsr.GsTsdfParams(float(voxel_size), float(trunc if trunc is not None else 6 * voxel_size),
                                    float(w_max), float(step if step is not None else voxel_size / 2),
                                    (gsr.C.c_int32 * 3)(*[int(x) for x in origin]))
        lib.tsdf_reset(self.vol)

    def integrate_frame(self, cam, depth):
        gcam = gsr.camera(cam)
        self.lib.tsdf_allocate(self.prm, self.vol, gcam, depth, self.new_blocks)
        self.lib.tsdf_integrate(self.prm, self.vol, gcam, depth, self.updated)

    def blocks(self):
        """(keys uint64 ascending, tsdf [n][512], weight [n][512]) on the host (sync)."""
        import numpy as np
        n = int(self.num_blocks.item())
        if n > self.block_cap:
            raise gsr.GsError("gs_tsdf_allocate", gsr.GS_ERR_CAPACITY, f"{n} blocks > capacity {self.block_cap}")
        keys = self.pool_keys[:n].cpu().numpy().view(np.uint64)
        order = np.argsort(keys)
        return keys[order], self.tsdf[:n].cpu().numpy()[order], self.weight[:n].cpu().numpy()[order]


def empty_model(capacity: int, sh_degree: int, device) -> GaussianModel:
    """A model with no Gaussians and room for `capacity` (the online map grows into it)."""
    import numpy as np

    class _S:
        pass
    sc = _S()
    S = (int(capacity) + 3) // 4 * 4
    sc.P, sc.sh_degree = 0, int(sh_degree)
    sc.params = np.zeros((11 + 3 * (sh_degree + 1) ** 2, S), np.float32)
    return GaussianModel(sc, device)


class Seeder:
    """NEXT-4: per frame, the contrast quadtree of the RGB image
    (gs_quadtree) and the weight-gated initialisation of new Gaussians at the leaves
    (gs_seed_gaussians, Eq. 10) against the TSDF grid fused with the same frame.
    seed_frame() appends to `model` and returns the number of new Gaussians (the
    keyframe signal of PAPER.md:149; one host sync)."""

    def __init__(self, lib, width: int, height: int, device, threshold=0.1, min_cell=4):
        self.lib, self.W, self.H = lib, int(width), int(height)
        self.threshold, self.min_cell = float(threshold), int(min_cell)
        self.ws = torch.empty(lib.quadtree_workspace(self.W, self.H, self.min_cell), dtype=torch.uint8, device=device)
        # worst case: a cell splits only while both sides exceed min_cell, so a leaf side
        # is at least ceil((min_cell + 1) / 2) pixels (gs_seed_gaussians reads every leaf
        # gs_quadtree counted, so the buffer must hold them all)
        side = (self.min_cell + 2) // 2
        cap = (self.W // side + 1) * (self.H // side + 1) + 16
        self.leaves = torch.empty((cap, 4), dtype=torch.int32, device=device)
        self.num_leaves = torch.zeros(1, dtype=torch.int64, device=device)
        self.num_new = torch.zeros(1, dtype=torch.int64, device=device)

    def leaves_of(self, rgb):
        self.lib.quadtree(self.W, self.H, rgb, self.threshold, self.min_cell, self.ws, self.leaves, self.num_leaves)

    def seed_frame(self, cam, depth, rgb, tsdf: "TsdfVolume", model: GaussianModel) -> int:
        self.leaves_of(rgb)
        self.lib.seed_gaussians(gsr.camera(cam), tsdf.prm, tsdf.vol, depth, rgb, self.leaves, self.num_leaves,
                                model.desc, model.params, self.num_new)
        n = int(self.num_new.item())
        n_fit = min(n, model.P_stride - model.P)
        model.P += n_fit
        model.desc = gsr.scene_desc(model.P, model.P_stride, model.sh_degree)
        return n


class OnlineMapper:
    """GSFusion's incremental mapping loop on the built GPU path, one
    RGB-D frame at a time:
      1. TSDF fusion of the depth frame (NEXT-3: band allocation + Eqs. 6-9);
      2. quadtree seeding of new Gaussians gated by the fused voxel weights (NEXT-4,
         Eq. 10) -- the number appended is the frame's keyframe signal;
      3. the keyframe strategy's iterations for this frame (NEXT-1: m on a keyframe, n +
         (m - n) shuffled keyframes otherwise), each one fwd + bwd + Adam step on one
         view with the colour L1 loss of Eq. 12 (w_depth = 0);
    and finish() runs the global passes over the keyframe list after the scan.  The
    plan of frame t is the host scheduler's plan of the prefix counts[0..t] (causal)."""

    def __init__(self, lib, cameras, device, capacity: int, sh_degree: int = 0, key_capacity: int = 8 << 20,
                 voxel_size=0.01, block_cap=1 << 20, threshold=0.1, min_cell=4, kf_threshold=50, m=5, n=3,
                 global_iters=10, store_all_frames=False, seed=0):
        self.lib, self.cameras, self.device = lib, cameras, device
        self.tsdf = TsdfVolume(lib, device, block_cap, voxel_size=voxel_size)
        c0 = cameras[0]
        self.seeder = Seeder(lib, c0.width, c0.height, device, threshold=threshold, min_cell=min_cell)
        self.model = empty_model(capacity, sh_degree, device)
        self.targets = [None] * len(cameras)
        self.trainer = Trainer(lib, self.model, cameras, self.targets, device, key_capacity, w_depth=0.0,
                               capacity=self.model.P_stride)
        self.kf = dict(threshold=kf_threshold, m=m, n=n, store_all_frames=store_all_frames, seed=seed)
        self.global_iters = global_iters
        self.counts = []
        self.iterations = 0

    def add_frame(self, t: int, rgb, depth):
        """Frame t (cameras[t]) with its colour [3][H][W] and depth [H][W] device images."""
        cam = self.cameras[t]
        self.targets[t] = (rgb, depth)
        self.tsdf.integrate_frame(cam, depth)
        n_new = self.seeder.seed_frame(cam, depth, rgb, self.tsdf, self.model)
        self.counts.append(n_new)
        views, frames, _ = self.lib.keyframe_schedule(self.counts, global_iters=0, **self.kf)
        if self.model.P > 0:
            for v in views[frames == t].tolist():
                self.trainer.step([v])
                self.iterations += 1
        return n_new

    def finish(self):
        views, frames, is_kf = self.lib.keyframe_schedule(self.counts, global_iters=self.global_iters, **self.kf)
        for v in views[frames < 0].tolist():
            self.trainer.step([v])
            self.iterations += 1
        return is_kf
