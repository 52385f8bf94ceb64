"""Thin ctypes binding of libgsr.so (include/gsr.h): argument marshalling only.

Every step of the hot path runs in the library's CUDA kernels; this module only
turns torch tensors into device pointers and the current torch stream into a
cudaStream_t.  There is no CPU fallback: if the library is missing or the call
fails, an exception is raised.
"""
from __future__ import annotations

import ctypes as C
import os

import torch

PKG = os.path.dirname(os.path.abspath(__file__))

GS_OK, GS_ERR_ARG, GS_ERR_ALIGN, GS_ERR_CAPACITY, GS_ERR_STATE, GS_ERR_EMPTY, GS_ERR_CUDA = 0, -1, -2, -3, -4, -5, -6
STATUS_NAMES = {0: "GS_OK", -1: "GS_ERR_ARG", -2: "GS_ERR_ALIGN", -3: "GS_ERR_CAPACITY", -4: "GS_ERR_STATE",
                -5: "GS_ERR_EMPTY", -6: "GS_ERR_CUDA"}
REC_FLOATS = 12
SGRAD_FLOATS = 12
TILE = 16
FLAG_CULLED = 128


class GsError(RuntimeError):
    def __init__(self, fn, status, msg):
        super().__init__(f"{fn} -> {STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


class GsCamera(C.Structure):
    _fields_ = [("width", C.c_int32), ("height", C.c_int32),
                ("fx", C.c_float), ("fy", C.c_float), ("cx", C.c_float), ("cy", C.c_float),
                ("R_cw", C.c_float * 9), ("t_cw", C.c_float * 3),
                ("z_near", C.c_float), ("bg", C.c_float * 3)]


class GsScene(C.Structure):
    _fields_ = [("P", C.c_int64), ("P_stride", C.c_int64), ("sh_degree", C.c_int32)]


class GsKfParams(C.Structure):
    _fields_ = [("threshold", C.c_int64), ("m", C.c_int32), ("n", C.c_int32), ("global_iters", C.c_int32),
                ("store_all_frames", C.c_int32), ("seed", C.c_uint64)]


class GsTsdfParams(C.Structure):
    _fields_ = [("voxel_size", C.c_float), ("trunc", C.c_float), ("w_max", C.c_float), ("step", C.c_float),
                ("origin", C.c_int32 * 3)]


class GsTsdfVolume(C.Structure):
    _fields_ = [("keys", C.c_void_p), ("slots", C.c_void_p), ("pool_keys", C.c_void_p), ("tsdf", C.c_void_p),
                ("weight", C.c_void_p), ("table_cap", C.c_int64), ("block_cap", C.c_int64),
                ("num_blocks", C.c_void_p)]


class GsProj(C.Structure):
    _fields_ = [("rec", C.c_void_p), ("radius", C.c_void_p), ("tiles", C.c_void_p), ("flags", C.c_void_p)]


class GsFwdState(C.Structure):
    """gs_fwd_state: written by gs_render_fwd, checked by the backward (GS_ERR_STATE)."""
    _fields_ = [("id", C.c_uint64), ("width", C.c_int32), ("height", C.c_int32), ("rec", C.c_void_p),
                ("sorted_ids", C.c_void_p), ("tile_ranges", C.c_void_p), ("rgb", C.c_void_p), ("depth", C.c_void_p),
                ("T_final", C.c_void_p), ("n_contrib", C.c_void_p), ("key_blocks", C.c_void_p)]


class GsBwdOpts(C.Structure):
    _fields_ = [("fwd", C.POINTER(GsFwdState)), ("det_ws", C.c_void_p), ("det_keys", C.c_int64)]


def bwd_opts(fwd=None, det=None):
    """gs_bwd_opts for the backward calls: fwd = a GsFwdState the forward filled,
    det = a float32 device tensor [keys][12] selecting the deterministic mode."""
    if fwd is None and det is None:
        return None
    o = GsBwdOpts()
    if fwd is not None:
        o.fwd = C.pointer(fwd)
    if det is not None:
        o.det_ws = det.data_ptr()
        o.det_keys = det.numel() // SGRAD_FLOATS
    return o


def _ref(x):
    return None if x is None else C.byref(x)


def camera(cam) -> GsCamera:
    """Marshal a scenegen.Camera (or any object with the same fields)."""
    g = GsCamera()
    g.width, g.height = int(cam.width), int(cam.height)
    g.fx, g.fy, g.cx, g.cy = float(cam.fx), float(cam.fy), float(cam.cx), float(cam.cy)
    R = [float(x) for x in list(getattr(cam.R_cw, "reshape", lambda n: cam.R_cw)(9))]
    t = [float(x) for x in list(cam.t_cw)]
    for i in range(9):
        g.R_cw[i] = R[i]
    for i in range(3):
        g.t_cw[i] = t[i]
        g.bg[i] = float(cam.bg[i])
    g.z_near = float(cam.z_near)
    return g


def scene_desc(P: int, P_stride: int, sh_degree: int) -> GsScene:
    return GsScene(int(P), int(P_stride), int(sh_degree))


def _ptr(t):
    if t is None:
        return None
    if isinstance(t, int):
        return t
    return C.c_void_p(t.data_ptr())


def _stream(stream=None):
    if stream is None:
        stream = torch.cuda.current_stream()
    return C.c_void_p(stream.cuda_stream)


class Library:
    """One loaded copy of libgsr (fast build) or libgsr_exact (GSR_EXACT_EXP)."""

    def __init__(self, path: str):
        if not os.path.exists(path):
            raise ImportError(f"{path} is missing: run __graft_entry__.build() (no CPU fallback exists)")
        self.path = path
        lib = C.CDLL(path)
        vp, i64, i32 = C.c_void_p, C.c_int64, C.c_int32
        lib.gs_version.restype = C.c_int
        lib.gs_last_error.restype = C.c_char_p
        lib.gs_launch_count.restype = i64
        lib.gs_exact_exp.restype = C.c_int
        lib.gs_set_render_rows.argtypes = [C.c_int]
        lib.gs_set_render_rows.restype = C.c_int
        lib.gs_render_rows.restype = C.c_int
        lib.gs_project.argtypes = [vp, vp, vp, GsProj, vp]
        lib.gs_bin_tiles_workspace.argtypes = [vp, i64, i64]
        lib.gs_bin_tiles_workspace.restype = C.c_size_t
        lib.gs_bin_tiles.argtypes = [vp, vp, GsProj, vp, C.c_size_t, i64, vp, vp, vp, vp, vp]
        lib.gs_render_fwd.argtypes = [vp, vp, GsProj, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp]
        lib.gs_render_bwd_workspace.argtypes = [vp]
        lib.gs_render_bwd_workspace.restype = C.c_size_t
        lib.gs_render_bwd.argtypes = [vp, vp, vp, GsProj, vp, vp, vp, vp, vp, vp, vp, vp, vp, C.c_size_t, vp, vp, vp]
        lib.gs_render_bwd_screen.argtypes = [vp, vp, GsProj, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp]
        lib.gs_tile_order.argtypes = [vp, vp, vp, vp]
        lib.gs_render_bwd_screen_l1.argtypes = [vp, vp, GsProj, vp, vp, vp, vp, vp, vp, vp, vp, vp, C.c_float, vp,
                                                vp, vp, vp, vp]
        lib.gs_naive_render_fwd.argtypes = [vp, vp, GsProj, vp, vp, vp, vp, vp, vp, vp, vp, vp]
        lib.gs_naive_render_bwd_screen.argtypes = [vp, vp, GsProj, vp, vp, vp, vp, vp, vp, vp, vp, vp]
        lib.gs_project_bwd_views.argtypes = [C.c_int, vp, vp, vp, vp, vp, vp, C.c_int, vp]
        lib.gs_project_bwd_views_adam_dev.argtypes = [C.c_int, vp, vp, vp, vp, vp, vp, C.c_int, vp, vp, vp,
                                                      C.c_float, C.c_float, C.c_float, vp, vp, vp]
        lib.gs_project_bwd_views_adam_dev.restype = i32
        lib.gs_adam_step.argtypes = [vp, vp, vp, vp, vp, vp, C.c_float, C.c_float, C.c_float, i64, C.c_int, vp]
        lib.gs_spatial_order_workspace.argtypes = [vp]
        lib.gs_spatial_order_workspace.restype = C.c_size_t
        lib.gs_spatial_order.argtypes = [vp, vp, vp, vp, vp, C.c_size_t, vp]
        lib.gs_l1_loss_grad.argtypes = [i64, vp, vp, vp, vp, C.c_float, vp, vp, vp, vp]
        lib.gs_adam_step_range.argtypes = [vp, vp, vp, vp, vp, vp, C.c_float, C.c_float, C.c_float, i64, i64, i64, vp]
        lib.gs_adam_step_peers.argtypes = [vp, C.c_int, C.c_int, vp, vp, vp, vp, vp, C.c_float, C.c_float, C.c_float,
                                           i64, i64, i64, vp]
        lib.gs_adam_step_dev.argtypes = [vp, vp, vp, vp, vp, vp, C.c_float, C.c_float, C.c_float, vp, C.c_int, vp]
        lib.gs_adam_step_multimem.argtypes = [vp, vp, vp, vp, vp, vp, vp, C.c_float, C.c_float, C.c_float, i64, vp,
                                              i64, i64, vp]
        lib.gs_adam_step_range_dev.argtypes = [vp, vp, vp, vp, vp, vp, C.c_float, C.c_float, C.c_float, vp, i64, i64,
                                               vp]
        lib.gs_adam_step_peers_dev.argtypes = [vp, C.c_int, C.c_int, vp, vp, vp, vp, vp, C.c_float, C.c_float,
                                               C.c_float, vp, i64, i64, vp]
        lib.gs_tsdf_reset.argtypes = [GsTsdfVolume, vp]
        lib.gs_tsdf_allocate.argtypes = [vp, GsTsdfVolume, vp, vp, vp, vp]
        lib.gs_tsdf_integrate.argtypes = [vp, GsTsdfVolume, vp, vp, vp, vp]
        lib.gs_quadtree_workspace.argtypes = [C.c_int32, C.c_int32, C.c_int32]
        lib.gs_quadtree_workspace.restype = C.c_size_t
        lib.gs_quadtree.argtypes = [C.c_int32, C.c_int32, vp, C.c_float, C.c_int32, vp, C.c_size_t, vp, i64, vp, vp]
        lib.gs_seed_gaussians.argtypes = [vp, vp, GsTsdfVolume, vp, vp, vp, vp, vp, vp, vp, vp]
        lib.gs_keyframe_schedule.argtypes = [vp, i64, vp, vp, vp, i64, vp, vp]
        lib.gs_decode_rgbd.argtypes = [C.c_int32, C.c_int32, vp, vp, C.c_float, vp, vp, vp]
        lib.gs_project_views.argtypes = [C.c_int, vp, vp, vp, vp, vp]
        lib.gs_visibility_union.argtypes = [C.c_int, vp, i64, C.c_int, vp, vp]
        lib.gs_compact_workspace.argtypes = [i64]
        lib.gs_compact_workspace.restype = C.c_size_t
        lib.gs_compact_index.argtypes = [vp, i64, vp, C.c_size_t, vp, vp, vp]
        lib.gs_gather_columns.argtypes = [vp, i64, i64, vp, i64, vp, vp]
        lib.gs_scatter_columns.argtypes = [vp, i64, i64, vp, i64, vp, vp]
        for fn in ("gs_project", "gs_bin_tiles", "gs_render_fwd", "gs_render_bwd", "gs_render_bwd_screen",  # noqa: E501
                   "gs_project_bwd_views", "gs_spatial_order", "gs_adam_step", "gs_l1_loss_grad",
                   "gs_naive_render_fwd", "gs_naive_render_bwd_screen", "gs_tile_order", "gs_render_bwd_screen_l1", "gs_keyframe_schedule", "gs_adam_step_range", "gs_adam_step_peers", "gs_adam_step_dev", "gs_adam_step_range_dev", "gs_adam_step_peers_dev", "gs_adam_step_multimem", "gs_tsdf_reset", "gs_tsdf_allocate",
                   "gs_tsdf_integrate", "gs_quadtree", "gs_seed_gaussians", "gs_decode_rgbd", "gs_visibility_union", "gs_compact_index",
                   "gs_gather_columns", "gs_scatter_columns", "gs_project_views"):
            getattr(lib, fn).restype = i32
        self.lib = lib
        self.exact = bool(lib.gs_exact_exp())

    # -- diagnostics ------------------------------------------------------
    def launch_count(self) -> int:
        return int(self.lib.gs_launch_count())

    # -- performance switch (results identical either way) -----------------
    def set_render_rows(self, enable: bool):
        return self._check("gs_set_render_rows", self.lib.gs_set_render_rows(1 if enable else 0))

    def render_rows(self) -> bool:
        return bool(self.lib.gs_render_rows())

    def last_error(self) -> str:
        return self.lib.gs_last_error().decode()

    def _check(self, fn, st, allow=()):
        if st != GS_OK and st not in allow:
            raise GsError(fn, st, self.last_error())
        return st

    # -- the five calls ----------------------------------------------------
    def project(self, cam: GsCamera, sc: GsScene, params, proj: GsProj, stream=None):
        return self._check("gs_project", self.lib.gs_project(C.byref(cam), C.byref(sc), _ptr(params), proj,
                                                             _stream(stream)))

    def project_views(self, cams, sc: GsScene, params, projs, stream=None):
        """cams: list of GsCamera; projs: list of GsProj (one per view)."""
        n = len(cams)
        cam_arr = (GsCamera * max(n, 1))(*cams)
        out_arr = (GsProj * max(n, 1))(*projs)
        return self._check("gs_project_views", self.lib.gs_project_views(n, cam_arr, C.byref(sc), _ptr(params),
                                                                         out_arr, _stream(stream)))

    def bin_tiles_workspace(self, cam: GsCamera, P: int, key_capacity: int) -> int:
        return int(self.lib.gs_bin_tiles_workspace(C.byref(cam), int(P), int(key_capacity)))

    def bin_tiles(self, cam, sc, proj, ws, key_capacity, sorted_ids, tile_ranges, num_keys_dev=None, sync=False,
                  stream=None, allow_capacity=False):
        k_host = C.c_int64(-1)
        st = self.lib.gs_bin_tiles(C.byref(cam), C.byref(sc), proj, _ptr(ws), ws.numel() * ws.element_size(),
                                   int(key_capacity), _ptr(sorted_ids), _ptr(tile_ranges), _ptr(num_keys_dev),
                                   C.byref(k_host) if sync else None, _stream(stream))
        self._check("gs_bin_tiles", st, allow=(GS_ERR_CAPACITY,) if allow_capacity else ())
        return (int(k_host.value) if sync else None), st

    def tile_order(self, cam, tile_ranges, tile_order, stream=None):
        return self._check("gs_tile_order", self.lib.gs_tile_order(C.byref(cam), _ptr(tile_ranges), _ptr(tile_order),
                                                                   _stream(stream)))

    def render_fwd(self, cam, sc, proj, sorted_ids, tile_ranges, rgb, depth, T_final, n_contrib, blended=None,
                   key_blocks=None, stream=None, tile_order=None, fwd_state=None):
        """fwd_state: optional GsFwdState (host) the call fills for the backward's check."""
        return self._check("gs_render_fwd", self.lib.gs_render_fwd(
            C.byref(cam), C.byref(sc), proj, _ptr(sorted_ids), _ptr(tile_ranges), _ptr(tile_order), _ptr(rgb),
            _ptr(depth),
            _ptr(T_final), _ptr(n_contrib), _ptr(blended), _ptr(key_blocks), _ref(fwd_state), _stream(stream)))

    def render_bwd_workspace(self, sc: GsScene) -> int:
        return int(self.lib.gs_render_bwd_workspace(C.byref(sc)))

    def render_bwd(self, cam, sc, params, proj, sorted_ids, tile_ranges, T_final, n_contrib, dL_drgb, dL_ddepth, ws,
                   grad, key_blocks=None, stream=None, tile_order=None, fwd=None, det=None):
        return self._check("gs_render_bwd", self.lib.gs_render_bwd(
            C.byref(cam), C.byref(sc), _ptr(params), proj, _ptr(sorted_ids), _ptr(tile_ranges), _ptr(tile_order),
            _ptr(T_final),
            _ptr(n_contrib), _ptr(dL_drgb), _ptr(dL_ddepth), _ptr(key_blocks), _ptr(ws),
            ws.numel() * ws.element_size(), _ptr(grad), _ref(bwd_opts(fwd, det)), _stream(stream)))

    def render_bwd_screen(self, cam, sc, proj, sorted_ids, tile_ranges, T_final, n_contrib, dL_drgb, dL_ddepth, sgrad,
                          key_blocks=None, stream=None, tile_order=None, fwd=None, det=None):
        return self._check("gs_render_bwd_screen", self.lib.gs_render_bwd_screen(
            C.byref(cam), C.byref(sc), proj, _ptr(sorted_ids), _ptr(tile_ranges), _ptr(tile_order), _ptr(T_final),
            _ptr(n_contrib),
            _ptr(dL_drgb), _ptr(dL_ddepth), _ptr(key_blocks), _ptr(sgrad), _ref(bwd_opts(fwd, det)),
            _stream(stream)))

    # -- K13 comparison baseline (per-pixel port; not the product path) ---
    def naive_render_fwd(self, cam, sc, proj, sorted_ids, tile_ranges, rgb, depth, T_final, n_contrib, blended=None,
                         stream=None, fwd_state=None):
        return self._check("gs_naive_render_fwd", self.lib.gs_naive_render_fwd(
            C.byref(cam), C.byref(sc), proj, _ptr(sorted_ids), _ptr(tile_ranges), _ptr(rgb), _ptr(depth),
            _ptr(T_final), _ptr(n_contrib), _ptr(blended), _ref(fwd_state), _stream(stream)))

    def naive_render_bwd_screen(self, cam, sc, proj, sorted_ids, tile_ranges, T_final, n_contrib, dL_drgb, dL_ddepth,
                                sgrad, stream=None, fwd=None, det=None):
        return self._check("gs_naive_render_bwd_screen", self.lib.gs_naive_render_bwd_screen(
            C.byref(cam), C.byref(sc), proj, _ptr(sorted_ids), _ptr(tile_ranges), _ptr(T_final), _ptr(n_contrib),
            _ptr(dL_drgb), _ptr(dL_ddepth), _ptr(sgrad), _ref(bwd_opts(fwd, det)), _stream(stream)))

    def render_bwd_screen_l1(self, cam, sc, proj, sorted_ids, tile_ranges, T_final, n_contrib, rgb, depth, t_rgb,
                             t_depth, w_depth, sgrad, loss=None, key_blocks=None, stream=None, tile_order=None,
                             fwd=None, det=None):
        return self._check("gs_render_bwd_screen_l1", self.lib.gs_render_bwd_screen_l1(
            C.byref(cam), C.byref(sc), proj, _ptr(sorted_ids), _ptr(tile_ranges), _ptr(tile_order), _ptr(T_final),
            _ptr(n_contrib), _ptr(rgb), _ptr(depth), _ptr(t_rgb), _ptr(t_depth), float(w_depth), _ptr(loss),
            _ptr(key_blocks), _ptr(sgrad), _ref(bwd_opts(fwd, det)), _stream(stream)))

    def project_bwd_views(self, cams, sc, params, flags, sgrads, grad, accumulate=True, stream=None):
        """cams: list of GsCamera; flags / sgrads: lists of device tensors (one per view)."""
        n = len(cams)
        cam_arr = (GsCamera * max(n, 1))(*cams)
        fl = (C.c_void_p * max(n, 1))(*[t.data_ptr() for t in flags])
        sg = (C.c_void_p * max(n, 1))(*[t.data_ptr() for t in sgrads])
        return self._check("gs_project_bwd_views", self.lib.gs_project_bwd_views(
            n, cam_arr, C.byref(sc), _ptr(params), fl, sg, _ptr(grad), 1 if accumulate else 0, _stream(stream)))

    def project_bwd_views_adam_dev(self, cams, sc, params, flags, sgrads, grad, m, v, lr_per_row, step_dev,
                                   accumulate=False, side_stream=None, beta1=0.9, beta2=0.999, eps=1e-15,
                                   stream=None):
        """gs_project_bwd_views + gs_adam_step_dev with the SH rows' update on side_stream
        (torch stream, None: no split) under the chain's geometry half."""
        n = len(cams)
        cam_arr = (GsCamera * max(n, 1))(*cams)
        fl = (C.c_void_p * max(n, 1))(*[t.data_ptr() for t in flags])
        sg = (C.c_void_p * max(n, 1))(*[t.data_ptr() for t in sgrads])
        lr = (C.c_float * len(lr_per_row))(*[float(x) for x in lr_per_row])
        side = C.c_void_p(side_stream.cuda_stream) if side_stream is not None else C.c_void_p(0)
        return self._check("gs_project_bwd_views_adam_dev", self.lib.gs_project_bwd_views_adam_dev(
            n, cam_arr, C.byref(sc), _ptr(params), fl, sg, _ptr(grad), 1 if accumulate else 0, _ptr(m), _ptr(v), lr,
            beta1, beta2, eps, _ptr(step_dev), _stream(stream), side))

    # -- visibility-sparse exchange (NEXT-2) -------------------------------
    def visibility_union(self, flags, P, visible, accumulate=False, stream=None):
        """flags: list of device uint8 tensors (gs_project flags); visible: uint8[P]."""
        n = len(flags)
        fl = (C.c_void_p * max(n, 1))(*[t.data_ptr() for t in flags])
        return self._check("gs_visibility_union", self.lib.gs_visibility_union(
            n, fl, int(P), 1 if accumulate else 0, _ptr(visible), _stream(stream)))

    def compact_workspace(self, P) -> int:
        return int(self.lib.gs_compact_workspace(int(P)))

    def compact_index(self, visible, P, ws, idx, count, stream=None):
        return self._check("gs_compact_index", self.lib.gs_compact_index(
            _ptr(visible), int(P), _ptr(ws), ws.numel() * ws.element_size(), _ptr(idx), _ptr(count), _stream(stream)))

    def gather_columns(self, full, F, S, idx, M, packed, stream=None):
        return self._check("gs_gather_columns", self.lib.gs_gather_columns(
            _ptr(full), int(F), int(S), _ptr(idx), int(M), _ptr(packed), _stream(stream)))

    def scatter_columns(self, packed, F, S, idx, M, full, stream=None):
        return self._check("gs_scatter_columns", self.lib.gs_scatter_columns(
            _ptr(packed), int(F), int(S), _ptr(idx), int(M), _ptr(full), _stream(stream)))

    def spatial_order(self, sc, params_in, params_out, perm=None, stream=None):
        ws = torch.empty(max(int(self.lib.gs_spatial_order_workspace(C.byref(sc))), 16), dtype=torch.uint8,
                         device=params_in.device)
        return self._check("gs_spatial_order", self.lib.gs_spatial_order(
            C.byref(sc), _ptr(params_in), _ptr(params_out), _ptr(perm), _ptr(ws), ws.numel(), _stream(stream)))

    def adam_step(self, sc, params, grad, m, v, lr_per_row, step, beta1=0.9, beta2=0.999, eps=1e-15, zero_grad=True,
                  stream=None):
        lr = (C.c_float * len(lr_per_row))(*[float(x) for x in lr_per_row])
        return self._check("gs_adam_step", self.lib.gs_adam_step(
            C.byref(sc), _ptr(params), _ptr(grad), _ptr(m), _ptr(v), lr, beta1, beta2, eps, int(step),
            1 if zero_grad else 0, _stream(stream)))

    def adam_step_dev(self, sc, params, grad, m, v, lr_per_row, step_dev, beta1=0.9, beta2=0.999, eps=1e-15,
                      zero_grad=False, stream=None):
        lr = (C.c_float * len(lr_per_row))(*[float(x) for x in lr_per_row])
        return self._check("gs_adam_step_dev", self.lib.gs_adam_step_dev(
            C.byref(sc), _ptr(params), _ptr(grad), _ptr(m), _ptr(v), lr, beta1, beta2, eps, _ptr(step_dev),
            1 if zero_grad else 0, _stream(stream)))

    def adam_step_range(self, sc, params, grad_range, m, v, lr_per_row, step, begin, end, beta1=0.9, beta2=0.999,
                        eps=1e-15, stream=None):
        """step: an int (host step counter) or an int64 device tensor (gs_adam_step_range_dev)."""
        lr = (C.c_float * len(lr_per_row))(*[float(x) for x in lr_per_row])
        if isinstance(step, torch.Tensor):
            return self._check("gs_adam_step_range_dev", self.lib.gs_adam_step_range_dev(
                C.byref(sc), _ptr(params), _ptr(grad_range), _ptr(m), _ptr(v), lr, beta1, beta2, eps, _ptr(step),
                int(begin), int(end), _stream(stream)))
        return self._check("gs_adam_step_range", self.lib.gs_adam_step_range(
            C.byref(sc), _ptr(params), _ptr(grad_range), _ptr(m), _ptr(v), lr, beta1, beta2, eps, int(step),
            int(begin), int(end), _stream(stream)))

    def adam_step_peers(self, sc, world, rank, grad_ptrs, param_ptrs, m, v, lr_per_row, step, begin, end, beta1=0.9,
                        beta2=0.999, eps=1e-15, stream=None):
        """grad_ptrs / param_ptrs: lists of `world` device addresses (ints); step: an int or
        an int64 device tensor (gs_adam_step_peers_dev)."""
        lr = (C.c_float * len(lr_per_row))(*[float(x) for x in lr_per_row])
        gp = (C.c_void_p * max(world, 1))(*grad_ptrs)
        pp = (C.c_void_p * max(world, 1))(*param_ptrs)
        if isinstance(step, torch.Tensor):
            return self._check("gs_adam_step_peers_dev", self.lib.gs_adam_step_peers_dev(
                C.byref(sc), int(world), int(rank), gp, pp, _ptr(m), _ptr(v), lr, beta1, beta2, eps, _ptr(step),
                int(begin), int(end), _stream(stream)))
        return self._check("gs_adam_step_peers", self.lib.gs_adam_step_peers(
            C.byref(sc), int(world), int(rank), gp, pp, _ptr(m), _ptr(v), lr, beta1, beta2, eps, int(step), int(begin),
            int(end), _stream(stream)))

    def adam_step_multimem(self, sc, mc_grad, mc_param, param, m, v, lr_per_row, step, begin, end, beta1=0.9,
                           beta2=0.999, eps=1e-15, stream=None):
        """NVLS variant: mc_grad / mc_param multicast device addresses (ints); step: int or
        int64 device tensor."""
        lr = (C.c_float * len(lr_per_row))(*[float(x) for x in lr_per_row])
        dev_step = isinstance(step, torch.Tensor)
        return self._check("gs_adam_step_multimem", self.lib.gs_adam_step_multimem(
            C.byref(sc), C.c_void_p(int(mc_grad)), C.c_void_p(int(mc_param)), _ptr(param), _ptr(m), _ptr(v), lr, beta1,
            beta2, eps, 0 if dev_step else int(step), _ptr(step) if dev_step else None, int(begin), int(end),
            _stream(stream)))

    # -- NEXT-3: TSDF fusion ---------------------------------------------
    def tsdf_reset(self, vol, stream=None):
        return self._check("gs_tsdf_reset", self.lib.gs_tsdf_reset(vol, _stream(stream)))

    def tsdf_allocate(self, prm, vol, cam, depth, new_blocks=None, stream=None):
        return self._check("gs_tsdf_allocate", self.lib.gs_tsdf_allocate(
            C.byref(prm), vol, C.byref(cam), _ptr(depth), _ptr(new_blocks), _stream(stream)))

    def tsdf_integrate(self, prm, vol, cam, depth, updated=None, stream=None):
        return self._check("gs_tsdf_integrate", self.lib.gs_tsdf_integrate(
            C.byref(prm), vol, C.byref(cam), _ptr(depth), _ptr(updated), _stream(stream)))

    # -- NEXT-4: quadtree seeding ------------------------------------------
    def quadtree_workspace(self, width, height, min_cell) -> int:
        return int(self.lib.gs_quadtree_workspace(int(width), int(height), int(min_cell)))

    def quadtree(self, width, height, rgb, threshold, min_cell, ws, leaves, num_leaves, stream=None):
        return self._check("gs_quadtree", self.lib.gs_quadtree(
            int(width), int(height), _ptr(rgb), float(threshold), int(min_cell), _ptr(ws), ws.numel() * ws.element_size(),
            _ptr(leaves), leaves.shape[0], _ptr(num_leaves), _stream(stream)))

    def seed_gaussians(self, cam, prm, vol, depth, rgb, leaves, num_leaves, sc, params, num_new, stream=None):
        return self._check("gs_seed_gaussians", self.lib.gs_seed_gaussians(
            C.byref(cam), C.byref(prm), vol, _ptr(depth), _ptr(rgb), _ptr(leaves), _ptr(num_leaves), C.byref(sc),
            _ptr(params), _ptr(num_new), _stream(stream)))

    def keyframe_schedule(self, new_prims, threshold=50, m=5, n=3, global_iters=10, store_all_frames=False, seed=0):
        """gs_keyframe_schedule (host): returns (iter_view, iter_frame, is_keyframe) numpy arrays."""
        import numpy as np
        prm = GsKfParams(int(threshold), int(m), int(n), int(global_iters), 1 if store_all_frames else 0, int(seed))
        counts = np.ascontiguousarray(new_prims, dtype=np.int64)
        T = counts.shape[0]
        kf = np.zeros(max(T, 1), np.uint8)
        need = C.c_int64(0)
        cp = counts.ctypes.data_as(C.c_void_p)
        st = self.lib.gs_keyframe_schedule(C.byref(prm), T, cp, None, None, 0, C.byref(need), kf.ctypes.data_as(C.c_void_p))
        if st not in (GS_OK, GS_ERR_CAPACITY):
            raise GsError("gs_keyframe_schedule", st, "invalid parameters")
        views = np.zeros(max(need.value, 1), np.int32)
        frames = np.zeros(max(need.value, 1), np.int32)
        self._check("gs_keyframe_schedule", self.lib.gs_keyframe_schedule(
            C.byref(prm), T, cp, views.ctypes.data_as(C.c_void_p), frames.ctypes.data_as(C.c_void_p), need.value,
            C.byref(need), kf.ctypes.data_as(C.c_void_p)))
        return views[:need.value], frames[:need.value], kf[:T].astype(bool)

    def l1_loss_grad(self, rgb, depth, t_rgb, t_depth, w_depth, g_rgb, g_depth, loss=None, stream=None):
        return self._check("gs_l1_loss_grad", self.lib.gs_l1_loss_grad(
            int(depth.numel()), _ptr(rgb), _ptr(depth), _ptr(t_rgb), _ptr(t_depth), float(w_depth), _ptr(g_rgb),
            _ptr(g_depth), _ptr(loss), _stream(stream)))

    def decode_rgbd(self, rgb_u8, depth_u16, depth_scale, out_rgb, out_depth, stream=None):
        """Sensor frame (uint8 [H][W][3], uint16 [H][W] -- or int16 holding the same bits)
        -> float [3][H][W] rgb / 255 and [H][W] depth x depth_scale (gs_decode_rgbd)."""
        H, W = int(depth_u16.shape[0]), int(depth_u16.shape[1])
        if tuple(rgb_u8.shape) != (H, W, 3) or rgb_u8.element_size() != 1 or depth_u16.element_size() != 2:
            raise ValueError("decode_rgbd: rgb must be uint8 [H][W][3] and depth 16-bit [H][W]")
        return self._check("gs_decode_rgbd", self.lib.gs_decode_rgbd(
            W, H, _ptr(rgb_u8), _ptr(depth_u16), float(depth_scale), _ptr(out_rgb), _ptr(out_depth),
            _stream(stream)))


_LIBS = {}


def load(exact: bool = False) -> Library:
    # GSR_LIB selects an in-tree build variant of the fast library (A/B experiments,
    # e.g. libgsr_w20.so from tools/build_variant.py); default libgsr.so
    name = "libgsr_exact.so" if exact else os.environ.get("GSR_LIB", "libgsr.so")
    if name not in _LIBS:
        _LIBS[name] = Library(os.path.join(PKG, name))
    return _LIBS[name]


def make_proj(P: int, device) -> tuple:
    """Allocate projection buffers for P Gaussians; returns (GsProj, dict of tensors)."""
    t = {
        "rec": torch.empty((max(P, 1), REC_FLOATS), dtype=torch.float32, device=device),
        "radius": torch.empty(max(P, 1), dtype=torch.int32, device=device),
        "tiles": torch.empty(max(P, 1), dtype=torch.int32, device=device),
        "flags": torch.empty(max(P, 1) + 16, dtype=torch.uint8, device=device),
    }
    proj = GsProj(t["rec"].data_ptr(), t["radius"].data_ptr(), t["tiles"].data_ptr(), t["flags"].data_ptr())
    proj._tensors = t  # the struct holds raw pointers: keep the storage alive as long as the struct
    return proj, t
