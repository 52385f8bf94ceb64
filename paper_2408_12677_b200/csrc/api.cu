// C-ABI entry points of libgsr.so (include/gsr.h): host-side argument validation,
// camera marshalling and kernel dispatch.  No device memory is allocated here.
#include <atomic>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <unordered_map>
#include <vector>

#include "gsr_internal.cuh"

namespace gsr {

namespace {
thread_local char g_err[512] = "";
std::atomic<long long> g_launches{0};
int g_sms[64] = {0};
}  // namespace

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

gs_status check_launch(const char* what) {
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("%s: %s", what, cudaGetErrorString(e));
    return GS_ERR_CUDA;
  }
  return GS_OK;
}

void count_launch(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

int sm_count() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
  if (g_sms[dev] == 0) {
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    g_sms[dev] = n > 0 ? n : 148;
  }
  return g_sms[dev];
}

DevCam make_devcam(const gs_camera& c) {
  DevCam d{};
  d.W = c.width, d.H = c.height;
  d.TX = (c.width + kTile - 1) / kTile;
  d.TY = (c.height + kTile - 1) / kTile;
  d.fx = c.fx, d.fy = c.fy, d.cx = c.cx, d.cy = c.cy;
  for (int i = 0; i < 9; ++i) d.R[i] = c.R_cw[i];
  for (int i = 0; i < 3; ++i) d.t[i] = c.t_cw[i], d.bg[i] = c.bg[i];
  d.z_near = c.z_near;
  // R7's tangent clamps, per camera instead of per Gaussian: the fixed fp32 order of
  // O5 (1.3 * (W / (2 fx))), each operation rounded (host SSE float arithmetic)
  {
    volatile float two_fx = 2.f * c.fx, two_fy = 2.f * c.fy;
    volatile float qx = (float)c.width / two_fx, qy = (float)c.height / two_fy;
    d.limx = 1.3f * qx;
    d.limy = 1.3f * qy;
  }
  for (int j = 0; j < 3; ++j) {  // camera centre -R^T t
    double acc = 0.0;
    for (int i = 0; i < 3; ++i) acc += (double)c.R_cw[3 * i + j] * (double)c.t_cw[i];
    d.ocam[j] = (float)(-acc);
  }
  return d;
}

}  // namespace gsr

using namespace gsr;

namespace {

gs_status check_camera(const gs_camera* cam, const char* fn) {
  if (!cam) {
    set_error("%s: camera is NULL", fn);
    return GS_ERR_ARG;
  }
  if (cam->width <= 0 || cam->height <= 0 || !(cam->fx > 0.f) || !(cam->fy > 0.f) || !std::isfinite(cam->cx) ||
      !std::isfinite(cam->cy) || !(cam->z_near >= 0.f)) {
    set_error("%s: invalid camera (width=%d height=%d fx=%g fy=%g z_near=%g)", fn, cam->width, cam->height,
              (double)cam->fx, (double)cam->fy, (double)cam->z_near);
    return GS_ERR_ARG;
  }
  const long long nt = (long long)((cam->width + kTile - 1) / kTile) * ((cam->height + kTile - 1) / kTile);
  if (nt > GS_MAX_TILES) {
    set_error("%s: %lld tiles exceed GS_MAX_TILES (%d)", fn, nt, GS_MAX_TILES);
    return GS_ERR_ARG;
  }
  return GS_OK;
}

gs_status check_scene(const gs_scene* sc, const char* fn) {
  if (!sc) {
    set_error("%s: scene is NULL", fn);
    return GS_ERR_ARG;
  }
  if (sc->P < 0 || sc->P_stride < sc->P || sc->sh_degree < 0 || sc->sh_degree > GS_MAX_SH_DEGREE ||
      sc->P >= (1ll << 31)) {
    set_error("%s: invalid scene (P=%lld P_stride=%lld sh_degree=%d)", fn, (long long)sc->P, (long long)sc->P_stride,
              sc->sh_degree);
    return GS_ERR_ARG;
  }
  if (sc->P_stride % 4 != 0) {
    set_error("%s: P_stride=%lld is not a multiple of 4", fn, (long long)sc->P_stride);
    return GS_ERR_ALIGN;
  }
  return GS_OK;
}

gs_status check_ptrs(const char* fn, std::initializer_list<std::pair<const void*, const char*>> ptrs) {
  for (const auto& p : ptrs) {
    if (!p.first) {
      set_error("%s: %s is NULL", fn, p.second);
      return GS_ERR_ARG;
    }
    if (!aligned16(p.first)) {
      set_error("%s: %s is not 16-byte aligned", fn, p.second);
      return GS_ERR_ALIGN;
    }
  }
  return GS_OK;
}

#define GS_TRY(x)                   \
  do {                              \
    const gs_status _s = (x);       \
    if (_s != GS_OK) return _s;     \
  } while (0)

int rows_of(const gs_scene* sc) { return 11 + 3 * (sc->sh_degree + 1) * (sc->sh_degree + 1); }

// ---- forward state (gs_fwd_state, GS_ERR_STATE): which forward call last wrote each
// n_contrib buffer.  Host-side, at call (or graph-capture) time.
std::mutex g_reg_mu;
std::unordered_map<const void*, uint64_t> g_last_fwd;
std::atomic<uint64_t> g_fwd_ids{0};

void record_forward(const gs_camera* cam, gs_proj proj, const int32_t* ids, const int32_t* ranges, const float* rgb,
                    const float* depth, const float* T, const int32_t* n, const uint8_t* kb, gs_fwd_state* out) {
  const uint64_t id = ++g_fwd_ids;
  {
    std::lock_guard<std::mutex> lk(g_reg_mu);
    g_last_fwd[n] = id;
  }
  if (out) {
    out->id = id;
    out->width = cam->width, out->height = cam->height;
    out->rec = proj.rec, out->sorted_ids = ids, out->tile_ranges = ranges;
    out->rgb = rgb, out->depth = depth, out->T_final = T, out->n_contrib = n, out->key_blocks = kb;
  }
}

gs_status check_forward(const gs_bwd_opts* opts, const char* fn, const gs_camera* cam, gs_proj proj,
                        const int32_t* ids, const int32_t* ranges, const float* T, const int32_t* n,
                        const uint8_t* kb, const float* rgb = nullptr, const float* depth = nullptr) {
  if (!opts || !opts->fwd) return GS_OK;
  const gs_fwd_state& f = *opts->fwd;
  const char* why = nullptr;
  if (f.id == 0) why = "the forward state was never written";
  else if (f.width != cam->width || f.height != cam->height) why = "image size differs from the forward's";
  else if (f.rec != proj.rec) why = "proj.rec is not the forward's";
  else if (f.sorted_ids != ids || f.tile_ranges != ranges) why = "sorted_ids / tile_ranges are not the forward's";
  else if (f.T_final != T || f.n_contrib != n) why = "T_final / n_contrib are not the forward's";
  else if (kb && kb != f.key_blocks) why = "key_blocks are not the forward's";
  else if ((rgb && rgb != f.rgb) || (depth && depth != f.depth)) why = "rgb / depth are not the forward's";
  else {
    std::lock_guard<std::mutex> lk(g_reg_mu);
    const auto it = g_last_fwd.find(n);
    if (it == g_last_fwd.end() || it->second != f.id) why = "n_contrib was rewritten by a later gs_render_fwd";
  }
  if (why) {
    set_error("%s: state mismatch: %s (forward id %llu)", fn, why, (unsigned long long)f.id);
    return GS_ERR_STATE;
  }
  return GS_OK;
}

// deterministic-mode workspace (gs_bwd_opts.det_ws)
gs_status check_det(const gs_bwd_opts* opts, const char* fn, float** det, int64_t* det_keys) {
  *det = nullptr;
  *det_keys = 0;
  if (!opts || !opts->det_ws) return GS_OK;
  if (opts->det_keys < 0 || opts->det_keys >= (1ll << 30)) {
    set_error("%s: det_keys=%lld out of range", fn, (long long)opts->det_keys);
    return GS_ERR_ARG;
  }
  if (!aligned16(opts->det_ws)) {
    set_error("%s: det_ws is not 16-byte aligned", fn);
    return GS_ERR_ALIGN;
  }
  *det = opts->det_ws;
  *det_keys = opts->det_keys;
  return GS_OK;
}

}  // namespace

// libgsr_check.so only (GSR_BOUNDS_CHECK): validate the lists a render call is given
static void check_lists(const gs_camera* cam, const gs_scene* scene, const int32_t* ids, const int32_t* ranges,
                        void* stream) {
#ifdef GSR_BOUNDS_CHECK
  const DevCam dc = make_devcam(*cam);
  launch_check_lists(dc.TX * dc.TY, scene->P, ids, ranges, static_cast<cudaStream_t>(stream));
#else
  (void)cam, (void)scene, (void)ids, (void)ranges, (void)stream;
#endif
}

extern "C" {

int gs_version(void) { return GSR_VERSION; }
const char* gs_last_error(void) { return g_err; }
int64_t gs_launch_count(void) { return (int64_t)g_launches.load(); }
gs_status gs_set_render_rows(int enable) {
  g_err[0] = 0;
  gsr::set_render_rows(enable);
  return GS_OK;
}
int gs_render_rows(void) { return gsr::render_rows(); }
int gs_exact_exp(void) {
#ifdef GSR_EXACT_EXP
  return 1;
#else
  return 0;
#endif
}

gs_status gs_project(const gs_camera* cam, const gs_scene* scene, const float* params, gs_proj out, void* stream) {
  g_err[0] = 0;
  GS_TRY(check_camera(cam, "gs_project"));
  GS_TRY(check_scene(scene, "gs_project"));
  if (scene->P == 0) return GS_OK;
  GS_TRY(check_ptrs("gs_project", {{params, "params"}, {out.rec, "out.rec"}, {out.radius, "out.radius"},
                                   {out.tiles, "out.tiles"}, {out.flags, "out.flags"}}));
  launch_project(make_devcam(*cam), scene->P, scene->P_stride, scene->sh_degree, params, out,
                 static_cast<cudaStream_t>(stream));
  return check_launch("gs_project");
}

gs_status gs_project_views(int n_views, const gs_camera* cams, const gs_scene* scene, const float* params,
                           const gs_proj* outs, void* stream) {
  g_err[0] = 0;
  if (n_views < 0 || (n_views > 0 && (!cams || !outs))) {
    set_error("gs_project_views: n_views=%d (NULL cams/outs)", n_views);
    return GS_ERR_ARG;
  }
  GS_TRY(check_scene(scene, "gs_project_views"));
  std::vector<DevCam> dc((size_t)n_views);
  for (int v = 0; v < n_views; ++v) {
    GS_TRY(check_camera(&cams[v], "gs_project_views"));
    if (scene->P > 0)
      GS_TRY(check_ptrs("gs_project_views", {{outs[v].rec, "outs.rec"}, {outs[v].radius, "outs.radius"},
                                             {outs[v].tiles, "outs.tiles"}, {outs[v].flags, "outs.flags"}}));
    dc[(size_t)v] = make_devcam(cams[v]);
  }
  if (scene->P == 0 || n_views == 0) return GS_OK;
  GS_TRY(check_ptrs("gs_project_views", {{params, "params"}}));
  launch_project_views(n_views, dc.data(), scene->P, scene->P_stride, scene->sh_degree, params, outs,
                       static_cast<cudaStream_t>(stream));
  return check_launch("gs_project_views");
}

size_t gs_bin_tiles_workspace(const gs_camera* cam, int64_t P, int64_t key_capacity) {
  if (!cam || P < 0 || key_capacity < 0) return 0;
  const int nt = ((cam->width + kTile - 1) / kTile) * ((cam->height + kTile - 1) / kTile);
  return bin_workspace_bytes(P, key_capacity, nt);
}

gs_status gs_bin_tiles(const gs_camera* cam, const gs_scene* scene, gs_proj proj, void* ws, size_t ws_bytes,
                       int64_t key_capacity, int32_t* sorted_ids, int32_t* tile_ranges, int64_t* num_keys_dev,
                       int64_t* num_keys_host, void* stream) {
  g_err[0] = 0;
  GS_TRY(check_camera(cam, "gs_bin_tiles"));
  GS_TRY(check_scene(scene, "gs_bin_tiles"));
  if (key_capacity < 0 || key_capacity >= (1ll << 30)) {
    set_error("gs_bin_tiles: key_capacity=%lld out of range [0, 2^30)", (long long)key_capacity);
    return GS_ERR_ARG;
  }
  GS_TRY(check_ptrs("gs_bin_tiles", {{ws, "ws"}, {tile_ranges, "tile_ranges"}}));
  if (scene->P > 0) {
    GS_TRY(check_ptrs("gs_bin_tiles", {{proj.rec, "proj.rec"}, {proj.tiles, "proj.tiles"}}));
    if (key_capacity > 0) GS_TRY(check_ptrs("gs_bin_tiles", {{sorted_ids, "sorted_ids"}}));
  }
  if (num_keys_dev && (reinterpret_cast<uintptr_t>(num_keys_dev) & 7u)) {
    set_error("gs_bin_tiles: num_keys_dev is not 8-byte aligned");
    return GS_ERR_ALIGN;
  }
  return launch_bin_tiles(make_devcam(*cam), scene->P, proj, ws, ws_bytes, key_capacity, sorted_ids, tile_ranges,
                          num_keys_dev, num_keys_host, static_cast<cudaStream_t>(stream));
}

gs_status gs_render_fwd(const gs_camera* cam, const gs_scene* scene, gs_proj proj, const int32_t* sorted_ids,
                        const int32_t* tile_ranges, const int32_t* tile_order, float* rgb, float* depth, float* T_final, int32_t* n_contrib,
                        unsigned long long* blended, uint8_t* key_blocks, gs_fwd_state* fwd_out, void* stream) {
  g_err[0] = 0;
  GS_TRY(check_camera(cam, "gs_render_fwd"));
  GS_TRY(check_scene(scene, "gs_render_fwd"));
  GS_TRY(check_ptrs("gs_render_fwd", {{tile_ranges, "tile_ranges"}, {rgb, "rgb"}, {depth, "depth"},
                                      {T_final, "T_final"}, {n_contrib, "n_contrib"}}));
  if (scene->P > 0) GS_TRY(check_ptrs("gs_render_fwd", {{proj.rec, "proj.rec"}}));
  if (blended && (reinterpret_cast<uintptr_t>(blended) & 7u)) {
    set_error("gs_render_fwd: blended is not 8-byte aligned");
    return GS_ERR_ALIGN;
  }
  check_lists(cam, scene, sorted_ids, tile_ranges, stream);
  launch_render_fwd(make_devcam(*cam), proj.rec, sorted_ids, tile_ranges, tile_order, rgb, depth, T_final, n_contrib, blended,
                    key_blocks, static_cast<cudaStream_t>(stream));
  GS_TRY(check_launch("gs_render_fwd"));
  record_forward(cam, proj, sorted_ids, tile_ranges, rgb, depth, T_final, n_contrib, key_blocks, fwd_out);
  return GS_OK;
}

size_t gs_render_bwd_workspace(const gs_scene* scene) {
  if (!scene || scene->P < 0) return 0;
  return (size_t)scene->P * GS_SGRAD_FLOATS * sizeof(float);
}

gs_status gs_render_bwd(const gs_camera* cam, const gs_scene* scene, const float* params, gs_proj proj,
                        const int32_t* sorted_ids, const int32_t* tile_ranges, const int32_t* tile_order,
                        const float* T_final,
                        const int32_t* n_contrib, const float* dL_drgb, const float* dL_ddepth,
                        const uint8_t* key_blocks, void* ws, size_t ws_bytes, float* grad, const gs_bwd_opts* opts,
                        void* stream) {
  g_err[0] = 0;
  GS_TRY(check_camera(cam, "gs_render_bwd"));
  GS_TRY(check_scene(scene, "gs_render_bwd"));
  GS_TRY(check_forward(opts, "gs_render_bwd", cam, proj, sorted_ids, tile_ranges, T_final, n_contrib, key_blocks));
  float* det;
  int64_t det_keys;
  GS_TRY(check_det(opts, "gs_render_bwd", &det, &det_keys));
  if (scene->P == 0) return GS_OK;
  GS_TRY(check_ptrs("gs_render_bwd", {{params, "params"}, {proj.rec, "proj.rec"}, {proj.radius, "proj.radius"},
                                      {proj.flags, "proj.flags"}, {tile_ranges, "tile_ranges"}, {T_final, "T_final"},
                                      {n_contrib, "n_contrib"}, {dL_drgb, "dL_drgb"}, {ws, "ws"}, {grad, "grad"}}));
  if (dL_ddepth && !aligned16(dL_ddepth)) {
    set_error("gs_render_bwd: dL_ddepth is not 16-byte aligned");
    return GS_ERR_ALIGN;
  }
  const size_t need = gs_render_bwd_workspace(scene);
  if (ws_bytes < need) {
    set_error("gs_render_bwd: workspace %zu B < required %zu B", ws_bytes, need);
    return GS_ERR_ARG;
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (cudaMemsetAsync(ws, 0, need, s) != cudaSuccess) return check_launch("gs_render_bwd memset");
  const DevCam dc = make_devcam(*cam);
  check_lists(cam, scene, sorted_ids, tile_ranges, stream);
  launch_render_bwd(dc, proj, scene->P, sorted_ids, tile_ranges, tile_order, T_final, n_contrib, dL_drgb, dL_ddepth,
                    key_blocks, static_cast<float*>(ws), s, nullptr, det, det_keys);
  const uint8_t* fl = proj.flags;
  float* sg = static_cast<float*>(ws);
  launch_project_bwd_views(1, &dc, &fl, &sg, scene->P, scene->P_stride, scene->sh_degree, params, grad, 1, s);
  return check_launch("gs_render_bwd");
}

gs_status gs_render_bwd_screen(const gs_camera* cam, const gs_scene* scene, gs_proj proj, const int32_t* sorted_ids,
                               const int32_t* tile_ranges, const int32_t* tile_order, const float* T_final, const int32_t* n_contrib,
                               const float* dL_drgb, const float* dL_ddepth, const uint8_t* key_blocks, float* sgrad,
                               const gs_bwd_opts* opts, void* stream) {
  g_err[0] = 0;
  GS_TRY(check_camera(cam, "gs_render_bwd_screen"));
  GS_TRY(check_scene(scene, "gs_render_bwd_screen"));
  GS_TRY(check_forward(opts, "gs_render_bwd_screen", cam, proj, sorted_ids, tile_ranges, T_final, n_contrib,
                       key_blocks));
  float* det;
  int64_t det_keys;
  GS_TRY(check_det(opts, "gs_render_bwd_screen", &det, &det_keys));
  if (scene->P == 0) return GS_OK;
  GS_TRY(check_ptrs("gs_render_bwd_screen", {{proj.rec, "proj.rec"}, {tile_ranges, "tile_ranges"},
                                             {T_final, "T_final"}, {n_contrib, "n_contrib"}, {dL_drgb, "dL_drgb"},
                                             {sgrad, "sgrad"}}));
  if (dL_ddepth && !aligned16(dL_ddepth)) {
    set_error("gs_render_bwd_screen: dL_ddepth is not 16-byte aligned");
    return GS_ERR_ALIGN;
  }
  check_lists(cam, scene, sorted_ids, tile_ranges, stream);
  launch_render_bwd(make_devcam(*cam), proj, scene->P, sorted_ids, tile_ranges, tile_order, T_final, n_contrib,
                    dL_drgb, dL_ddepth, key_blocks, sgrad, static_cast<cudaStream_t>(stream), nullptr, det, det_keys);
  return check_launch("gs_render_bwd_screen");
}

gs_status gs_render_bwd_screen_l1(const gs_camera* cam, const gs_scene* scene, gs_proj proj,
                                  const int32_t* sorted_ids, const int32_t* tile_ranges, const int32_t* tile_order,
                                  const float* T_final, const int32_t* n_contrib, const float* rgb, const float* depth,
                                  const float* target_rgb, const float* target_depth, float w_depth, float* loss,
                                  const uint8_t* key_blocks, float* sgrad, const gs_bwd_opts* opts, void* stream) {
  g_err[0] = 0;
  GS_TRY(check_camera(cam, "gs_render_bwd_screen_l1"));
  GS_TRY(check_scene(scene, "gs_render_bwd_screen_l1"));
  GS_TRY(check_forward(opts, "gs_render_bwd_screen_l1", cam, proj, sorted_ids, tile_ranges, T_final, n_contrib,
                       key_blocks, rgb, depth));
  float* det;
  int64_t det_keys;
  GS_TRY(check_det(opts, "gs_render_bwd_screen_l1", &det, &det_keys));
  GS_TRY(check_ptrs("gs_render_bwd_screen_l1", {{tile_ranges, "tile_ranges"}, {T_final, "T_final"},
                                                {n_contrib, "n_contrib"}, {rgb, "rgb"}, {depth, "depth"},
                                                {target_rgb, "target_rgb"}, {target_depth, "target_depth"},
                                                {sgrad, "sgrad"}}));
  if (scene->P > 0) GS_TRY(check_ptrs("gs_render_bwd_screen_l1", {{proj.rec, "proj.rec"}}));
  const L1Targets l1{rgb, depth, target_rgb, target_depth, w_depth, loss};
  check_lists(cam, scene, sorted_ids, tile_ranges, stream);
  launch_render_bwd(make_devcam(*cam), proj, scene->P, sorted_ids, tile_ranges, tile_order, T_final, n_contrib,
                    nullptr, nullptr, key_blocks, sgrad, static_cast<cudaStream_t>(stream), &l1, det, det_keys);
  return check_launch("gs_render_bwd_screen_l1");
}

gs_status gs_tile_order(const gs_camera* cam, const int32_t* tile_ranges, int32_t* tile_order, void* stream) {
  g_err[0] = 0;
  GS_TRY(check_camera(cam, "gs_tile_order"));
  GS_TRY(check_ptrs("gs_tile_order", {{tile_ranges, "tile_ranges"}, {tile_order, "tile_order"}}));
  const DevCam dc = make_devcam(*cam);
  launch_tile_order(dc.TX * dc.TY, tile_ranges, tile_order, static_cast<cudaStream_t>(stream));
  return check_launch("gs_tile_order");
}

gs_status gs_naive_render_fwd(const gs_camera* cam, const gs_scene* scene, gs_proj proj, const int32_t* sorted_ids,
                              const int32_t* tile_ranges, float* rgb, float* depth, float* T_final,
                              int32_t* n_contrib, unsigned long long* blended, gs_fwd_state* fwd_out, void* stream) {
  g_err[0] = 0;
  GS_TRY(check_camera(cam, "gs_naive_render_fwd"));
  GS_TRY(check_scene(scene, "gs_naive_render_fwd"));
  GS_TRY(check_ptrs("gs_naive_render_fwd", {{tile_ranges, "tile_ranges"}, {rgb, "rgb"}, {depth, "depth"},
                                            {T_final, "T_final"}, {n_contrib, "n_contrib"}}));
  if (scene->P > 0) GS_TRY(check_ptrs("gs_naive_render_fwd", {{proj.rec, "proj.rec"}}));
  if (blended && (reinterpret_cast<uintptr_t>(blended) & 7u)) {
    set_error("gs_naive_render_fwd: blended is not 8-byte aligned");
    return GS_ERR_ALIGN;
  }
  check_lists(cam, scene, sorted_ids, tile_ranges, stream);
  launch_naive_fwd(make_devcam(*cam), proj.rec, sorted_ids, tile_ranges, rgb, depth, T_final, n_contrib, blended,
                   static_cast<cudaStream_t>(stream));
  GS_TRY(check_launch("gs_naive_render_fwd"));
  record_forward(cam, proj, sorted_ids, tile_ranges, rgb, depth, T_final, n_contrib, nullptr, fwd_out);
  return GS_OK;
}

gs_status gs_naive_render_bwd_screen(const gs_camera* cam, const gs_scene* scene, gs_proj proj,
                                     const int32_t* sorted_ids, const int32_t* tile_ranges, const float* T_final,
                                     const int32_t* n_contrib, const float* dL_drgb, const float* dL_ddepth,
                                     float* sgrad, const gs_bwd_opts* opts, void* stream) {
  g_err[0] = 0;
  GS_TRY(check_camera(cam, "gs_naive_render_bwd_screen"));
  GS_TRY(check_scene(scene, "gs_naive_render_bwd_screen"));
  GS_TRY(check_forward(opts, "gs_naive_render_bwd_screen", cam, proj, sorted_ids, tile_ranges, T_final, n_contrib,
                       nullptr));
  if (opts && opts->det_ws) {
    set_error("gs_naive_render_bwd_screen: the K13 port has no deterministic mode");
    return GS_ERR_ARG;
  }
  if (scene->P == 0) return GS_OK;
  GS_TRY(check_ptrs("gs_naive_render_bwd_screen", {{proj.rec, "proj.rec"}, {tile_ranges, "tile_ranges"},
                                                   {T_final, "T_final"}, {n_contrib, "n_contrib"},
                                                   {dL_drgb, "dL_drgb"}, {sgrad, "sgrad"}}));
  check_lists(cam, scene, sorted_ids, tile_ranges, stream);
  launch_naive_bwd(make_devcam(*cam), proj.rec, sorted_ids, tile_ranges, T_final, n_contrib, dL_drgb, dL_ddepth,
                   sgrad, static_cast<cudaStream_t>(stream));
  return check_launch("gs_naive_render_bwd_screen");
}

gs_status gs_project_bwd_views(int n_views, const gs_camera* cams, const gs_scene* scene, const float* params,
                               const uint8_t* const* flags, float* const* sgrads, float* grad, int accumulate,
                               void* stream) {
  g_err[0] = 0;
  GS_TRY(check_scene(scene, "gs_project_bwd_views"));
  if (n_views < 0 || (n_views > 0 && (!cams || !flags || !sgrads))) {
    set_error("gs_project_bwd_views: invalid view arrays (n_views=%d)", n_views);
    return GS_ERR_ARG;
  }
  if (scene->P == 0 || (n_views == 0 && accumulate)) return GS_OK;
  if (n_views == 0) {  // overwrite with an empty batch: grad := 0
    GS_TRY(check_ptrs("gs_project_bwd_views", {{grad, "grad"}}));
    if (cudaMemsetAsync(grad, 0, (size_t)rows_of(scene) * scene->P_stride * sizeof(float),
                        static_cast<cudaStream_t>(stream)) != cudaSuccess)
      return check_launch("gs_project_bwd_views memset");
    return GS_OK;
  }
  GS_TRY(check_ptrs("gs_project_bwd_views", {{params, "params"}, {grad, "grad"}}));
  std::vector<DevCam> dc((size_t)n_views);
  for (int v = 0; v < n_views; ++v) {
    GS_TRY(check_camera(cams + v, "gs_project_bwd_views"));
    if (!flags[v] || !sgrads[v]) {
      set_error("gs_project_bwd_views: view %d has a NULL flags or sgrad pointer", v);
      return GS_ERR_ARG;
    }
    if (!aligned16(sgrads[v])) {
      set_error("gs_project_bwd_views: sgrads[%d] is not 16-byte aligned", v);
      return GS_ERR_ALIGN;
    }
    dc[v] = make_devcam(cams[v]);
  }
  launch_project_bwd_views(n_views, dc.data(), flags, sgrads, scene->P, scene->P_stride, scene->sh_degree, params,
                           grad, accumulate ? 1 : 0, static_cast<cudaStream_t>(stream));
  return check_launch("gs_project_bwd_views");
}

gs_status gs_project_bwd_views_adam_dev(int n_views, const gs_camera* cams, const gs_scene* scene, float* params,
                                        const uint8_t* const* flags, float* const* sgrads, float* grad, int accumulate,
                                        float* m, float* v, const float* lr_per_row, float beta1, float beta2,
                                        float eps, int64_t* step_dev, void* stream, void* side_stream) {
  static const char* fn = "gs_project_bwd_views_adam_dev";
  g_err[0] = 0;
  GS_TRY(check_scene(scene, fn));
  if (n_views < 1 || !cams || !flags || !sgrads || !step_dev || !lr_per_row || !(beta1 >= 0.f && beta1 < 1.f) ||
      !(beta2 >= 0.f && beta2 < 1.f) || !(eps >= 0.f)) {
    set_error("%s: invalid arguments (n_views=%d)", fn, n_views);
    return GS_ERR_ARG;
  }
  if (scene->P == 0) return GS_OK;
  GS_TRY(check_ptrs(fn, {{params, "params"}, {grad, "grad"}, {m, "m"}, {v, "v"}}));
  std::vector<DevCam> dc((size_t)n_views);
  for (int i = 0; i < n_views; ++i) {
    GS_TRY(check_camera(cams + i, fn));
    if (!flags[i] || !sgrads[i]) {
      set_error("%s: view %d has a NULL flags or sgrad pointer", fn, i);
      return GS_ERR_ARG;
    }
    if (!aligned16(sgrads[i])) {
      set_error("%s: sgrads[%d] is not 16-byte aligned", fn, i);
      return GS_ERR_ALIGN;
    }
    dc[i] = make_devcam(cams[i]);
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream), side = static_cast<cudaStream_t>(side_stream);
  // library-owned events (created once; only ordering, no timing): the colour half's end
  // and the side stream's Adam end.  Recorded / waited in stream order, so they also work
  // inside a CUDA-graph capture (the side stream forks from and joins the captured one).
  static cudaEvent_t ev_colour = nullptr, ev_side = nullptr;
  if (!ev_colour) {
    if (cudaEventCreateWithFlags(&ev_colour, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&ev_side, cudaEventDisableTiming) != cudaSuccess)
      return check_launch(fn);
  }
  const int64_t F = rows_of(scene), S = scene->P_stride, split = 11 * S;  // rows 0..10 | SH rows 11..F-1
  launch_step_inc(step_dev, s);  // t += 1 once, before either half reads it
  launch_project_bwd_views(n_views, dc.data(), flags, sgrads, scene->P, S, scene->sh_degree, params, grad,
                           accumulate ? 1 : 0, s, side ? ev_colour : nullptr);
  if (side) {  // the SH rows' Adam on the side stream, under the geometry half
    cudaStreamWaitEvent(side, ev_colour, 0);
    launch_adam(F, S, params, grad + split, m, v, lr_per_row, beta1, beta2, eps, 1.f, 1.f, 0, side, split, F * S, -1,
                step_dev, false);
    cudaEventRecord(ev_side, side);
    launch_adam(F, S, params, grad, m, v, lr_per_row, beta1, beta2, eps, 1.f, 1.f, 0, s, 0, split, -1, step_dev,
                false);
    cudaStreamWaitEvent(s, ev_side, 0);
  } else {
    launch_adam(F, S, params, grad, m, v, lr_per_row, beta1, beta2, eps, 1.f, 1.f, 0, s, 0, F * S, -1, step_dev,
                false);
  }
  return check_launch(fn);
}

size_t gs_spatial_order_workspace(const gs_scene* scene) {
  if (!scene || scene->P < 0) return 0;
  return spatial_order_workspace_bytes(scene->P);
}

gs_status gs_spatial_order(const gs_scene* scene, const float* params_in, float* params_out, int32_t* perm, void* ws,
                           size_t ws_bytes, void* stream) {
  g_err[0] = 0;
  GS_TRY(check_scene(scene, "gs_spatial_order"));
  if (scene->P == 0) return GS_OK;
  GS_TRY(check_ptrs("gs_spatial_order", {{params_in, "params_in"}, {params_out, "params_out"}, {ws, "ws"}}));
  if (params_in == params_out) {
    set_error("gs_spatial_order: params_in and params_out must not alias");
    return GS_ERR_ARG;
  }
  return launch_spatial_order(rows_of(scene), scene->P, scene->P_stride, params_in, params_out, perm, ws, ws_bytes,
                              static_cast<cudaStream_t>(stream));
}

gs_status gs_adam_step(const gs_scene* scene, float* params, float* grad, float* m, float* v, const float* lr_per_row,
                       float beta1, float beta2, float eps, int64_t step, int zero_grad, void* stream) {
  g_err[0] = 0;
  GS_TRY(check_scene(scene, "gs_adam_step"));
  if (scene->P == 0) {
    set_error("gs_adam_step: no Gaussians (P == 0)");
    return GS_ERR_EMPTY;
  }
  if (!lr_per_row || step < 1 || !(beta1 >= 0.f && beta1 < 1.f) || !(beta2 >= 0.f && beta2 < 1.f) || !(eps >= 0.f)) {
    set_error("gs_adam_step: invalid hyper-parameters (step=%lld beta1=%g beta2=%g eps=%g)", (long long)step,
              (double)beta1, (double)beta2, (double)eps);
    return GS_ERR_ARG;
  }
  GS_TRY(check_ptrs("gs_adam_step", {{params, "params"}, {grad, "grad"}, {m, "m"}, {v, "v"}}));
  const double bc1 = 1.0 - std::pow((double)beta1, (double)step);
  const double bc2 = 1.0 - std::pow((double)beta2, (double)step);
  launch_adam(rows_of(scene), scene->P_stride, params, grad, m, v, lr_per_row, beta1, beta2, eps, (float)bc1,
              (float)bc2, zero_grad, static_cast<cudaStream_t>(stream), 0, -1, scene->P);
  return check_launch("gs_adam_step");
}

gs_status gs_adam_step_dev(const gs_scene* scene, float* params, float* grad, float* m, float* v,
                           const float* lr_per_row, float beta1, float beta2, float eps, int64_t* step_dev,
                           int zero_grad, void* stream) {
  g_err[0] = 0;
  GS_TRY(check_scene(scene, "gs_adam_step_dev"));
  if (scene->P == 0) {
    set_error("gs_adam_step_dev: no Gaussians (P == 0)");
    return GS_ERR_EMPTY;
  }
  if (!lr_per_row || !step_dev || !(beta1 >= 0.f && beta1 < 1.f) || !(beta2 >= 0.f && beta2 < 1.f) || !(eps >= 0.f)) {
    set_error("gs_adam_step_dev: invalid arguments");
    return GS_ERR_ARG;
  }
  GS_TRY(check_ptrs("gs_adam_step_dev", {{params, "params"}, {grad, "grad"}, {m, "m"}, {v, "v"}}));
  launch_adam_dev(rows_of(scene), scene->P_stride, params, grad, m, v, lr_per_row, beta1, beta2, eps, step_dev,
                  zero_grad, static_cast<cudaStream_t>(stream), scene->P);
  return check_launch("gs_adam_step_dev");
}

namespace {
// gs_adam_step_range / gs_adam_step_peers with the step on the host (step_dev NULL) or on
// the device (the *_dev calls: *step_dev is incremented first, graph-capturable).
gs_status adam_range_impl(const char* fn, const gs_scene* scene, float* params, const float* grad_range, float* m,
                          float* v, const float* lr_per_row, float beta1, float beta2, float eps, int64_t step,
                          int64_t* step_dev, int64_t begin, int64_t end, void* stream) {
  g_err[0] = 0;
  GS_TRY(check_scene(scene, fn));
  const int64_t n = (int64_t)rows_of(scene) * scene->P_stride;
  if (!lr_per_row || (!step_dev && step < 1) || !(beta1 >= 0.f && beta1 < 1.f) || !(beta2 >= 0.f && beta2 < 1.f) ||
      !(eps >= 0.f) || begin < 0 || end < begin || end > n) {
    set_error("%s: invalid arguments (step=%lld begin=%lld end=%lld n=%lld)", fn, (long long)step, (long long)begin,
              (long long)end, (long long)n);
    return GS_ERR_ARG;
  }
  if ((begin & 3) || (end & 3)) {
    set_error("%s: begin/end must be multiples of 4", fn);
    return GS_ERR_ALIGN;
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (end == begin) {
    if (step_dev) launch_adam(rows_of(scene), scene->P_stride, nullptr, nullptr, nullptr, nullptr, lr_per_row, beta1,
                              beta2, eps, 1.f, 1.f, 0, s, 0, 0, -1, step_dev);  // only advances the counter
    return step_dev ? check_launch(fn) : GS_OK;
  }
  GS_TRY(check_ptrs(fn, {{params, "params"}, {grad_range, "grad_range"}, {m, "m"}, {v, "v"}}));
  const double bc1 = step_dev ? 1.0 : 1.0 - std::pow((double)beta1, (double)step);
  const double bc2 = step_dev ? 1.0 : 1.0 - std::pow((double)beta2, (double)step);
  launch_adam(rows_of(scene), scene->P_stride, params, const_cast<float*>(grad_range), m, v, lr_per_row, beta1, beta2,
              eps, (float)bc1, (float)bc2, 0, s, begin, end, -1, step_dev);
  return check_launch(fn);
}

gs_status adam_peers_impl(const char* fn, const gs_scene* scene, int world, int rank, const float* const* grad_peers,
                          float* const* param_peers, float* m, float* v, const float* lr_per_row, float beta1,
                          float beta2, float eps, int64_t step, int64_t* step_dev, int64_t begin, int64_t end,
                          void* stream) {
  g_err[0] = 0;
  GS_TRY(check_scene(scene, fn));
  const int64_t n = (int64_t)rows_of(scene) * scene->P_stride;
  if (!grad_peers || !param_peers || !lr_per_row || (!step_dev && step < 1) || !(beta1 >= 0.f && beta1 < 1.f) ||
      !(beta2 >= 0.f && beta2 < 1.f) || !(eps >= 0.f) || begin < 0 || end < begin || end > n) {
    set_error("%s: invalid arguments (step=%lld begin=%lld end=%lld n=%lld)", fn, (long long)step, (long long)begin,
              (long long)end, (long long)n);
    return GS_ERR_ARG;
  }
  if ((begin & 3) || (end & 3)) {
    set_error("%s: begin/end must be multiples of 4", fn);
    return GS_ERR_ALIGN;
  }
  if (end > begin) GS_TRY(check_ptrs(fn, {{m, "m"}, {v, "v"}}));
  const double bc1 = step_dev ? 1.0 : 1.0 - std::pow((double)beta1, (double)step);
  const double bc2 = step_dev ? 1.0 : 1.0 - std::pow((double)beta2, (double)step);
  GS_TRY(launch_adam_peers(rows_of(scene), scene->P_stride, world, rank, grad_peers, param_peers, m, v, lr_per_row,
                           beta1, beta2, eps, (float)bc1, (float)bc2, begin, end, static_cast<cudaStream_t>(stream),
                           step_dev));
  return check_launch(fn);
}
}  // namespace

gs_status gs_adam_step_range(const gs_scene* scene, float* params, const float* grad_range, float* m, float* v,
                             const float* lr_per_row, float beta1, float beta2, float eps, int64_t step, int64_t begin,
                             int64_t end, void* stream) {
  return adam_range_impl("gs_adam_step_range", scene, params, grad_range, m, v, lr_per_row, beta1, beta2, eps, step,
                         nullptr, begin, end, stream);
}

gs_status gs_adam_step_range_dev(const gs_scene* scene, float* params, const float* grad_range, float* m, float* v,
                                 const float* lr_per_row, float beta1, float beta2, float eps, int64_t* step_dev,
                                 int64_t begin, int64_t end, void* stream) {
  if (!step_dev) {
    set_error("gs_adam_step_range_dev: step_dev is NULL");
    return GS_ERR_ARG;
  }
  return adam_range_impl("gs_adam_step_range_dev", scene, params, grad_range, m, v, lr_per_row, beta1, beta2, eps, 0,
                         step_dev, begin, end, stream);
}

gs_status gs_adam_step_peers(const gs_scene* scene, int world, int rank, const float* const* grad_peers,
                             float* const* param_peers, float* m, float* v, const float* lr_per_row, float beta1,
                             float beta2, float eps, int64_t step, int64_t begin, int64_t end, void* stream) {
  return adam_peers_impl("gs_adam_step_peers", scene, world, rank, grad_peers, param_peers, m, v, lr_per_row, beta1,
                         beta2, eps, step, nullptr, begin, end, stream);
}

gs_status gs_adam_step_peers_dev(const gs_scene* scene, int world, int rank, const float* const* grad_peers,
                                 float* const* param_peers, float* m, float* v, const float* lr_per_row, float beta1,
                                 float beta2, float eps, int64_t* step_dev, int64_t begin, int64_t end, void* stream) {
  if (!step_dev) {
    set_error("gs_adam_step_peers_dev: step_dev is NULL");
    return GS_ERR_ARG;
  }
  return adam_peers_impl("gs_adam_step_peers_dev", scene, world, rank, grad_peers, param_peers, m, v, lr_per_row,
                         beta1, beta2, eps, 0, step_dev, begin, end, stream);
}

gs_status gs_adam_step_multimem(const gs_scene* scene, const float* mc_grad, float* mc_param, const float* param,
                                float* m, float* v, const float* lr_per_row, float beta1, float beta2, float eps,
                                int64_t step, int64_t* step_dev, int64_t begin, int64_t end, void* stream) {
  g_err[0] = 0;
  GS_TRY(check_scene(scene, "gs_adam_step_multimem"));
  const int64_t n = (int64_t)rows_of(scene) * scene->P_stride;
  if (!lr_per_row || (!step_dev && step < 1) || !(beta1 >= 0.f && beta1 < 1.f) || !(beta2 >= 0.f && beta2 < 1.f) ||
      !(eps >= 0.f) || begin < 0 || end < begin || end > n) {
    set_error("gs_adam_step_multimem: invalid arguments (step=%lld begin=%lld end=%lld n=%lld)", (long long)step,
              (long long)begin, (long long)end, (long long)n);
    return GS_ERR_ARG;
  }
  if ((begin & 3) || (end & 3)) {
    set_error("gs_adam_step_multimem: begin/end must be multiples of 4");
    return GS_ERR_ALIGN;
  }
  if (end > begin)
    GS_TRY(check_ptrs("gs_adam_step_multimem",
                      {{mc_grad, "mc_grad"}, {mc_param, "mc_param"}, {param, "param"}, {m, "m"}, {v, "v"}}));
  const double bc1 = step_dev ? 1.0 : 1.0 - std::pow((double)beta1, (double)step);
  const double bc2 = step_dev ? 1.0 : 1.0 - std::pow((double)beta2, (double)step);
  GS_TRY(launch_adam_multimem(rows_of(scene), scene->P_stride, mc_grad, mc_param, param, m, v, lr_per_row, beta1,
                              beta2, eps, (float)bc1, (float)bc2, begin, end, static_cast<cudaStream_t>(stream),
                              step_dev));
  return check_launch("gs_adam_step_multimem");
}

gs_status gs_l1_loss_grad(int64_t npix, const float* rgb, const float* depth, const float* target_rgb,
                          const float* target_depth, float w_depth, float* dL_drgb, float* dL_ddepth, float* loss,
                          void* stream) {
  g_err[0] = 0;
  if (npix <= 0) {
    set_error("gs_l1_loss_grad: npix=%lld", (long long)npix);
    return GS_ERR_ARG;
  }
  GS_TRY(check_ptrs("gs_l1_loss_grad", {{rgb, "rgb"}, {depth, "depth"}, {target_rgb, "target_rgb"},
                                        {target_depth, "target_depth"}, {dL_drgb, "dL_drgb"},
                                        {dL_ddepth, "dL_ddepth"}}));
  launch_l1(npix, rgb, depth, target_rgb, target_depth, w_depth, dL_drgb, dL_ddepth, loss,
            static_cast<cudaStream_t>(stream));
  return check_launch("gs_l1_loss_grad");
}

gs_status gs_visibility_union(int n_views, const uint8_t* const* flags, int64_t P, int accumulate, uint8_t* visible,
                              void* stream) {
  g_err[0] = 0;
  if (n_views < 0 || P < 0 || (P > 0 && !visible) || (n_views > 0 && !flags)) {
    set_error("gs_visibility_union: n_views=%d P=%lld", n_views, (long long)P);
    return GS_ERR_ARG;
  }
  for (int v = 0; v < n_views; ++v)
    if (P > 0 && !flags[v]) {
      set_error("gs_visibility_union: flags[%d] is NULL", v);
      return GS_ERR_ARG;
    }
  if (P == 0) return GS_OK;
  if (n_views == 0 && accumulate) return GS_OK;
  launch_vis_union(n_views, flags, P, accumulate != 0, visible, static_cast<cudaStream_t>(stream));
  return check_launch("gs_visibility_union");
}

size_t gs_compact_workspace(int64_t P) { return P < 0 ? 0 : compact_workspace(P); }

gs_status gs_compact_index(const uint8_t* visible, int64_t P, void* ws, size_t ws_bytes, int32_t* idx,
                           int64_t* count_dev, void* stream) {
  g_err[0] = 0;
  if (P < 0 || !count_dev || !ws || (P > 0 && (!visible || !idx))) {
    set_error("gs_compact_index: P=%lld (NULL pointer)", (long long)P);
    return GS_ERR_ARG;
  }
  if (ws_bytes < compact_workspace(P)) {
    set_error("gs_compact_index: workspace %zu B < required %zu B", ws_bytes, compact_workspace(P));
    return GS_ERR_ARG;
  }
  launch_compact_index(visible, P, static_cast<uint32_t*>(ws), idx, count_dev, static_cast<cudaStream_t>(stream));
  return check_launch("gs_compact_index");
}

gs_status gs_gather_columns(const float* full, int64_t F, int64_t S, const int32_t* idx, int64_t M, float* packed,
                            void* stream) {
  g_err[0] = 0;
  if (F < 0 || S < 0 || M < 0 || M > S || (F > 0 && M > 0 && (!full || !idx || !packed))) {
    set_error("gs_gather_columns: F=%lld S=%lld M=%lld", (long long)F, (long long)S, (long long)M);
    return GS_ERR_ARG;
  }
  launch_gather_cols(full, F, S, idx, M, packed, static_cast<cudaStream_t>(stream));
  return check_launch("gs_gather_columns");
}

gs_status gs_scatter_columns(const float* packed, int64_t F, int64_t S, const int32_t* idx, int64_t M, float* full,
                             void* stream) {
  g_err[0] = 0;
  if (F < 0 || S < 0 || M < 0 || M > S || (F > 0 && M > 0 && (!full || !idx || !packed))) {
    set_error("gs_scatter_columns: F=%lld S=%lld M=%lld", (long long)F, (long long)S, (long long)M);
    return GS_ERR_ARG;
  }
  launch_scatter_cols(packed, F, S, idx, M, full, static_cast<cudaStream_t>(stream));
  return check_launch("gs_scatter_columns");
}

gs_status gs_decode_rgbd(int32_t width, int32_t height, const uint8_t* rgb, const uint16_t* depth, float depth_scale,
                         float* out_rgb, float* out_depth, void* stream) {
  g_err[0] = 0;
  if (width <= 0 || height <= 0 || !(depth_scale > 0.f) || !std::isfinite(depth_scale)) {
    set_error("gs_decode_rgbd: width=%d height=%d depth_scale=%g", width, height, (double)depth_scale);
    return GS_ERR_ARG;
  }
  // any alignment is accepted (the aligned case takes the vectorised kernel)
  for (const auto& p : {std::make_pair((const void*)rgb, "rgb"), std::make_pair((const void*)depth, "depth"),
                        std::make_pair((const void*)out_rgb, "out_rgb"), std::make_pair((const void*)out_depth, "out_depth")})
    if (!p.first) {
      set_error("gs_decode_rgbd: %s is NULL", p.second);
      return GS_ERR_ARG;
    }
  launch_decode_rgbd((int64_t)width * height, rgb, depth, depth_scale, out_rgb, out_depth,
                     static_cast<cudaStream_t>(stream));
  return check_launch("gs_decode_rgbd");
}

}  // extern "C"
