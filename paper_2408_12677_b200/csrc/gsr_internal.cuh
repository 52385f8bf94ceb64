// Internal helpers shared by the libgsr.so translation units (product path only).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstdio>
#include <utility>

#include "gsr.h"

namespace gsr {

constexpr int kTile = GS_TILE;
constexpr unsigned kFull = 0xffffffffu;

// Per-view camera constants passed to kernels by value.
struct DevCam {
  int W, H, TX, TY;
  float fx, fy, cx, cy;
  float R[9], t[3];
  float z_near;
  float bg[3];
  float ocam[3];  // camera centre in world coordinates, -R^T t (SH view direction)
  float limx, limy;  // R7 tangent clamps 1.3 W / (2 fx), 1.3 H / (2 fy), fp32 in that order
};

DevCam make_devcam(const gs_camera& c);

// Bounds-checked build (libgsr_check.so, -DGSR_BOUNDS_CHECK; compute-sanitizer is
// closed on the GPU pool): device-side index asserts in the kernels that scatter
// through computed indices, plus validation of the caller's lists at the ABI
// (launch_check_lists).  A failed check prints its condition and traps, which turns
// into cudaErrorLaunchFailure at the next check_launch.  Compiled out otherwise.
#ifdef GSR_BOUNDS_CHECK
#define GSR_CHECK(cond)                                                                        \
  do {                                                                                         \
    if (!(cond)) {                                                                             \
      printf("GSR_CHECK failed %s:%d block %d thread %d: %s\n", __FILE__, __LINE__, (int)blockIdx.x, \
             (int)threadIdx.x, #cond);                                                         \
      __trap();                                                                                \
    }                                                                                          \
  } while (0)
#else
#define GSR_CHECK(cond) \
  do {                  \
  } while (0)
#endif
// every id of every tile's list in [0, P), 0 <= start <= end <= K (K = the largest end)
void launch_check_lists(int NT, int64_t P, const int32_t* ids, const int32_t* ranges, cudaStream_t s);

// error plumbing (api.cu)
void set_error(const char* fmt, ...);
gs_status check_launch(const char* what);
void count_launch(int n = 1);
int sm_count();  // SMs of the current device (cached per device)

// Lanes of the warp holding the same 8-bit digit as this lane (stable multisplit
// ranking): 8 bit-sliced ballots instead of __match_any_sync, whose SASS MATCH.ANY
// measured ~40 cycles/warp of SM throughput on B200.  Invalid lanes
// are nobody's peers; an invalid lane gets an arbitrary mask (callers ignore it).
__device__ __forceinline__ uint32_t digit_peers(uint32_t d, bool valid) {
  uint32_t peers = __ballot_sync(kFull, valid);
#pragma unroll
  for (int b = 0; b < 8; ++b) {
    const uint32_t bits = __ballot_sync(kFull, (d >> b) & 1u);
    peers &= ((d >> b) & 1u) ? bits : ~bits;
  }
  return peers;
}

// One Adam update of a scalar (R20), in a fixed fp32 operation order shared by every
// kernel that applies it (k_adam, k_adam_dev, k_adam_peers), so the single-rank,
// graph and multi-GPU paths give bit-identical parameters.
__device__ __forceinline__ void adam_update(float& p, float& m, float& v, float g, float b1, float b2, float c1,
                                            float c2, float step, float rs_bc2, float eps) {
  m = __fmaf_rn(b1, m, __fmul_rn(c1, g));
  v = __fmaf_rn(b2, v, __fmul_rn(__fmul_rn(c2, g), g));
  p = __fsub_rn(p, __fdiv_rn(__fmul_rn(step, m), __fmaf_rn(__fsqrt_rn(v), rs_bc2, eps)));
}

// Eq. 12 residual of one target sample (reading R43): a target that is not a
// measurement -- a non-finite colour, or a depth that is <= 0 (the sensor's
// "invalid", R41) or non-finite -- gives residual 0: no loss term and no gradient
// (sign(0) = 0, R19).  Shared by k_l1 and the fused backward so both are identical.
__device__ __forceinline__ float l1_res_rgb(float x, float t) { return fabsf(t) <= 3.402823466e+38f ? x - t : 0.f; }
__device__ __forceinline__ float l1_res_depth(float x, float t) {
  return (t > 0.f && t <= 3.402823466e+38f) ? x - t : 0.f;
}

inline int ceil_div(long long a, long long b) { return (int)((a + b - 1) / b); }
inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// ------------------------------------------------------------------ launchers
// project.cu
void launch_project(const DevCam& cam, int64_t P, int64_t P_stride, int deg, const float* params, gs_proj out,
                    cudaStream_t s);
constexpr int kMaxViews = 8;  // views chained per pass of the projection backward
void launch_project_views(int n_views, const DevCam* cams, int64_t P, int64_t S, int deg, const float* params,
                          const gs_proj* outs, cudaStream_t s);
void launch_project_bwd_views(int n_views, const DevCam* cams, const uint8_t* const* flags, float* const* sgrads,
                              int64_t P, int64_t S, int deg, const float* params, float* grad, int accumulate,
                              cudaStream_t s, cudaEvent_t colour_done = nullptr);
// binning.cu
size_t bin_workspace_bytes(int64_t P, int64_t key_capacity, int num_tiles);
gs_status launch_bin_tiles(const DevCam& cam, int64_t P, gs_proj proj, void* ws, size_t ws_bytes,
                           int64_t key_capacity, int32_t* sorted_ids, int32_t* tile_ranges, int64_t* num_keys_dev,
                           int64_t* num_keys_host, cudaStream_t s);
void launch_tile_order(int NT, const int32_t* tile_ranges, int32_t* order, cudaStream_t s);
size_t spatial_order_workspace_bytes(int64_t P);
gs_status launch_spatial_order(int64_t F, int64_t P, int64_t S, const float* params_in, float* params_out,
                               int32_t* perm, void* ws, size_t ws_bytes, cudaStream_t s);
// render.cu
// performance switch of the render kernels (gs_set_render_rows): 1 = block-row walk
void set_render_rows(int v);
int render_rows();
void launch_render_fwd(const DevCam& cam, const float* rec, const int32_t* ids, const int32_t* ranges,
                       const int32_t* order, float* rgb,
                       float* depth, float* T_final, int32_t* n_contrib, unsigned long long* blended,
                       uint8_t* key_blocks, cudaStream_t s);
// Fused Eq. 12 upstream for the backward (gs_render_bwd_screen_l1): rendered and target
// images, the depth weight and the loss accumulator.
struct L1Targets {
  const float *rgb, *depth, *target_rgb, *target_depth;
  float w_depth;
  float* loss;
};
// det != nullptr: deterministic reduction (gs_bwd_opts.det_ws): per-key partials to
// det[key][12] (zeroed here), then a fixed-order per-Gaussian sum into sgrad.
void launch_render_bwd(const DevCam& cam, gs_proj proj, int64_t P, const int32_t* ids, const int32_t* ranges,
                       const int32_t* order, const float* T_final, const int32_t* n_contrib, const float* g_rgb,
                       const float* g_depth, const uint8_t* key_blocks, float* sgrad, cudaStream_t s,
                       const L1Targets* l1 = nullptr, float* det = nullptr, int64_t det_keys = 0);
// naive.cu (K13 comparison baseline, not the product path)
void launch_naive_fwd(const DevCam& cam, const float* rec, const int32_t* ids, const int32_t* ranges, float* rgb,
                      float* depth, float* T_final, int32_t* n_contrib, unsigned long long* blended, cudaStream_t s);
void launch_naive_bwd(const DevCam& cam, const float* rec, const int32_t* ids, const int32_t* ranges,
                      const float* T_final, const int32_t* n_contrib, const float* g_rgb, const float* g_depth,
                      float* sgrad, cudaStream_t s);
// optim.cu
void launch_adam(int64_t F, int64_t P_stride, float* params, float* grad, float* m, float* v, const float* lr,
                 float beta1, float beta2, float eps, float bc1, float bc2, int zero_grad, cudaStream_t s,
                 int64_t begin = 0, int64_t end = -1, int64_t live = -1, int64_t* step_dev = nullptr,
                 bool inc_step = true);
void launch_step_inc(int64_t* step_dev, cudaStream_t s);
void launch_adam_dev(int64_t F, int64_t S, float* params, float* grad, float* m, float* v, const float* lr, float beta1,
                     float beta2, float eps, int64_t* step_dev, int zero_grad, cudaStream_t s, int64_t live = -1);
gs_status launch_adam_peers(int64_t F, int64_t S, int world, int rank, const float* const* grad_peers,
                            float* const* param_peers, float* m, float* v, const float* lr, float beta1, float beta2,
                            float eps, float bc1, float bc2, int64_t begin, int64_t end, cudaStream_t s,
                            int64_t* step_dev = nullptr);
gs_status launch_adam_multimem(int64_t F, int64_t S, const float* mc_grad, float* mc_param, const float* param,
                               float* m, float* v, const float* lr, float beta1, float beta2, float eps, float bc1,
                               float bc2, int64_t begin, int64_t end, cudaStream_t s, int64_t* step_dev = nullptr);
void launch_l1(int64_t npix, const float* rgb, const float* depth, const float* t_rgb, const float* t_depth,
               float w_depth, float* g_rgb, float* g_depth, float* loss, cudaStream_t s);

// exchange.cu
size_t compact_workspace(int64_t P);
void launch_vis_union(int n_views, const uint8_t* const* flags, int64_t P, bool accumulate, uint8_t* visible,
                      cudaStream_t s);
void launch_compact_index(const uint8_t* visible, int64_t P, uint32_t* tile_cnt, int32_t* idx, int64_t* count,
                          cudaStream_t s);
void launch_gather_cols(const float* full, int64_t F, int64_t S, const int32_t* idx, int64_t M, float* packed,
                        cudaStream_t s);
void launch_scatter_cols(const float* packed, int64_t F, int64_t S, const int32_t* idx, int64_t M, float* full,
                         cudaStream_t s);

// frame.cu
void launch_decode_rgbd(int64_t npix, const uint8_t* rgb, const uint16_t* depth, float scale, float* out_rgb,
                        float* out_d, cudaStream_t s);

}  // namespace gsr
