// K9 adam_step (first-order update; Adam per north_star, R20) and
// K10 the Eq. 12 L1 harness (R19).  Both are HBM-streaming kernels:
// 128-bit vector loads/stores, grid-stride loops over a grid of a few waves.
#include "gsr_internal.cuh"

namespace gsr {
namespace {

struct LrTable {
  float step[64];  // lr_row / (1 - beta1^t)   (raw lr_row when the step is on the device)
};

// Per-row step sizes and 1/sqrt(1 - beta2^t) of one Adam step, in shared memory.  With
// step_dev == nullptr they come from the host (lr already divided by bc1, rs_bc2
// given); otherwise every block derives them from the device step counter t = *step_dev
// (CUDA-graph replays, gs_adam_step*_dev), with the same arithmetic as the host (t in
// double, bias corrections rounded to fp32), so both give bit-identical updates.
__device__ __forceinline__ void adam_steps(const LrTable& lr, int F, float b1, float b2, float rs_host,
                                           const int64_t* __restrict__ step_dev, float* s_step, float& s_rs) {
  __shared__ float rs;
  if (threadIdx.x < 64) {
    if (step_dev) {
      const double t = (double)*step_dev;
      const float bc1 = (float)(1.0 - pow((double)b1, t));
      s_step[threadIdx.x] = threadIdx.x < F ? lr.step[threadIdx.x] / bc1 : 0.f;
      if (threadIdx.x == 0) rs = 1.f / sqrtf((float)(1.0 - pow((double)b2, t)));
    } else {
      s_step[threadIdx.x] = lr.step[threadIdx.x];
      if (threadIdx.x == 0) rs = rs_host;
    }
  }
  __syncthreads();
  s_rs = rs;
}

// Scalars [4 b4, 4 e4) of the flattened [F][P_stride] arrays; g holds the gradient of
// that range (g[i - b4]), so a rank of the sharded optimiser passes its reduce-scattered
// shard and the full step passes b4 = 0, g = grad.
// cl4 < S4 (full step only): just the first cl4 float4 columns of every row -- the live
// Gaussians [0, P) of a map that grows into its capacity P_stride.
__global__ void __launch_bounds__(256) k_adam(float4* __restrict__ p, float4* __restrict__ g, float4* __restrict__ m,
                                              float4* __restrict__ v, int64_t b4, int64_t e4, int64_t S4, int64_t cl4,
                                              LrTable lr_in, int F, float b1, float b2, float eps, float rs_host,
                                              const int64_t* __restrict__ step_dev, int zero_grad) {
  __shared__ float s_step[64];
  float rs_bc2;
  adam_steps(lr_in, F, b1, b2, rs_host, step_dev, s_step, rs_bc2);
  const float c1 = 1.f - b1, c2 = 1.f - b2;
  const int64_t count = cl4 < S4 ? (e4 / S4) * cl4 : e4 - b4;
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < count; j += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = cl4 < S4 ? (j / cl4) * S4 + j % cl4 : b4 + j;
    const float step = s_step[i / S4];
    const float4 gg = g[i - b4];
    float4 mm = m[i], vv = v[i], pp = p[i];
    adam_update(pp.x, mm.x, vv.x, gg.x, b1, b2, c1, c2, step, rs_bc2, eps);
    adam_update(pp.y, mm.y, vv.y, gg.y, b1, b2, c1, c2, step, rs_bc2, eps);
    adam_update(pp.z, mm.z, vv.z, gg.z, b1, b2, c1, c2, step, rs_bc2, eps);
    adam_update(pp.w, mm.w, vv.w, gg.w, b1, b2, c1, c2, step, rs_bc2, eps);
    p[i] = pp;
    m[i] = mm;
    v[i] = vv;
    if (zero_grad) g[i - b4] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
}

// Graph-capturable Adam: the step counter lives on the device (k_step_inc advances it,
// then every block derives its bias corrections from it), so a captured iteration
// replays with the right t.  Same arithmetic as k_adam (t in double, rounded to fp32).
__global__ void k_step_inc(int64_t* t) { *t += 1; }

__global__ void __launch_bounds__(256) k_adam_dev(float4* __restrict__ p, float4* __restrict__ g,
                                                  float4* __restrict__ m, float4* __restrict__ v, int64_t n4,
                                                  int64_t S4, int64_t cl4, LrTable lr_raw, int F, float b1, float b2,
                                                  float eps, const int64_t* __restrict__ step_dev, int zero_grad) {
  __shared__ float s_step[64];
  __shared__ float s_rs;
  if (threadIdx.x < 64) {
    const double t = (double)*step_dev;
    const float bc1 = (float)(1.0 - pow((double)b1, t));
    s_step[threadIdx.x] = threadIdx.x < F ? lr_raw.step[threadIdx.x] / bc1 : 0.f;
    if (threadIdx.x == 0) s_rs = 1.f / sqrtf((float)(1.0 - pow((double)b2, t)));
  }
  __syncthreads();
  const float rs_bc2 = s_rs;
  const float c1 = 1.f - b1, c2 = 1.f - b2;
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n4; j += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = cl4 < S4 ? (j / cl4) * S4 + j % cl4 : j;
    const float step = s_step[i / S4];
    const float4 gg = g[i];
    float4 mm = m[i], vv = v[i], pp = p[i];
    adam_update(pp.x, mm.x, vv.x, gg.x, b1, b2, c1, c2, step, rs_bc2, eps);
    adam_update(pp.y, mm.y, vv.y, gg.y, b1, b2, c1, c2, step, rs_bc2, eps);
    adam_update(pp.z, mm.z, vv.z, gg.z, b1, b2, c1, c2, step, rs_bc2, eps);
    adam_update(pp.w, mm.w, vv.w, gg.w, b1, b2, c1, c2, step, rs_bc2, eps);
    p[i] = pp;
    m[i] = mm;
    v[i] = vv;
    if (zero_grad) g[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
}

// Fused reduce-scatter + Adam + all-gather over peer memory (NEXT-2): this rank owns
// scalars [4 b4, 4 e4) of the flattened arrays; it pulls that range of every rank's
// gradient over NVLink (P2P loads, summed in rank order: deterministic), applies Adam
// to its local m, v and parameters, and pushes the new parameters into every rank's
// parameter buffer (P2P stores).  Peer buffers come from symmetric memory; the caller
// fences the ranks before (gradients final) and after (parameters delivered).
constexpr int kMaxPeers = 8;
struct Peers {
  const float4* grad[kMaxPeers];
  float4* param[kMaxPeers];
  int world, rank;
};

__global__ void __launch_bounds__(256) k_adam_peers(const __grid_constant__ Peers pr, float4* __restrict__ m,
                                                    float4* __restrict__ v, int64_t b4, int64_t e4, int64_t S4,
                                                    LrTable lr_in, int F, float b1, float b2, float eps, float rs_host,
                                                    const int64_t* __restrict__ step_dev) {
  __shared__ float s_step[64];
  float rs_bc2;
  adam_steps(lr_in, F, b1, b2, rs_host, step_dev, s_step, rs_bc2);
  const float c1 = 1.f - b1, c2 = 1.f - b2;
  for (int64_t i = b4 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < e4; i += (int64_t)gridDim.x * blockDim.x) {
    const float step = s_step[i / S4];
    float4 gs[kMaxPeers];
#pragma unroll
    for (int r = 0; r < kMaxPeers; ++r)
      if (r < pr.world) gs[r] = pr.grad[r][i];  // all peers' loads in flight at once
    float4 gg = gs[0];
#pragma unroll
    for (int r = 1; r < kMaxPeers; ++r)
      if (r < pr.world) gg.x += gs[r].x, gg.y += gs[r].y, gg.z += gs[r].z, gg.w += gs[r].w;
    float4 mm = m[i], vv = v[i], pp = pr.param[pr.rank][i];
    adam_update(pp.x, mm.x, vv.x, gg.x, b1, b2, c1, c2, step, rs_bc2, eps);
    adam_update(pp.y, mm.y, vv.y, gg.y, b1, b2, c1, c2, step, rs_bc2, eps);
    adam_update(pp.z, mm.z, vv.z, gg.z, b1, b2, c1, c2, step, rs_bc2, eps);
    adam_update(pp.w, mm.w, vv.w, gg.w, b1, b2, c1, c2, step, rs_bc2, eps);
    m[i] = mm;
    v[i] = vv;
#pragma unroll
    for (int r = 0; r < kMaxPeers; ++r)
      if (r < pr.world) pr.param[r][i] = pp;
  }
}

// NVLS (in-switch) variant of k_adam_peers (SURVEY.md §8(f) NEXT-2 remainder): this
// rank's shard of the SUM of every rank's gradient arrives in ONE multicast load-reduce
// (multimem.ld_reduce: the NVSwitch adds the ranks' values, fp32), Adam runs on the
// local m, v and parameters, and ONE multicast store (multimem.st) writes the new
// parameters into every rank's copy.  mc_grad / mc_param: multicast addresses of the
// symmetric gradient / parameter buffers; param: this rank's own copy (unicast).  Each
// scalar is reduced and stored once, by its owner: the ranks stay bit-identical.
__device__ __forceinline__ float4 mc_ld_reduce_add(const float4* mc) {
  float4 r;
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
               : "l"(mc)
               : "memory");
  return r;
}
__device__ __forceinline__ void mc_st(float4* mc, const float4& v) {
  asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(mc), "f"(v.x), "f"(v.y), "f"(v.z),
               "f"(v.w)
               : "memory");
}

__global__ void __launch_bounds__(256) k_adam_multimem(const float4* __restrict__ mc_grad, float4* __restrict__ mc_param,
                                                       const float4* __restrict__ param, float4* __restrict__ m,
                                                       float4* __restrict__ v, int64_t b4, int64_t e4, int64_t S4,
                                                       LrTable lr_in, int F, float b1, float b2, float eps,
                                                       float rs_host, const int64_t* __restrict__ step_dev) {
  __shared__ float s_step[64];
  float rs_bc2;
  adam_steps(lr_in, F, b1, b2, rs_host, step_dev, s_step, rs_bc2);
  const float c1 = 1.f - b1, c2 = 1.f - b2;
  for (int64_t i = b4 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < e4; i += (int64_t)gridDim.x * blockDim.x) {
    const float step = s_step[i / S4];
    const float4 gg = mc_ld_reduce_add(mc_grad + i);
    float4 mm = m[i], vv = v[i], pp = param[i];
    adam_update(pp.x, mm.x, vv.x, gg.x, b1, b2, c1, c2, step, rs_bc2, eps);
    adam_update(pp.y, mm.y, vv.y, gg.y, b1, b2, c1, c2, step, rs_bc2, eps);
    adam_update(pp.z, mm.z, vv.z, gg.z, b1, b2, c1, c2, step, rs_bc2, eps);
    adam_update(pp.w, mm.w, vv.w, gg.w, b1, b2, c1, c2, step, rs_bc2, eps);
    m[i] = mm;
    v[i] = vv;
    mc_st(mc_param + i, pp);
  }
}

__global__ void __launch_bounds__(256) k_l1(int64_t npix, const float* __restrict__ rgb, const float* __restrict__ dep,
                                            const float* __restrict__ trgb, const float* __restrict__ tdep, float sc,
                                            float sd, float* __restrict__ grgb, float* __restrict__ gdep,
                                            float* loss) {
  float L = 0.f;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < npix; i += (int64_t)gridDim.x * blockDim.x) {
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) {
      const int64_t j = ch * npix + i;
      const float r = l1_res_rgb(rgb[j], trgb[j]);
      L += fabsf(r) * sc;
      grgb[j] = r > 0.f ? sc : (r < 0.f ? -sc : 0.f);
    }
    const float r = l1_res_depth(dep[i], tdep[i]);
    L += fabsf(r) * sd;
    gdep[i] = r > 0.f ? sd : (r < 0.f ? -sd : 0.f);
  }
  if (loss) {
    for (int o = 16; o > 0; o >>= 1) L += __shfl_xor_sync(kFull, L, o);
    if ((threadIdx.x & 31) == 0 && L != 0.f) atomicAdd(loss, L);
  }
}

}  // namespace

void launch_adam(int64_t F, int64_t S, float* params, float* grad, float* m, float* v, const float* lr, float beta1,
                 float beta2, float eps, float bc1, float bc2, int zero_grad, cudaStream_t s, int64_t begin,
                 int64_t end, int64_t live, int64_t* step_dev, bool inc_step) {
  LrTable t{};
  for (int64_t r = 0; r < F && r < 64; ++r) t.step[r] = step_dev ? lr[r] : lr[r] / bc1;
  if (step_dev && inc_step) {
    k_step_inc<<<1, 1, 0, s>>>(step_dev);
    count_launch();
  }
  int64_t cl4 = S / 4;
  if (end < 0) {
    end = F * S;
    if (live >= 0) cl4 = std::min<int64_t>((live + 3) / 4, S / 4);
  }
  const int64_t n4 = cl4 < S / 4 ? F * cl4 : (end - begin) / 4;
  const int grid = (int)std::min<int64_t>((n4 + 255) / 256, (int64_t)sm_count() * 8);
  k_adam<<<std::max(grid, 1), 256, 0, s>>>(reinterpret_cast<float4*>(params), reinterpret_cast<float4*>(grad),
                                           reinterpret_cast<float4*>(m), reinterpret_cast<float4*>(v), begin / 4,
                                           end / 4, S / 4, cl4, t, (int)F, beta1, beta2, eps,
                                           step_dev ? 0.f : 1.f / sqrtf(bc2), step_dev, zero_grad);
  count_launch();
}

void launch_step_inc(int64_t* step_dev, cudaStream_t s) {
  k_step_inc<<<1, 1, 0, s>>>(step_dev);
  count_launch();
}

void launch_adam_dev(int64_t F, int64_t S, float* params, float* grad, float* m, float* v, const float* lr, float beta1,
                     float beta2, float eps, int64_t* step_dev, int zero_grad, cudaStream_t s, int64_t live) {
  LrTable t{};
  for (int64_t r = 0; r < F && r < 64; ++r) t.step[r] = lr[r];
  const int64_t cl4 = live >= 0 ? std::min<int64_t>((live + 3) / 4, S / 4) : S / 4;
  const int64_t n4 = F * cl4;
  const int grid = (int)std::min<int64_t>((n4 + 255) / 256, (int64_t)sm_count() * 8);
  k_step_inc<<<1, 1, 0, s>>>(step_dev);
  k_adam_dev<<<std::max(grid, 1), 256, 0, s>>>(reinterpret_cast<float4*>(params), reinterpret_cast<float4*>(grad),
                                               reinterpret_cast<float4*>(m), reinterpret_cast<float4*>(v), n4, S / 4, cl4,
                                               t, (int)F, beta1, beta2, eps, step_dev, zero_grad);
  count_launch(2);
}

gs_status launch_adam_peers(int64_t F, int64_t S, int world, int rank, const float* const* grad_peers,
                            float* const* param_peers, float* m, float* v, const float* lr, float beta1, float beta2,
                            float eps, float bc1, float bc2, int64_t begin, int64_t end, cudaStream_t s,
                            int64_t* step_dev) {
  if (world < 1 || world > kMaxPeers || rank < 0 || rank >= world) {
    set_error("gs_adam_step_peers: world %d / rank %d outside [1, %d]", world, rank, kMaxPeers);
    return GS_ERR_ARG;
  }
  Peers pr{};
  pr.world = world, pr.rank = rank;
  for (int r = 0; r < world; ++r) {
    if (!grad_peers[r] || !param_peers[r] || !aligned16(grad_peers[r]) || !aligned16(param_peers[r])) {
      set_error("gs_adam_step_peers: peer %d buffers NULL or not 16-byte aligned", r);
      return GS_ERR_ALIGN;
    }
    pr.grad[r] = reinterpret_cast<const float4*>(grad_peers[r]);
    pr.param[r] = reinterpret_cast<float4*>(param_peers[r]);
  }
  LrTable t{};
  for (int64_t r = 0; r < F && r < 64; ++r) t.step[r] = step_dev ? lr[r] : lr[r] / bc1;
  if (step_dev) {  // every rank advances its own counter, whether or not it owns scalars
    k_step_inc<<<1, 1, 0, s>>>(step_dev);
    count_launch();
  }
  const int64_t n4 = (end - begin) / 4;
  const int grid = (int)std::min<int64_t>((n4 + 255) / 256, (int64_t)sm_count() * 8);
  if (n4 > 0) {
    k_adam_peers<<<std::max(grid, 1), 256, 0, s>>>(pr, reinterpret_cast<float4*>(m), reinterpret_cast<float4*>(v),
                                                    begin / 4, end / 4, S / 4, t, (int)F, beta1, beta2, eps,
                                                    step_dev ? 0.f : 1.f / sqrtf(bc2), step_dev);
    count_launch();
  }
  return GS_OK;
}

gs_status launch_adam_multimem(int64_t F, int64_t S, const float* mc_grad, float* mc_param, const float* param,
                               float* m, float* v, const float* lr, float beta1, float beta2, float eps, float bc1,
                               float bc2, int64_t begin, int64_t end, cudaStream_t s, int64_t* step_dev) {
  LrTable t{};
  for (int64_t r = 0; r < F && r < 64; ++r) t.step[r] = step_dev ? lr[r] : lr[r] / bc1;
  if (step_dev) {
    k_step_inc<<<1, 1, 0, s>>>(step_dev);
    count_launch();
  }
  const int64_t n4 = (end - begin) / 4;
  const int grid = (int)std::min<int64_t>((n4 + 255) / 256, (int64_t)sm_count() * 8);
  if (n4 > 0) {
    k_adam_multimem<<<std::max(grid, 1), 256, 0, s>>>(
        reinterpret_cast<const float4*>(mc_grad), reinterpret_cast<float4*>(mc_param),
        reinterpret_cast<const float4*>(param), reinterpret_cast<float4*>(m), reinterpret_cast<float4*>(v), begin / 4,
        end / 4, S / 4, t, (int)F, beta1, beta2, eps, step_dev ? 0.f : 1.f / sqrtf(bc2), step_dev);
    count_launch();
  }
  return GS_OK;
}

void launch_l1(int64_t npix, const float* rgb, const float* depth, const float* t_rgb, const float* t_depth,
               float w_depth, float* g_rgb, float* g_depth, float* loss, cudaStream_t s) {
  const float sc = (float)(1.0 / (3.0 * (double)npix)), sd = (float)((double)w_depth / (double)npix);
  const int grid = (int)std::min<int64_t>((npix + 255) / 256, (int64_t)sm_count() * 8);
  k_l1<<<std::max(grid, 1), 256, 0, s>>>(npix, rgb, depth, t_rgb, t_depth, sc, sd, g_rgb, g_depth, loss);
  count_launch();
}

}  // namespace gsr
