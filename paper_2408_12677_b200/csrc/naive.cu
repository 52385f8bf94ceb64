// K13: the "straightforward per-pixel GPU port" the north_star's >= 10x target is
// measured against (BASELINE.json north_star; SURVEY.md §8(d) "Targets").  It is a
// COMPARISON BASELINE, not the product path: same projection, binning, projection
// backward and Adam as the product, but
//  * forward: one thread per pixel (16x16 threads = one tile per CTA) walks its tile's
//    depth-sorted list reading every Gaussian record straight from global memory --
//    no shared-memory staging, no warp cooperation, no block masks (Eq. 11,
//    PAPER.md:140-142, with the R15-R17 skip / cap / stop rules);
//  * backward: one thread per pixel walks its list back to front from n_contrib,
//    recovering T_k = T_{k+1} / (1 - alpha_k), and issues 10 atomicAdd per composited
//    (pixel, Gaussian) pair into the screen-space gradient (R18).
// Both compute exactly the quantities of k_render_fwd / k_render_bwd (same record
// layout, same screen-gradient layout), so bench.py credits both with the same
// blended-pair count and the ratio is one of times at identical work.
#include "gsr_internal.cuh"

namespace gsr {
namespace {

constexpr float kAlphaMinN = 1.0f / 255.0f;
constexpr float kTStopN = 1e-4f;
constexpr float kAlphaCapN = 0.99f;

struct NaiveRec {
  float mx, my, z, o, A, B, C, r, g, b;
};

__device__ __forceinline__ NaiveRec naive_load(const float4* __restrict__ rec, int id) {
  const float4 q0 = rec[3 * (int64_t)id], q1 = rec[3 * (int64_t)id + 1], q2 = rec[3 * (int64_t)id + 2];
  return {q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, q1.z, q1.w, q2.x, q2.y};
}

__global__ void __launch_bounds__(256) k_naive_fwd(DevCam cam, const float4* __restrict__ rec,
                                                   const int32_t* __restrict__ ids, const int2* __restrict__ ranges,
                                                   float* __restrict__ out_rgb, float* __restrict__ out_d,
                                                   float* __restrict__ out_T, int32_t* __restrict__ out_n,
                                                   unsigned long long* blended) {
  const int x = blockIdx.x * kTile + threadIdx.x, y = blockIdx.y * kTile + threadIdx.y;
  const bool inside = x < cam.W && y < cam.H;
  const int2 rg = ranges[blockIdx.y * cam.TX + blockIdx.x];
  const float px = (float)x, py = (float)y;
  float T = 1.f, cr = 0.f, cg = 0.f, cb = 0.f, d = 0.f;
  int n = 0;
  uint32_t nb = 0;
  if (inside) {
    for (int i = rg.x; i < rg.y; ++i) {
      const NaiveRec q = naive_load(rec, ids[i]);
      const float dx = q.mx - px, dy = q.my - py;
      const float power = -0.5f * (q.A * dx * dx + q.C * dy * dy) - q.B * dx * dy;
      if (power > 0.f) continue;
      const float alpha = fminf(kAlphaCapN, q.o * __expf(power));
      if (alpha < kAlphaMinN) continue;
      const float Tn = T * (1.f - alpha);
      if (Tn < kTStopN) break;
      const float w = alpha * T;
      cr += q.r * w, cg += q.g * w, cb += q.b * w, d += q.z * w;
      T = Tn;
      n = i - rg.x + 1;
      ++nb;
    }
    const int64_t npix = (int64_t)cam.W * cam.H, p = (int64_t)y * cam.W + x;
    out_rgb[p] = cr + T * cam.bg[0];
    out_rgb[npix + p] = cg + T * cam.bg[1];
    out_rgb[2 * npix + p] = cb + T * cam.bg[2];
    out_d[p] = d;
    out_T[p] = T;
    out_n[p] = n;
  }
  if (blended) {
    const uint32_t tot = __reduce_add_sync(kFull, nb);
    if ((threadIdx.x & 31) == 0 && (threadIdx.y & 1) == 0 && tot) atomicAdd(blended, (unsigned long long)tot);
  }
}

__global__ void __launch_bounds__(256) k_naive_bwd(DevCam cam, const float4* __restrict__ rec,
                                                   const int32_t* __restrict__ ids, const int2* __restrict__ ranges,
                                                   const float* __restrict__ T_final,
                                                   const int32_t* __restrict__ n_contrib,
                                                   const float* __restrict__ g_rgb, const float* __restrict__ g_dep,
                                                   float* __restrict__ sgrad) {
  const int x = blockIdx.x * kTile + threadIdx.x, y = blockIdx.y * kTile + threadIdx.y;
  if (x >= cam.W || y >= cam.H) return;
  const int2 rg = ranges[blockIdx.y * cam.TX + blockIdx.x];
  const int64_t npix = (int64_t)cam.W * cam.H, p = (int64_t)y * cam.W + x;
  const float px = (float)x, py = (float)y;
  float T = T_final[p];
  const float gr = g_rgb[p], gg = g_rgb[npix + p], gb = g_rgb[2 * npix + p];
  const float gd = g_dep ? g_dep[p] : 0.f;
  // suffix term Q_k = sum_ch g_ch S^C_ch + g_D S^D, starting with the background
  float Q = T * (gr * cam.bg[0] + gg * cam.bg[1] + gb * cam.bg[2]);
  for (int i = rg.x + n_contrib[p] - 1; i >= rg.x; --i) {
    const int id = ids[i];
    const NaiveRec q = naive_load(rec, id);
    const float dx = q.mx - px, dy = q.my - py;
    const float power = -0.5f * (q.A * dx * dx + q.C * dy * dy) - q.B * dx * dy;
    if (power > 0.f) continue;
    const float G = __expf(power);
    const float raw = q.o * G;
    const float alpha = fminf(kAlphaCapN, raw);
    if (alpha < kAlphaMinN) continue;
    const float inv = 1.f / (1.f - alpha);
    const float Tk = T * inv;
    const float w = alpha * Tk;
    const float u = gr * q.r + gg * q.g + gb * q.b + gd * q.z;
    const float dal = raw > kAlphaCapN ? 0.f : (Tk * u - inv * Q);  // capped alpha: no derivative (R18)
    Q += w * u;
    T = Tk;
    const float dp = raw * dal;  // dL/dpower
    float* s = sgrad + (int64_t)GS_SGRAD_FLOATS * id;
    atomicAdd(s + 0, -dp * (q.A * dx + q.B * dy));
    atomicAdd(s + 1, -dp * (q.B * dx + q.C * dy));
    atomicAdd(s + 2, -0.5f * dp * dx * dx);
    atomicAdd(s + 3, -dp * dx * dy);
    atomicAdd(s + 4, -0.5f * dp * dy * dy);
    atomicAdd(s + 5, G * dal);
    atomicAdd(s + 6, gr * w);
    atomicAdd(s + 7, gg * w);
    atomicAdd(s + 8, gb * w);
    atomicAdd(s + 9, gd * w);
  }
}

}  // namespace

void launch_naive_fwd(const DevCam& cam, const float* rec, const int32_t* ids, const int32_t* ranges, float* rgb,
                      float* depth, float* T_final, int32_t* n_contrib, unsigned long long* blended, cudaStream_t s) {
  k_naive_fwd<<<dim3(cam.TX, cam.TY), dim3(kTile, kTile), 0, s>>>(
      cam, reinterpret_cast<const float4*>(rec), ids, reinterpret_cast<const int2*>(ranges), rgb, depth, T_final,
      n_contrib, blended);
  count_launch();
}

void launch_naive_bwd(const DevCam& cam, const float* rec, const int32_t* ids, const int32_t* ranges,
                      const float* T_final, const int32_t* n_contrib, const float* g_rgb, const float* g_depth,
                      float* sgrad, cudaStream_t s) {
  k_naive_bwd<<<dim3(cam.TX, cam.TY), dim3(kTile, kTile), 0, s>>>(
      cam, reinterpret_cast<const float4*>(rec), ids, reinterpret_cast<const int2*>(ranges), T_final, n_contrib,
      g_rgb, g_depth, sgrad);
  count_launch();
}

}  // namespace gsr
