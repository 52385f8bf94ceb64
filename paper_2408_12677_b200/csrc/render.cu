// K6 render_fwd and K7 render_bwd (Eq. 11; backward PAPER.md:147).
//
// Work decomposition (B200-first): one warp per 16x16 tile, each
// lane owns a column of 8 pixels (lane & 15 = column, lane >> 4 = upper/lower half).
// A warp stages 32 of its tile's Gaussian records (48 B each, gathered from L2 by
// id) into shared memory, then every lane evaluates each record against its 8
// pixels.  Because the 8 pixels share x, the per-record part of the Gaussian
// exponent (A dx^2, B dx) is computed once per lane and each pixel costs one FADD +
// two FFMA + one MUFU.EX2 for its exponent.  The backward reverses the composite
// with T_k = T_{k+1} / (1 - alpha_k), keeps the suffix term as one scalar per pixel
// (Q = sum_ch g_ch S^C_ch + g_D S^D), accumulates the 10 screen-space gradient
// components of the current Gaussian over the lane's 8 pixels in registers, and
// reduces them across the warp (= the whole tile) with a 13-shuffle transpose
// reduction so that 10 lanes issue ONE red.global.add.f32 instruction per (tile,
// Gaussian): one atomic per warp per component, as the north_star asks.
//
// GSR_EXACT_EXP builds (libgsr_exact.so) evaluate the exponent, alpha, transmittance
// and accumulation in the oracle's fp32 operation order with exp computed in double
// (reading R9): the forward is then bit-identical to the fp32 oracle.
#include "gsr_internal.cuh"

namespace gsr {
namespace {

constexpr int kWarpsPerCta = 4;
constexpr int kPix = 8;  // pixels per lane
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kAlphaMin = 1.0f / 255.0f;
constexpr float kTStop = 1e-4f;
constexpr float kAlphaCap = 0.99f;

#ifdef GSR_EXACT_EXP
constexpr bool kExact = true;
#else
constexpr bool kExact = false;
#endif

__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// Per-(record, lane) constants for evaluating the Gaussian on the lane's column.
struct Eval {
  float a0, b0, c2;  // fast path: p2 = a0 + dy (b0 + c2 dy) = log2(e) * power
  float A, B, C, dx; // exact path
};

__device__ __forceinline__ Eval make_eval(float mx, float A, float B, float C, float pxf) {
  Eval e;
  e.dx = mx - pxf;
  e.A = A, e.B = B, e.C = C;
  if (!kExact) {
    e.a0 = (-0.5f * kLog2e) * A * e.dx * e.dx;
    e.b0 = (-kLog2e * B) * e.dx;
    e.c2 = -0.5f * kLog2e * C;
  }
  return e;
}

// Returns the power test result ("power <= 0") and G = exp(power).
__device__ __forceinline__ bool eval_gauss(const Eval& e, float my, float pyf, float& G, float& dy) {
  if (kExact) {
    const float dxx = e.dx;
    dy = __fsub_rn(my, pyf);
    const float power = __fsub_rn(
        __fmul_rn(-0.5f, __fadd_rn(__fmul_rn(__fmul_rn(e.A, dxx), dxx), __fmul_rn(__fmul_rn(e.C, dy), dy))),
        __fmul_rn(__fmul_rn(e.B, dxx), dy));
    G = (float)exp((double)power);
    return !(power > 0.f);
  } else {
    dy = my - pyf;
    const float p2 = fmaf(dy, fmaf(e.c2, dy, e.b0), e.a0);
    G = ex2_approx(p2);
    return !(p2 > 0.f);
  }
}

__device__ __forceinline__ void load_rec(const float4* s, float& mx, float& my, float& z, float& o, float& A, float& B,
                                         float& C, float& r, float& g, float& b) {
  const float4 q0 = s[0], q1 = s[1], q2 = s[2];
  mx = q0.x, my = q0.y, z = q0.z, o = q0.w;
  A = q1.x, B = q1.y, C = q1.z, r = q1.w;
  g = q2.x, b = q2.y;
}

// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kWarpsPerCta * 32) k_render_fwd(DevCam cam, const float4* __restrict__ rec,
                                                                   const int32_t* __restrict__ ids,
                                                                   const int2* __restrict__ ranges,
                                                                   float* __restrict__ out_rgb,
                                                                   float* __restrict__ out_d, float* __restrict__ out_T,
                                                                   int32_t* __restrict__ out_n,
                                                                   unsigned long long* blended) {
  __shared__ float4 s_rec[kWarpsPerCta][32][3];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tile = blockIdx.x * kWarpsPerCta + warp;
  if (tile >= cam.TX * cam.TY) return;
  const int tx = tile % cam.TX, ty = tile / cam.TX;
  const int px = tx * kTile + (lane & 15);
  const int py0 = ty * kTile + (lane >> 4) * kPix;
  const float pxf = (float)px;
  const int2 rg = ranges[tile];

  float T[kPix], Cr[kPix], Cg[kPix], Cb[kPix], D[kPix];
  int n[kPix];
  uint32_t done = 0;
#pragma unroll
  for (int i = 0; i < kPix; ++i) {
    T[i] = 1.f, Cr[i] = Cg[i] = Cb[i] = D[i] = 0.f, n[i] = 0;
    if (px >= cam.W || py0 + i >= cam.H) done |= 1u << i;
  }
  uint32_t nblend = 0;
  bool all_done = __all_sync(kFull, done == 0xffu);
  for (int b = rg.x; b < rg.y && !all_done; b += 32) {
    const int idx = b + lane;
    if (idx < rg.y) {
      const float4* r = rec + 3 * (int64_t)ids[idx];
      s_rec[warp][lane][0] = r[0];
      s_rec[warp][lane][1] = r[1];
      s_rec[warp][lane][2] = r[2];
    }
    __syncwarp();
    const int cnt = min(32, rg.y - b);
    for (int j = 0; j < cnt; ++j) {
      float mx, my, z, o, A, B, C, cr, cg, cb;
      load_rec(s_rec[warp][j], mx, my, z, o, A, B, C, cr, cg, cb);
      const Eval e = make_eval(mx, A, B, C, pxf);
      const int pos1 = b + j - rg.x + 1;
#pragma unroll
      for (int i = 0; i < kPix; ++i) {
        float G, dy;
        const bool pok = eval_gauss(e, my, (float)(py0 + i), G, dy);
        const float alpha = fminf(kAlphaCap, kExact ? __fmul_rn(o, G) : o * G);
        const bool act = !((done >> i) & 1u) && pok && !(alpha < kAlphaMin);
        const float Tn = kExact ? __fmul_rn(T[i], __fsub_rn(1.f, alpha)) : T[i] * (1.f - alpha);
        const bool stop = act && (Tn < kTStop);
        if (stop) done |= 1u << i;
        if (act && !stop) {
          if (kExact) {
            const float w = __fmul_rn(alpha, T[i]);
            Cr[i] = __fadd_rn(Cr[i], __fmul_rn(cr, w));
            Cg[i] = __fadd_rn(Cg[i], __fmul_rn(cg, w));
            Cb[i] = __fadd_rn(Cb[i], __fmul_rn(cb, w));
            D[i] = __fadd_rn(D[i], __fmul_rn(z, w));
          } else {
            const float w = alpha * T[i];
            Cr[i] = fmaf(cr, w, Cr[i]);
            Cg[i] = fmaf(cg, w, Cg[i]);
            Cb[i] = fmaf(cb, w, Cb[i]);
            D[i] = fmaf(z, w, D[i]);
          }
          T[i] = Tn;
          n[i] = pos1;
          ++nblend;
        }
      }
      all_done = __all_sync(kFull, done == 0xffu);
      if (all_done) break;
    }
    __syncwarp();
  }
  const int64_t npix = (int64_t)cam.W * cam.H;
#pragma unroll
  for (int i = 0; i < kPix; ++i) {
    const int py = py0 + i;
    if (px < cam.W && py < cam.H) {
      const int64_t p = (int64_t)py * cam.W + px;
      if (kExact) {
        out_rgb[p] = __fadd_rn(Cr[i], __fmul_rn(T[i], cam.bg[0]));
        out_rgb[npix + p] = __fadd_rn(Cg[i], __fmul_rn(T[i], cam.bg[1]));
        out_rgb[2 * npix + p] = __fadd_rn(Cb[i], __fmul_rn(T[i], cam.bg[2]));
      } else {
        out_rgb[p] = fmaf(T[i], cam.bg[0], Cr[i]);
        out_rgb[npix + p] = fmaf(T[i], cam.bg[1], Cg[i]);
        out_rgb[2 * npix + p] = fmaf(T[i], cam.bg[2], Cb[i]);
      }
      out_d[p] = D[i];
      out_T[p] = T[i];
      out_n[p] = n[i];
    }
  }
  if (blended) {
    const uint32_t tot = __reduce_add_sync(kFull, nblend);
    if (lane == 0 && tot) atomicAdd(blended, (unsigned long long)tot);
  }
}

// ---------------------------------------------------------------------------
// Transpose reduction of 10 per-lane values over the warp: 13 shuffles (vs 50 for
// ten butterfly reductions).  On return, the 10 lanes with slot >= 0 hold the warp
// total of component `slot`.
__device__ __forceinline__ void warp_reduce10(const float (&v)[10], int lane, float& out, int& slot) {
  const bool b4 = lane & 16, b3 = lane & 8, b2 = lane & 4, b1 = lane & 2;
  float w6[6];
#pragma unroll
  for (int k = 0; k < 6; ++k) {
    const float lo = v[k], hi = (k + 6 < 10) ? v[k + 6] : 0.f;
    const float send = b4 ? lo : hi, keep = b4 ? hi : lo;
    w6[k] = keep + __shfl_xor_sync(kFull, send, 16);
  }
  float w3[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const float lo = w6[k], hi = w6[k + 3];
    const float send = b3 ? lo : hi, keep = b3 ? hi : lo;
    w3[k] = keep + __shfl_xor_sync(kFull, send, 8);
  }
  float w2[2];
  {
    const float send0 = b2 ? w3[0] : w3[2], keep0 = b2 ? w3[2] : w3[0];
    const float send1 = b2 ? w3[1] : 0.f, keep1 = b2 ? 0.f : w3[1];
    w2[0] = keep0 + __shfl_xor_sync(kFull, send0, 4);
    w2[1] = keep1 + __shfl_xor_sync(kFull, send1, 4);
  }
  float w1;
  {
    const float send = b1 ? w2[0] : w2[1], keep = b1 ? w2[1] : w2[0];
    w1 = keep + __shfl_xor_sync(kFull, send, 2);
  }
  w1 += __shfl_xor_sync(kFull, w1, 1);
  const int gi = (b2 ? 2 : 0) + (b1 ? 1 : 0);
  const int s = (b4 ? 6 : 0) + (b3 ? 3 : 0) + gi;
  out = w1;
  slot = (gi < 3 && s < 10 && !(lane & 1)) ? s : -1;
}

__global__ void __launch_bounds__(kWarpsPerCta * 32) k_render_bwd(DevCam cam, const float4* __restrict__ rec,
                                                                   const int32_t* __restrict__ ids,
                                                                   const int2* __restrict__ ranges,
                                                                   const float* __restrict__ T_final,
                                                                   const int32_t* __restrict__ n_contrib,
                                                                   const float* __restrict__ g_rgb,
                                                                   const float* __restrict__ g_dep,
                                                                   float* __restrict__ sgrad) {
  __shared__ float4 s_rec[kWarpsPerCta][32][3];
  __shared__ int s_gid[kWarpsPerCta][32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tile = blockIdx.x * kWarpsPerCta + warp;
  if (tile >= cam.TX * cam.TY) return;
  const int tx = tile % cam.TX, ty = tile / cam.TX;
  const int px = tx * kTile + (lane & 15);
  const int py0 = ty * kTile + (lane >> 4) * kPix;
  const float pxf = (float)px;
  const int2 rg = ranges[tile];
  const int64_t npix = (int64_t)cam.W * cam.H;

  float T[kPix], Q[kPix], gr[kPix], gg[kPix], gb[kPix], gd[kPix];
  int n[kPix];
  int maxn = 0;
#pragma unroll
  for (int i = 0; i < kPix; ++i) {
    const int py = py0 + i;
    if (px < cam.W && py < cam.H) {
      const int64_t p = (int64_t)py * cam.W + px;
      T[i] = T_final[p];
      n[i] = n_contrib[p];
      gr[i] = g_rgb[p];
      gg[i] = g_rgb[npix + p];
      gb[i] = g_rgb[2 * npix + p];
      gd[i] = g_dep ? g_dep[p] : 0.f;
    } else {
      T[i] = 1.f, n[i] = 0, gr[i] = gg[i] = gb[i] = gd[i] = 0.f;
    }
    Q[i] = T[i] * (gr[i] * cam.bg[0] + gg[i] * cam.bg[1] + gb[i] * cam.bg[2]);
    maxn = max(maxn, n[i]);
  }
  maxn = __reduce_max_sync(kFull, maxn);
  for (int hi = rg.x + maxn; hi > rg.x; hi -= 32) {
    const int lo = max(rg.x, hi - 32);
    const int idx = lo + lane;
    if (idx < hi) {
      const int g = ids[idx];
      const float4* r = rec + 3 * (int64_t)g;
      s_gid[warp][lane] = g;
      s_rec[warp][lane][0] = r[0];
      s_rec[warp][lane][1] = r[1];
      s_rec[warp][lane][2] = r[2];
    }
    __syncwarp();
    for (int j = hi - 1 - lo; j >= 0; --j) {
      float mx, my, z, o, A, B, C, cr, cg, cb;
      load_rec(s_rec[warp][j], mx, my, z, o, A, B, C, cr, cg, cb);
      const Eval e = make_eval(mx, A, B, C, pxf);
      const int pos = lo + j - rg.x;
      float acc_r = 0.f, acc_g = 0.f, acc_b = 0.f, acc_z = 0.f, acc_o = 0.f, s0 = 0.f, s1 = 0.f, s2 = 0.f;
      bool any = false;
#pragma unroll
      for (int i = 0; i < kPix; ++i) {
        float G, dy;
        const bool pok = eval_gauss(e, my, (float)(py0 + i), G, dy);
        const float raw = kExact ? __fmul_rn(o, G) : o * G;
        const float alpha = fminf(kAlphaCap, raw);
        if (pos < n[i] && pok && !(alpha < kAlphaMin)) {
          any = true;
          const float inv = __fdividef(1.f, 1.f - alpha);
          const float Tk = T[i] * inv;
          const float w = alpha * Tk;
          const float u = fmaf(gr[i], cr, fmaf(gg[i], cg, fmaf(gb[i], cb, gd[i] * z)));
          const float dal = Tk * u - inv * Q[i];
          Q[i] = fmaf(w, u, Q[i]);
          T[i] = Tk;
          acc_r = fmaf(gr[i], w, acc_r);
          acc_g = fmaf(gg[i], w, acc_g);
          acc_b = fmaf(gb[i], w, acc_b);
          acc_z = fmaf(gd[i], w, acc_z);
          if (!(raw > kAlphaCap)) {  // capped alpha has no derivative (R18)
            acc_o = fmaf(G, dal, acc_o);
            const float dp = raw * dal;
            const float t = dp * dy;
            s0 += dp;
            s1 += t;
            s2 = fmaf(t, dy, s2);
          }
        }
      }
      if (__any_sync(kFull, any)) {
        const float dx = e.dx;
        float v[10];
        v[0] = -(A * dx * s0 + B * s1);
        v[1] = -(B * dx * s0 + C * s1);
        v[2] = -0.5f * dx * dx * s0;
        v[3] = -dx * s1;
        v[4] = -0.5f * s2;
        v[5] = acc_o;
        v[6] = acc_r;
        v[7] = acc_g;
        v[8] = acc_b;
        v[9] = acc_z;
        float out;
        int slot;
        warp_reduce10(v, lane, out, slot);
        if (slot >= 0) atomicAdd(sgrad + (int64_t)GS_SGRAD_FLOATS * s_gid[warp][j] + slot, out);
      }
    }
    __syncwarp();
  }
}

}  // namespace

void launch_render_fwd(const DevCam& cam, const float* rec, const int32_t* ids, const int32_t* ranges, float* rgb,
                       float* depth, float* T_final, int32_t* n_contrib, unsigned long long* blended,
                       cudaStream_t s) {
  const int NT = cam.TX * cam.TY;
  k_render_fwd<<<ceil_div(NT, kWarpsPerCta), kWarpsPerCta * 32, 0, s>>>(
      cam, reinterpret_cast<const float4*>(rec), ids, reinterpret_cast<const int2*>(ranges), rgb, depth, T_final,
      n_contrib, blended);
  count_launch();
}

void launch_render_bwd(const DevCam& cam, const float* rec, const int32_t* ids, const int32_t* ranges,
                       const float* T_final, const int32_t* n_contrib, const float* g_rgb, const float* g_depth,
                       float* sgrad, cudaStream_t s) {
  const int NT = cam.TX * cam.TY;
  k_render_bwd<<<ceil_div(NT, kWarpsPerCta), kWarpsPerCta * 32, 0, s>>>(
      cam, reinterpret_cast<const float4*>(rec), ids, reinterpret_cast<const int2*>(ranges), T_final, n_contrib,
      g_rgb, g_depth, sgrad);
  count_launch();
}

}  // namespace gsr
