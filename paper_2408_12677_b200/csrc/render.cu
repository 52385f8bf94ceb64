// K6 render_fwd and K7 render_bwd (Eq. 11; backward PAPER.md:147).
//
// Work decomposition (B200-first): one warp per 16x16 tile, split into
// eight 8x4 pixel blocks; lane (lx, ly) owns pixel (lx + 8 (b & 1), ly + 4 (b >> 1))
// of every block b.  A warp gathers 32 of its tile's Gaussian records (48 B each, by
// id, from L2) into shared memory with cp.async, one batch ahead of the one being
// composited; on arrival each lane computes, for its record, the 8-bit mask of the
// blocks the record's alpha >= 1/255 support can reach (exact ellipse-rectangle
// test).  Blocks outside the mask, and blocks whose pixels have all terminated, are
// skipped warp-uniformly; records reaching >= 3 blocks run a branch-free path over
// all 8 blocks (8 independent chains), the others a per-block path.  Each lane's two
// columns share x, so the x part of the exponent (A dx^2, B dx) is computed once per
// record and a pixel costs one FADD + two FFMA + one MUFU.EX2.  The backward reverses the composite
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
constexpr int kDenseBlocks = 3;     // fwd: masks with >= this many 8x4 blocks take the branch-free path
constexpr int kDenseBlocksBwd = 6;  // bwd: same (its per-block body is ~4x longer)
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

// Support box of alpha >= 1/255: {d : 0.5 d^T Sigma_hat^{-1} d <= ln(255 o)} has
// half-extents sqrt(2 L Sigma_hat_xx), sqrt(2 L Sigma_hat_yy).  Returns the 8-bit mask
// of the tile's 8x4 pixel blocks (block b = (b & 1, b >> 1): x offset 8 (b & 1), y
// offset 4 (b >> 1)) that intersect it, with a relative 1% + 1 px safety margin so
// that a skipped pixel can never pass the alpha test (the result is identical to
// evaluating every pixel; the oracle parity tests check it).
__device__ __forceinline__ uint32_t block_mask(float mx, float my, float A, float B, float C, float o, int ox,
                                               int oy) {
  const float L = __logf(255.f * o);
  if (!(L >= -1e-3f)) return 0u;  // o < 1/255: alpha can never reach 1/255
  const float detc = A * C - B * B;
  if (!(detc > 0.f) || !(A > 0.f) || !(C > 0.f)) return 0xffu;
  const float two_l = 2.f * fmaxf(L, 0.f) * 1.0201f;  // (1.01)^2
  const float idet = __fdividef(1.f, detc);
  const float tx = two_l * C * idet, ty = two_l * A * idet;
  const float hx = tx * rsqrtf(fmaxf(tx, 1e-30f)) + 1.f, hy = ty * rsqrtf(fmaxf(ty, 1e-30f)) + 1.f;
  if (!(hx < 1e6f) || !(hy < 1e6f)) return 0xffu;
  // exact test: min over the block of q(d) = A dx^2 + 2 B dx dy + C dy^2 (power = -q/2)
  // against 2 L (with the 1% margin), the block taken as the rectangle of its pixel
  // centres grown by 0.5 px.  The minimum of a convex quadratic over a rectangle is 0
  // if the mean is inside, else on an edge, where it is a 1-D convex quadratic.
  const float qmax = two_l + 1e-3f;
  const float iA = __fdividef(1.f, A), iC = __fdividef(1.f, C);
  const float fx0 = (float)ox - 0.5f - mx, fy0 = (float)oy - 0.5f - my;
  uint32_t m = 0;
#pragma unroll
  for (int b = 0; b < 8; ++b) {
    const float ax0 = fx0 + 8.f * (b & 1), ax1 = ax0 + 8.f;
    const float ay0 = fy0 + 4.f * (b >> 1), ay1 = ay0 + 4.f;
    bool hit = (ax1 >= -hx) && (ax0 <= hx) && (ay1 >= -hy) && (ay0 <= hy);  // bounding-box pre-test
    if (hit && !(ax0 <= 0.f && ax1 >= 0.f && ay0 <= 0.f && ay1 >= 0.f)) {
      float qmin = 3.4e38f;
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const float dx = e ? ax1 : ax0;  // vertical edge dx = const
        const float dy = fminf(fmaxf(-B * dx * iC, ay0), ay1);
        qmin = fminf(qmin, fmaf(A * dx, dx, fmaf(2.f * B * dx, dy, C * dy * dy)));
        const float ey = e ? ay1 : ay0;  // horizontal edge dy = const
        const float ex = fminf(fmaxf(-B * ey * iA, ax0), ax1);
        qmin = fminf(qmin, fmaf(A * ex, ex, fmaf(2.f * B * ex, ey, C * ey * ey)));
      }
      hit = qmin <= qmax;
    }
    m |= hit ? (1u << b) : 0u;
  }
  return m;
}

struct StagedRec {
  float mx, my, z, o, A, B, C, r, g, b;
  uint32_t mask;
};

__device__ __forceinline__ StagedRec load_staged(const float4* s) {
  const float4 q0 = s[0], q1 = s[1], q2 = s[2];
  StagedRec r;
  r.mx = q0.x, r.my = q0.y, r.z = q0.z, r.o = q0.w;
  r.A = q1.x, r.B = q1.y, r.C = q1.z, r.r = q1.w;
  r.g = q2.x, r.b = q2.y, r.mask = __float_as_uint(q2.w);
  return r;
}

// Asynchronous gather of one 48-B record into shared memory (cp.async, L2 -> SMEM,
// bypassing registers) so that batch k+1's gathers are in flight while batch k is
// composited; finish_stage then replaces the rect word with the block mask.
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const uint32_t s = (uint32_t)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void gather_rec_async(const float4* __restrict__ rec, int id, float4* dst) {
  const float4* src = rec + 3 * (int64_t)id;
  cp_async16(dst + 0, src + 0);
  cp_async16(dst + 1, src + 1);
  cp_async16(dst + 2, src + 2);
}
__device__ __forceinline__ void finish_stage(float4* dst, int ox, int oy) {
  const float4 q0 = dst[0], q1 = dst[1];
  reinterpret_cast<float*>(dst + 2)[3] = __uint_as_float(block_mask(q0.x, q0.y, q1.x, q1.y, q1.z, q0.w, ox, oy));
}

// Blocks (8x4) all of whose pixels in this warp have bit set in `bits`.
__device__ __forceinline__ uint32_t blocks_all(uint32_t bits) {
  uint32_t m = 0;
#pragma unroll
  for (int b = 0; b < 8; ++b) m |= __all_sync(kFull, (bits >> b) & 1u) ? (1u << b) : 0u;
  return m;
}

// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kWarpsPerCta * 32) k_render_fwd(DevCam cam, const float4* __restrict__ rec,
                                                                   const int32_t* __restrict__ ids,
                                                                   const int2* __restrict__ ranges,
                                                                   float* __restrict__ out_rgb,
                                                                   float* __restrict__ out_d, float* __restrict__ out_T,
                                                                   int32_t* __restrict__ out_n,
                                                                   unsigned long long* blended,
                                                                   uint8_t* __restrict__ key_blocks) {
  __shared__ float4 s_rec[kWarpsPerCta][2][32][3];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tile = blockIdx.x * kWarpsPerCta + warp;
  if (tile >= cam.TX * cam.TY) return;
  const int tx = tile % cam.TX, ty = tile / cam.TX;
  const int ox = tx * kTile, oy = ty * kTile;
  const int lx = lane & 7, ly = lane >> 3;
  // pixel b of this lane: x = ox + lx + 8 (b & 1), y = oy + ly + 4 (b >> 1)
  const float pxf0 = (float)(ox + lx), pxf1 = pxf0 + 8.f, pyf0 = (float)(oy + ly);
  const int2 rg = ranges[tile];

  float T[kPix], Cr[kPix], Cg[kPix], Cb[kPix], D[kPix];
  int n[kPix];
  uint32_t done = 0;
#pragma unroll
  for (int b = 0; b < kPix; ++b) {
    T[b] = 1.f, Cr[b] = Cg[b] = Cb[b] = D[b] = 0.f, n[b] = 0;
    if (ox + lx + 8 * (b & 1) >= cam.W || oy + ly + 4 * (b >> 1) >= cam.H) done |= 1u << b;
  }
  uint32_t nblend = 0;
  uint32_t bdone = blocks_all(done);
  // double-buffered staging: ids two batches ahead, records one batch ahead
  if (rg.x + lane < rg.y) gather_rec_async(rec, ids[rg.x + lane], s_rec[warp][0][lane]);
  cp_async_commit();
  int nxt_id = (rg.x + 32 + lane < rg.y) ? ids[rg.x + 32 + lane] : -1;
  int buf = 0;
  for (int b0 = rg.x; b0 < rg.y && bdone != 0xffu; b0 += 32, buf ^= 1) {
    if (nxt_id >= 0) gather_rec_async(rec, nxt_id, s_rec[warp][buf ^ 1][lane]);
    cp_async_commit();
    nxt_id = (b0 + 64 + lane < rg.y) ? ids[b0 + 64 + lane] : -1;
    cp_async_wait<1>();
    __syncwarp();
    if (b0 + lane < rg.y) finish_stage(s_rec[warp][buf][lane], ox, oy);
    __syncwarp();
    const int cnt = min(32, rg.y - b0);
    uint32_t kb_mine = 0;  // lane j: 8x4 blocks in which key b0 + j composited >= 1 pixel
    for (int j = 0; j < cnt; ++j) {
      const StagedRec q = load_staged(s_rec[warp][buf][j]);
      const uint32_t m = q.mask & ~bdone;
      if (m == 0) continue;
      const int pos1 = b0 + j - rg.x + 1;
      const Eval e0 = make_eval(q.mx, q.A, q.B, q.C, pxf0);
      const Eval e1 = make_eval(q.mx, q.A, q.B, q.C, pxf1);
      uint32_t lm = 0;  // this lane's composited blocks for this key
      if (kExact) {
#pragma unroll
        for (int b = 0; b < kPix; ++b) {
          if (!((m >> b) & 1u)) continue;
          float G, dy;
          const bool pok = eval_gauss((b & 1) ? e1 : e0, q.my, pyf0 + 4.f * (b >> 1), G, dy);
          const float alpha = fminf(kAlphaCap, __fmul_rn(q.o, G));
          const bool act = !((done >> b) & 1u) && pok && !(alpha < kAlphaMin);
          const float Tn = __fmul_rn(T[b], __fsub_rn(1.f, alpha));
          const bool stop = act && (Tn < kTStop);
          if (stop) done |= 1u << b;
          if (act && !stop) {
            const float w = __fmul_rn(alpha, T[b]);
            Cr[b] = __fadd_rn(Cr[b], __fmul_rn(q.r, w));
            Cg[b] = __fadd_rn(Cg[b], __fmul_rn(q.g, w));
            Cb[b] = __fadd_rn(Cb[b], __fmul_rn(q.b, w));
            D[b] = __fadd_rn(D[b], __fmul_rn(q.z, w));
            T[b] = Tn;
            n[b] = pos1;
            ++nblend;
            lm |= 1u << b;
          }
        }
      } else {
        const float dy0 = q.my - pyf0;
        if (__popc(m) >= kDenseBlocks) {
          // dense: all 8 blocks without branches (8 independent chains for the
          // scheduler); masked-out blocks and failing pixels contribute exact zeros
          float al[kPix];
          bool ac[kPix];
#pragma unroll
          for (int b = 0; b < kPix; ++b) {
            const Eval& e = (b & 1) ? e1 : e0;
            const float dy = dy0 - 4.f * (b >> 1);
            const float p2 = fmaf(dy, fmaf(e.c2, dy, e.b0), e.a0);
            al[b] = fminf(kAlphaCap, q.o * ex2_approx(p2));
            ac[b] = ((m >> b) & 1u) && (p2 <= 0.f) && (al[b] >= kAlphaMin) && !((done >> b) & 1u);
          }
#pragma unroll
          for (int b = 0; b < kPix; ++b) {
            const float Tn = fmaf(-al[b], T[b], T[b]);
            const bool stop = ac[b] && (Tn < kTStop);
            const bool comp = ac[b] && !stop;
            done |= stop ? (1u << b) : 0u;
            lm |= comp ? (1u << b) : 0u;
            const float w = comp ? al[b] * T[b] : 0.f;
            Cr[b] = fmaf(q.r, w, Cr[b]);
            Cg[b] = fmaf(q.g, w, Cg[b]);
            Cb[b] = fmaf(q.b, w, Cb[b]);
            D[b] = fmaf(q.z, w, D[b]);
            T[b] = comp ? Tn : T[b];
            n[b] = comp ? pos1 : n[b];
            nblend += comp ? 1u : 0u;
          }
        } else {
          // sparse: per block, skipped (warp-uniform) when masked out or no lane passes
#pragma unroll
          for (int b = 0; b < kPix; ++b) {
            if (!((m >> b) & 1u)) continue;
            const Eval& e = (b & 1) ? e1 : e0;
            const float dy = dy0 - 4.f * (b >> 1);
            const float p2 = fmaf(dy, fmaf(e.c2, dy, e.b0), e.a0);
            const float alpha = fminf(kAlphaCap, q.o * ex2_approx(p2));
            const bool act = (p2 <= 0.f) && (alpha >= kAlphaMin) && !((done >> b) & 1u);
            if (!__any_sync(kFull, act)) continue;
            const float Tn = fmaf(-alpha, T[b], T[b]);
            const bool stop = act && (Tn < kTStop);
            const bool comp = act && !stop;
            done |= stop ? (1u << b) : 0u;
            lm |= comp ? (1u << b) : 0u;
            const float w = comp ? alpha * T[b] : 0.f;
            Cr[b] = fmaf(q.r, w, Cr[b]);
            Cg[b] = fmaf(q.g, w, Cg[b]);
            Cb[b] = fmaf(q.b, w, Cb[b]);
            D[b] = fmaf(q.z, w, D[b]);
            T[b] = comp ? Tn : T[b];
            n[b] = comp ? pos1 : n[b];
            nblend += comp ? 1u : 0u;
          }
        }
      }
      const uint32_t cm = __reduce_or_sync(kFull, lm);
      kb_mine = (lane == j) ? cm : kb_mine;
      if ((j & 7) == 7) bdone = blocks_all(done);
    }
    if (key_blocks && b0 + lane < rg.y) key_blocks[b0 + lane] = (uint8_t)kb_mine;
    bdone = blocks_all(done);
    __syncwarp();
  }
  cp_async_wait<0>();
  const int64_t npix = (int64_t)cam.W * cam.H;
#pragma unroll
  for (int b = 0; b < kPix; ++b) {
    const int px = ox + lx + 8 * (b & 1), py = oy + ly + 4 * (b >> 1);
    if (px < cam.W && py < cam.H) {
      const int64_t p = (int64_t)py * cam.W + px;
      if (kExact) {
        out_rgb[p] = __fadd_rn(Cr[b], __fmul_rn(T[b], cam.bg[0]));
        out_rgb[npix + p] = __fadd_rn(Cg[b], __fmul_rn(T[b], cam.bg[1]));
        out_rgb[2 * npix + p] = __fadd_rn(Cb[b], __fmul_rn(T[b], cam.bg[2]));
      } else {
        out_rgb[p] = fmaf(T[b], cam.bg[0], Cr[b]);
        out_rgb[npix + p] = fmaf(T[b], cam.bg[1], Cg[b]);
        out_rgb[2 * npix + p] = fmaf(T[b], cam.bg[2], Cb[b]);
      }
      out_d[p] = D[b];
      out_T[p] = T[b];
      out_n[p] = n[b];
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
                                                                   const uint8_t* __restrict__ key_blocks,
                                                                   float* __restrict__ sgrad) {
  __shared__ float4 s_rec[kWarpsPerCta][2][32][3];
  __shared__ int s_gid[kWarpsPerCta][2][32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tile = blockIdx.x * kWarpsPerCta + warp;
  if (tile >= cam.TX * cam.TY) return;
  const int tx = tile % cam.TX, ty = tile / cam.TX;
  const int ox = tx * kTile, oy = ty * kTile;
  const int lx = lane & 7, ly = lane >> 3;
  const float pxf0 = (float)(ox + lx), pxf1 = pxf0 + 8.f, pyf0 = (float)(oy + ly);
  const int2 rg = ranges[tile];
  const int64_t npix = (int64_t)cam.W * cam.H;

  float T[kPix], Q[kPix], gr[kPix], gg[kPix], gb[kPix], gd[kPix];
  int n[kPix];
  int bmaxn[kPix];  // per 8x4 block: max n_contrib over its 32 pixels (warp-uniform)
  int maxn = 0;
#pragma unroll
  for (int b = 0; b < kPix; ++b) {
    const int px = ox + lx + 8 * (b & 1), py = oy + ly + 4 * (b >> 1);
    if (px < cam.W && py < cam.H) {
      const int64_t p = (int64_t)py * cam.W + px;
      T[b] = T_final[p];
      n[b] = n_contrib[p];
      gr[b] = g_rgb[p];
      gg[b] = g_rgb[npix + p];
      gb[b] = g_rgb[2 * npix + p];
      gd[b] = g_dep ? g_dep[p] : 0.f;
    } else {
      T[b] = 1.f, n[b] = 0, gr[b] = gg[b] = gb[b] = gd[b] = 0.f;
    }
    Q[b] = T[b] * (gr[b] * cam.bg[0] + gg[b] * cam.bg[1] + gb[b] * cam.bg[2]);
    bmaxn[b] = __reduce_max_sync(kFull, n[b]);
    maxn = max(maxn, bmaxn[b]);
  }
  // double-buffered staging (back to front): ids + key masks two batches ahead,
  // records one ahead.  With the forward's key masks, keys that composited nothing
  // in this tile are neither gathered nor visited.
  int hi = rg.x + maxn;
  auto load_key = [&](int h, int& id, uint32_t& kb) {
    id = -1, kb = 0;
    if (h > rg.x) {
      const int l = max(rg.x, h - 32);
      if (l + lane < h) {
        id = ids[l + lane];
        kb = key_blocks ? (uint32_t)key_blocks[l + lane] : 0xffu;
      }
    }
  };
  auto stage = [&](int b, int id, uint32_t kb) {
    if (id >= 0 && kb) {
      s_gid[warp][b][lane] = id;
      gather_rec_async(rec, id, s_rec[warp][b][lane]);
    }
  };
  int id1;
  uint32_t kb_cur, kb1;
  load_key(hi, id1, kb_cur);
  stage(0, id1, kb_cur);
  cp_async_commit();
  load_key(hi - 32, id1, kb1);
  int buf = 0;
  for (; hi > rg.x; hi -= 32, buf ^= 1) {
    const int lo = max(rg.x, hi - 32);
    stage(buf ^ 1, id1, kb1);
    cp_async_commit();
    int id2;
    uint32_t kb2;
    load_key(hi - 64, id2, kb2);
    cp_async_wait<1>();
    __syncwarp();
    if (!key_blocks && lo + lane < hi) finish_stage(s_rec[warp][buf][lane], ox, oy);
    __syncwarp();
    uint32_t live = __ballot_sync(kFull, kb_cur != 0);
    while (live) {
      const int j = 31 - __clz(live);  // back to front
      live &= ~(1u << j);
      const StagedRec q = load_staged(s_rec[warp][buf][j]);
      const int pos = lo + j - rg.x;
      uint32_t m;
      if (key_blocks) {
        m = __shfl_sync(kFull, kb_cur, j);  // blocks the forward composited this key in
      } else {
        m = q.mask;
#pragma unroll
        for (int b = 0; b < kPix; ++b)
          if (pos >= bmaxn[b]) m &= ~(1u << b);
        if (m == 0) continue;
      }
      const Eval e0 = make_eval(q.mx, q.A, q.B, q.C, pxf0);
      const Eval e1 = make_eval(q.mx, q.A, q.B, q.C, pxf1);
      float acc_r = 0.f, acc_g = 0.f, acc_b = 0.f, acc_z = 0.f, acc_o = 0.f;
      float s0[2] = {0.f, 0.f}, s1[2] = {0.f, 0.f}, s2 = 0.f;
      bool any = false;  // warp-uniform
      if (!kExact && __popc(m) >= kDenseBlocksBwd) {
        // dense: all 8 blocks without branches; invalid pixels contribute exact zeros
        const float dy0 = q.my - pyf0;
        float Gv[kPix], rawv[kPix];
        bool vv[kPix];
        bool lane_any = false;
#pragma unroll
        for (int b = 0; b < kPix; ++b) {
          const Eval& e = (b & 1) ? e1 : e0;
          const float dy = dy0 - 4.f * (b >> 1);
          const float p2 = fmaf(dy, fmaf(e.c2, dy, e.b0), e.a0);
          Gv[b] = ex2_approx(p2);
          rawv[b] = q.o * Gv[b];
          vv[b] = ((m >> b) & 1u) && pos < n[b] && (p2 <= 0.f) && (fminf(kAlphaCap, rawv[b]) >= kAlphaMin);
          lane_any |= vv[b];
        }
#pragma unroll
        for (int b = 0; b < kPix; ++b) {
          const bool valid = vv[b];
          const float dy = dy0 - 4.f * (b >> 1);
          const float alpha = fminf(kAlphaCap, rawv[b]);
          const float inv = __fdividef(1.f, 1.f - alpha);
          const float Tk = T[b] * inv;
          const float w = valid ? alpha * Tk : 0.f;
          const float u = fmaf(gr[b], q.r, fmaf(gg[b], q.g, fmaf(gb[b], q.b, gd[b] * q.z)));
          const bool unc = valid && !(rawv[b] > kAlphaCap);
          const float dal = unc ? (Tk * u - inv * Q[b]) : 0.f;
          Q[b] = fmaf(w, u, Q[b]);
          T[b] = valid ? Tk : T[b];
          acc_r = fmaf(gr[b], w, acc_r);
          acc_g = fmaf(gg[b], w, acc_g);
          acc_b = fmaf(gb[b], w, acc_b);
          acc_z = fmaf(gd[b], w, acc_z);
          acc_o = fmaf(Gv[b], dal, acc_o);
          const float dp = rawv[b] * dal;
          const float t = dp * dy;
          s0[b & 1] += dp;
          s1[b & 1] += t;
          s2 = fmaf(t, dy, s2);
        }
        any = __any_sync(kFull, lane_any);
        m = 0;  // skip the sparse loop below
      }
#pragma unroll
      for (int b = 0; b < kPix; ++b) {
        if (!((m >> b) & 1u)) continue;
        float G, dy;
        const bool pok = eval_gauss((b & 1) ? e1 : e0, q.my, pyf0 + 4.f * (b >> 1), G, dy);
        const float raw = kExact ? __fmul_rn(q.o, G) : q.o * G;
        const float alpha = fminf(kAlphaCap, raw);
        const bool valid = pos < n[b] && pok && !(alpha < kAlphaMin);
        if (!__any_sync(kFull, valid)) continue;
        any = true;
        // predicated body: invalid lanes contribute exact zeros and keep their state
        const float inv = __fdividef(1.f, 1.f - alpha);
        const float Tk = T[b] * inv;
        const float w = valid ? alpha * Tk : 0.f;
        const float u = fmaf(gr[b], q.r, fmaf(gg[b], q.g, fmaf(gb[b], q.b, gd[b] * q.z)));
        const bool unc = valid && !(raw > kAlphaCap);  // capped alpha has no derivative (R18)
        const float dal = unc ? (Tk * u - inv * Q[b]) : 0.f;
        Q[b] = fmaf(w, u, Q[b]);
        T[b] = valid ? Tk : T[b];
        acc_r = fmaf(gr[b], w, acc_r);
        acc_g = fmaf(gg[b], w, acc_g);
        acc_b = fmaf(gb[b], w, acc_b);
        acc_z = fmaf(gd[b], w, acc_z);
        acc_o = fmaf(G, dal, acc_o);
        const float dp = raw * dal;
        const float t = dp * dy;
        s0[b & 1] += dp;
        s1[b & 1] += t;
        s2 = fmaf(t, dy, s2);
      }
      if (any) {
        const float dx0 = e0.dx, dx1 = e1.dx;
        const float sx = dx0 * s0[0] + dx1 * s0[1];        // sum dp dx
        const float sxx = dx0 * dx0 * s0[0] + dx1 * dx1 * s0[1];  // sum dp dx^2
        const float sy = s1[0] + s1[1];                      // sum dp dy
        const float sxy = dx0 * s1[0] + dx1 * s1[1];         // sum dp dx dy
        float v[10];
        v[0] = -(q.A * sx + q.B * sy);
        v[1] = -(q.B * sx + q.C * sy);
        v[2] = -0.5f * sxx;
        v[3] = -sxy;
        v[4] = -0.5f * s2;
        v[5] = acc_o;
        v[6] = acc_r;
        v[7] = acc_g;
        v[8] = acc_b;
        v[9] = acc_z;
        float out;
        int slot;
        warp_reduce10(v, lane, out, slot);
        if (slot >= 0) atomicAdd(sgrad + (int64_t)GS_SGRAD_FLOATS * s_gid[warp][buf][j] + slot, out);
      }
    }
    __syncwarp();
    kb_cur = kb1, id1 = id2, kb1 = kb2;
  }
  cp_async_wait<0>();
}

}  // namespace

void launch_render_fwd(const DevCam& cam, const float* rec, const int32_t* ids, const int32_t* ranges, float* rgb,
                       float* depth, float* T_final, int32_t* n_contrib, unsigned long long* blended,
                       uint8_t* key_blocks, cudaStream_t s) {
  const int NT = cam.TX * cam.TY;
  k_render_fwd<<<ceil_div(NT, kWarpsPerCta), kWarpsPerCta * 32, 0, s>>>(
      cam, reinterpret_cast<const float4*>(rec), ids, reinterpret_cast<const int2*>(ranges), rgb, depth, T_final,
      n_contrib, blended, key_blocks);
  count_launch();
}

void launch_render_bwd(const DevCam& cam, const float* rec, const int32_t* ids, const int32_t* ranges,
                       const float* T_final, const int32_t* n_contrib, const float* g_rgb, const float* g_depth,
                       const uint8_t* key_blocks, float* sgrad, cudaStream_t s) {
  const int NT = cam.TX * cam.TY;
  k_render_bwd<<<ceil_div(NT, kWarpsPerCta), kWarpsPerCta * 32, 0, s>>>(
      cam, reinterpret_cast<const float4*>(rec), ids, reinterpret_cast<const int2*>(ranges), T_final, n_contrib,
      g_rgb, g_depth, key_blocks, sgrad);
  count_launch();
}

}  // namespace gsr
