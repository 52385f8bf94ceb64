#include <atomic>
// K6 render_fwd and K7 render_bwd (Eq. 11; backward PAPER.md:147).
//
// Work decomposition (B200-first): one warp per 16x16 tile, split into
// eight 8x4 pixel blocks; lane (lx, ly) owns pixel (lx + 8 (b & 1), ly + 4 (b >> 1))
// of every block b.  A warp gathers 32 of its tile's Gaussian records (48 B each, by
// id, from L2) into shared memory with cp.async, one batch ahead of the one being
// composited; on arrival each lane rewrites its record into the form the inner loops
// consume and computes the 8-bit mask of the blocks the record's alpha >= 1/255
// support can reach (exact ellipse-rectangle test).  Only keys whose mask meets a
// block with live pixels are visited; records reaching >= kDenseBlocks blocks run a
// branch-free path over all 8 blocks (8 independent chains), the others a per-block
// path skipped warp-uniformly where no lane passes.
//
// The inner loops are shaped by the measured B200 issue rates (profiles/r01/
// pipe_rates.txt): FP32 FMA-pipe 1 warp-instruction/clk/SMSP, ALU pipe (compares,
// selects, logic, FMNMX) 1/2, MUFU 1/8, and FFMA2 no faster than two FFMAs.  So:
//  * log2(alpha) = lo2 + Ah dx^2 + Bh dx dy + Ch dy^2 with lo2 = log2(o) folded in
//    (one FADD + two FFMA + one MUFU.EX2 per pixel, no FMUL by o);
//  * a terminated pixel is marked by the sign of T (T := -|T|), which makes every
//    later T - alpha T negative and so fails the same T >= 1e-4 test that decides
//    compositing: no per-pixel "done" bit tests or selects;
//  * the composite updates are predicated on one compare; the blended count is
//    popc of the per-key lane mask, not a per-pixel add;
//  * opacity <= 0.9 records skip the 0.99 cap (alpha cannot reach it), positive-
//    definite conics skip the "power > 0" test (it cannot fire in exact arithmetic:
//    reading R27); the rare others take a general per-block path with both.
// The backward reverses the composite with T_k = T_{k+1} / (1 - alpha_k), keeps the
// suffix term as one scalar per pixel (Q = sum_ch g_ch S^C_ch + g_D S^D), accumulates
// the moments of dL/dpower over the lane's pixels per column (sum dp, dp dy, dp dy^2)
// and forms the 10 screen-space gradient components once per key, reduces them across
// the warp (= the whole tile) with a 13-shuffle transpose reduction so that 10 lanes
// issue ONE red.global.add.f32 instruction per (tile, Gaussian).
//
// GSR_EXACT_EXP builds (libgsr_exact.so) run separate kernels that evaluate the
// exponent, alpha, transmittance and accumulation in the oracle's fp32 operation
// order with exp computed in double (reading R9): the forward is then bit-identical
// to the fp32 oracle.
#include <cstdlib>

#include "gsr_internal.cuh"

namespace gsr {
namespace {

[[maybe_unused]] constexpr int kWarpsPerCta = 4;
// Resident warps per SM the fast kernels are compiled for (register cap 65536 /
// (32 x warps)); the register file is split per SM sub-partition, so 16 warps = 4
// per SMSP at <= 128 registers, 20 = 5 per SMSP at <= 102 (measured: 16 -> 20 warps
// gives 7.28 -> 6.92 ms per scannetpp step, 24 spills and loses).  A/B: -DGSR_FWD_MINW=...
#ifndef GSR_FWD_MINW
#define GSR_FWD_MINW 20
#endif
#ifndef GSR_BWD_MINW
#define GSR_BWD_MINW 20
#endif
[[maybe_unused]] constexpr int kFwdMinWarps = GSR_FWD_MINW, kBwdMinWarps = GSR_BWD_MINW;
[[maybe_unused]] constexpr int kPix = 8;             // pixels per lane
#ifndef GSR_BWD_PAIR
#define GSR_BWD_PAIR 1
#endif
#ifndef GSR_DEAD_EVERY
#define GSR_DEAD_EVERY 0  // forward: keys between mid-batch re-checks of the blocks whose pixels all terminated (0: batch ends only; r02: 8 -> 16 -> 0)
#endif
#ifndef GSR_FWD_KB_SMEM
#define GSR_FWD_KB_SMEM 0  // 1: the per-key block masks collected in shared memory (one STS per key; measured slower)
#endif
#ifndef GSR_DENSE_FWD
#define GSR_DENSE_FWD 1  // r02: 1 (every non-general key branch-free) -> fwd -3.5% at config 4 and scannetpp vs 2
#endif
// Dense (branch-free) paths on packed FP32 pairs (FFMA2 / FMUL2, fma.rn.f32x2 etc.):
// the two pixels of a lane in one block row (columns lx, lx + 8) share dy, so their
// per-pixel arithmetic is issued as one paired instruction -- the same IEEE fp32
// operations per element, half the issue slots (the render kernels are issue-bound).
#ifndef GSR_FFMA2
#define GSR_FFMA2 1
#endif
#ifndef GSR_FFMA2_FWD
#define GSR_FFMA2_FWD GSR_FFMA2
#endif
#ifndef GSR_FFMA2_GEO
#define GSR_FFMA2_GEO GSR_FFMA2  // forward: the per-key column / row terms (make_geo) as packed pairs
#endif
#ifndef GSR_FFMA2_GEO_BWD
#define GSR_FFMA2_GEO_BWD 0  // backward: measured slower (+24 B of spills in the register-capped kernel)
#endif
#ifndef GSR_DENSE_BWD
#define GSR_DENSE_BWD 5
#endif
[[maybe_unused]] constexpr int kDenseBlocks = GSR_DENSE_FWD;     // fwd: masks with >= this many 8x4 blocks take the branch-free path
[[maybe_unused]] constexpr int kDenseBlocksBwd = GSR_DENSE_BWD;  // bwd: same (its per-block body is ~2x longer)
[[maybe_unused]] constexpr float kLog2e = 1.4426950408889634f;
[[maybe_unused]] constexpr float kAlphaMin = 1.0f / 255.0f;
[[maybe_unused]] constexpr float kTStop = 1e-4f;
[[maybe_unused]] constexpr float kAlphaCap = 0.99f;
[[maybe_unused]] constexpr float kUncappedO = 0.9f;         // o <= this: alpha = o exp(power) < 0.99 (no cap)
[[maybe_unused]] constexpr uint32_t kFlagGeneral = 1u << 8;  // conic not positive definite: keep the power > 0 test
[[maybe_unused]] constexpr uint32_t kFlagCap = 1u << 9;      // o > kUncappedO: the 0.99 cap may bind
[[maybe_unused]] constexpr int kGidShift = 10;                // backward, kPack: Gaussian id in bits 10-31
#ifndef GSR_BWD_PAIR_INPLACE
#define GSR_BWD_PAIR_INPLACE 1
#endif
#ifndef GSR_BWD_PACK
#define GSR_BWD_PACK 1
#endif
[[maybe_unused]] constexpr float kHalfL2e = -0.5f * kLog2e;  // Ah = kHalfL2e A, Ch = kHalfL2e C
[[maybe_unused]] constexpr float kNegL2e = -kLog2e;          // Bh = kNegL2e B

[[maybe_unused]] __device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
[[maybe_unused]] __device__ __forceinline__ float lg2_approx(float x) {
  float y;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
[[maybe_unused]] __device__ __forceinline__ float rcp_approx(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// one MUFU.SQRT (relative error ~2^-22); only for the conservative block masks, whose
// 1% quadratic margin and 0.01 px slack dwarf it -- never for a value the oracle checks
[[maybe_unused]] __device__ __forceinline__ float sqrt_approx(float x) {
  float y;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
#ifndef GSR_MASK_SQRT_APPROX
#define GSR_MASK_SQRT_APPROX 1
#endif
#if GSR_MASK_SQRT_APPROX
#define GSR_MASK_SQRT sqrt_approx
#else
#define GSR_MASK_SQRT sqrtf
#endif

// Support box of alpha >= 1/255: {d : 0.5 d^T Sigma_hat^{-1} d <= ln(255 o)} has
// half-extents sqrt(2 L Sigma_hat_xx), sqrt(2 L Sigma_hat_yy).  Returns the 8-bit mask
// of the tile's 8x4 pixel blocks (block b = (b & 1, b >> 1): x offset 8 (b & 1), y
// offset 4 (b >> 1)) that intersect it, with a relative 1% + 1 px safety margin so
// that a skipped pixel can never pass the alpha test (the result is identical to
// evaluating every pixel; the oracle parity tests check it).
[[maybe_unused]] __device__ __forceinline__ uint32_t block_mask(float mx, float my, float A, float B, float C, float o, int ox,
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

// Same contract as block_mask (a superset of the blocks holding a pixel with alpha >=
// 1/255, the same 1% margin), computed per row of blocks instead of per block: the
// ellipse E = {q(d) <= qmax} meets the horizontal slab y in [y0, y1] exactly over
// the x-interval [xl, xr] with xr = hx if the rightmost point of E (y = -B hx / C) lies
// in the slab, else the larger right end of E's chords on the slab's two edge lines
// (x_right(y) is concave, so off its peak it is monotone on the slab); xl likewise.
// Five edge-line chords (one sqrt each) serve the four block rows: ~1/2 the
// instructions of block_mask's per-block edge minimisation.
[[maybe_unused]] __device__ __forceinline__ uint32_t block_mask_rows(float mx, float my, float A, float B, float C, float o, int ox,
                                                    int oy) {
  const float L = __logf(255.f * o);
  if (!(L >= -1e-3f)) return 0u;  // o < 1/255: alpha can never reach 1/255
  const float det = A * C - B * B;
  if (!(det > 0.f) || !(A > 0.f) || !(C > 0.f)) return 0xffu;
  const float qmax = 2.f * fmaxf(L, 0.f) * 1.0201f + 1e-3f;  // (1.01)^2 margin, as block_mask
  const float idet = __fdividef(1.f, det), iA = __fdividef(1.f, A);
  const float hx = GSR_MASK_SQRT(qmax * C * idet), hy = GSR_MASK_SQRT(qmax * A * idet);
  if (!(hx < 1e6f) || !(hy < 1e6f)) return 0xffu;
  const float yR = -B * hx * __fdividef(1.f, C);  // y of the rightmost point; leftmost at -yR
  const float fx0 = (float)ox - 0.5f - mx, fy0 = (float)oy - 0.5f - my;
  const float kSlack = 1e-2f;  // px, on top of the 1% quadratic margin
  float xr[5], xl[5];
#pragma unroll
  for (int k = 0; k < 5; ++k) {
    const float y = fy0 + 4.f * k;
    const float s = GSR_MASK_SQRT(fmaxf(fmaf(-det, y * y, A * qmax), 0.f));
    const bool in = fabsf(y) <= hy + kSlack;
    xr[k] = in ? (s - B * y) * iA : -3.4e38f;
    xl[k] = in ? (-s - B * y) * iA : 3.4e38f;
  }
  uint32_t m = 0;
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const float y0 = fy0 + 4.f * r, y1 = y0 + 4.f;
    if (!(y1 >= -hy - kSlack && y0 <= hy + kSlack)) continue;
    const float r_hi = (yR >= y0 && yR <= y1) ? hx : fmaxf(xr[r], xr[r + 1]);
    const float l_lo = (-yR >= y0 && -yR <= y1) ? -hx : fminf(xl[r], xl[r + 1]);
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      const float x0 = fx0 + 8.f * c, x1 = x0 + 8.f;
      if (r_hi + kSlack >= x0 && l_lo - kSlack <= x1) m |= 1u << (2 * r + c);
    }
  }
  return m;
}

// Asynchronous gather of one 48-B record into shared memory (cp.async, L2 -> SMEM,
// bypassing registers) so that batch k+1's gathers are in flight while batch k is
// composited.
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

// Transpose reduction of 10 per-lane values over the warp: 13 shuffles (vs 50 for
// ten butterfly reductions).  On return, the 10 lanes with slot >= 0 hold the warp
// total of component `slot`.
[[maybe_unused]] __device__ __forceinline__ void warp_reduce10(const float (&v)[10], int lane, float& out, int& slot) {
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

// Upstream gradient of one pixel: dL/drgb, dL/ddepth read from the caller's buffers, or,
// with the fused Eq. 12 loss (gs_render_bwd_screen_l1), computed here from the rendered
// and target images exactly as gs_l1_loss_grad does (sign(residual) x 1/(3 npix), x
// w_depth/npix for depth, sign(0) = 0, invalid targets masked per R43), the pixel's
// loss terms added to `lsum`.
struct L1Fuse {
  const float *rgb, *depth, *trgb, *tdep;
  float sc, sd;
  float* loss;
};
__device__ __forceinline__ float l1_sign(float r, float s) { return r > 0.f ? s : (r < 0.f ? -s : 0.f); }
__device__ __forceinline__ void upstream(const L1Fuse& l1, const float* __restrict__ g_rgb,
                                         const float* __restrict__ g_dep, int64_t npix, int64_t p, float& gr,
                                         float& gg, float& gb, float& gd, float& lsum) {
  if (l1.trgb) {
    const float r0 = l1_res_rgb(l1.rgb[p], l1.trgb[p]), r1 = l1_res_rgb(l1.rgb[npix + p], l1.trgb[npix + p]);
    const float r2 = l1_res_rgb(l1.rgb[2 * npix + p], l1.trgb[2 * npix + p]);
    const float rd = l1_res_depth(l1.depth[p], l1.tdep[p]);
    gr = l1_sign(r0, l1.sc), gg = l1_sign(r1, l1.sc), gb = l1_sign(r2, l1.sc), gd = l1_sign(rd, l1.sd);
    lsum += fabsf(r0) * l1.sc + fabsf(r1) * l1.sc + fabsf(r2) * l1.sc + fabsf(rd) * l1.sd;
  } else {
    gr = g_rgb[p], gg = g_rgb[npix + p], gb = g_rgb[2 * npix + p];
    gd = g_dep ? g_dep[p] : 0.f;
  }
}
__device__ __forceinline__ void l1_commit(const L1Fuse& l1, float lsum, int lane) {
  if (l1.loss) {
    for (int o = 16; o > 0; o >>= 1) lsum += __shfl_xor_sync(kFull, lsum, o);
    if (lane == 0 && lsum != 0.f) atomicAdd(l1.loss, lsum);
  }
}

#ifndef GSR_EXACT_EXP
// ===========================================================================
// Fast path (libgsr.so)
// ===========================================================================

// Two keys' 10-component reductions in one transpose (GSR_BWD_PAIR): the first stage
// (xor 16) of each key alone -- 5 shuffles, leaving components k (lanes with bit 4
// clear) or k + 5 (set) -- then both keys' 5 + 5 halves together (xor 8, 4, 2, 1: 11
// shuffles), 21 in all instead of 26, and one RED instruction for both keys' 20 values.
__device__ __forceinline__ void reduce_half10(const float (&v)[10], int lane, float (&h)[5]) {
  const bool b4 = lane & 16;
#pragma unroll
  for (int k = 0; k < 5; ++k) {
    const float send = b4 ? v[k] : v[k + 5], keep = b4 ? v[k + 5] : v[k];
    h[k] = keep + __shfl_xor_sync(kFull, send, 16);
  }
}
// Keys a (gid ga) and b (gid gb; gb < 0: none) reduced to their warp totals and added to
// the screen gradients: 20 lanes, component (bit 4 ? 5 : 0) + d of key (bit 3 ? b : a).
__device__ __forceinline__ void reduce_pair_commit(const float (&a)[5], const float (&b)[5], int ga, int gb, int lane,
                                                   float* __restrict__ sgrad) {
  const bool b3 = lane & 8, b2 = lane & 4, b1 = lane & 2, b0 = lane & 1;
  float d[5];
#pragma unroll
  for (int k = 0; k < 5; ++k) {
    const float send = b3 ? a[k] : b[k], keep = b3 ? b[k] : a[k];
    d[k] = keep + __shfl_xor_sync(kFull, send, 8);
  }
  float e[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const float lo = d[k], hi = (k + 3 < 5) ? d[k + 3] : 0.f;
    const float send = b2 ? lo : hi, keep = b2 ? hi : lo;
    e[k] = keep + __shfl_xor_sync(kFull, send, 4);
  }
  float f[2];
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const float lo = e[k], hi = (k + 2 < 3) ? e[k + 2] : 0.f;
    const float send = b1 ? lo : hi, keep = b1 ? hi : lo;
    f[k] = keep + __shfl_xor_sync(kFull, send, 2);
  }
  const float send = b0 ? f[0] : f[1], keep = b0 ? f[1] : f[0];
  const float out = keep + __shfl_xor_sync(kFull, send, 1);
  const int ei = (b1 ? 2 : 0) + (b0 ? 1 : 0), di = (b2 ? 3 : 0) + ei;
  const int g = b3 ? gb : ga;
  if (ei < 3 && di < 5 && g >= 0) atomicAdd(sgrad + (int64_t)GS_SGRAD_FLOATS * g + ((lane & 16) ? 5 : 0) + di, out);
}

// Staged record (3 x float4 in shared memory), rewritten in place by its lane:
//   (mx, my, z, lo2) (Ah, Bh, Ch, r) (g, b, 1/o, mask | flags)
// lo2 = log2(o), Ah = -log2(e)/2 A, Bh = -log2(e) B, Ch = -log2(e)/2 C, so that
// log2(alpha) = lo2 + Ah dx^2 + Bh dx dy + Ch dy^2 = lo2 + log2(e) power.  Every value
// is computed by one fixed instruction sequence, so the forward and the backward
// take identical decisions.
template <bool kMask>
__device__ __forceinline__ void stage_fast(float4* dst, int ox, int oy) {
  const float4 q0 = dst[0], q1 = dst[1];
  const float A = q1.x, B = q1.y, C = q1.z, o = q0.w;
  uint32_t fl = kMask ? block_mask_rows(q0.x, q0.y, A, B, C, o, ox, oy) : 0xffu;
  const float detc = __fsub_rn(__fmul_rn(A, C), __fmul_rn(B, B));
  if (!(detc > 0.f && A > 0.f && C > 0.f)) fl |= kFlagGeneral;
  if (!(o <= kUncappedO)) fl |= kFlagCap;
  dst[0].w = lg2_approx(o);
  dst[1] = make_float4(__fmul_rn(kHalfL2e, A), __fmul_rn(kNegL2e, B), __fmul_rn(kHalfL2e, C), q1.w);
  float* q2 = reinterpret_cast<float*>(dst + 2);
  q2[2] = rcp_approx(o);  // the backward's dalpha/do = alpha / o (keys with o < 1/255 are never visited)
  q2[3] = __uint_as_float(fl);
}

// Per (key, lane): the column terms of log2(alpha) for the lane's two pixel columns
// and the four row offsets.  p2(b) = fma(dy_r, fma(Ch, dy_r, b0_e), a0_e), e = b & 1,
// r = b >> 1.
struct Geo {
  float dx[2], a0[2], b0[2], dy[4];
};
template <bool kPair>
__device__ __forceinline__ Geo make_geo(const float4& q0, const float4& q1, float pxf0, float pyf0) {
  Geo g;
  g.dx[0] = __fsub_rn(q0.x, pxf0);
  g.dx[1] = __fsub_rn(g.dx[0], 8.f);
  if constexpr (kPair) {
  // the two columns' terms as packed pairs (per element the same IEEE operations)
  const float2 dx = make_float2(g.dx[0], g.dx[1]);
  const float2 a0 = __ffma2_rn(__fmul2_rn(make_float2(q1.x, q1.x), dx), dx, make_float2(q0.w, q0.w));
  const float2 b0 = __fmul2_rn(make_float2(q1.y, q1.y), dx);
  g.a0[0] = a0.x, g.a0[1] = a0.y, g.b0[0] = b0.x, g.b0[1] = b0.y;
  g.dy[0] = __fsub_rn(q0.y, pyf0);
  const float2 d12 = __fadd2_rn(make_float2(g.dy[0], g.dy[0]), make_float2(-4.f, -8.f));
  g.dy[1] = d12.x, g.dy[2] = d12.y;
  g.dy[3] = __fsub_rn(g.dy[0], 12.f);
  } else {
#pragma unroll
  for (int e = 0; e < 2; ++e) {
    g.a0[e] = __fmaf_rn(__fmul_rn(q1.x, g.dx[e]), g.dx[e], q0.w);
    g.b0[e] = __fmul_rn(q1.y, g.dx[e]);
  }
  g.dy[0] = __fsub_rn(q0.y, pyf0);
#pragma unroll
  for (int r = 1; r < 4; ++r) g.dy[r] = __fsub_rn(g.dy[0], 4.f * r);
  }
  return g;
}
__device__ __forceinline__ float geo_p2(const Geo& g, float Ch, int b) {
  const float dy = g.dy[b >> 1];
  return __fmaf_rn(dy, __fmaf_rn(Ch, dy, g.b0[b & 1]), g.a0[b & 1]);
}

// Per-lane pixel state; pixels 2r and 2r + 1 (one block row, columns lx and lx + 8)
// are the two halves of one float2 so that the dense paths can use packed FP32 ops.
struct FwdPix {
  float2 T2[kPix / 2], Cr2[kPix / 2], Cg2[kPix / 2], Cb2[kPix / 2], D2[kPix / 2];  // T < 0: terminated (|T| final)
  int n[kPix];
  __device__ __forceinline__ float& T(int b) { return (b & 1) ? T2[b >> 1].y : T2[b >> 1].x; }
  __device__ __forceinline__ float& Cr(int b) { return (b & 1) ? Cr2[b >> 1].y : Cr2[b >> 1].x; }
  __device__ __forceinline__ float& Cg(int b) { return (b & 1) ? Cg2[b >> 1].y : Cg2[b >> 1].x; }
  __device__ __forceinline__ float& Cb(int b) { return (b & 1) ? Cb2[b >> 1].y : Cb2[b >> 1].x; }
  __device__ __forceinline__ float& D(int b) { return (b & 1) ? D2[b >> 1].y : D2[b >> 1].x; }
  __device__ __forceinline__ float Tc(int b) const { return (b & 1) ? T2[b >> 1].y : T2[b >> 1].x; }
};

// alpha of pixel b and the composite test "alpha >= 1/255 (and power <= 0)".
template <bool kCap, bool kGen>
__device__ __forceinline__ bool fwd_alpha(float p2, float lo2, float& al) {
  al = ex2_approx(p2);
  if (kCap) al = fminf(al, kAlphaCap);
  bool c = al >= kAlphaMin;
  if (kGen) c = c && (p2 <= lo2);
  return c;
}

// Front-to-back step for pixel b: composite if T - alpha T stays >= 1e-4, else stop
// the pixel (R16).  A terminated pixel (T < 0) fails the test forever.
__device__ __forceinline__ void fwd_blend(FwdPix& px, int b, bool cond, float al, const float4& q0, float r,
                                          float g, float bl, int pos1, uint32_t& lm) {
  // Predicated PTX (the C form compiles to branches): with c = cond,
  //   Tn = T - alpha T;  comp = c && Tn >= 1e-4;
  //   if comp: C += col alpha T, D += z alpha T, n = pos1, lm |= bit
  //   if c:    T = comp ? Tn : -|T|
  asm("{\n\t"
      ".reg .pred pc, pcomp, pstop;\n\t"
      ".reg .f32 tn, w, na, ta;\n\t"
      "setp.ne.u32 pc, %7, 0;\n\t"
      "neg.f32 na, %8;\n\t"
      "fma.rn.f32 tn, na, %0, %0;\n\t"
      "setp.ge.and.f32 pcomp|pstop, tn, 0f38D1B717, pc;\n\t"
      "mul.f32 w, %8, %0;\n\t"
      "@pcomp fma.rn.f32 %1, %9, w, %1;\n\t"
      "@pcomp fma.rn.f32 %2, %10, w, %2;\n\t"
      "@pcomp fma.rn.f32 %3, %11, w, %3;\n\t"
      "@pcomp fma.rn.f32 %4, %12, w, %4;\n\t"
      "@pcomp mov.b32 %5, %13;\n\t"
      "@pcomp or.b32 %6, %6, %14;\n\t"
      "abs.f32 ta, %0;\n\t"
      "neg.f32 ta, ta;\n\t"
      "@pc selp.f32 %0, tn, ta, pcomp;\n\t"
      "}"
      : "+f"(px.T(b)), "+f"(px.Cr(b)), "+f"(px.Cg(b)), "+f"(px.Cb(b)), "+f"(px.D(b)), "+r"(px.n[b]), "+r"(lm)
      : "r"((uint32_t)cond), "f"(al), "f"(r), "f"(g), "f"(bl), "f"(q0.z), "r"(pos1), "r"(1u << b));
}

#if GSR_FFMA2_FWD
// fwd_blend for the pixel pair (2r, 2r + 1) on packed FP32 ops: the composited pixels
// get w = alpha T, the others w = 0 (C + col x 0 == C exactly), so the colour / depth
// accumulations need no predicate; per element the same fp32 operations as fwd_blend.
__device__ __forceinline__ void fwd_blend2(FwdPix& px, int r, bool c0, bool c1, float al0, float al1, float z,
                                           float cr, float cg, float cb, int pos1, uint32_t& lm) {
  const float2 T = px.T2[r];
  const float2 tn = __ffma2_rn(make_float2(-al0, -al1), T, T);
  const bool k0 = c0 && tn.x >= kTStop, k1 = c1 && tn.y >= kTStop;
  float a0z, a1z, t0, t1;
  asm("{\n\t.reg .pred pk;\n\tsetp.ne.u32 pk, %2, 0;\n\tselp.f32 %0, %1, 0f00000000, pk;\n\t}"
      : "=f"(a0z) : "f"(al0), "r"((uint32_t)k0));
  asm("{\n\t.reg .pred pk;\n\tsetp.ne.u32 pk, %2, 0;\n\tselp.f32 %0, %1, 0f00000000, pk;\n\t}"
      : "=f"(a1z) : "f"(al1), "r"((uint32_t)k1));
  const float2 w = __fmul2_rn(make_float2(a0z, a1z), T);
  px.Cr2[r] = __ffma2_rn(make_float2(cr, cr), w, px.Cr2[r]);
  px.Cg2[r] = __ffma2_rn(make_float2(cg, cg), w, px.Cg2[r]);
  px.Cb2[r] = __ffma2_rn(make_float2(cb, cb), w, px.Cb2[r]);
  px.D2[r] = __ffma2_rn(make_float2(z, z), w, px.D2[r]);
  // T := composited ? tn : (tested ? -|T| : T)
  asm("{\n\t.reg .pred pc, pk;\n\t.reg .f32 ta;\n\t"
      "setp.ne.u32 pc, %2, 0;\n\tsetp.ne.u32 pk, %3, 0;\n\t"
      "abs.f32 ta, %1;\n\tneg.f32 ta, ta;\n\t"
      "selp.f32 ta, %4, ta, pk;\n\t"
      "selp.f32 %0, ta, %1, pc;\n\t}"
      : "=f"(t0) : "f"(T.x), "r"((uint32_t)c0), "r"((uint32_t)k0), "f"(tn.x));
  asm("{\n\t.reg .pred pc, pk;\n\t.reg .f32 ta;\n\t"
      "setp.ne.u32 pc, %2, 0;\n\tsetp.ne.u32 pk, %3, 0;\n\t"
      "abs.f32 ta, %1;\n\tneg.f32 ta, ta;\n\t"
      "selp.f32 ta, %4, ta, pk;\n\t"
      "selp.f32 %0, ta, %1, pc;\n\t}"
      : "=f"(t1) : "f"(T.y), "r"((uint32_t)c1), "r"((uint32_t)k1), "f"(tn.y));
  px.T2[r] = make_float2(t0, t1);
  asm("{\n\t.reg .pred pk;\n\tsetp.ne.u32 pk, %2, 0;\n\t@pk mov.b32 %0, %3;\n\t@pk or.b32 %1, %1, %4;\n\t}"
      : "+r"(px.n[2 * r]), "+r"(lm) : "r"((uint32_t)k0), "r"(pos1), "r"(1u << (2 * r)));
  asm("{\n\t.reg .pred pk;\n\tsetp.ne.u32 pk, %2, 0;\n\t@pk mov.b32 %0, %3;\n\t@pk or.b32 %1, %1, %4;\n\t}"
      : "+r"(px.n[2 * r + 1]), "+r"(lm) : "r"((uint32_t)k1), "r"(pos1), "r"(1u << (2 * r + 1)));
}
#endif

template <bool kCap>
__device__ __forceinline__ void fwd_dense(FwdPix& px, const Geo& g, const float4& q0, const float4& q1,
                                          const float4& q2, int pos1, uint32_t& lm) {
  float al[kPix];
  bool c[kPix];
#if GSR_FFMA2_FWD
  // p2 of both columns of a block row at once: fma(dy, fma(Ch, dy, b0_e), a0_e)
  const float2 a0 = make_float2(g.a0[0], g.a0[1]), b0 = make_float2(g.b0[0], g.b0[1]);
  const float2 ch = make_float2(q1.z, q1.z);
#pragma unroll
  for (int r = 0; r < kPix / 2; ++r) {
    const float2 dy = make_float2(g.dy[r], g.dy[r]);
    const float2 p2 = __ffma2_rn(dy, __ffma2_rn(ch, dy, b0), a0);
    c[2 * r] = fwd_alpha<kCap, false>(p2.x, q0.w, al[2 * r]);
    c[2 * r + 1] = fwd_alpha<kCap, false>(p2.y, q0.w, al[2 * r + 1]);
  }
#pragma unroll
  for (int r = 0; r < kPix / 2; ++r)
    fwd_blend2(px, r, c[2 * r], c[2 * r + 1], al[2 * r], al[2 * r + 1], q0.z, q1.w, q2.x, q2.y, pos1, lm);
#else
#pragma unroll
  for (int b = 0; b < kPix; ++b) c[b] = fwd_alpha<kCap, false>(geo_p2(g, q1.z, b), q0.w, al[b]);
#pragma unroll
  for (int b = 0; b < kPix; ++b) fwd_blend(px, b, c[b], al[b], q0, q1.w, q2.x, q2.y, pos1, lm);
#endif
}

#if GSR_FFMA2_FWD
// fwd_dense restricted to the block rows the key's mask touches (bit 2r or 2r + 1 of m2 =
// m | m >> 1): both pixels of a touched row as in fwd_dense, untouched rows skipped by a
// warp-uniform branch.  Pixels of a touched row's other block lie outside the
// conservative mask and fail the alpha test exactly as in fwd_dense: same results.
template <bool kCap>
__device__ __forceinline__ void fwd_rows(FwdPix& px, uint32_t m2, const Geo& g, const float4& q0, const float4& q1,
                                         const float4& q2, int pos1, uint32_t& lm) {
  const float2 a0 = make_float2(g.a0[0], g.a0[1]), b0 = make_float2(g.b0[0], g.b0[1]);
  const float2 ch = make_float2(q1.z, q1.z);
#pragma unroll
  for (int r = 0; r < kPix / 2; ++r) {
    if (!((m2 >> (2 * r)) & 1u)) continue;
    const float2 dy = make_float2(g.dy[r], g.dy[r]);
    const float2 p2 = __ffma2_rn(dy, __ffma2_rn(ch, dy, b0), a0);
    float al0, al1;
    const bool c0 = fwd_alpha<kCap, false>(p2.x, q0.w, al0);
    const bool c1 = fwd_alpha<kCap, false>(p2.y, q0.w, al1);
    fwd_blend2(px, r, c0, c1, al0, al1, q0.z, q1.w, q2.x, q2.y, pos1, lm);
  }
}
#endif

template <bool kGen>
__device__ __forceinline__ void fwd_sparse(FwdPix& px, uint32_t m, const Geo& g, const float4& q0, const float4& q1,
                                           const float4& q2, int pos1, uint32_t& lm) {
#pragma unroll
  for (int b = 0; b < kPix; ++b) {
    if (!((m >> b) & 1u)) continue;
    float al;
    const bool c = fwd_alpha<true, kGen>(geo_p2(g, q1.z, b), q0.w, al);
    if (!__any_sync(kFull, c)) continue;
    fwd_blend(px, b, c, al, q0, q1.w, q2.x, q2.y, pos1, lm);
  }
}

// Blocks (8x4) all of whose pixels in this warp have terminated.
__device__ __forceinline__ uint32_t dead_blocks(const FwdPix& px) {
  uint32_t d = 0;
#pragma unroll
  for (int b = 0; b < kPix; ++b) d |= (__float_as_uint(px.Tc(b)) >> 31) << b;
  return __reduce_and_sync(kFull, d);
}

// kRows (gs_set_render_rows): every non-general key visits only the block rows its mask
// touches (fwd_rows) instead of all four (fwd_dense); same results.
template <int WPC, bool kRows = false>
__global__ void __launch_bounds__(WPC * 32, kFwdMinWarps / WPC) k_render_fwd(DevCam cam, const float4* __restrict__ rec,
                                                                   const int32_t* __restrict__ ids,
                                                                   const int2* __restrict__ ranges, const int32_t* __restrict__ order,
                                                                   float* __restrict__ out_rgb,
                                                                   float* __restrict__ out_d, float* __restrict__ out_T,
                                                                   int32_t* __restrict__ out_n,
                                                                   unsigned long long* blended,
                                                                   uint8_t* __restrict__ key_blocks) {
  __shared__ float4 s_rec[WPC][2][32][3];
#if GSR_FWD_KB_SMEM
  __shared__ uint8_t s_kb[WPC][32];  // the batch's key masks (key j's byte written by the whole warp)
#endif
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wslot = blockIdx.x * WPC + warp;
  if (wslot >= cam.TX * cam.TY) return;
  const int tile = order ? order[wslot] : wslot;  // work order (gs_tile_order)
  const int tx = tile % cam.TX, ty = tile / cam.TX;
  const int ox = tx * kTile, oy = ty * kTile;
  const int lx = lane & 7, ly = lane >> 3;
  // pixel b of this lane: x = ox + lx + 8 (b & 1), y = oy + ly + 4 (b >> 1)
  const float pxf0 = (float)(ox + lx), pyf0 = (float)(oy + ly);
  const int2 rg = ranges[tile];

  FwdPix px;
#pragma unroll
  for (int b = 0; b < kPix; ++b) {
    const bool inside = ox + lx + 8 * (b & 1) < cam.W && oy + ly + 4 * (b >> 1) < cam.H;
    px.T(b) = inside ? 1.f : -1.f;  // pixels outside the image start terminated
    px.Cr(b) = px.Cg(b) = px.Cb(b) = px.D(b) = 0.f;
    px.n[b] = 0;
  }
  uint32_t nblend = 0;
  uint32_t bdone = dead_blocks(px);
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
    uint32_t my_fl = 0;
    if (b0 + lane < rg.y) {
      stage_fast<true>(s_rec[warp][buf][lane], ox, oy);
      my_fl = __float_as_uint(reinterpret_cast<const float*>(&s_rec[warp][buf][lane][2])[3]);
    }
#if GSR_FWD_KB_SMEM
    s_kb[warp][lane] = 0;
#endif
    __syncwarp();
    uint32_t live = __ballot_sync(kFull, (my_fl & ~bdone & 0xffu) != 0u);
#if !GSR_FWD_KB_SMEM
    uint32_t kb_mine = 0;  // lane j: 8x4 blocks in which key b0 + j composited >= 1 pixel
#endif
    [[maybe_unused]] int since = 0;
    const int pos0 = b0 - rg.x + 1;  // 1-based position of the batch's key 0 in the tile's list
    while (live) {
      const int j = __ffs(live) - 1;
      live &= live - 1;
      const float4 q0 = s_rec[warp][buf][j][0], q1 = s_rec[warp][buf][j][1], q2 = s_rec[warp][buf][j][2];
      const uint32_t fl = __float_as_uint(q2.w);
      const uint32_t m = fl & ~bdone & 0xffu;
      if (m == 0) continue;
      const int pos1 = pos0 + j;
      const Geo g = make_geo<GSR_FFMA2_GEO>(q0, q1, pxf0, pyf0);
      uint32_t lm = 0;  // this lane's composited pixels (bit b = block b) for this key
      if (fl & kFlagGeneral) {
        fwd_sparse<true>(px, m, g, q0, q1, q2, pos1, lm);
      } else if (__popc(m) >= kDenseBlocks) {
#if GSR_FFMA2_FWD
        if constexpr (kRows) {
          const uint32_t m2 = m | (m >> 1);
          if (fl & kFlagCap)
            fwd_rows<true>(px, m2, g, q0, q1, q2, pos1, lm);
          else
            fwd_rows<false>(px, m2, g, q0, q1, q2, pos1, lm);
        } else
#endif
        if (fl & kFlagCap)
          fwd_dense<true>(px, g, q0, q1, q2, pos1, lm);
        else
          fwd_dense<false>(px, g, q0, q1, q2, pos1, lm);
      } else {
        fwd_sparse<false>(px, m, g, q0, q1, q2, pos1, lm);
      }
      const uint32_t cm = __reduce_or_sync(kFull, lm);
#ifndef GSR_COUNT_EVAL
      nblend += __popc(lm);
#else  // diagnostics build: the blended counter counts work units instead (lane 0)
      if (lane == 0) {
        const bool dense = !(fl & kFlagGeneral) && __popc(m) >= kDenseBlocks;
        nblend += GSR_COUNT_EVAL == 1 ? (dense ? 8u : (uint32_t)__popc(m)) : GSR_COUNT_EVAL == 2 ? 1u : (uint32_t)__popc(cm);
      }
#endif
#if GSR_FWD_KB_SMEM
      s_kb[warp][j] = (uint8_t)cm;  // every lane stores the same (warp-uniform) byte: one STS, no lane test
#else
      kb_mine = (lane == j) ? cm : kb_mine;
#endif
      if (GSR_DEAD_EVERY > 0 && ++since == GSR_DEAD_EVERY) {
        since = 0;
        bdone = dead_blocks(px);
        if (bdone == 0xffu) break;
      }
    }
#if GSR_FWD_KB_SMEM
    __syncwarp();
    if (key_blocks && b0 + lane < rg.y) key_blocks[b0 + lane] = s_kb[warp][lane];
#else
    if (key_blocks && b0 + lane < rg.y) key_blocks[b0 + lane] = (uint8_t)kb_mine;
#endif
    bdone = dead_blocks(px);
    __syncwarp();
  }
  cp_async_wait<0>();
  const int64_t npix = (int64_t)cam.W * cam.H;
#pragma unroll
  for (int b = 0; b < kPix; ++b) {
    const int x = ox + lx + 8 * (b & 1), y = oy + ly + 4 * (b >> 1);
    if (x < cam.W && y < cam.H) {
      const int64_t p = (int64_t)y * cam.W + x;
      const float T = fabsf(px.T(b));
      out_rgb[p] = fmaf(T, cam.bg[0], px.Cr(b));
      out_rgb[npix + p] = fmaf(T, cam.bg[1], px.Cg(b));
      out_rgb[2 * npix + p] = fmaf(T, cam.bg[2], px.Cb(b));
      out_d[p] = px.D(b);
      out_T[p] = T;
      out_n[p] = px.n[b];
    }
  }
  if (blended) {
    const uint32_t tot = __reduce_add_sync(kFull, nblend);
    if (lane == 0 && tot) atomicAdd(blended, (unsigned long long)tot);
  }
}

// ---------------------------------------------------------------------------
// Pixel pairs (2r, 2r + 1) in float2 halves, as FwdPix.
struct BwdPix {
  float2 T2[kPix / 2], Q2[kPix / 2], gr2[kPix / 2], gg2[kPix / 2], gb2[kPix / 2], gd2[kPix / 2];
  int n[kPix];
  __device__ __forceinline__ float& T(int b) { return (b & 1) ? T2[b >> 1].y : T2[b >> 1].x; }
  __device__ __forceinline__ float& Q(int b) { return (b & 1) ? Q2[b >> 1].y : Q2[b >> 1].x; }
  __device__ __forceinline__ float& gr(int b) { return (b & 1) ? gr2[b >> 1].y : gr2[b >> 1].x; }
  __device__ __forceinline__ float& gg(int b) { return (b & 1) ? gg2[b >> 1].y : gg2[b >> 1].x; }
  __device__ __forceinline__ float& gb(int b) { return (b & 1) ? gb2[b >> 1].y : gb2[b >> 1].x; }
  __device__ __forceinline__ float& gd(int b) { return (b & 1) ? gd2[b >> 1].y : gd2[b >> 1].x; }
};
// Lane partial sums over the key's pixels, per pixel column (x: lx, y: lx + 8):
// colour / depth  sum g_ch w;  s0 = sum dp, s1 = sum dp dy, s2 = sum dp dy^2
// (dp = dL/dpower).  The two columns are added before the warp reduction.
struct BwdAcc {
  float r, g, b, z, s2;
  float2 s0, s1;
  __device__ __forceinline__ float& c(float2& v, int b) { return (b & 1) ? v.y : v.x; }
};

// One pixel's reverse step (alpha_k, T_{k+1} = T, suffix Q): dL/dalpha =
// (T u - Q) / (1 - alpha) with u = g . (c, z); capped alpha has no derivative (R18).
template <bool kCap>
__device__ __forceinline__ void bwd_pixel(BwdPix& px, int b, bool valid, float raw, float dy, float dy2,
                                          const float4& q0, const float4& q1, const float4& q2, BwdAcc& a) {
  const float al = kCap ? fminf(raw, kAlphaCap) : raw;
  const float inv = rcp_approx(1.f - al);
  const float ai = al * inv;
  const float T = px.T(b);
  const float Tk = T * inv;
  const float u = fmaf(px.gr(b), q1.w, fmaf(px.gg(b), q2.x, fmaf(px.gb(b), q2.y, px.gd(b) * q0.z)));
  const float x = fmaf(T, u, -px.Q(b));
  float dp = ai * x;
  if (kCap) dp = (raw > kAlphaCap) ? 0.f : dp;
  const float w = ai * T;
  // predicated PTX (the C form compiles to branches)
  asm("{\n\t"
      ".reg .pred p;\n\t"
      "setp.ne.u32 p, %9, 0;\n\t"
      "@p fma.rn.f32 %0, %10, %11, %0;\n\t"
      "@p mov.b32 %1, %12;\n\t"
      "@p fma.rn.f32 %2, %13, %10, %2;\n\t"
      "@p fma.rn.f32 %3, %14, %10, %3;\n\t"
      "@p fma.rn.f32 %4, %15, %10, %4;\n\t"
      "@p fma.rn.f32 %5, %16, %10, %5;\n\t"
      "@p add.f32 %6, %6, %17;\n\t"
      "@p fma.rn.f32 %7, %17, %18, %7;\n\t"
      "@p fma.rn.f32 %8, %17, %19, %8;\n\t"
      "}"
      : "+f"(px.Q(b)), "+f"(px.T(b)), "+f"(a.r), "+f"(a.g), "+f"(a.b), "+f"(a.z), "+f"(a.c(a.s0, b)),
        "+f"(a.c(a.s1, b)), "+f"(a.s2)
      : "r"((uint32_t)valid), "f"(w), "f"(u), "f"(Tk), "f"(px.gr(b)), "f"(px.gg(b)), "f"(px.gb(b)), "f"(px.gd(b)),
        "f"(dp), "f"(dy), "f"(dy2));
}

#if GSR_FFMA2
__device__ __forceinline__ float sel0(bool p, float v) {  // p ? v : +0
  float r;
  asm("{\n\t.reg .pred pk;\n\tsetp.ne.u32 pk, %2, 0;\n\tselp.f32 %0, %1, 0f00000000, pk;\n\t}"
      : "=f"(r) : "f"(v), "r"((uint32_t)p));
  return r;
}
__device__ __forceinline__ float selv(bool p, float v, float w) {  // p ? v : w
  float r;
  asm("{\n\t.reg .pred pk;\n\tsetp.ne.u32 pk, %3, 0;\n\tselp.f32 %0, %1, %2, pk;\n\t}"
      : "=f"(r) : "f"(v), "f"(w), "r"((uint32_t)p));
  return r;
}
// bwd_pixel for the pixel pair (2r, 2r + 1) on packed FP32 ops: a pixel that does not
// take part gets ai = 0, hence dp = w = 0, and adds exact zeros to every sum; T keeps
// its value by a select.  Per element the same fp32 operations as bwd_pixel.
template <bool kCap>
__device__ __forceinline__ void bwd_pixel2(BwdPix& px, int r, bool v0, bool v1, float raw0, float raw1, float dy,
                                           float dy2, const float4& q0, const float4& q1, const float4& q2,
                                           BwdAcc& a) {
  const float2 al = kCap ? make_float2(fminf(raw0, kAlphaCap), fminf(raw1, kAlphaCap)) : make_float2(raw0, raw1);
  const float2 om = __fadd2_rn(make_float2(1.f, 1.f), make_float2(-al.x, -al.y));
  const float2 inv = make_float2(rcp_approx(om.x), rcp_approx(om.y));
  float2 ai = __fmul2_rn(al, inv);
  ai = make_float2(sel0(v0, ai.x), sel0(v1, ai.y));
  const float2 T = px.T2[r];
  const float2 Tk = __fmul2_rn(T, inv);
  const float2 u = __ffma2_rn(px.gr2[r], make_float2(q1.w, q1.w),
                              __ffma2_rn(px.gg2[r], make_float2(q2.x, q2.x),
                                         __ffma2_rn(px.gb2[r], make_float2(q2.y, q2.y),
                                                    __fmul2_rn(px.gd2[r], make_float2(q0.z, q0.z)))));
  const float2 x = __ffma2_rn(T, u, make_float2(-px.Q2[r].x, -px.Q2[r].y));
  float2 dp = __fmul2_rn(ai, x);
  if (kCap) dp = make_float2(sel0(!(raw0 > kAlphaCap), dp.x), sel0(!(raw1 > kAlphaCap), dp.y));
  const float2 w = __fmul2_rn(ai, T);
  px.Q2[r] = __ffma2_rn(w, u, px.Q2[r]);
  px.T2[r] = make_float2(selv(v0, Tk.x, T.x), selv(v1, Tk.y, T.y));
  // the column-independent sums stay scalar (pixel 2r, then 2r + 1, as bwd_pixel):
  // paired accumulators would cost 5 more registers in the register-capped kernel
  a.r = fmaf(px.gr2[r].x, w.x, a.r);
  a.g = fmaf(px.gg2[r].x, w.x, a.g);
  a.b = fmaf(px.gb2[r].x, w.x, a.b);
  a.z = fmaf(px.gd2[r].x, w.x, a.z);
  a.s2 = fmaf(dp.x, dy2, a.s2);
  a.r = fmaf(px.gr2[r].y, w.y, a.r);
  a.g = fmaf(px.gg2[r].y, w.y, a.g);
  a.b = fmaf(px.gb2[r].y, w.y, a.b);
  a.z = fmaf(px.gd2[r].y, w.y, a.z);
  a.s2 = fmaf(dp.y, dy2, a.s2);
  a.s0 = __fadd2_rn(a.s0, dp);
  a.s1 = __ffma2_rn(dp, make_float2(dy, dy), a.s1);
}
#endif

template <bool kCap>
__device__ __forceinline__ bool bwd_dense(BwdPix& px, int pos, const Geo& g, const float (&dy2)[4], const float4& q0,
                                          const float4& q1, const float4& q2, BwdAcc& a) {
  float raw[kPix];
#if GSR_FFMA2
  const float2 a0 = make_float2(g.a0[0], g.a0[1]), b0 = make_float2(g.b0[0], g.b0[1]);
  const float2 ch = make_float2(q1.z, q1.z);
#pragma unroll
  for (int r = 0; r < kPix / 2; ++r) {
    const float2 dy = make_float2(g.dy[r], g.dy[r]);
    const float2 p2 = __ffma2_rn(dy, __ffma2_rn(ch, dy, b0), a0);
    raw[2 * r] = ex2_approx(p2.x);
    raw[2 * r + 1] = ex2_approx(p2.y);
  }
#pragma unroll
  for (int r = 0; r < kPix / 2; ++r)
    bwd_pixel2<kCap>(px, r, pos < px.n[2 * r] && raw[2 * r] >= kAlphaMin, pos < px.n[2 * r + 1] && raw[2 * r + 1] >= kAlphaMin,
                     raw[2 * r], raw[2 * r + 1], g.dy[r], dy2[r], q0, q1, q2, a);
#else
#pragma unroll
  for (int b = 0; b < kPix; ++b) raw[b] = ex2_approx(geo_p2(g, q1.z, b));
#pragma unroll
  for (int b = 0; b < kPix; ++b)
    bwd_pixel<kCap>(px, b, pos < px.n[b] && raw[b] >= kAlphaMin, raw[b], g.dy[b >> 1], dy2[b >> 1], q0, q1, q2, a);
#endif
  return true;  // dense keys (>= 6 blocks composited in the forward) practically always contribute
}

#if GSR_FFMA2
// bwd_dense restricted to the block rows the key's mask touches (as fwd_rows): a pixel of
// an untouched block of a touched row is invalid (the forward composited the key in no
// pixel of that block) and adds exact zeros, in the same ascending pixel order as
// bwd_sparse's per-block walk.
template <bool kCap>
__device__ __forceinline__ void bwd_rows(BwdPix& px, uint32_t m2, int pos, const Geo& g, const float (&dy2)[4],
                                         const float4& q0, const float4& q1, const float4& q2, BwdAcc& a) {
  const float2 a0 = make_float2(g.a0[0], g.a0[1]), b0 = make_float2(g.b0[0], g.b0[1]);
  const float2 ch = make_float2(q1.z, q1.z);
#pragma unroll
  for (int r = 0; r < kPix / 2; ++r) {
    if (!((m2 >> (2 * r)) & 1u)) continue;
    const float2 dy = make_float2(g.dy[r], g.dy[r]);
    const float2 p2 = __ffma2_rn(dy, __ffma2_rn(ch, dy, b0), a0);
    const float raw0 = ex2_approx(p2.x), raw1 = ex2_approx(p2.y);
    bwd_pixel2<kCap>(px, r, pos < px.n[2 * r] && raw0 >= kAlphaMin, pos < px.n[2 * r + 1] && raw1 >= kAlphaMin, raw0,
                     raw1, g.dy[r], dy2[r], q0, q1, q2, a);
  }
}
#endif

template <bool kGen>
__device__ __forceinline__ bool bwd_sparse(BwdPix& px, uint32_t m, int pos, const Geo& g, const float (&dy2)[4],
                                           const float4& q0, const float4& q1, const float4& q2, BwdAcc& a) {
  bool any = false;
#pragma unroll
  for (int b = 0; b < kPix; ++b) {
    if (!((m >> b) & 1u)) continue;
    const float p2 = geo_p2(g, q1.z, b);
    const float raw = ex2_approx(p2);
    bool valid = pos < px.n[b] && raw >= kAlphaMin;
    if (kGen) valid = valid && (p2 <= q0.w);
    if (!__any_sync(kFull, valid)) continue;
    any = true;
    bwd_pixel<true>(px, b, valid, raw, g.dy[b >> 1], dy2[b >> 1], q0, q1, q2, a);
  }
  return any;
}

// kMasks: the forward's per-key block masks are given (key_blocks != NULL; the
// product path) -- a compile-time switch, so the key loop carries no test for it.
// kDet: deterministic mode (gs_bwd_opts.det_ws): each (tile, key) pair's reduced 10
// components are stored to det[key][12] instead of atomically added (k_det_reduce sums
// them per Gaussian in a fixed order).
// kPack (product path, P < 2^22): each staged record carries its Gaussian id in bits
// 10-31 of its flag word (the block-mask bits are unused with the forward's key
// masks), so a key's id is one shift of a value already loaded instead of a shared-memory
// read per key.
// kRows (with the forward's key masks): every non-general key through bwd_rows.
template <int WPC, bool kMasks, bool kDet, bool kPack = false, bool kRows = false>
__global__ void __launch_bounds__(WPC * 32, kBwdMinWarps / WPC) k_render_bwd(DevCam cam, const float4* __restrict__ rec,
                                                                   const int32_t* __restrict__ ids,
                                                                   const int2* __restrict__ ranges, const int32_t* __restrict__ order,
                                                                   const float* __restrict__ T_final,
                                                                   const int32_t* __restrict__ n_contrib,
                                                                   const float* __restrict__ g_rgb,
                                                                   const float* __restrict__ g_dep,
                                                                   const uint8_t* __restrict__ key_blocks,
                                                                   float* __restrict__ sgrad, L1Fuse l1,
                                                                   float* __restrict__ det, int64_t det_keys) {
  __shared__ float4 s_rec[WPC][2][32][3];
  __shared__ int s_gid[WPC][2][32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wslot = blockIdx.x * WPC + warp;
  if (wslot >= cam.TX * cam.TY) return;
  const int tile = order ? order[wslot] : wslot;  // work order (gs_tile_order)
  const int tx = tile % cam.TX, ty = tile / cam.TX;
  const int ox = tx * kTile, oy = ty * kTile;
  const int lx = lane & 7, ly = lane >> 3;
  const float pxf0 = (float)(ox + lx), pyf0 = (float)(oy + ly);
  const int2 rg = ranges[tile];
  const int64_t npix = (int64_t)cam.W * cam.H;

  BwdPix px;
  int bmaxn[kPix];  // per 8x4 block: max n_contrib over its 32 pixels (warp-uniform)
  int maxn = 0;
  float lsum = 0.f;
#pragma unroll
  for (int b = 0; b < kPix; ++b) {
    const int x = ox + lx + 8 * (b & 1), y = oy + ly + 4 * (b >> 1);
    if (x < cam.W && y < cam.H) {
      const int64_t p = (int64_t)y * cam.W + x;
      px.T(b) = T_final[p];
      px.n[b] = n_contrib[p];
      upstream(l1, g_rgb, g_dep, npix, p, px.gr(b), px.gg(b), px.gb(b), px.gd(b), lsum);
    } else {
      px.T(b) = 1.f, px.n[b] = 0, px.gr(b) = px.gg(b) = px.gb(b) = px.gd(b) = 0.f;
    }
    px.Q(b) = px.T(b) * (px.gr(b) * cam.bg[0] + px.gg(b) * cam.bg[1] + px.gb(b) * cam.bg[2]);
    bmaxn[b] = __reduce_max_sync(kFull, px.n[b]);
    maxn = max(maxn, bmaxn[b]);
  }
  l1_commit(l1, lsum, lane);
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
        kb = kMasks ? (uint32_t)key_blocks[l + lane] : 0xffu;
      }
    }
  };
  auto stage = [&](int b, int id, uint32_t kb) {
    if (id >= 0 && kb) {
      s_gid[warp][b][lane] = id;
      gather_rec_async(rec, id, s_rec[warp][b][lane]);
    }
  };
#if GSR_BWD_PAIR
  float h_p[5];  // first stage of the pending key's reduction (gid_p >= 0)
  int gid_p = -1;
#endif
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
    if (lo + lane < hi && kb_cur) {
      stage_fast<!kMasks>(s_rec[warp][buf][lane], ox, oy);
      if constexpr (kPack)
        reinterpret_cast<uint32_t*>(&s_rec[warp][buf][lane][2])[3] |= (uint32_t)s_gid[warp][buf][lane] << kGidShift;
    }
    __syncwarp();
    uint32_t live = __ballot_sync(kFull, kb_cur != 0);
    while (live) {
      const int j = 31 - __clz(live);  // back to front
      live &= ~(1u << j);
      const float4 q0 = s_rec[warp][buf][j][0], q1 = s_rec[warp][buf][j][1], q2 = s_rec[warp][buf][j][2];
      const uint32_t fl = __float_as_uint(q2.w);
      const int pos = lo + j - rg.x;
      uint32_t m;
      if constexpr (kMasks) {
        m = __shfl_sync(kFull, kb_cur, j);  // blocks the forward composited this key in
      } else {
        m = fl & 0xffu;
#pragma unroll
        for (int b = 0; b < kPix; ++b)
          if (pos >= bmaxn[b]) m &= ~(1u << b);
        if (m == 0) continue;
      }
      const Geo g = make_geo<GSR_FFMA2_GEO_BWD>(q0, q1, pxf0, pyf0);
      float dy2[4];
#if GSR_FFMA2_GEO_BWD
      {
        const float2 d01 = make_float2(g.dy[0], g.dy[1]), d23 = make_float2(g.dy[2], g.dy[3]);
        const float2 s01 = __fmul2_rn(d01, d01), s23 = __fmul2_rn(d23, d23);
        dy2[0] = s01.x, dy2[1] = s01.y, dy2[2] = s23.x, dy2[3] = s23.y;
      }
#else
#pragma unroll
      for (int r = 0; r < 4; ++r) dy2[r] = g.dy[r] * g.dy[r];
#endif
      BwdAcc a;
      a.r = a.g = a.b = a.z = a.s2 = 0.f;
      a.s0 = a.s1 = make_float2(0.f, 0.f);
      bool any;
      if (fl & kFlagGeneral)
        any = bwd_sparse<true>(px, m, pos, g, dy2, q0, q1, q2, a);
#if GSR_FFMA2
      else if (kRows && kMasks) {  // the forward composited this key in >= 1 pixel: some pixel is valid
        const uint32_t m2 = m | (m >> 1);
        if (fl & kFlagCap)
          bwd_rows<true>(px, m2, pos, g, dy2, q0, q1, q2, a);
        else
          bwd_rows<false>(px, m2, pos, g, dy2, q0, q1, q2, a);
        any = true;
      }
#endif
      else if (__popc(m) >= kDenseBlocksBwd)
        any = (fl & kFlagCap) ? bwd_dense<true>(px, pos, g, dy2, q0, q1, q2, a)
                              : bwd_dense<false>(px, pos, g, dy2, q0, q1, q2, a);
      else
        any = bwd_sparse<false>(px, m, pos, g, dy2, q0, q1, q2, a);
      if (any) {
        // conic and mean gradients from the moments of dp over the tile:
        // dpower/dA = -dx^2/2, dpower/dB = -dx dy, dpower/dC = -dy^2/2,
        // dpower/dmu = -(A dx + B dy, B dx + C dy)
        const float A = q1.x * (1.f / kHalfL2e), B = q1.y * (1.f / kNegL2e), C = q1.z * (1.f / kHalfL2e);
        const float dx0 = g.dx[0], dx1 = g.dx[1];
        const float sx = dx0 * a.s0.x + dx1 * a.s0.y;
        const float sxx = dx0 * dx0 * a.s0.x + dx1 * dx1 * a.s0.y;
        const float sy = a.s1.x + a.s1.y;
        const float sxy = dx0 * a.s1.x + dx1 * a.s1.y;
        float v[10];
        v[0] = -(A * sx + B * sy);
        v[1] = -(B * sx + C * sy);
        v[2] = -0.5f * sxx;
        v[3] = -sxy;
        v[4] = -0.5f * a.s2;
        v[5] = (a.s0.x + a.s0.y) * q2.z;  // dalpha/do = exp(power) = alpha / o; q2.z = 1/o
        v[6] = a.r;
        v[7] = a.g;
        v[8] = a.b;
        v[9] = a.z;
        if constexpr (kDet) {
          float out;
          int slot;
          warp_reduce10(v, lane, out, slot);
          const int64_t kpos = (int64_t)lo + j;
          if (slot >= 0 && kpos < det_keys) det[(int64_t)GS_SGRAD_FLOATS * kpos + slot] = out;
        } else {
#if GSR_BWD_PAIR
          const int gid = kPack ? (int)(fl >> kGidShift) : s_gid[warp][buf][j];
#if GSR_BWD_PAIR_INPLACE
          // the pending key's first stage is reduced straight into h_p (no register copies)
          if (gid_p >= 0) {
            float h[5];
            reduce_half10(v, lane, h);
            reduce_pair_commit(h_p, h, gid_p, gid, lane, sgrad);
            gid_p = -1;
          } else {
            reduce_half10(v, lane, h_p);
            gid_p = gid;
          }
#else
          float h[5];
          reduce_half10(v, lane, h);
          if (gid_p >= 0) {
            reduce_pair_commit(h_p, h, gid_p, gid, lane, sgrad);
            gid_p = -1;
          } else {
#pragma unroll
            for (int k = 0; k < 5; ++k) h_p[k] = h[k];
            gid_p = gid;
          }
#endif
#else
          float out;
          int slot;
          warp_reduce10(v, lane, out, slot);
          if (slot >= 0) atomicAdd(sgrad + (int64_t)GS_SGRAD_FLOATS * s_gid[warp][buf][j] + slot, out);
#endif
        }
      }
    }
    __syncwarp();
    kb_cur = kb1, id1 = id2, kb1 = kb2;
  }
  cp_async_wait<0>();
#if GSR_BWD_PAIR
  if (gid_p >= 0) {
    const float z[5] = {0.f, 0.f, 0.f, 0.f, 0.f};
    reduce_pair_commit(h_p, z, gid_p, -1, lane, sgrad);
  }
#endif
}

#else  // GSR_EXACT_EXP
// ===========================================================================
// Exact path (libgsr_exact.so): the oracle's fp32 operation order, exp in double.
// ===========================================================================
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

// replaces the rect word with the block mask
__device__ __forceinline__ void finish_stage(float4* dst, int ox, int oy) {
  const float4 q0 = dst[0], q1 = dst[1];
  reinterpret_cast<float*>(dst + 2)[3] = __uint_as_float(block_mask(q0.x, q0.y, q1.x, q1.y, q1.z, q0.w, ox, oy));
}

// Blocks (8x4) all of whose pixels in this warp have bit set in `bits`.
__device__ __forceinline__ uint32_t blocks_all(uint32_t bits) { return __reduce_and_sync(kFull, bits); }

// power in the oracle's order; returns the "power <= 0" test and G = exp(power)
__device__ __forceinline__ bool eval_gauss(float mx, float my, float A, float B, float C, float pxf, float pyf,
                                           float& G, float& dx, float& dy) {
  dx = __fsub_rn(mx, pxf);
  dy = __fsub_rn(my, pyf);
  const float power =
      __fsub_rn(__fmul_rn(-0.5f, __fadd_rn(__fmul_rn(__fmul_rn(A, dx), dx), __fmul_rn(__fmul_rn(C, dy), dy))),
                __fmul_rn(__fmul_rn(B, dx), dy));
  G = (float)exp((double)power);
  return !(power > 0.f);
}

__global__ void __launch_bounds__(kWarpsPerCta * 32) k_render_fwd(DevCam cam, const float4* __restrict__ rec,
                                                                   const int32_t* __restrict__ ids,
                                                                   const int2* __restrict__ ranges, const int32_t* __restrict__ order,
                                                                   float* __restrict__ out_rgb,
                                                                   float* __restrict__ out_d, float* __restrict__ out_T,
                                                                   int32_t* __restrict__ out_n,
                                                                   unsigned long long* blended,
                                                                   uint8_t* __restrict__ key_blocks) {
  __shared__ float4 s_rec[kWarpsPerCta][2][32][3];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wslot = blockIdx.x * kWarpsPerCta + warp;
  if (wslot >= cam.TX * cam.TY) return;
  const int tile = order ? order[wslot] : wslot;  // work order (gs_tile_order)
  const int tx = tile % cam.TX, ty = tile / cam.TX;
  const int ox = tx * kTile, oy = ty * kTile;
  const int lx = lane & 7, ly = lane >> 3;
  const float pxf0 = (float)(ox + lx), pyf0 = (float)(oy + ly);
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
    uint32_t kb_mine = 0;
    for (int j = 0; j < cnt; ++j) {
      const StagedRec q = load_staged(s_rec[warp][buf][j]);
      const uint32_t m = q.mask & ~bdone;
      if (m == 0) continue;
      const int pos1 = b0 + j - rg.x + 1;
      uint32_t lm = 0;
#pragma unroll
      for (int b = 0; b < kPix; ++b) {
        if (!((m >> b) & 1u)) continue;
        float G, dx, dy;
        const bool pok = eval_gauss(q.mx, q.my, q.A, q.B, q.C, pxf0 + 8.f * (b & 1), pyf0 + 4.f * (b >> 1), G, dx, dy);
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
    const int x = ox + lx + 8 * (b & 1), y = oy + ly + 4 * (b >> 1);
    if (x < cam.W && y < cam.H) {
      const int64_t p = (int64_t)y * cam.W + x;
      out_rgb[p] = __fadd_rn(Cr[b], __fmul_rn(T[b], cam.bg[0]));
      out_rgb[npix + p] = __fadd_rn(Cg[b], __fmul_rn(T[b], cam.bg[1]));
      out_rgb[2 * npix + p] = __fadd_rn(Cb[b], __fmul_rn(T[b], cam.bg[2]));
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

__global__ void __launch_bounds__(kWarpsPerCta * 32) k_render_bwd(DevCam cam, const float4* __restrict__ rec,
                                                                   const int32_t* __restrict__ ids,
                                                                   const int2* __restrict__ ranges, const int32_t* __restrict__ order,
                                                                   const float* __restrict__ T_final,
                                                                   const int32_t* __restrict__ n_contrib,
                                                                   const float* __restrict__ g_rgb,
                                                                   const float* __restrict__ g_dep,
                                                                   const uint8_t* __restrict__ key_blocks,
                                                                   float* __restrict__ sgrad, L1Fuse l1,
                                                                   float* __restrict__ det, int64_t det_keys) {
  __shared__ float4 s_rec[kWarpsPerCta][2][32][3];
  __shared__ int s_gid[kWarpsPerCta][2][32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wslot = blockIdx.x * kWarpsPerCta + warp;
  if (wslot >= cam.TX * cam.TY) return;
  const int tile = order ? order[wslot] : wslot;  // work order (gs_tile_order)
  const int tx = tile % cam.TX, ty = tile / cam.TX;
  const int ox = tx * kTile, oy = ty * kTile;
  const int lx = lane & 7, ly = lane >> 3;
  const float pxf0 = (float)(ox + lx), pyf0 = (float)(oy + ly);
  const int2 rg = ranges[tile];
  const int64_t npix = (int64_t)cam.W * cam.H;

  float T[kPix], Q[kPix], gr[kPix], gg[kPix], gb[kPix], gd[kPix];
  int n[kPix];
  int bmaxn[kPix];
  int maxn = 0;
  float lsum = 0.f;
#pragma unroll
  for (int b = 0; b < kPix; ++b) {
    const int x = ox + lx + 8 * (b & 1), y = oy + ly + 4 * (b >> 1);
    if (x < cam.W && y < cam.H) {
      const int64_t p = (int64_t)y * cam.W + x;
      T[b] = T_final[p];
      n[b] = n_contrib[p];
      upstream(l1, g_rgb, g_dep, npix, p, gr[b], gg[b], gb[b], gd[b], lsum);
    } else {
      T[b] = 1.f, n[b] = 0, gr[b] = gg[b] = gb[b] = gd[b] = 0.f;
    }
    Q[b] = T[b] * (gr[b] * cam.bg[0] + gg[b] * cam.bg[1] + gb[b] * cam.bg[2]);
    bmaxn[b] = __reduce_max_sync(kFull, n[b]);
    maxn = max(maxn, bmaxn[b]);
  }
  l1_commit(l1, lsum, lane);
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
      const int j = 31 - __clz(live);
      live &= ~(1u << j);
      const StagedRec q = load_staged(s_rec[warp][buf][j]);
      const int pos = lo + j - rg.x;
      uint32_t m;
      if (key_blocks) {
        m = __shfl_sync(kFull, kb_cur, j);
      } else {
        m = q.mask;
#pragma unroll
        for (int b = 0; b < kPix; ++b)
          if (pos >= bmaxn[b]) m &= ~(1u << b);
        if (m == 0) continue;
      }
      float acc_r = 0.f, acc_g = 0.f, acc_b = 0.f, acc_z = 0.f, acc_o = 0.f;
      float s0[2] = {0.f, 0.f}, s1[2] = {0.f, 0.f}, s2 = 0.f;
      bool any = false;
#pragma unroll
      for (int b = 0; b < kPix; ++b) {
        if (!((m >> b) & 1u)) continue;
        float G, dx, dy;
        const bool pok = eval_gauss(q.mx, q.my, q.A, q.B, q.C, pxf0 + 8.f * (b & 1), pyf0 + 4.f * (b >> 1), G, dx, dy);
        const float raw = __fmul_rn(q.o, G);
        const float alpha = fminf(kAlphaCap, raw);
        const bool valid = pos < n[b] && pok && !(alpha < kAlphaMin);
        if (!__any_sync(kFull, valid)) continue;
        any = true;
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
        const float dx0 = __fsub_rn(q.mx, pxf0), dx1 = __fsub_rn(q.mx, pxf0 + 8.f);
        const float sx = dx0 * s0[0] + dx1 * s0[1];
        const float sxx = dx0 * dx0 * s0[0] + dx1 * dx1 * s0[1];
        const float sy = s1[0] + s1[1];
        const float sxy = dx0 * s1[0] + dx1 * s1[1];
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
        if (det) {
          const int64_t kpos = (int64_t)lo + j;
          if (slot >= 0 && kpos < det_keys) det[(int64_t)GS_SGRAD_FLOATS * kpos + slot] = out;
        } else if (slot >= 0) {
          atomicAdd(sgrad + (int64_t)GS_SGRAD_FLOATS * s_gid[warp][buf][j] + slot, out);
        }
      }
    }
    __syncwarp();
    kb_cur = kb1, id1 = id2, kb1 = kb2;
  }
  cp_async_wait<0>();
}
#endif  // GSR_EXACT_EXP

// Deterministic mode, second pass: one thread per visible Gaussian sums its (tile, key)
// partials in a fixed order -- the tiles of its rectangle, row-major -- and adds them to
// its screen-gradient entry (no atomics: one writer per entry).  Its key in tile t is
// found by a binary search of t's list on the sort key (depth bits, index) (R12).
__global__ void __launch_bounds__(256) k_det_reduce(DevCam cam, const float4* __restrict__ rec,
                                                    const int32_t* __restrict__ radius,
                                                    const int32_t* __restrict__ ids, const int2* __restrict__ ranges,
                                                    const float* __restrict__ det, int64_t det_keys, int64_t P,
                                                    float* __restrict__ sgrad) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= P || radius[i] <= 0) return;
  const float4 q0 = rec[3 * i], q2 = rec[3 * i + 2];
  const uint32_t zb = __float_as_uint(q0.z);
  const uint32_t rx = __float_as_uint(q2.z), ry = __float_as_uint(q2.w);
  const int x0 = (int)(rx & 0xffffu), x1 = (int)(rx >> 16), y0 = (int)(ry & 0xffffu), y1 = (int)(ry >> 16);
  float acc[10];
#pragma unroll
  for (int k = 0; k < 10; ++k) acc[k] = 0.f;
  for (int ty = y0; ty < y1; ++ty)
    for (int tx = x0; tx < x1; ++tx) {
      const int2 rg = ranges[ty * cam.TX + tx];
      int lo = rg.x, hi = rg.y;
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        const int g = ids[mid];
        const uint32_t zg = __float_as_uint(rec[3 * (int64_t)g].z);
        if (zg < zb || (zg == zb && g < i)) lo = mid + 1;
        else hi = mid;
      }
      if (lo < rg.y && ids[lo] == i && lo < det_keys) {
        const float* d = det + (int64_t)GS_SGRAD_FLOATS * lo;
#pragma unroll
        for (int k = 0; k < 10; ++k) acc[k] += d[k];
      }
    }
  float* o = sgrad + (int64_t)GS_SGRAD_FLOATS * i;
#pragma unroll
  for (int k = 0; k < 10; ++k) o[k] += acc[k];
}

// gs_set_render_rows (process-wide, performance only: both settings give the same results)
std::atomic<int> g_render_rows{0};

#ifndef GSR_EXACT_EXP
// Warps (= tiles) per CTA of the fast kernels.  Tile work is very uneven (list lengths
// and early termination), and a CTA's slot is held until its slowest warp ends, so
// small CTAs let the block scheduler balance tiles dynamically.  GSR_RENDER_WPC
// (1, 2 or 4) overrides the default for A/B runs.
int render_wpc() {
  static const int wpc = [] {
    const char* e = getenv("GSR_RENDER_WPC");
    const int v = e ? atoi(e) : 1;
    return (v == 2 || v == 4) ? v : 1;
  }();
  return wpc;
}

template <int WPC>
void launch_fwd_wpc(const DevCam& cam, const float* rec, const int32_t* ids, const int32_t* ranges, const int32_t* order, float* rgb,
                    float* depth, float* T_final, int32_t* n_contrib, unsigned long long* blended,
                    uint8_t* key_blocks, cudaStream_t s) {
  if constexpr (WPC == 1) {
    if (g_render_rows.load(std::memory_order_relaxed)) {
      k_render_fwd<1, true><<<cam.TX * cam.TY, 32, 0, s>>>(
          cam, reinterpret_cast<const float4*>(rec), ids, reinterpret_cast<const int2*>(ranges), order, rgb, depth,
          T_final, n_contrib, blended, key_blocks);
      return;
    }
  }
  k_render_fwd<WPC><<<ceil_div(cam.TX * cam.TY, WPC), WPC * 32, 0, s>>>(
      cam, reinterpret_cast<const float4*>(rec), ids, reinterpret_cast<const int2*>(ranges), order, rgb, depth, T_final,
      n_contrib, blended, key_blocks);
}
template <int WPC, bool kDet>
void launch_bwd_wpc(const DevCam& cam, const float* rec, const int32_t* ids, const int32_t* ranges, const int32_t* order,
                    const float* T_final, const int32_t* n_contrib, const float* g_rgb, const float* g_depth,
                    const uint8_t* key_blocks, float* sgrad, cudaStream_t s, const L1Fuse& l1, float* det,
                    int64_t det_keys, int64_t P) {
#define GSR_BWD_ARGS                                                                                              \
  cam, reinterpret_cast<const float4*>(rec), ids, reinterpret_cast<const int2*>(ranges), order, T_final, n_contrib, \
      g_rgb, g_depth, key_blocks, sgrad, l1, det, det_keys
  const bool rows = WPC == 1 && key_blocks && g_render_rows.load(std::memory_order_relaxed);
  if constexpr (!kDet) {
    if (GSR_BWD_PACK && key_blocks && P < (int64_t(1) << (32 - kGidShift))) {
      if (rows)
        k_render_bwd<1, true, false, true, true><<<cam.TX * cam.TY, 32, 0, s>>>(GSR_BWD_ARGS);
      else
        k_render_bwd<WPC, true, false, true><<<ceil_div(cam.TX * cam.TY, WPC), WPC * 32, 0, s>>>(GSR_BWD_ARGS);
      return;
    }
  }
  if (rows) {
    k_render_bwd<1, true, kDet, false, true><<<cam.TX * cam.TY, 32, 0, s>>>(GSR_BWD_ARGS);
    return;
  }
#undef GSR_BWD_ARGS
  if (key_blocks)
    k_render_bwd<WPC, true, kDet><<<ceil_div(cam.TX * cam.TY, WPC), WPC * 32, 0, s>>>(
        cam, reinterpret_cast<const float4*>(rec), ids, reinterpret_cast<const int2*>(ranges), order, T_final, n_contrib,
        g_rgb, g_depth, key_blocks, sgrad, l1, det, det_keys);
  else
    k_render_bwd<WPC, false, kDet><<<ceil_div(cam.TX * cam.TY, WPC), WPC * 32, 0, s>>>(
        cam, reinterpret_cast<const float4*>(rec), ids, reinterpret_cast<const int2*>(ranges), order, T_final, n_contrib,
        g_rgb, g_depth, key_blocks, sgrad, l1, det, det_keys);
}
#endif

}  // namespace

void set_render_rows(int v) { g_render_rows.store(v ? 1 : 0); }
int render_rows() { return g_render_rows.load(); }

void launch_render_fwd(const DevCam& cam, const float* rec, const int32_t* ids, const int32_t* ranges, const int32_t* order, float* rgb,
                       float* depth, float* T_final, int32_t* n_contrib, unsigned long long* blended,
                       uint8_t* key_blocks, cudaStream_t s) {
#ifndef GSR_EXACT_EXP
  switch (render_wpc()) {
    case 4: launch_fwd_wpc<4>(cam, rec, ids, ranges, order, rgb, depth, T_final, n_contrib, blended, key_blocks, s); break;
    case 2: launch_fwd_wpc<2>(cam, rec, ids, ranges, order, rgb, depth, T_final, n_contrib, blended, key_blocks, s); break;
    default: launch_fwd_wpc<1>(cam, rec, ids, ranges, order, rgb, depth, T_final, n_contrib, blended, key_blocks, s);
  }
#else
  k_render_fwd<<<ceil_div(cam.TX * cam.TY, kWarpsPerCta), kWarpsPerCta * 32, 0, s>>>(
      cam, reinterpret_cast<const float4*>(rec), ids, reinterpret_cast<const int2*>(ranges), order, rgb, depth, T_final,
      n_contrib, blended, key_blocks);
#endif
  count_launch();
}

void launch_render_bwd(const DevCam& cam, gs_proj proj, int64_t P, const int32_t* ids, const int32_t* ranges,
                       const int32_t* order, const float* T_final, const int32_t* n_contrib, const float* g_rgb,
                       const float* g_depth, const uint8_t* key_blocks, float* sgrad, cudaStream_t s,
                       const L1Targets* l1t, float* det, int64_t det_keys) {
  const float* rec = proj.rec;
  if (det && det_keys > 0) cudaMemsetAsync(det, 0, (size_t)det_keys * GS_SGRAD_FLOATS * sizeof(float), s);
  L1Fuse l1{};
  if (l1t) {
    const int64_t npix = (int64_t)cam.W * cam.H;
    l1.rgb = l1t->rgb, l1.depth = l1t->depth, l1.trgb = l1t->target_rgb, l1.tdep = l1t->target_depth;
    l1.sc = (float)(1.0 / (3.0 * (double)npix));  // as launch_l1
    l1.sd = (float)((double)l1t->w_depth / (double)npix);
    l1.loss = l1t->loss;
  }
#ifndef GSR_EXACT_EXP
  if (det) {  // deterministic mode: one warp per CTA
    launch_bwd_wpc<1, true>(cam, rec, ids, ranges, order, T_final, n_contrib, g_rgb, g_depth, key_blocks, sgrad, s, l1,
                            det, det_keys, P);
  } else {
    switch (render_wpc()) {
      case 4: launch_bwd_wpc<4, false>(cam, rec, ids, ranges, order, T_final, n_contrib, g_rgb, g_depth, key_blocks, sgrad, s, l1, nullptr, 0, P); break;
      case 2: launch_bwd_wpc<2, false>(cam, rec, ids, ranges, order, T_final, n_contrib, g_rgb, g_depth, key_blocks, sgrad, s, l1, nullptr, 0, P); break;
      default: launch_bwd_wpc<1, false>(cam, rec, ids, ranges, order, T_final, n_contrib, g_rgb, g_depth, key_blocks, sgrad, s, l1, nullptr, 0, P);
    }
  }
#else
  k_render_bwd<<<ceil_div(cam.TX * cam.TY, kWarpsPerCta), kWarpsPerCta * 32, 0, s>>>(
      cam, reinterpret_cast<const float4*>(rec), ids, reinterpret_cast<const int2*>(ranges), order, T_final, n_contrib,
      g_rgb, g_depth, key_blocks, sgrad, l1, det, det_keys);
#endif
  count_launch();
  if (det && P > 0) {
    k_det_reduce<<<ceil_div(P, 256), 256, 0, s>>>(cam, reinterpret_cast<const float4*>(rec), proj.radius, ids,
                                                   reinterpret_cast<const int2*>(ranges), det, det_keys, P, sgrad);
    count_launch();
  }
}

}  // namespace gsr
