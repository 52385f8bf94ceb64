// K1 project_fwd and K8 project_bwd (Eqs. 2-5; backward PAPER.md:147).
//
// HBM-bound streaming kernels: one thread per Gaussian, SoA parameter rows read
// with coalesced 32-bit loads (each warp touches one 128-B line per row), records
// written as three 16-B vector stores.  Culled Gaussians stop after the 24-B mean
// read and write only radius/tiles/flags (8 + 1 B).
//
// The forward chain up to the tile rectangle uses explicitly rounded fp32
// intrinsics in a fixed order and computes the activations exp/sigmoid in double
// (reading R9), so that mu, z, conic, opacity, radius, rect and tile counts are
// bit-identical to the fp32 CPU oracle.  The colour (SH) and the backward are free
// to use FMA contraction: their parity is a tolerance.
#include <cstdlib>

#include "gsr_internal.cuh"
#include "bulk_copy.cuh"
#include "sh_basis.cuh"

namespace gsr {
namespace {

#define FM(a, b) __fmul_rn((a), (b))
#define FA(a, b) __fadd_rn((a), (b))
#define FS(a, b) __fsub_rn((a), (b))
#define FD(a, b) __fdiv_rn((a), (b))

__device__ __forceinline__ float act_exp(float x) { return (float)exp((double)x); }
__device__ __forceinline__ float act_sigmoid(float x) { return (float)(1.0 / (1.0 + exp(-(double)x))); }

__device__ __forceinline__ void quat_to_rot(float w, float x, float y, float z, float R[3][3]) {
  R[0][0] = FS(1.f, FM(2.f, FA(FM(y, y), FM(z, z))));
  R[0][1] = FM(2.f, FS(FM(x, y), FM(w, z)));
  R[0][2] = FM(2.f, FA(FM(x, z), FM(w, y)));
  R[1][0] = FM(2.f, FA(FM(x, y), FM(w, z)));
  R[1][1] = FS(1.f, FM(2.f, FA(FM(x, x), FM(z, z))));
  R[1][2] = FM(2.f, FS(FM(y, z), FM(w, x)));
  R[2][0] = FM(2.f, FS(FM(x, z), FM(w, y)));
  R[2][1] = FM(2.f, FA(FM(y, z), FM(w, x)));
  R[2][2] = FS(1.f, FM(2.f, FA(FM(x, x), FM(y, y))));
}

__device__ __forceinline__ bool finitef(float v) { return isfinite(v); }

// ---------------------------------------------------------------------------
// O1-O7 for one Gaussian (mean already read): the fixed-order fp32 chain of R9.
// fetch(row) returns parameter row 3..10 of this Gaussian (read only if z_c > z_near).
// ---------------------------------------------------------------------------
struct Geom {
  float4 q0, q1;  // (mu_x, mu_y, z, opacity), (conic A, B, C, -)
  uint32_t rx, ry;
  int32_t rad, ntiles;
  uint8_t flags;
};

// O1-O2 (view independent): activations and Sigma.  ok = false for a degenerate
// quaternion (culled in every view).
struct Act {
  float Sig[3][3];
  float opa;
  bool ok;
};

template <class Fetch>
__device__ __forceinline__ Act project_act(Fetch fetch) {
  Act a;
  a.ok = false;
  // O1: activations (R3-R5, R9)
  const float l0 = fetch(3), l1 = fetch(4), l2 = fetch(5);
  const float qw = fetch(6), qx = fetch(7), qy = fetch(8), qz = fetch(9);
  const float logit = fetch(10);
  float s[3];
  s[0] = act_exp(l0);
  s[1] = act_exp(l1);
  s[2] = act_exp(l2);
  const float qn = __fsqrt_rn(FA(FA(FA(FM(qw, qw), FM(qx, qx)), FM(qy, qy)), FM(qz, qz)));
  if (!(qn > 0.f) || !finitef(qn)) return a;
  a.opa = act_sigmoid(logit);
  float R[3][3];
  quat_to_rot(FD(qw, qn), FD(qx, qn), FD(qy, qn), FD(qz, qn), R);
  // O2: Sigma = (R S)(R S)^T  (Eq. 2)
  float M[3][3];
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c) M[r][c] = FM(R[r][c], s[c]);
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c) a.Sig[r][c] = FA(FA(FM(M[r][0], M[c][0]), FM(M[r][1], M[c][1])), FM(M[r][2], M[c][2]));
  a.ok = true;
  return a;
}

// O3 and O4-O7 of one view.  act(): the Gaussian's Act, called only if z_c > z_near
// (so a Gaussian behind every camera never evaluates its activations).
// Conservative frustum pre-cull of a Gaussian in front of the near plane, BEFORE its
// activations (R9's IEEE chain and the double-precision exp / sigmoid): true only if
// the exact chain is certain to cull it at O7's rectangle test.  The O7 radius is
// rf = ceil(3 sqrt(lam)), lam the larger eigenvalue of T Sigma T^T + 0.3 I, and
// lam <= ||T||_F^2 max_k s_k^2 + 0.3 = ||J||_F^2 exp(2 lmax) + 0.3 (T = J W, W a
// rotation; Sigma = R S^2 R^T).  The bound is inflated (1% on each factor, +2 px) so
// that the fast fp32 evaluation here can only over-estimate; the mean's position is
// approximated to well under the 1 px slack.  A NaN anywhere fails every comparison
// and leaves the Gaussian to the exact chain.  Bit-identical outputs.
__device__ __forceinline__ bool precull(const DevCam& cam, float xc, float yc, float zc, float lmax) {
  const float iz = __frcp_rn(zc);
  const float ux = xc * iz, uy = yc * iz;
  const float uxc = fminf(fmaxf(ux, -cam.limx), cam.limx), uyc = fminf(fmaxf(uy, -cam.limy), cam.limy);
  const float jn2 = (cam.fx * cam.fx * fmaf(uxc, uxc, 1.f) + cam.fy * cam.fy * fmaf(uyc, uyc, 1.f)) * (iz * iz);
  const float smax = __expf(fminf(lmax, 80.f)) * 1.01f;
  const float R = fmaf(3.03f, sqrtf(fmaf(jn2 * 1.01f, smax * smax, 0.31f)), 2.f);
  const float mx = fmaf(cam.fx, ux, cam.cx), my = fmaf(cam.fy, uy, cam.cy);
  return (mx + R < -1.f) || (mx - R > (float)cam.W) || (my + R < -1.f) || (my - R > (float)cam.H);
}

template <class ActFn, class LmaxFn>
__device__ __forceinline__ Geom project_view(const DevCam& cam, float px, float py, float pz, ActFn act, LmaxFn lmax) {
  Geom g;
  // O3: p_c = W p + t  (Eq. 4)
  const float* W = cam.R;
  const float xc = FA(FA(FA(FM(W[0], px), FM(W[1], py)), FM(W[2], pz)), cam.t[0]);
  const float yc = FA(FA(FA(FM(W[3], px), FM(W[4], py)), FM(W[5], pz)), cam.t[1]);
  const float zc = FA(FA(FA(FM(W[6], px), FM(W[7], py)), FM(W[8], pz)), cam.t[2]);
  g.rad = 0, g.ntiles = 0;
  g.flags = GS_FLAG_CULLED;
  do {
    if (!(zc > cam.z_near)) break;  // R6, R23
    if (precull(cam, xc, yc, zc, lmax())) break;
    const Act& A = act();
    if (!A.ok) break;
    const float (&Sig)[3][3] = A.Sig;
    // O4: mean projection (Eq. 4), R1
    const float ux = FD(xc, zc), uy = FD(yc, zc);
    const float mux = FA(FM(cam.fx, ux), cam.cx);
    const float muy = FA(FM(cam.fy, uy), cam.cy);
    // O5: EWA (Eq. 5) with the 1.3x tangent clamp (R7) and the 0.3 low-pass (R8)
    const float limx = cam.limx, limy = cam.limy;  // 1.3 W / (2 fx), 1.3 H / (2 fy) (make_devcam)
    const float uxc = fminf(fmaxf(ux, -limx), limx);
    const float uyc = fminf(fmaxf(uy, -limy), limy);
    const float J00 = FD(cam.fx, zc), J02 = FD(-FM(cam.fx, uxc), zc);
    const float J11 = FD(cam.fy, zc), J12 = FD(-FM(cam.fy, uyc), zc);
    float T[2][3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      T[0][c] = FA(FM(J00, W[c]), FM(J02, W[6 + c]));
      T[1][c] = FA(FM(J11, W[3 + c]), FM(J12, W[6 + c]));
    }
    float MT[2][3];
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
      for (int c = 0; c < 3; ++c) MT[r][c] = FA(FA(FM(T[r][0], Sig[0][c]), FM(T[r][1], Sig[1][c])), FM(T[r][2], Sig[2][c]));
    const float a = FA(FA(FA(FM(MT[0][0], T[0][0]), FM(MT[0][1], T[0][1])), FM(MT[0][2], T[0][2])), 0.3f);
    const float b = FA(FA(FM(MT[0][0], T[1][0]), FM(MT[0][1], T[1][1])), FM(MT[0][2], T[1][2]));
    const float c = FA(FA(FA(FM(MT[1][0], T[1][0]), FM(MT[1][1], T[1][1])), FM(MT[1][2], T[1][2])), 0.3f);
    // O6: conic
    const float det = FS(FM(a, c), FM(b, b));
    if (!(det > 0.f) || !finitef(det)) break;
    const float cA = FD(c, det), cB = FD(-b, det), cC = FD(a, det);
    if (!finitef(cA) || !finitef(cB) || !finitef(cC) || !finitef(mux) || !finitef(muy)) break;
    // O7: radius and tile rectangle (R10, R11)
    const float mid = FM(0.5f, FA(a, c));
    const float disc = FS(FM(mid, mid), det);
    const float lam = FA(mid, __fsqrt_rn(fmaxf(disc, 0.f)));
    const float rf = ceilf(FM(3.f, __fsqrt_rn(lam)));
    float xlo = ceilf(FS(mux, rf)), xhi = floorf(FA(mux, rf));
    float ylo = ceilf(FS(muy, rf)), yhi = floorf(FA(muy, rf));
    xlo = fmaxf(xlo, 0.f);
    ylo = fmaxf(ylo, 0.f);
    xhi = fminf(xhi, (float)(cam.W - 1));
    yhi = fminf(yhi, (float)(cam.H - 1));
    if (!(xlo <= xhi) || !(ylo <= yhi)) break;
    const int x0 = (int)xlo / kTile, x1 = (int)xhi / kTile + 1;
    const int y0 = (int)ylo / kTile, y1 = (int)yhi / kTile + 1;
    g.rad = (int32_t)fminf(rf, (float)(1 << 30));
    g.ntiles = (x1 - x0) * (y1 - y0);
    g.flags = ((uxc != ux) ? GS_FLAG_JCLAMP_X : 0) | ((uyc != uy) ? GS_FLAG_JCLAMP_Y : 0);
    const uint32_t rx = (uint32_t)x0 | ((uint32_t)x1 << 16);
    const uint32_t ry = (uint32_t)y0 | ((uint32_t)y1 << 16);
    g.q0 = make_float4(mux, muy, zc, A.opa);
    g.q1 = make_float4(cA, cB, cC, 0.f);
    g.rx = rx, g.ry = ry;
  } while (0);
  return g;
}

template <class Fetch>
__device__ __forceinline__ Geom project_geom_one(const DevCam& cam, float px, float py, float pz, Fetch fetch) {
  Act a;
  return project_view(
      cam, px, py, pz,
      [&]() -> const Act& {
        a = project_act(fetch);
        return a;
      },
      [&]() { return fmaxf(fmaxf(fetch(3), fetch(4)), fetch(5)); });
}

// ---------------------------------------------------------------------------
// K1a (legacy, GSR_PROJECT=legacy): geometry of the projection (O1-O7), one thread
// per Gaussian with direct loads; K1b below adds the colour.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256, 3) k_project_geom(DevCam cam, int64_t P, int64_t S, const float* __restrict__ prm,
                                                          float4* __restrict__ rec, int32_t* __restrict__ radius_out,
                                                          int32_t* __restrict__ tiles_out,
                                                          uint8_t* __restrict__ flags_out) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < P; i += stride) {
    const float px = __ldg(prm + i), py = __ldg(prm + S + i), pz = __ldg(prm + 2 * S + i);
    const Geom g = project_geom_one(cam, px, py, pz, [&](int row) { return __ldg(prm + row * S + i); });
    if (g.rad > 0) {
      float4* r4 = rec + 3 * i;
      r4[0] = g.q0;
      reinterpret_cast<float2*>(r4 + 1)[0] = make_float2(g.q1.x, g.q1.y);
      reinterpret_cast<float*>(r4 + 1)[2] = g.q1.z;
      reinterpret_cast<float2*>(r4 + 2)[1] = make_float2(__uint_as_float(g.rx), __uint_as_float(g.ry));
    }
    radius_out[i] = g.rad;
    tiles_out[i] = g.ntiles;
    flags_out[i] = g.flags;
  }
}

// ---------------------------------------------------------------------------
// K1b: view-dependent SH colour of the visible Gaussians (O8, R13).
// ---------------------------------------------------------------------------
template <int DEG>
__global__ void __launch_bounds__(256, 4) k_project_color(DevCam cam, int64_t P, int64_t S,
                                                           const float* __restrict__ prm, float* __restrict__ rec,
                                                           const int32_t* __restrict__ radius,
                                                           uint8_t* __restrict__ flags) {
  constexpr int NK = (DEG + 1) * (DEG + 1);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < P; i += stride) {
    if (radius[i] == 0) continue;
    const float vx = __ldg(prm + i) - cam.ocam[0], vy = __ldg(prm + S + i) - cam.ocam[1],
                vz = __ldg(prm + 2 * S + i) - cam.ocam[2];
    const float inv = rsqrtf(vx * vx + vy * vy + vz * vz);
    const float x = vx * inv, y = vy * inv, z = vz * inv;
    float acc[3] = {0.f, 0.f, 0.f};
#pragma unroll
    for (int k = 0; k < NK; ++k) {
      float Y, gx, gy, gz;
      sh_term(k, x, y, z, Y, gx, gy, gz);
#pragma unroll
      for (int ch = 0; ch < 3; ++ch) acc[ch] = fmaf(__ldg(prm + (11 + 3 * k + ch) * S + i), Y, acc[ch]);
    }
    uint8_t fl = flags[i];
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) {
      acc[ch] += 0.5f;
      if (acc[ch] < 0.f) fl |= (uint8_t)(1u << ch);
      acc[ch] = fmaxf(acc[ch], 0.f);
    }
    flags[i] = fl;
    rec[12 * i + 7] = acc[0];
    *reinterpret_cast<float2*>(rec + 12 * i + 8) = make_float2(acc[1], acc[2]);
  }
}

// ---------------------------------------------------------------------------
// K1 (default): the whole projection (O1-O8) in one pass.  A CTA owns 128
// consecutive Gaussians; one thread stages their 11 geometry rows into shared
// memory with 1-D TMA bulk copies (11 x 512 B in flight per CTA, no register
// staging), the CTA computes O1-O7, and only if any of its Gaussians is visible
// (Morton order makes CTAs mostly all-visible or all-culled) it bulk-copies the
// 3 (deg+1)^2 SH rows and computes the colour (O8).  Each visible Gaussian's 48-B
// record is written once with three 16-B stores.
// ---------------------------------------------------------------------------
constexpr int kPjThreads = 128;

template <int DEG>
__global__ void __launch_bounds__(kPjThreads) k_project(DevCam cam, int64_t P, int64_t S,
                                                        const float* __restrict__ prm, float4* __restrict__ rec,
                                                        int32_t* __restrict__ radius_out,
                                                        int32_t* __restrict__ tiles_out,
                                                        uint8_t* __restrict__ flags_out) {
  constexpr int NK = (DEG + 1) * (DEG + 1), NSH = 3 * NK;
  __shared__ __align__(16) float s_geo[11][kPjThreads];
  __shared__ __align__(16) float s_sh[NSH][kPjThreads];
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x;
  const int64_t i0 = (int64_t)blockIdx.x * kPjThreads;
  // columns i0 .. i0 + ncol - 1 exist in every row (P_stride = S is a multiple of 4,
  // so the byte count is a multiple of 16 and every row segment is 16-B aligned)
  const int64_t ncol = S - i0 < kPjThreads ? S - i0 : (int64_t)kPjThreads;
  const uint32_t bytes = (uint32_t)ncol * 4u;
  if (tid == 0) mbar_init(&bar, 1);
  __syncthreads();
  if (tid == 0) {
    mbar_arrive_expect_tx(&bar, 11u * bytes);
#pragma unroll 1
    for (int r = 0; r < 11; ++r) bulk_g2s(s_geo[r], prm + r * S + i0, bytes, &bar);
  }
  mbar_wait(&bar, 0);
  const int64_t i = i0 + tid;
  Geom g;
  g.rad = 0, g.ntiles = 0, g.flags = GS_FLAG_CULLED;
  if (i < P) g = project_geom_one(cam, s_geo[0][tid], s_geo[1][tid], s_geo[2][tid], [&](int row) { return s_geo[row][tid]; });
  const bool vis = g.rad > 0;
  if (__syncthreads_or(vis)) {
    if (tid == 0) {
      mbar_arrive_expect_tx(&bar, (uint32_t)NSH * bytes);
#pragma unroll 1
      for (int r = 0; r < NSH; ++r) bulk_g2s(s_sh[r], prm + (11 + r) * S + i0, bytes, &bar);
    }
    mbar_wait(&bar, 1);
    if (vis) {
      // O8: SH colour at the mean's viewing direction (R13); same arithmetic as K1b
      const float vx = s_geo[0][tid] - cam.ocam[0], vy = s_geo[1][tid] - cam.ocam[1], vz = s_geo[2][tid] - cam.ocam[2];
      const float inv = rsqrtf(vx * vx + vy * vy + vz * vz);
      const float x = vx * inv, y = vy * inv, z = vz * inv;
      float acc[3] = {0.f, 0.f, 0.f};
#pragma unroll
      for (int k = 0; k < NK; ++k) {
        float Y, gx, gy, gz;
        sh_term(k, x, y, z, Y, gx, gy, gz);
#pragma unroll
        for (int ch = 0; ch < 3; ++ch) acc[ch] = fmaf(s_sh[3 * k + ch][tid], Y, acc[ch]);
      }
#pragma unroll
      for (int ch = 0; ch < 3; ++ch) {
        acc[ch] += 0.5f;
        if (acc[ch] < 0.f) g.flags |= (uint8_t)(1u << ch);
        acc[ch] = fmaxf(acc[ch], 0.f);
      }
      float4* r4 = rec + 3 * i;
      r4[0] = g.q0;
      r4[1] = make_float4(g.q1.x, g.q1.y, g.q1.z, acc[0]);
      r4[2] = make_float4(acc[1], acc[2], __uint_as_float(g.rx), __uint_as_float(g.ry));
    }
  }
  if (i < P) {
    radius_out[i] = g.rad;
    tiles_out[i] = g.ntiles;
    flags_out[i] = g.flags;
  }
}

// K1 over a batch of <= 8 views (gs_project_views): the 11 geometry rows (and, if a
// Gaussian of the CTA is visible in any view, the SH rows) are staged ONCE for all the
// views, instead of once per view, and the activations / Sigma (O1-O2) are evaluated
// once per Gaussian.  Pass 1 computes O1-O7 for every view and writes
// each view's record geometry, radius and tiles; pass 2 computes the colour (O8) of
// every view's visible Gaussians and writes the colour and the flags.  The per-view
// arithmetic is k_project's, so every output is bit-identical to gs_project's.
struct ViewOuts {
  DevCam cam[kMaxViews];
  float4* rec[kMaxViews];
  int32_t* radius[kMaxViews];
  int32_t* tiles[kMaxViews];
  uint8_t* flags[kMaxViews];
  int n;
};

template <int DEG>
__global__ void __launch_bounds__(kPjThreads) k_project_views(const __grid_constant__ ViewOuts vo, int64_t P, int64_t S,
                                                              const float* __restrict__ prm) {
  constexpr int NK = (DEG + 1) * (DEG + 1), NSH = 3 * NK;
  __shared__ __align__(16) float s_geo[11][kPjThreads];
  __shared__ __align__(16) float s_sh[NSH][kPjThreads];
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x;
  const int64_t i0 = (int64_t)blockIdx.x * kPjThreads;
  const int64_t ncol = S - i0 < kPjThreads ? S - i0 : (int64_t)kPjThreads;
  const uint32_t bytes = (uint32_t)ncol * 4u;
  if (tid == 0) mbar_init(&bar, 1);
  __syncthreads();
  if (tid == 0) {
    mbar_arrive_expect_tx(&bar, 11u * bytes);
#pragma unroll 1
    for (int r = 0; r < 11; ++r) bulk_g2s(s_geo[r], prm + r * S + i0, bytes, &bar);
  }
  mbar_wait(&bar, 0);
  const int64_t i = i0 + tid;
  uint64_t fl8 = 0;  // view v's flags in byte v
  bool any = false;
  Act act;  // O1-O2, computed once (at the first view that needs them) for all views
  bool have_act = false;
#pragma unroll 1
  for (int v = 0; v < vo.n; ++v) {
    Geom g;
    g.rad = 0, g.ntiles = 0, g.flags = GS_FLAG_CULLED;
    if (i < P)
      g = project_view(
          vo.cam[v], s_geo[0][tid], s_geo[1][tid], s_geo[2][tid],
          [&]() -> const Act& {
            if (!have_act) {
              act = project_act([&](int row) { return s_geo[row][tid]; });
              have_act = true;
            }
            return act;
          },
          [&]() { return fmaxf(fmaxf(s_geo[3][tid], s_geo[4][tid]), s_geo[5][tid]); });
    fl8 |= (uint64_t)g.flags << (8 * v);
    if (g.rad > 0) {
      any = true;
      float4* r4 = vo.rec[v] + 3 * i;
      r4[0] = g.q0;
      r4[1] = make_float4(g.q1.x, g.q1.y, g.q1.z, 0.f);
      r4[2] = make_float4(0.f, 0.f, __uint_as_float(g.rx), __uint_as_float(g.ry));
    }
    if (i < P) {
      vo.radius[v][i] = g.rad;
      vo.tiles[v][i] = g.ntiles;
    }
  }
  if (__syncthreads_or(any)) {
    if (tid == 0) {
      mbar_arrive_expect_tx(&bar, (uint32_t)NSH * bytes);
#pragma unroll 1
      for (int r = 0; r < NSH; ++r) bulk_g2s(s_sh[r], prm + (11 + r) * S + i0, bytes, &bar);
    }
    mbar_wait(&bar, 1);
#pragma unroll 1
    for (int v = 0; v < vo.n; ++v) {
      uint8_t f = (uint8_t)(fl8 >> (8 * v));
      if (f & GS_FLAG_CULLED) continue;
      // O8: SH colour at the mean's viewing direction (R13); k_project's arithmetic
      const DevCam& cam = vo.cam[v];
      const float vx = s_geo[0][tid] - cam.ocam[0], vy = s_geo[1][tid] - cam.ocam[1], vz = s_geo[2][tid] - cam.ocam[2];
      const float inv = rsqrtf(vx * vx + vy * vy + vz * vz);
      const float x = vx * inv, y = vy * inv, z = vz * inv;
      float acc[3] = {0.f, 0.f, 0.f};
#pragma unroll
      for (int k = 0; k < NK; ++k) {
        float Y, gx, gy, gz;
        sh_term(k, x, y, z, Y, gx, gy, gz);
#pragma unroll
        for (int ch = 0; ch < 3; ++ch) acc[ch] = fmaf(s_sh[3 * k + ch][tid], Y, acc[ch]);
      }
#pragma unroll
      for (int ch = 0; ch < 3; ++ch) {
        acc[ch] += 0.5f;
        if (acc[ch] < 0.f) f |= (uint8_t)(1u << ch);
        acc[ch] = fmaxf(acc[ch], 0.f);
      }
      float* r = reinterpret_cast<float*>(vo.rec[v] + 3 * i);
      r[7] = acc[0];
      *reinterpret_cast<float2*>(r + 8) = make_float2(acc[1], acc[2]);
      fl8 = (fl8 & ~((uint64_t)0xff << (8 * v))) | ((uint64_t)f << (8 * v));
    }
  }
  if (i < P)
    for (int v = 0; v < vo.n; ++v) vo.flags[v][i] = (uint8_t)(fl8 >> (8 * v));
}

// O8 of one visible Gaussian: SH colour at the mean's viewing direction (R13),
// coefficients fetched by sh(row) (row = 3k + ch); +0.5, clamp at 0, clamp flags.
// The arithmetic of every projection kernel (gs_project and gs_project_views agree).
template <int DEG, class ShFetch>
__device__ __forceinline__ void sh_colour(const DevCam& cam, float px, float py, float pz, ShFetch sh, float (&acc)[3],
                                          uint8_t& flags) {
  constexpr int NK = (DEG + 1) * (DEG + 1);
  const float vx = px - cam.ocam[0], vy = py - cam.ocam[1], vz = pz - cam.ocam[2];
  const float inv = rsqrtf(vx * vx + vy * vy + vz * vz);
  const float x = vx * inv, y = vy * inv, z = vz * inv;
  acc[0] = acc[1] = acc[2] = 0.f;
#pragma unroll
  for (int k = 0; k < NK; ++k) {
    float Y, gx, gy, gz;
    sh_term(k, x, y, z, Y, gx, gy, gz);
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) acc[ch] = fmaf(sh(3 * k + ch), Y, acc[ch]);
  }
#pragma unroll
  for (int ch = 0; ch < 3; ++ch) {
    acc[ch] += 0.5f;
    if (acc[ch] < 0.f) flags |= (uint8_t)(1u << ch);
    acc[ch] = fmaxf(acc[ch], 0.f);
  }
}

// O3's camera z of a mean (the fixed-order chain of project_view).
__device__ __forceinline__ float cam_z(const DevCam& cam, float px, float py, float pz) {
  const float* W = cam.R;
  return FA(FA(FA(FM(W[6], px), FM(W[7], py)), FM(W[8], pz)), cam.t[2]);
}

#ifndef GSR_PROJ_SPEC
#define GSR_PROJ_SPEC 1
#endif
#ifndef GSR_PROJV_SPEC
#define GSR_PROJV_SPEC 1  // scannetpp 8 views 139 -> 117 us, config 4 416 -> 343 us (bit-identical)
#endif
#ifndef GSR_PROJ_MINB
#define GSR_PROJ_MINB 10  // k_project2 CTAs per SM (register cap)
#endif
#ifndef GSR_PROJV_MINB
#define GSR_PROJV_MINB 8  // k_project_views2 CTAs per SM (register cap)
#endif
// ---------------------------------------------------------------------------
// K1 v2 (default): as K1, with the bytes a view does not need left in HBM and twice
// the Gaussians in flight per SM.
//  * The 3 mean rows are staged first (TMA bulk, 1.5 KB); only if a Gaussian of the
//    CTA lies in front of the near plane (R6) are the other 8 geometry rows staged:
//    with the Morton layout whole CTAs lie behind the camera, and they move 12 B per
//    Gaussian instead of 44.
//  * The SH coefficients are read straight from the parameter rows by the visible
//    threads only (coalesced 128-B rows per warp, no shared staging): no 24 KB of
//    shared memory per CTA, so 16 instead of 7 CTAs fit on an SM, and a partly
//    visible CTA reads no coefficient of its culled Gaussians.
// Same arithmetic as K1 (outputs bit-identical).
// ---------------------------------------------------------------------------
template <int DEG>
__global__ void __launch_bounds__(kPjThreads, GSR_PROJ_MINB) k_project2(DevCam cam, int64_t P, int64_t S,
                                                             const float* __restrict__ prm, float4* __restrict__ rec,
                                                             int32_t* __restrict__ radius_out,
                                                             int32_t* __restrict__ tiles_out,
                                                             uint8_t* __restrict__ flags_out) {
  __shared__ __align__(16) float s_geo[11][kPjThreads];
  __shared__ __align__(8) uint64_t bar[2];
  const int tid = threadIdx.x;
  const int64_t i0 = (int64_t)blockIdx.x * kPjThreads;
  const int64_t ncol = S - i0 < kPjThreads ? S - i0 : (int64_t)kPjThreads;
  const uint32_t bytes = (uint32_t)ncol * 4u;
  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
  }
  __syncthreads();
  if (tid == 0) {
    mbar_arrive_expect_tx(&bar[0], 3u * bytes);
#pragma unroll 1
    for (int r = 0; r < 3; ++r) bulk_g2s(s_geo[r], prm + r * S + i0, bytes, &bar[0]);
#if GSR_PROJ_SPEC
    // the 8 other rows speculatively in the same round trip (a CTA behind the camera
    // moves 32 B per Gaussian it does not need, every other CTA saves a round trip)
    mbar_arrive_expect_tx(&bar[1], 8u * bytes);
#pragma unroll 1
    for (int r = 3; r < 11; ++r) bulk_g2s(s_geo[r], prm + r * S + i0, bytes, &bar[1]);
#endif
  }
  mbar_wait(&bar[0], 0);
  const int64_t i = i0 + tid;
  const bool front = i < P && cam_z(cam, s_geo[0][tid], s_geo[1][tid], s_geo[2][tid]) > cam.z_near;
  Geom g;
  g.rad = 0, g.ntiles = 0, g.flags = GS_FLAG_CULLED;
  const bool any_front = __syncthreads_or(front);
#if GSR_PROJ_SPEC
  mbar_wait(&bar[1], 0);  // also when nothing is in front: no copy may outlive the CTA
#endif
  if (any_front) {
#if !GSR_PROJ_SPEC
    if (tid == 0) {
      mbar_arrive_expect_tx(&bar[1], 8u * bytes);
#pragma unroll 1
      for (int r = 3; r < 11; ++r) bulk_g2s(s_geo[r], prm + r * S + i0, bytes, &bar[1]);
    }
    mbar_wait(&bar[1], 0);
#endif
    if (front) g = project_geom_one(cam, s_geo[0][tid], s_geo[1][tid], s_geo[2][tid], [&](int row) { return s_geo[row][tid]; });
    if (g.rad > 0) {
      float acc[3];
      sh_colour<DEG>(cam, s_geo[0][tid], s_geo[1][tid], s_geo[2][tid],
                     [&](int row) { return __ldg(prm + (int64_t)(11 + row) * S + i); }, acc, g.flags);
      float4* r4 = rec + 3 * i;
      r4[0] = g.q0;
      r4[1] = make_float4(g.q1.x, g.q1.y, g.q1.z, acc[0]);
      r4[2] = make_float4(acc[1], acc[2], __uint_as_float(g.rx), __uint_as_float(g.ry));
    }
  }
  if (i < P) {
    radius_out[i] = g.rad;
    tiles_out[i] = g.ntiles;
    flags_out[i] = g.flags;
  }
}

// gs_project_views, v2: the same two changes for a batch of <= 8 views (the 8 other
// geometry rows staged if a Gaussian of the CTA is in front of ANY view's near plane;
// the SH coefficients read per visible (Gaussian, view) straight from the rows -- the
// second and later views hit L1 / L2).  Bit-identical to gs_project.
template <int DEG>
__global__ void __launch_bounds__(kPjThreads, GSR_PROJV_MINB) k_project_views2(const __grid_constant__ ViewOuts vo, int64_t P,
                                                                   int64_t S, const float* __restrict__ prm) {
  __shared__ __align__(16) float s_geo[11][kPjThreads];
  __shared__ __align__(8) uint64_t bar[2];
  const int tid = threadIdx.x;
  const int64_t i0 = (int64_t)blockIdx.x * kPjThreads;
  const int64_t ncol = S - i0 < kPjThreads ? S - i0 : (int64_t)kPjThreads;
  const uint32_t bytes = (uint32_t)ncol * 4u;
  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
  }
  __syncthreads();
  if (tid == 0) {
    mbar_arrive_expect_tx(&bar[0], 3u * bytes);
#pragma unroll 1
    for (int r = 0; r < 3; ++r) bulk_g2s(s_geo[r], prm + r * S + i0, bytes, &bar[0]);
#if GSR_PROJV_SPEC
    // the 8 other rows in the same round trip: with a batch of views around the scene
    // nearly every CTA has a Gaussian in front of some view
    mbar_arrive_expect_tx(&bar[1], 8u * bytes);
#pragma unroll 1
    for (int r = 3; r < 11; ++r) bulk_g2s(s_geo[r], prm + r * S + i0, bytes, &bar[1]);
#endif
  }
  mbar_wait(&bar[0], 0);
  const int64_t i = i0 + tid;
  bool front = false;
  if (i < P)
    for (int v = 0; v < vo.n; ++v) front = front || cam_z(vo.cam[v], s_geo[0][tid], s_geo[1][tid], s_geo[2][tid]) > vo.cam[v].z_near;
#if GSR_PROJV_SPEC
  mbar_wait(&bar[1], 0);  // also when nothing is in front: no copy may outlive the CTA
#endif
  const bool any_front = __syncthreads_or(front);
  if (!GSR_PROJV_SPEC && any_front) {
    if (tid == 0) {
      mbar_arrive_expect_tx(&bar[1], 8u * bytes);
#pragma unroll 1
      for (int r = 3; r < 11; ++r) bulk_g2s(s_geo[r], prm + r * S + i0, bytes, &bar[1]);
    }
    mbar_wait(&bar[1], 0);
  }
  Act act;
  bool have_act = false;
#pragma unroll 1
  for (int v = 0; v < vo.n; ++v) {
    Geom g;
    g.rad = 0, g.ntiles = 0, g.flags = GS_FLAG_CULLED;
    if (front)
      g = project_view(
          vo.cam[v], s_geo[0][tid], s_geo[1][tid], s_geo[2][tid],
          [&]() -> const Act& {
            if (!have_act) {
              act = project_act([&](int row) { return s_geo[row][tid]; });
              have_act = true;
            }
            return act;
          },
          [&]() { return fmaxf(fmaxf(s_geo[3][tid], s_geo[4][tid]), s_geo[5][tid]); });
    if (g.rad > 0) {
      float acc[3];
      sh_colour<DEG>(vo.cam[v], s_geo[0][tid], s_geo[1][tid], s_geo[2][tid],
                     [&](int row) { return __ldg(prm + (int64_t)(11 + row) * S + i); }, acc, g.flags);
      float4* r4 = vo.rec[v] + 3 * i;
      r4[0] = g.q0;
      r4[1] = make_float4(g.q1.x, g.q1.y, g.q1.z, acc[0]);
      r4[2] = make_float4(acc[1], acc[2], __uint_as_float(g.rx), __uint_as_float(g.ry));
    }
    if (i < P) {
      vo.radius[v][i] = g.rad;
      vo.tiles[v][i] = g.ntiles;
      vo.flags[v][i] = g.flags;
    }
  }
}

// Persistent, software-pipelined variant (GSR_PROJECT=pipe; slower, kept for A/B): grid = a few CTAs per SM, each
// walking tiles blockIdx.x, blockIdx.x + gridDim.x, ...  The geometry rows of the NEXT
// tile are bulk-copied (double buffer, one mbarrier per buffer) while the current
// tile computes O1-O7 and waits for its SH rows, so every CTA keeps a transfer in
// flight through its whole life instead of two exposed latency rounds per tile.
#ifndef GSR_PJ_CTAS
#define GSR_PJ_CTAS 4
#endif
constexpr int kPjCtasPerSm = GSR_PJ_CTAS;

template <int DEG>
__global__ void __launch_bounds__(kPjThreads) k_project_pipe(DevCam cam, int64_t P, int64_t S,
                                                             const float* __restrict__ prm, float4* __restrict__ rec,
                                                             int32_t* __restrict__ radius_out,
                                                             int32_t* __restrict__ tiles_out,
                                                             uint8_t* __restrict__ flags_out) {
  constexpr int NK = (DEG + 1) * (DEG + 1), NSH = 3 * NK;
  __shared__ __align__(16) float s_geo[2][11][kPjThreads];
  __shared__ __align__(16) float s_sh[NSH][kPjThreads];
  __shared__ __align__(8) uint64_t bar_g[2];
  __shared__ __align__(8) uint64_t bar_s;
  const int tid = threadIdx.x;
  const int64_t ntile = (P + kPjThreads - 1) / kPjThreads;
  auto tile_bytes = [&](int64_t t) {
    const int64_t i0 = t * kPjThreads;
    return (uint32_t)((S - i0 < kPjThreads ? S - i0 : (int64_t)kPjThreads) * 4);
  };
  auto issue_geo = [&](int64_t t, int b) {
    const uint32_t bytes = tile_bytes(t);
    fence_proxy_async_smem();  // the buffer's previous tile was read by the generic proxy
    mbar_arrive_expect_tx(&bar_g[b], 11u * bytes);
#pragma unroll 1
    for (int r = 0; r < 11; ++r) bulk_g2s(s_geo[b][r], prm + r * S + t * kPjThreads, bytes, &bar_g[b]);
  };
  if (tid == 0) {
    mbar_init(&bar_g[0], 1);
    mbar_init(&bar_g[1], 1);
    mbar_init(&bar_s, 1);
  }
  __syncthreads();
  int64_t t = blockIdx.x;
  if (tid == 0 && t < ntile) issue_geo(t, 0);
  uint32_t sh_uses = 0;
  for (int k = 0; t < ntile; ++k, t += gridDim.x) {
    const int b = k & 1;
    const int64_t tn = t + gridDim.x;
    if (tid == 0 && tn < ntile) issue_geo(tn, b ^ 1);  // buffer b ^ 1 was released by the last __syncthreads
    mbar_wait(&bar_g[b], (uint32_t)(k >> 1) & 1u);
    const int64_t i = t * kPjThreads + tid;
    Geom g;
    g.rad = 0, g.ntiles = 0, g.flags = GS_FLAG_CULLED;
    if (i < P)
      g = project_geom_one(cam, s_geo[b][0][tid], s_geo[b][1][tid], s_geo[b][2][tid],
                           [&](int row) { return s_geo[b][row][tid]; });
    const bool vis = g.rad > 0;
    if (__syncthreads_or(vis)) {
      if (tid == 0) {
        const uint32_t bytes = tile_bytes(t);
        fence_proxy_async_smem();
        mbar_arrive_expect_tx(&bar_s, (uint32_t)NSH * bytes);
#pragma unroll 1
        for (int r = 0; r < NSH; ++r) bulk_g2s(s_sh[r], prm + (11 + r) * S + t * kPjThreads, bytes, &bar_s);
      }
      mbar_wait(&bar_s, sh_uses & 1u);
      ++sh_uses;
      if (vis) {
        const float vx = s_geo[b][0][tid] - cam.ocam[0], vy = s_geo[b][1][tid] - cam.ocam[1],
                    vz = s_geo[b][2][tid] - cam.ocam[2];
        const float inv = rsqrtf(vx * vx + vy * vy + vz * vz);
        const float x = vx * inv, y = vy * inv, z = vz * inv;
        float acc[3] = {0.f, 0.f, 0.f};
#pragma unroll
        for (int kk = 0; kk < NK; ++kk) {
          float Y, gx, gy, gz;
          sh_term(kk, x, y, z, Y, gx, gy, gz);
#pragma unroll
          for (int ch = 0; ch < 3; ++ch) acc[ch] = fmaf(s_sh[3 * kk + ch][tid], Y, acc[ch]);
        }
#pragma unroll
        for (int ch = 0; ch < 3; ++ch) {
          acc[ch] += 0.5f;
          if (acc[ch] < 0.f) g.flags |= (uint8_t)(1u << ch);
          acc[ch] = fmaxf(acc[ch], 0.f);
        }
        float4* r4 = rec + 3 * i;
        r4[0] = g.q0;
        r4[1] = make_float4(g.q1.x, g.q1.y, g.q1.z, acc[0]);
        r4[2] = make_float4(acc[1], acc[2], __uint_as_float(g.rx), __uint_as_float(g.ry));
      }
    }
    if (i < P) {
      radius_out[i] = g.rad;
      tiles_out[i] = g.ntiles;
      flags_out[i] = g.flags;
    }
    __syncthreads();  // s_geo[b] and s_sh are free again
  }
}

// GSR_PROJECT: "legacy" (two kernels, direct loads), "pipe" (persistent pipelined),
// default "tma" (one 128-Gaussian tile per CTA).  Measured per scannetpp view:
// legacy 54 us, pipe 53 us (4 CTAs/SM; 41 us at 6), tma 38 us -- the one-tile CTAs
// keep 7 independent latency chains per SM, the persistent ones only 4-6.
int project_mode() {
  static const int mode = [] {
    const char* e = getenv("GSR_PROJECT");
    if (e && e[0] == 'l') return 0;
    if (e && e[0] == 'p') return 2;
    if (e && e[0] == 't') return 1;
    return 3;
  }();
  return mode;
}

}  // namespace

void launch_project_views(int n_views, const DevCam* cams, int64_t P, int64_t S, int deg, const float* params,
                          const gs_proj* outs, cudaStream_t s) {
  const int grid = (int)((P + kPjThreads - 1) / kPjThreads);
  for (int v0 = 0; v0 < n_views; v0 += kMaxViews) {
    ViewOuts vo{};
    vo.n = std::min(kMaxViews, n_views - v0);
    for (int v = 0; v < vo.n; ++v) {
      vo.cam[v] = cams[v0 + v];
      vo.rec[v] = reinterpret_cast<float4*>(outs[v0 + v].rec);
      vo.radius[v] = outs[v0 + v].radius;
      vo.tiles[v] = outs[v0 + v].tiles;
      vo.flags[v] = outs[v0 + v].flags;
    }
    if (project_mode() == 3) {
      switch (deg) {
        case 0: k_project_views2<0><<<grid, kPjThreads, 0, s>>>(vo, P, S, params); break;
        case 1: k_project_views2<1><<<grid, kPjThreads, 0, s>>>(vo, P, S, params); break;
        case 2: k_project_views2<2><<<grid, kPjThreads, 0, s>>>(vo, P, S, params); break;
        default: k_project_views2<3><<<grid, kPjThreads, 0, s>>>(vo, P, S, params); break;
      }
    } else {
      switch (deg) {
        case 0: k_project_views<0><<<grid, kPjThreads, 0, s>>>(vo, P, S, params); break;
        case 1: k_project_views<1><<<grid, kPjThreads, 0, s>>>(vo, P, S, params); break;
        case 2: k_project_views<2><<<grid, kPjThreads, 0, s>>>(vo, P, S, params); break;
        default: k_project_views<3><<<grid, kPjThreads, 0, s>>>(vo, P, S, params); break;
      }
    }
    count_launch();
  }
}

void launch_project(const DevCam& cam, int64_t P, int64_t S, int deg, const float* params, gs_proj out,
                    cudaStream_t s) {
  if (project_mode() == 2) {
    const int64_t ntile = (P + kPjThreads - 1) / kPjThreads;
    const int grid = (int)std::min<int64_t>(ntile, (int64_t)sm_count() * kPjCtasPerSm);
    float4* rec = reinterpret_cast<float4*>(out.rec);
    switch (deg) {
      case 0: k_project_pipe<0><<<grid, kPjThreads, 0, s>>>(cam, P, S, params, rec, out.radius, out.tiles, out.flags); break;
      case 1: k_project_pipe<1><<<grid, kPjThreads, 0, s>>>(cam, P, S, params, rec, out.radius, out.tiles, out.flags); break;
      case 2: k_project_pipe<2><<<grid, kPjThreads, 0, s>>>(cam, P, S, params, rec, out.radius, out.tiles, out.flags); break;
      default: k_project_pipe<3><<<grid, kPjThreads, 0, s>>>(cam, P, S, params, rec, out.radius, out.tiles, out.flags);
    }
    count_launch();
    return;
  }
  if (project_mode() == 3) {
    const int grid = (int)((P + kPjThreads - 1) / kPjThreads);
    float4* rec = reinterpret_cast<float4*>(out.rec);
    switch (deg) {
      case 0: k_project2<0><<<grid, kPjThreads, 0, s>>>(cam, P, S, params, rec, out.radius, out.tiles, out.flags); break;
      case 1: k_project2<1><<<grid, kPjThreads, 0, s>>>(cam, P, S, params, rec, out.radius, out.tiles, out.flags); break;
      case 2: k_project2<2><<<grid, kPjThreads, 0, s>>>(cam, P, S, params, rec, out.radius, out.tiles, out.flags); break;
      default: k_project2<3><<<grid, kPjThreads, 0, s>>>(cam, P, S, params, rec, out.radius, out.tiles, out.flags);
    }
    count_launch();
    return;
  }
  if (project_mode() == 1) {
    const int grid = (int)((P + kPjThreads - 1) / kPjThreads);
    float4* rec = reinterpret_cast<float4*>(out.rec);
    switch (deg) {
      case 0: k_project<0><<<grid, kPjThreads, 0, s>>>(cam, P, S, params, rec, out.radius, out.tiles, out.flags); break;
      case 1: k_project<1><<<grid, kPjThreads, 0, s>>>(cam, P, S, params, rec, out.radius, out.tiles, out.flags); break;
      case 2: k_project<2><<<grid, kPjThreads, 0, s>>>(cam, P, S, params, rec, out.radius, out.tiles, out.flags); break;
      default: k_project<3><<<grid, kPjThreads, 0, s>>>(cam, P, S, params, rec, out.radius, out.tiles, out.flags);
    }
    count_launch();
    return;
  }
  const int block = 256;
  const int grid = (int)std::min<int64_t>((P + block - 1) / block, (int64_t)sm_count() * 12);
  float4* rec = reinterpret_cast<float4*>(out.rec);
  k_project_geom<<<grid, block, 0, s>>>(cam, P, S, params, rec, out.radius, out.tiles, out.flags);
  const int gridc = (int)std::min<int64_t>((P + block - 1) / block, (int64_t)sm_count() * 16);
  switch (deg) {
    case 0: k_project_color<0><<<gridc, block, 0, s>>>(cam, P, S, params, out.rec, out.radius, out.flags); break;
    case 1: k_project_color<1><<<gridc, block, 0, s>>>(cam, P, S, params, out.rec, out.radius, out.flags); break;
    case 2: k_project_color<2><<<gridc, block, 0, s>>>(cam, P, S, params, out.rec, out.radius, out.flags); break;
    default: k_project_color<3><<<gridc, block, 0, s>>>(cam, P, S, params, out.rec, out.radius, out.flags); break;
  }
  count_launch(2);
}

}  // namespace gsr
