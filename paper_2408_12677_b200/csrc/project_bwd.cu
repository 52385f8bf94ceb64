// K8: the projection backward (exact derivative of k_project_geom / k_project_color,
// PAPER.md:147, readings R7, R13, R18), batched over up to kMaxViews views per pass.
//
// Per-view screen-space gradients (float[P][12], written by gs_render_bwd_screen) are
// chained to the parameter rows with every parameter row read and every gradient
// row written ONCE per batch of views instead of once per view: dL/dSigma and
// dL/dopacity are summed over the views before the view-independent Sigma -> (s, q)
// and sigmoid chains, and each SH gradient row accumulates all views in registers.
// In overwrite mode (accumulate == 0) the gradient rows are written without being
// read, which also makes a separate zeroing pass unnecessary.  Both kernels are
// HBM-streaming: one thread per Gaussian, coalesced SoA rows, every view's per-Gaussian
// loads issued before they are consumed (views fully unrolled).
#include "gsr_internal.cuh"
#include "sh_basis.cuh"

namespace gsr {
namespace {

// Reciprocals of the wide projection backward: rcp.approx (~1 ulp) instead of the IEEE
// division and its slow-path subroutine (gradients carry a 1e-3 relative tolerance;
// nothing here decides a bit-exact output): config 4 chain 2.76 -> 2.58 ms.  The <= 8
// view kernels keep IEEE divisions (there the change re-allocates registers and costs
// 224 -> 324 us).  GSR_PBWD_IEEE_DIV=1 restores IEEE.
#ifndef GSR_PBWD_IEEE_DIV
#define GSR_PBWD_IEEE_DIV 0
#endif
__device__ __forceinline__ float pb_rcp(float x) {
#if GSR_PBWD_IEEE_DIV
  return 1.f / x;
#else
  return __fdividef(1.f, x);
#endif
}


struct ViewBatch {
  DevCam cam[kMaxViews];
  const uint8_t* flags[kMaxViews];
  float* sgrad[kMaxViews];
  int n;
};

// K8a: SH rows and the view-direction term of the mean gradient (rows 0-2).
template <int DEG>
__global__ void __launch_bounds__(256, 2) k_project_bwd_color(const __grid_constant__ ViewBatch vb, int64_t P, int64_t S,
                                                               const float* __restrict__ prm, float* __restrict__ grad,
                                                               int accumulate) {
  constexpr int NK = (DEG + 1) * (DEG + 1);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < P; i += stride) {
    uint32_t fl[kMaxViews];
#pragma unroll
    for (int v = 0; v < kMaxViews; ++v) fl[v] = v < vb.n ? vb.flags[v][i] : (uint32_t)GS_FLAG_CULLED;
    float gc[kMaxViews][3];
#pragma unroll
    for (int v = 0; v < kMaxViews; ++v) {
      gc[v][0] = gc[v][1] = gc[v][2] = 0.f;
      if (!(fl[v] & GS_FLAG_CULLED)) {
        const float* sg = vb.sgrad[v] + 12 * i;
        const float2 g67 = *reinterpret_cast<const float2*>(sg + 6);
        const float g8 = sg[8];
        gc[v][0] = (fl[v] & 1) ? 0.f : g67.x;
        gc[v][1] = (fl[v] & 2) ? 0.f : g67.y;
        gc[v][2] = (fl[v] & 4) ? 0.f : g8;
      }
    }
    uint32_t live = 0;
#pragma unroll
    for (int v = 0; v < kMaxViews; ++v)
      live |= (gc[v][0] != 0.f || gc[v][1] != 0.f || gc[v][2] != 0.f) ? (1u << v) : 0u;
    if (!live) {
      if (!accumulate) {
#pragma unroll
        for (int r = 0; r < 3; ++r) grad[r * S + i] = 0.f;
#pragma unroll
        for (int r = 11; r < 11 + 3 * NK; ++r) grad[(int64_t)r * S + i] = 0.f;
      }
      continue;
    }
    const float px = prm[i], py = prm[S + i], pz = prm[2 * S + i];
    float d[kMaxViews][3], ivn[kMaxViews], gd[kMaxViews][3];
#pragma unroll
    for (int v = 0; v < kMaxViews; ++v) {
      const float vx = px - vb.cam[v].ocam[0], vy = py - vb.cam[v].ocam[1], vz = pz - vb.cam[v].ocam[2];
      ivn[v] = ((live >> v) & 1u) ? rsqrtf(vx * vx + vy * vy + vz * vz) : 0.f;
      d[v][0] = vx * ivn[v], d[v][1] = vy * ivn[v], d[v][2] = vz * ivn[v];
      gd[v][0] = gd[v][1] = gd[v][2] = 0.f;
    }
    // SH rows in groups of 4 coefficients: 12 (or 24) loads in flight per group
#pragma unroll
    for (int k0 = 0; k0 < NK; k0 += 4) {
      float sh[4][3], old[4][3];
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        const int k = k0 + kk;
#pragma unroll
        for (int ch = 0; ch < 3; ++ch) {
          const int64_t row = (int64_t)(11 + 3 * k + ch) * S + i;
          sh[kk][ch] = (k < NK && k > 0) ? prm[row] : 0.f;
          old[kk][ch] = (k < NK && accumulate) ? grad[row] : 0.f;
        }
      }
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        const int k = k0 + kk;
        if (k >= NK) break;
        float a0 = old[kk][0], a1 = old[kk][1], a2 = old[kk][2];
#pragma unroll
        for (int v = 0; v < kMaxViews; ++v) {
          if (!((live >> v) & 1u)) continue;
          float Y, gx, gy, gz;
          sh_term(k, d[v][0], d[v][1], d[v][2], Y, gx, gy, gz);
          a0 = fmaf(Y, gc[v][0], a0);
          a1 = fmaf(Y, gc[v][1], a1);
          a2 = fmaf(Y, gc[v][2], a2);
          if (k > 0) {
            const float w = sh[kk][0] * gc[v][0] + sh[kk][1] * gc[v][1] + sh[kk][2] * gc[v][2];
            gd[v][0] = fmaf(w, gx, gd[v][0]);
            gd[v][1] = fmaf(w, gy, gd[v][1]);
            gd[v][2] = fmaf(w, gz, gd[v][2]);
          }
        }
        float* g = grad + (int64_t)(11 + 3 * k) * S + i;
        g[0] = a0;
        g[S] = a1;
        g[2 * S] = a2;
      }
    }
    // d = v/|v|: dL/dv = (I - d d^T) dL/dd / |v|
    float gp0 = 0.f, gp1 = 0.f, gp2 = 0.f;
#pragma unroll
    for (int v = 0; v < kMaxViews; ++v) {
      const float dd = d[v][0] * gd[v][0] + d[v][1] * gd[v][1] + d[v][2] * gd[v][2];
      gp0 += (gd[v][0] - d[v][0] * dd) * ivn[v];
      gp1 += (gd[v][1] - d[v][1] * dd) * ivn[v];
      gp2 += (gd[v][2] - d[v][2] * dd) * ivn[v];
    }
    if (accumulate) {
      grad[i] += gp0;
      grad[S + i] += gp1;
      grad[2 * S + i] += gp2;
    } else {
      grad[i] = gp0;
      grad[S + i] = gp1;
      grad[2 * S + i] = gp2;
    }
  }
}

// K8b: geometry rows -- mean (via mu, J and depth; rows 0-2 always +=, after K8a),
// log-scale, quaternion and opacity (rows 3-10).  Consumes and clears every visible
// view's screen-gradient entry.
__global__ void __launch_bounds__(256, 2) k_project_bwd_geom(const __grid_constant__ ViewBatch vb, int64_t P, int64_t S,
                                                              const float* __restrict__ prm, float* __restrict__ grad,
                                                              int accumulate) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < P; i += stride) {
    uint32_t fl[kMaxViews];
#pragma unroll
    for (int v = 0; v < kMaxViews; ++v) fl[v] = v < vb.n ? vb.flags[v][i] : (uint32_t)GS_FLAG_CULLED;
    uint32_t vis = 0;
#pragma unroll
    for (int v = 0; v < kMaxViews; ++v) vis |= (fl[v] & GS_FLAG_CULLED) ? 0u : (1u << v);
    if (!vis) {
      if (!accumulate) {
#pragma unroll
        for (int r = 3; r < 11; ++r) grad[r * S + i] = 0.f;
      }
      continue;
    }
    const float px = prm[i], py = prm[S + i], pz = prm[2 * S + i];
    // Sigma = R diag(s)^2 R^T (view independent)
    const float q0 = prm[6 * S + i], q1 = prm[7 * S + i], q2 = prm[8 * S + i], q3 = prm[9 * S + i];
    const float iqn = rsqrtf(q0 * q0 + q1 * q1 + q2 * q2 + q3 * q3);
    const float w = q0 * iqn, x = q1 * iqn, y = q2 * iqn, z = q3 * iqn;
    float R[3][3];
    R[0][0] = 1.f - 2.f * (y * y + z * z), R[0][1] = 2.f * (x * y - w * z), R[0][2] = 2.f * (x * z + w * y);
    R[1][0] = 2.f * (x * y + w * z), R[1][1] = 1.f - 2.f * (x * x + z * z), R[1][2] = 2.f * (y * z - w * x);
    R[2][0] = 2.f * (x * z - w * y), R[2][1] = 2.f * (y * z + w * x), R[2][2] = 1.f - 2.f * (x * x + y * y);
    float s[3];
#pragma unroll
    for (int j = 0; j < 3; ++j) s[j] = __expf(prm[(3 + j) * S + i]);
    float Sig[6];
    {
      const float s0 = s[0] * s[0], s1 = s[1] * s[1], s2 = s[2] * s[2];
      Sig[0] = R[0][0] * R[0][0] * s0 + R[0][1] * R[0][1] * s1 + R[0][2] * R[0][2] * s2;
      Sig[1] = R[0][0] * R[1][0] * s0 + R[0][1] * R[1][1] * s1 + R[0][2] * R[1][2] * s2;
      Sig[2] = R[0][0] * R[2][0] * s0 + R[0][1] * R[2][1] * s1 + R[0][2] * R[2][2] * s2;
      Sig[3] = R[1][0] * R[1][0] * s0 + R[1][1] * R[1][1] * s1 + R[1][2] * R[1][2] * s2;
      Sig[4] = R[1][0] * R[2][0] * s0 + R[1][1] * R[2][1] * s1 + R[1][2] * R[2][2] * s2;
      Sig[5] = R[2][0] * R[2][0] * s0 + R[2][1] * R[2][1] * s1 + R[2][2] * R[2][2] * s2;
    }
    float gSig[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f};  // xx, xy, xz, yy, yz, zz
    float gp[3] = {0.f, 0.f, 0.f};
    float gop = 0.f;
    // every view's entry is loaded before any is cleared: the clearing stores could
    // alias later views' loads, which would otherwise serialise 8 round trips
    float4 sg0[kMaxViews];
    float2 sg1[kMaxViews];
    float sgz[kMaxViews];
#pragma unroll
    for (int v = 0; v < kMaxViews; ++v) {
      sg0[v] = make_float4(0.f, 0.f, 0.f, 0.f), sg1[v] = make_float2(0.f, 0.f), sgz[v] = 0.f;
      if ((vis >> v) & 1u) {
        const float4* sg4 = reinterpret_cast<const float4*>(vb.sgrad[v] + 12 * i);
        sg0[v] = sg4[0];
        sg1[v] = *reinterpret_cast<const float2*>(sg4 + 1);
        sgz[v] = reinterpret_cast<const float*>(sg4 + 2)[1];
      }
    }
#pragma unroll
    for (int v = 0; v < kMaxViews; ++v) {
      if ((vis >> v) & 1u) {  // consume and clear
        float4* sg4 = reinterpret_cast<float4*>(vb.sgrad[v] + 12 * i);
        sg4[0] = sg4[1] = sg4[2] = make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
#pragma unroll
    for (int v = 0; v < kMaxViews; ++v) {
      if (!((vis >> v) & 1u)) continue;
      const float4 g0 = sg0[v];
      const float2 g1 = sg1[v];
      const float gz = sgz[v];
      const float gmx = g0.x, gmy = g0.y, gA = g0.z, gB = g0.w, gC = g1.x;
      gop += g1.y;
      if (gmx == 0.f && gmy == 0.f && gA == 0.f && gB == 0.f && gC == 0.f && gz == 0.f) continue;
      const DevCam& cam = vb.cam[v];
      const float* W = cam.R;
      const float xc = W[0] * px + W[1] * py + W[2] * pz + cam.t[0];
      const float yc = W[3] * px + W[4] * py + W[5] * pz + cam.t[1];
      const float zc = W[6] * px + W[7] * py + W[8] * pz + cam.t[2];
      const float iz = 1.f / zc, iz2 = iz * iz;
      const float ux = xc * iz, uy = yc * iz;
      const float limx = cam.limx, limy = cam.limy;
      const bool jx = fl[v] & GS_FLAG_JCLAMP_X, jy = fl[v] & GS_FLAG_JCLAMP_Y;
      const float uxc = jx ? fminf(fmaxf(ux, -limx), limx) : ux;
      const float uyc = jy ? fminf(fmaxf(uy, -limy), limy) : uy;
      const float J00 = cam.fx * iz, J02 = -cam.fx * uxc * iz, J11 = cam.fy * iz, J12 = -cam.fy * uyc * iz;
      float T[2][3];
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        T[0][c] = J00 * W[c] + J02 * W[6 + c];
        T[1][c] = J11 * W[3 + c] + J12 * W[6 + c];
      }
      float TS[2][3];  // T Sigma
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        TS[r][0] = T[r][0] * Sig[0] + T[r][1] * Sig[1] + T[r][2] * Sig[2];
        TS[r][1] = T[r][0] * Sig[1] + T[r][1] * Sig[3] + T[r][2] * Sig[4];
        TS[r][2] = T[r][0] * Sig[2] + T[r][1] * Sig[4] + T[r][2] * Sig[5];
      }
      const float a = TS[0][0] * T[0][0] + TS[0][1] * T[0][1] + TS[0][2] * T[0][2] + 0.3f;
      const float b = TS[0][0] * T[1][0] + TS[0][1] * T[1][1] + TS[0][2] * T[1][2];
      const float c = TS[1][0] * T[1][0] + TS[1][1] * T[1][1] + TS[1][2] * T[1][2] + 0.3f;
      const float det = a * c - b * b;
      const float id2 = 1.f / (det * det);
      // conic (A, B, C) = (c, -b, a)/det  ->  Sigma_hat entries (a, b, c)
      const float ga = (-gA * c * c + gB * b * c - gC * b * b) * id2;
      const float gb = (2.f * gA * b * c - gB * (det + 2.f * b * b) + 2.f * gC * a * b) * id2;
      const float gc = (-gA * b * b + gB * a * b - gC * a * a) * id2;
      const float h = 0.5f * gb;
      // dL/dSigma += T^T G2 T with G2 = [[ga, h], [h, gc]]
      {
        float G2T[2][3];
#pragma unroll
        for (int cc = 0; cc < 3; ++cc) {
          G2T[0][cc] = ga * T[0][cc] + h * T[1][cc];
          G2T[1][cc] = h * T[0][cc] + gc * T[1][cc];
        }
        gSig[0] += T[0][0] * G2T[0][0] + T[1][0] * G2T[1][0];
        gSig[1] += T[0][0] * G2T[0][1] + T[1][0] * G2T[1][1];
        gSig[2] += T[0][0] * G2T[0][2] + T[1][0] * G2T[1][2];
        gSig[3] += T[0][1] * G2T[0][1] + T[1][1] * G2T[1][1];
        gSig[4] += T[0][1] * G2T[0][2] + T[1][1] * G2T[1][2];
        gSig[5] += T[0][2] * G2T[0][2] + T[1][2] * G2T[1][2];
      }
      // dL/dT = 2 G2 (T Sigma); dL/dJ = dL/dT W^T (entries 00, 02, 11, 12)
      float gT[2][3];
#pragma unroll
      for (int cc = 0; cc < 3; ++cc) {
        gT[0][cc] = 2.f * (ga * TS[0][cc] + h * TS[1][cc]);
        gT[1][cc] = 2.f * (h * TS[0][cc] + gc * TS[1][cc]);
      }
      const float gJ00 = gT[0][0] * W[0] + gT[0][1] * W[1] + gT[0][2] * W[2];
      const float gJ02 = gT[0][0] * W[6] + gT[0][1] * W[7] + gT[0][2] * W[8];
      const float gJ11 = gT[1][0] * W[3] + gT[1][1] * W[4] + gT[1][2] * W[5];
      const float gJ12 = gT[1][0] * W[6] + gT[1][1] * W[7] + gT[1][2] * W[8];
      float gx = gmx * cam.fx * iz, gy = gmy * cam.fy * iz;
      float gzc = gz - (gJ00 * cam.fx + gJ11 * cam.fy) * iz2 - (gmx * cam.fx * xc + gmy * cam.fy * yc) * iz2;
      if (!jx) {
        gx -= gJ02 * cam.fx * iz2;
        gzc += gJ02 * 2.f * cam.fx * xc * iz2 * iz;
      } else {
        gzc += gJ02 * cam.fx * uxc * iz2;
      }
      if (!jy) {
        gy -= gJ12 * cam.fy * iz2;
        gzc += gJ12 * 2.f * cam.fy * yc * iz2 * iz;
      } else {
        gzc += gJ12 * cam.fy * uyc * iz2;
      }
#pragma unroll
      for (int cc = 0; cc < 3; ++cc) gp[cc] += W[cc] * gx + W[3 + cc] * gy + W[6 + cc] * gzc;
    }
    // rows 0-2: K8a already wrote them this batch, always accumulate
#pragma unroll
    for (int cc = 0; cc < 3; ++cc) grad[cc * S + i] += gp[cc];
    // Sigma = M M^T, M = R diag(s): dL/dM = 2 gSig M;  dL/ds, dL/dR
    const float G[3][3] = {{gSig[0], gSig[1], gSig[2]}, {gSig[1], gSig[3], gSig[4]}, {gSig[2], gSig[4], gSig[5]}};
    float gR[3][3];
#pragma unroll
    for (int cc = 0; cc < 3; ++cc) {
      float gs = 0.f;
#pragma unroll
      for (int r = 0; r < 3; ++r) {
        const float gM = 2.f * (G[r][0] * R[0][cc] + G[r][1] * R[1][cc] + G[r][2] * R[2][cc]) * s[cc];
        gs += gM * R[r][cc];
        gR[r][cc] = gM * s[cc];
      }
      const float v = gs * s[cc];
      grad[(3 + cc) * S + i] = accumulate ? grad[(3 + cc) * S + i] + v : v;
    }
    // R(q_hat) -> q_hat -> q
    float gw = 0.f, gqx = 0.f, gqy = 0.f, gqz = 0.f;
    gqy += -4.f * y * gR[0][0], gqz += -4.f * z * gR[0][0];
    gw += -2.f * z * gR[0][1], gqx += 2.f * y * gR[0][1], gqy += 2.f * x * gR[0][1], gqz += -2.f * w * gR[0][1];
    gw += 2.f * y * gR[0][2], gqx += 2.f * z * gR[0][2], gqy += 2.f * w * gR[0][2], gqz += 2.f * x * gR[0][2];
    gw += 2.f * z * gR[1][0], gqx += 2.f * y * gR[1][0], gqy += 2.f * x * gR[1][0], gqz += 2.f * w * gR[1][0];
    gqx += -4.f * x * gR[1][1], gqz += -4.f * z * gR[1][1];
    gw += -2.f * x * gR[1][2], gqx += -2.f * w * gR[1][2], gqy += 2.f * z * gR[1][2], gqz += 2.f * y * gR[1][2];
    gw += -2.f * y * gR[2][0], gqx += 2.f * z * gR[2][0], gqy += -2.f * w * gR[2][0], gqz += 2.f * x * gR[2][0];
    gw += 2.f * x * gR[2][1], gqx += 2.f * w * gR[2][1], gqy += 2.f * z * gR[2][1], gqz += 2.f * y * gR[2][1];
    gqx += -4.f * x * gR[2][2], gqy += -4.f * y * gR[2][2];
    const float qd = gw * w + gqx * x + gqy * y + gqz * z;
    const float gq[4] = {(gw - w * qd) * iqn, (gqx - x * qd) * iqn, (gqy - y * qd) * iqn, (gqz - z * qd) * iqn};
#pragma unroll
    for (int j = 0; j < 4; ++j) grad[(6 + j) * S + i] = accumulate ? grad[(6 + j) * S + i] + gq[j] : gq[j];
    const float o = 1.f / (1.f + __expf(-prm[10 * S + i]));
    const float go = gop * o * (1.f - o);
    grad[10 * S + i] = accumulate ? grad[10 * S + i] + go : go;
  }
}

// ---------------------------------------------------------------------------
// K8 wide (n > 8 views in one call, up to kMaxWide): the same chain with the views in
// the inner loop of each Gaussian instead of unrolled register arrays, so that a whole
// iteration's views (config 4: 64) are chained in one pass -- every parameter row
// read and every gradient row written once per iteration instead of once per 8 views.
// A thread first loads the flag byte of every view (all loads in flight at once) into
// a visibility mask, then walks only its visible views, kWideGroup (geometry:
// kWideGroupGeom) at a time with the
// group's screen-gradient loads issued together: a Gaussian is seen by few of the
// views, and no dependent load chain runs over all of them.
// ---------------------------------------------------------------------------
#ifndef GSR_WIDE_VIS_HANDOFF
#define GSR_WIDE_VIS_HANDOFF 1
#endif
#ifndef GSR_WIDE_GROUP
#define GSR_WIDE_GROUP 2  // r02: 2 (was 4; config 4 chain 3.10 -> 2.86 ms with GEOM min blocks 6)
#endif
#ifndef GSR_WIDE_GROUP_GEOM
#define GSR_WIDE_GROUP_GEOM GSR_WIDE_GROUP
#endif
#ifndef GSR_WIDE_MINB_COLOR
#define GSR_WIDE_MINB_COLOR 4
#endif
#ifndef GSR_WIDE_MINB_GEOM
#define GSR_WIDE_MINB_GEOM 6
#endif
constexpr int kMaxWide = 64, kWideGroup = GSR_WIDE_GROUP, kWideGroupGeom = GSR_WIDE_GROUP_GEOM;
struct WideBatch {
  DevCam cam[kMaxWide];
  const uint8_t* flags[kMaxWide];
  float* sgrad[kMaxWide];
  int n;
};

__device__ __forceinline__ uint64_t wide_visible(const WideBatch& vb, int64_t i) {
  uint32_t f[kMaxWide];
#pragma unroll
  for (int v = 0; v < kMaxWide; ++v) f[v] = v < vb.n ? (uint32_t)vb.flags[v][i] : (uint32_t)GS_FLAG_CULLED;
  uint64_t vis = 0;
#pragma unroll
  for (int v = 0; v < kMaxWide; ++v) vis |= (f[v] & GS_FLAG_CULLED) ? 0ull : (1ull << v);
  return vis;
}

// the next up-to-G views of the mask (removed from it); -1 = none
template <int G>
__device__ __forceinline__ void wide_take(uint64_t& vis, int (&vv)[G]) {
#pragma unroll
  for (int j = 0; j < G; ++j) {
    vv[j] = vis ? __ffsll((long long)vis) - 1 : -1;
    vis &= vis - 1;
  }
}

template <int DEG>
__global__ void __launch_bounds__(128, GSR_WIDE_MINB_COLOR) k_project_bwd_color_wide(const __grid_constant__ WideBatch vb, int64_t P,
                                                                    int64_t S, const float* __restrict__ prm,
                                                                    float* __restrict__ grad, int accumulate) {
  constexpr int NK = (DEG + 1) * (DEG + 1);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < P; i += stride) {
    uint64_t vis = wide_visible(vb, i);
#if GSR_WIDE_VIS_HANDOFF
    // hand the mask to the geometry kernel in the two spare floats (10, 11) of view 0's
    // screen-gradient record (the render backward writes floats 0-9 only); the geometry
    // kernel reads one 8-B word instead of 64 flag bytes and zeroes it again
    *reinterpret_cast<uint64_t*>(vb.sgrad[0] + 12 * i + 10) = vis;
#endif
    float acc[NK][3];  // the SH gradient rows, in registers across the views
    bool loaded = false;
    float gp0 = 0.f, gp1 = 0.f, gp2 = 0.f, px = 0.f, py = 0.f, pz = 0.f;
    while (vis) {
      int vv[kWideGroup];
      wide_take(vis, vv);
      float gc[kWideGroup][3];
#pragma unroll
      for (int j = 0; j < kWideGroup; ++j) {  // the group's loads in flight together
        gc[j][0] = gc[j][1] = gc[j][2] = 0.f;
        if (vv[j] >= 0) {
          const uint32_t fl = vb.flags[vv[j]][i];
          const float* sg = vb.sgrad[vv[j]] + 12 * i;
          const float2 g67 = *reinterpret_cast<const float2*>(sg + 6);
          const float g8 = sg[8];
          gc[j][0] = (fl & 1) ? 0.f : g67.x;
          gc[j][1] = (fl & 2) ? 0.f : g67.y;
          gc[j][2] = (fl & 4) ? 0.f : g8;
        }
      }
#pragma unroll
      for (int j = 0; j < kWideGroup; ++j) {
        if (gc[j][0] == 0.f && gc[j][1] == 0.f && gc[j][2] == 0.f) continue;
        if (!loaded) {  // the Gaussian's mean and gradient rows, once, at its first contributing view
          px = prm[i], py = prm[S + i], pz = prm[2 * S + i];
#pragma unroll
          for (int k = 0; k < NK; ++k)
#pragma unroll
            for (int ch = 0; ch < 3; ++ch) acc[k][ch] = accumulate ? grad[(int64_t)(11 + 3 * k + ch) * S + i] : 0.f;
          loaded = true;
        }
        const DevCam& cam = vb.cam[vv[j]];
        const float vx = px - cam.ocam[0], vy = py - cam.ocam[1], vz = pz - cam.ocam[2];
        const float ivn = rsqrtf(vx * vx + vy * vy + vz * vz);
        const float d0 = vx * ivn, d1 = vy * ivn, d2 = vz * ivn;
        float gd0 = 0.f, gd1 = 0.f, gd2 = 0.f;
#pragma unroll
        for (int k = 0; k < NK; ++k) {
          float Y, gx, gy, gz;
          sh_term(k, d0, d1, d2, Y, gx, gy, gz);
          acc[k][0] = fmaf(Y, gc[j][0], acc[k][0]);
          acc[k][1] = fmaf(Y, gc[j][1], acc[k][1]);
          acc[k][2] = fmaf(Y, gc[j][2], acc[k][2]);
          if (k > 0) {  // coefficients re-read per view: L1 / L2 hits after the first
            const float* c = prm + (int64_t)(11 + 3 * k) * S + i;
            const float w = __ldg(c) * gc[j][0] + __ldg(c + S) * gc[j][1] + __ldg(c + 2 * S) * gc[j][2];
            gd0 = fmaf(w, gx, gd0);
            gd1 = fmaf(w, gy, gd1);
            gd2 = fmaf(w, gz, gd2);
          }
        }
        // d = v/|v|: dL/dv = (I - d d^T) dL/dd / |v|
        const float dd = d0 * gd0 + d1 * gd1 + d2 * gd2;
        gp0 += (gd0 - d0 * dd) * ivn;
        gp1 += (gd1 - d1 * dd) * ivn;
        gp2 += (gd2 - d2 * dd) * ivn;
      }
    }
    if (loaded) {
#pragma unroll
      for (int k = 0; k < NK; ++k)
#pragma unroll
        for (int ch = 0; ch < 3; ++ch) grad[(int64_t)(11 + 3 * k + ch) * S + i] = acc[k][ch];
    } else if (!accumulate) {
#pragma unroll
      for (int r = 11; r < 11 + 3 * NK; ++r) grad[(int64_t)r * S + i] = 0.f;
    }
    if (accumulate) {
      if (loaded) {
        grad[i] += gp0;
        grad[S + i] += gp1;
        grad[2 * S + i] += gp2;
      }
    } else {
      grad[i] = gp0;
      grad[S + i] = gp1;
      grad[2 * S + i] = gp2;
    }
  }
}

__global__ void __launch_bounds__(128, GSR_WIDE_MINB_GEOM) k_project_bwd_geom_wide(const __grid_constant__ WideBatch vb, int64_t P,
                                                                   int64_t S, const float* __restrict__ prm,
                                                                   float* __restrict__ grad, int accumulate) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < P; i += stride) {
#if GSR_WIDE_VIS_HANDOFF
    uint64_t* vslot = reinterpret_cast<uint64_t*>(vb.sgrad[0] + 12 * i + 10);
    const uint64_t vis_all = *vslot;
    if (!(vis_all & 1ull)) *vslot = 0ull;  // (view 0 visible: its whole record is cleared below)
#else
    const uint64_t vis_all = wide_visible(vb, i);
#endif
    uint64_t vis = vis_all;
    bool loaded = false;
    float px = 0.f, py = 0.f, pz = 0.f, iqn = 0.f, w = 0.f, x = 0.f, y = 0.f, z = 0.f;
    float R[3][3], s[3], Sig[6];
    float gSig[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f};  // xx, xy, xz, yy, yz, zz
    float gp[3] = {0.f, 0.f, 0.f};
    float gop = 0.f;
    while (vis) {
      int vv[kWideGroupGeom];
      wide_take(vis, vv);
      float4 g0[kWideGroupGeom];
      float2 g1[kWideGroupGeom];
      float gzz[kWideGroupGeom];
      uint32_t flv[kWideGroupGeom];
#pragma unroll
      for (int j = 0; j < kWideGroupGeom; ++j) {  // the group's loads in flight together (clears after the loop)
        g0[j] = make_float4(0.f, 0.f, 0.f, 0.f), g1[j] = make_float2(0.f, 0.f), gzz[j] = 0.f, flv[j] = 0;
        if (vv[j] >= 0) {
          const float4* sg4 = reinterpret_cast<const float4*>(vb.sgrad[vv[j]] + 12 * i);
          g0[j] = sg4[0];
          g1[j] = *reinterpret_cast<const float2*>(sg4 + 1);
          gzz[j] = reinterpret_cast<const float*>(sg4 + 2)[1];
          flv[j] = vb.flags[vv[j]][i];
        }
      }
#pragma unroll
      for (int j = 0; j < kWideGroupGeom; ++j) {
        if (vv[j] < 0) continue;
        gop += g1[j].y;
        const float gmx = g0[j].x, gmy = g0[j].y, gA = g0[j].z, gB = g0[j].w, gC = g1[j].x, gz = gzz[j];
        if (gmx == 0.f && gmy == 0.f && gA == 0.f && gB == 0.f && gC == 0.f && gz == 0.f) continue;
        if (!loaded) {  // Sigma = R diag(s)^2 R^T (view independent), once
          px = prm[i], py = prm[S + i], pz = prm[2 * S + i];
          const float q0 = prm[6 * S + i], q1 = prm[7 * S + i], q2 = prm[8 * S + i], q3 = prm[9 * S + i];
          iqn = rsqrtf(q0 * q0 + q1 * q1 + q2 * q2 + q3 * q3);
          w = q0 * iqn, x = q1 * iqn, y = q2 * iqn, z = q3 * iqn;
          R[0][0] = 1.f - 2.f * (y * y + z * z), R[0][1] = 2.f * (x * y - w * z), R[0][2] = 2.f * (x * z + w * y);
          R[1][0] = 2.f * (x * y + w * z), R[1][1] = 1.f - 2.f * (x * x + z * z), R[1][2] = 2.f * (y * z - w * x);
          R[2][0] = 2.f * (x * z - w * y), R[2][1] = 2.f * (y * z + w * x), R[2][2] = 1.f - 2.f * (x * x + y * y);
#pragma unroll
          for (int jj = 0; jj < 3; ++jj) s[jj] = __expf(prm[(3 + jj) * S + i]);
          const float s0 = s[0] * s[0], s1 = s[1] * s[1], s2 = s[2] * s[2];
          Sig[0] = R[0][0] * R[0][0] * s0 + R[0][1] * R[0][1] * s1 + R[0][2] * R[0][2] * s2;
          Sig[1] = R[0][0] * R[1][0] * s0 + R[0][1] * R[1][1] * s1 + R[0][2] * R[1][2] * s2;
          Sig[2] = R[0][0] * R[2][0] * s0 + R[0][1] * R[2][1] * s1 + R[0][2] * R[2][2] * s2;
          Sig[3] = R[1][0] * R[1][0] * s0 + R[1][1] * R[1][1] * s1 + R[1][2] * R[1][2] * s2;
          Sig[4] = R[1][0] * R[2][0] * s0 + R[1][1] * R[2][1] * s1 + R[1][2] * R[2][2] * s2;
          Sig[5] = R[2][0] * R[2][0] * s0 + R[2][1] * R[2][1] * s1 + R[2][2] * R[2][2] * s2;
          loaded = true;
        }
        const DevCam& cam = vb.cam[vv[j]];
        const float* W = cam.R;
        const float xc = W[0] * px + W[1] * py + W[2] * pz + cam.t[0];
        const float yc = W[3] * px + W[4] * py + W[5] * pz + cam.t[1];
        const float zc = W[6] * px + W[7] * py + W[8] * pz + cam.t[2];
        const float iz = pb_rcp(zc), iz2 = iz * iz;
        const float ux = xc * iz, uy = yc * iz;
        const bool jx = flv[j] & GS_FLAG_JCLAMP_X, jy = flv[j] & GS_FLAG_JCLAMP_Y;
        const float uxc = jx ? fminf(fmaxf(ux, -cam.limx), cam.limx) : ux;
        const float uyc = jy ? fminf(fmaxf(uy, -cam.limy), cam.limy) : uy;
        const float J00 = cam.fx * iz, J02 = -cam.fx * uxc * iz, J11 = cam.fy * iz, J12 = -cam.fy * uyc * iz;
        float T[2][3];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          T[0][c] = J00 * W[c] + J02 * W[6 + c];
          T[1][c] = J11 * W[3 + c] + J12 * W[6 + c];
        }
        float TS[2][3];
#pragma unroll
        for (int r = 0; r < 2; ++r) {
          TS[r][0] = T[r][0] * Sig[0] + T[r][1] * Sig[1] + T[r][2] * Sig[2];
          TS[r][1] = T[r][0] * Sig[1] + T[r][1] * Sig[3] + T[r][2] * Sig[4];
          TS[r][2] = T[r][0] * Sig[2] + T[r][1] * Sig[4] + T[r][2] * Sig[5];
        }
        const float a = TS[0][0] * T[0][0] + TS[0][1] * T[0][1] + TS[0][2] * T[0][2] + 0.3f;
        const float b = TS[0][0] * T[1][0] + TS[0][1] * T[1][1] + TS[0][2] * T[1][2];
        const float c = TS[1][0] * T[1][0] + TS[1][1] * T[1][1] + TS[1][2] * T[1][2] + 0.3f;
        const float det = a * c - b * b;
        const float id2 = pb_rcp(det * det);
        const float ga = (-gA * c * c + gB * b * c - gC * b * b) * id2;
        const float gb = (2.f * gA * b * c - gB * (det + 2.f * b * b) + 2.f * gC * a * b) * id2;
        const float gcc = (-gA * b * b + gB * a * b - gC * a * a) * id2;
        const float h = 0.5f * gb;
        {
          float G2T[2][3];
#pragma unroll
          for (int cc = 0; cc < 3; ++cc) {
            G2T[0][cc] = ga * T[0][cc] + h * T[1][cc];
            G2T[1][cc] = h * T[0][cc] + gcc * T[1][cc];
          }
          gSig[0] += T[0][0] * G2T[0][0] + T[1][0] * G2T[1][0];
          gSig[1] += T[0][0] * G2T[0][1] + T[1][0] * G2T[1][1];
          gSig[2] += T[0][0] * G2T[0][2] + T[1][0] * G2T[1][2];
          gSig[3] += T[0][1] * G2T[0][1] + T[1][1] * G2T[1][1];
          gSig[4] += T[0][1] * G2T[0][2] + T[1][1] * G2T[1][2];
          gSig[5] += T[0][2] * G2T[0][2] + T[1][2] * G2T[1][2];
        }
        float gT[2][3];
#pragma unroll
        for (int cc = 0; cc < 3; ++cc) {
          gT[0][cc] = 2.f * (ga * TS[0][cc] + h * TS[1][cc]);
          gT[1][cc] = 2.f * (h * TS[0][cc] + gcc * TS[1][cc]);
        }
        const float gJ00 = gT[0][0] * W[0] + gT[0][1] * W[1] + gT[0][2] * W[2];
        const float gJ02 = gT[0][0] * W[6] + gT[0][1] * W[7] + gT[0][2] * W[8];
        const float gJ11 = gT[1][0] * W[3] + gT[1][1] * W[4] + gT[1][2] * W[5];
        const float gJ12 = gT[1][0] * W[6] + gT[1][1] * W[7] + gT[1][2] * W[8];
        float gx = gmx * cam.fx * iz, gy = gmy * cam.fy * iz;
        float gzc = gz - (gJ00 * cam.fx + gJ11 * cam.fy) * iz2 - (gmx * cam.fx * xc + gmy * cam.fy * yc) * iz2;
        if (!jx) {
          gx -= gJ02 * cam.fx * iz2;
          gzc += gJ02 * 2.f * cam.fx * xc * iz2 * iz;
        } else {
          gzc += gJ02 * cam.fx * uxc * iz2;
        }
        if (!jy) {
          gy -= gJ12 * cam.fy * iz2;
          gzc += gJ12 * 2.f * cam.fy * yc * iz2 * iz;
        } else {
          gzc += gJ12 * cam.fy * uyc * iz2;
        }
#pragma unroll
        for (int cc = 0; cc < 3; ++cc) gp[cc] += W[cc] * gx + W[3 + cc] * gy + W[6 + cc] * gzc;
      }
    }
    for (uint64_t m = vis_all; m; m &= m - 1) {  // consume: clear every visible view's entry
      float4* sg4 = reinterpret_cast<float4*>(vb.sgrad[__ffsll((long long)m) - 1] + 12 * i);
      sg4[0] = sg4[1] = sg4[2] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    if (!loaded) {  // no contributing view: zero (overwrite) or unchanged, plus the opacity sum
      if (!accumulate) {
#pragma unroll
        for (int r = 3; r < 11; ++r) grad[r * S + i] = 0.f;
      }
      if (gop != 0.f) {
        const float o = pb_rcp(1.f + __expf(-prm[10 * S + i]));
        grad[10 * S + i] = (accumulate ? grad[10 * S + i] : 0.f) + gop * o * (1.f - o);
      }
      continue;
    }
#pragma unroll
    for (int cc = 0; cc < 3; ++cc) grad[cc * S + i] += gp[cc];  // rows 0-2: K8a wrote them, accumulate
    const float G[3][3] = {{gSig[0], gSig[1], gSig[2]}, {gSig[1], gSig[3], gSig[4]}, {gSig[2], gSig[4], gSig[5]}};
    float gR[3][3];
#pragma unroll
    for (int cc = 0; cc < 3; ++cc) {
      float gs = 0.f;
#pragma unroll
      for (int r = 0; r < 3; ++r) {
        const float gM = 2.f * (G[r][0] * R[0][cc] + G[r][1] * R[1][cc] + G[r][2] * R[2][cc]) * s[cc];
        gs += gM * R[r][cc];
        gR[r][cc] = gM * s[cc];
      }
      const float vv = gs * s[cc];
      grad[(3 + cc) * S + i] = accumulate ? grad[(3 + cc) * S + i] + vv : vv;
    }
    float gw = 0.f, gqx = 0.f, gqy = 0.f, gqz = 0.f;
    gqy += -4.f * y * gR[0][0], gqz += -4.f * z * gR[0][0];
    gw += -2.f * z * gR[0][1], gqx += 2.f * y * gR[0][1], gqy += 2.f * x * gR[0][1], gqz += -2.f * w * gR[0][1];
    gw += 2.f * y * gR[0][2], gqx += 2.f * z * gR[0][2], gqy += 2.f * w * gR[0][2], gqz += 2.f * x * gR[0][2];
    gw += 2.f * z * gR[1][0], gqx += 2.f * y * gR[1][0], gqy += 2.f * x * gR[1][0], gqz += 2.f * w * gR[1][0];
    gqx += -4.f * x * gR[1][1], gqz += -4.f * z * gR[1][1];
    gw += -2.f * x * gR[1][2], gqx += -2.f * w * gR[1][2], gqy += 2.f * z * gR[1][2], gqz += 2.f * y * gR[1][2];
    gw += -2.f * y * gR[2][0], gqx += 2.f * z * gR[2][0], gqy += -2.f * w * gR[2][0], gqz += 2.f * x * gR[2][0];
    gw += 2.f * x * gR[2][1], gqx += 2.f * w * gR[2][1], gqy += 2.f * z * gR[2][1], gqz += 2.f * y * gR[2][1];
    gqx += -4.f * x * gR[2][2], gqy += -4.f * y * gR[2][2];
    const float qd = gw * w + gqx * x + gqy * y + gqz * z;
    const float gq[4] = {(gw - w * qd) * iqn, (gqx - x * qd) * iqn, (gqy - y * qd) * iqn, (gqz - z * qd) * iqn};
#pragma unroll
    for (int j = 0; j < 4; ++j) grad[(6 + j) * S + i] = accumulate ? grad[(6 + j) * S + i] + gq[j] : gq[j];
    const float o = pb_rcp(1.f + __expf(-prm[10 * S + i]));
    const float go = gop * o * (1.f - o);
    grad[10 * S + i] = accumulate ? grad[10 * S + i] + go : go;
  }
}

}  // namespace

void launch_project_bwd_views(int n_views, const DevCam* cams, const uint8_t* const* flags, float* const* sgrads,
                              int64_t P, int64_t S, int deg, const float* params, float* grad, int accumulate,
                              cudaStream_t s, cudaEvent_t colour_done) {
  const int block = 256;
  const int grid = (int)std::min<int64_t>((P + block - 1) / block, (int64_t)sm_count() * 8);
  if (n_views > kMaxViews) {  // one pass per kMaxWide views (the views in the inner loop)
    const int gridw = (int)std::min<int64_t>((P + 127) / 128, (int64_t)sm_count() * 16);
    for (int v0 = 0; v0 < n_views; v0 += kMaxWide) {
      WideBatch vb{};
      vb.n = std::min(kMaxWide, n_views - v0);
      for (int v = 0; v < vb.n; ++v) {
        vb.cam[v] = cams[v0 + v];
        vb.flags[v] = flags[v0 + v];
        vb.sgrad[v] = sgrads[v0 + v];
      }
      const int acc = (v0 == 0) ? accumulate : 1;
      switch (deg) {
        case 0: k_project_bwd_color_wide<0><<<gridw, 128, 0, s>>>(vb, P, S, params, grad, acc); break;
        case 1: k_project_bwd_color_wide<1><<<gridw, 128, 0, s>>>(vb, P, S, params, grad, acc); break;
        case 2: k_project_bwd_color_wide<2><<<gridw, 128, 0, s>>>(vb, P, S, params, grad, acc); break;
        default: k_project_bwd_color_wide<3><<<gridw, 128, 0, s>>>(vb, P, S, params, grad, acc); break;
      }
      // the SH rows (11..F-1) are final after the last pass's colour kernel
      if (colour_done && v0 + kMaxWide >= n_views) cudaEventRecord(colour_done, s);
      k_project_bwd_geom_wide<<<gridw, 128, 0, s>>>(vb, P, S, params, grad, acc);
      count_launch(2);
    }
    return;
  }
  for (int v0 = 0; v0 < n_views; v0 += kMaxViews) {
    ViewBatch vb{};
    vb.n = std::min(kMaxViews, n_views - v0);
    for (int v = 0; v < vb.n; ++v) {
      vb.cam[v] = cams[v0 + v];
      vb.flags[v] = flags[v0 + v];
      vb.sgrad[v] = sgrads[v0 + v];
    }
    const int acc = (v0 == 0) ? accumulate : 1;
    switch (deg) {
      case 0: k_project_bwd_color<0><<<grid, block, 0, s>>>(vb, P, S, params, grad, acc); break;
      case 1: k_project_bwd_color<1><<<grid, block, 0, s>>>(vb, P, S, params, grad, acc); break;
      case 2: k_project_bwd_color<2><<<grid, block, 0, s>>>(vb, P, S, params, grad, acc); break;
      default: k_project_bwd_color<3><<<grid, block, 0, s>>>(vb, P, S, params, grad, acc); break;
    }
    if (colour_done && v0 + kMaxViews >= n_views) cudaEventRecord(colour_done, s);
    k_project_bwd_geom<<<grid, block, 0, s>>>(vb, P, S, params, grad, acc);
    count_launch(2);
  }
}

}  // namespace gsr
