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
#include "gsr_internal.cuh"

namespace gsr {
namespace {

#define FM(a, b) __fmul_rn((a), (b))
#define FA(a, b) __fadd_rn((a), (b))
#define FS(a, b) __fsub_rn((a), (b))
#define FD(a, b) __fdiv_rn((a), (b))

__device__ __forceinline__ float act_exp(float x) { return (float)exp((double)x); }
__device__ __forceinline__ float act_sigmoid(float x) { return (float)(1.0 / (1.0 + exp(-(double)x))); }

// Real SH basis (Condon-Shortley phase, k = l^2 + l + m), unrolled polynomials.
constexpr float kC0 = 0.28209479177387814f;
constexpr float kC1 = 0.4886025119029199f;
constexpr float kC2_0 = 1.0925484305920792f, kC2_1 = -1.0925484305920792f, kC2_2 = 0.31539156525252005f,
                kC2_3 = -1.0925484305920792f, kC2_4 = 0.5462742152960396f;
constexpr float kC3_0 = -0.5900435899266435f, kC3_1 = 2.890611442640554f, kC3_2 = -0.4570457994644658f,
                kC3_3 = 0.3731763325901154f, kC3_4 = -0.4570457994644658f, kC3_5 = 1.445305721320277f,
                kC3_6 = -0.5900435899266435f;

template <int DEG>
__device__ __forceinline__ void sh_basis(float x, float y, float z, float* Y) {
  Y[0] = kC0;
  if (DEG >= 1) {
    Y[1] = -kC1 * y;
    Y[2] = kC1 * z;
    Y[3] = -kC1 * x;
  }
  if (DEG >= 2) {
    const float xx = x * x, yy = y * y, zz = z * z;
    Y[4] = kC2_0 * x * y;
    Y[5] = kC2_1 * y * z;
    Y[6] = kC2_2 * (2.f * zz - xx - yy);
    Y[7] = kC2_3 * x * z;
    Y[8] = kC2_4 * (xx - yy);
    if (DEG >= 3) {
      Y[9] = kC3_0 * y * (3.f * xx - yy);
      Y[10] = kC3_1 * x * y * z;
      Y[11] = kC3_2 * y * (4.f * zz - xx - yy);
      Y[12] = kC3_3 * z * (2.f * zz - 3.f * xx - 3.f * yy);
      Y[13] = kC3_4 * x * (4.f * zz - xx - yy);
      Y[14] = kC3_5 * z * (xx - yy);
      Y[15] = kC3_6 * x * (xx - 3.f * yy);
    }
  }
}

// Cartesian gradient of each basis polynomial (only its tangential part matters).
template <int DEG>
__device__ __forceinline__ void sh_basis_grad(float x, float y, float z, float (*G)[3]) {
  G[0][0] = G[0][1] = G[0][2] = 0.f;
  if (DEG >= 1) {
    G[1][0] = 0.f, G[1][1] = -kC1, G[1][2] = 0.f;
    G[2][0] = 0.f, G[2][1] = 0.f, G[2][2] = kC1;
    G[3][0] = -kC1, G[3][1] = 0.f, G[3][2] = 0.f;
  }
  if (DEG >= 2) {
    const float xx = x * x, yy = y * y, zz = z * z;
    G[4][0] = kC2_0 * y, G[4][1] = kC2_0 * x, G[4][2] = 0.f;
    G[5][0] = 0.f, G[5][1] = kC2_1 * z, G[5][2] = kC2_1 * y;
    G[6][0] = -2.f * kC2_2 * x, G[6][1] = -2.f * kC2_2 * y, G[6][2] = 4.f * kC2_2 * z;
    G[7][0] = kC2_3 * z, G[7][1] = 0.f, G[7][2] = kC2_3 * x;
    G[8][0] = 2.f * kC2_4 * x, G[8][1] = -2.f * kC2_4 * y, G[8][2] = 0.f;
    if (DEG >= 3) {
      G[9][0] = 6.f * kC3_0 * x * y, G[9][1] = kC3_0 * (3.f * xx - 3.f * yy), G[9][2] = 0.f;
      G[10][0] = kC3_1 * y * z, G[10][1] = kC3_1 * x * z, G[10][2] = kC3_1 * x * y;
      G[11][0] = -2.f * kC3_2 * x * y, G[11][1] = kC3_2 * (4.f * zz - xx - 3.f * yy),
      G[11][2] = 8.f * kC3_2 * y * z;
      G[12][0] = -6.f * kC3_3 * x * z, G[12][1] = -6.f * kC3_3 * y * z,
      G[12][2] = kC3_3 * (6.f * zz - 3.f * xx - 3.f * yy);
      G[13][0] = kC3_4 * (4.f * zz - 3.f * xx - yy), G[13][1] = -2.f * kC3_4 * x * y,
      G[13][2] = 8.f * kC3_4 * x * z;
      G[14][0] = 2.f * kC3_5 * x * z, G[14][1] = -2.f * kC3_5 * y * z, G[14][2] = kC3_5 * (xx - yy);
      G[15][0] = kC3_6 * (3.f * xx - 3.f * yy), G[15][1] = -6.f * kC3_6 * x * y, G[15][2] = 0.f;
    }
  }
}

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

template <int DEG>
__global__ void __launch_bounds__(256) k_project(DevCam cam, int64_t P, int64_t S, const float* __restrict__ prm,
                                                 float4* __restrict__ rec, int32_t* __restrict__ radius_out,
                                                 int32_t* __restrict__ tiles_out, uint8_t* __restrict__ flags_out) {
  constexpr int NK = (DEG + 1) * (DEG + 1);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < P; i += stride) {
    const float px = __ldg(prm + i), py = __ldg(prm + S + i), pz = __ldg(prm + 2 * S + i);
    // O3: p_c = W p + t  (Eq. 4)
    const float* W = cam.R;
    const float xc = FA(FA(FA(FM(W[0], px), FM(W[1], py)), FM(W[2], pz)), cam.t[0]);
    const float yc = FA(FA(FA(FM(W[3], px), FM(W[4], py)), FM(W[5], pz)), cam.t[1]);
    const float zc = FA(FA(FA(FM(W[6], px), FM(W[7], py)), FM(W[8], pz)), cam.t[2]);
    int32_t rad = 0, ntiles = 0;
    uint8_t flags = GS_FLAG_CULLED;
    do {
      if (!(zc > cam.z_near)) break;  // R6, R23
      // O1: activations
      float s[3];
      s[0] = act_exp(__ldg(prm + 3 * S + i));
      s[1] = act_exp(__ldg(prm + 4 * S + i));
      s[2] = act_exp(__ldg(prm + 5 * S + i));
      const float qw = __ldg(prm + 6 * S + i), qx = __ldg(prm + 7 * S + i), qy = __ldg(prm + 8 * S + i),
                  qz = __ldg(prm + 9 * S + i);
      const float qn = __fsqrt_rn(FA(FA(FA(FM(qw, qw), FM(qx, qx)), FM(qy, qy)), FM(qz, qz)));
      if (!(qn > 0.f) || !finitef(qn)) break;
      const float opa = act_sigmoid(__ldg(prm + 10 * S + i));
      float R[3][3];
      quat_to_rot(FD(qw, qn), FD(qx, qn), FD(qy, qn), FD(qz, qn), R);
      // O2: Sigma = (R S)(R S)^T  (Eq. 2)
      float M[3][3], Sig[3][3];
#pragma unroll
      for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c) M[r][c] = FM(R[r][c], s[c]);
#pragma unroll
      for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c) Sig[r][c] = FA(FA(FM(M[r][0], M[c][0]), FM(M[r][1], M[c][1])), FM(M[r][2], M[c][2]));
      // O4: mean projection (Eq. 4), R1
      const float ux = FD(xc, zc), uy = FD(yc, zc);
      const float mux = FA(FM(cam.fx, ux), cam.cx);
      const float muy = FA(FM(cam.fy, uy), cam.cy);
      // O5: EWA (Eq. 5) with the 1.3x tangent clamp (R7) and the 0.3 low-pass (R8)
      const float limx = FM(1.3f, FD((float)cam.W, FM(2.f, cam.fx)));
      const float limy = FM(1.3f, FD((float)cam.H, FM(2.f, cam.fy)));
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
      rad = (int32_t)fminf(rf, (float)(1 << 30));
      ntiles = (x1 - x0) * (y1 - y0);
      // O8: SH colour at the mean (R13): +0.5, clamp at 0 per channel
      const float vx = px - cam.ocam[0], vy = py - cam.ocam[1], vz = pz - cam.ocam[2];
      const float inv = rsqrtf(vx * vx + vy * vy + vz * vz);
      float Y[NK];
      sh_basis<DEG>(vx * inv, vy * inv, vz * inv, Y);
      float col[3];
      flags = ((uxc != ux) ? GS_FLAG_JCLAMP_X : 0) | ((uyc != uy) ? GS_FLAG_JCLAMP_Y : 0);
#pragma unroll
      for (int ch = 0; ch < 3; ++ch) {
        float acc = 0.f;
#pragma unroll
        for (int k = 0; k < NK; ++k) acc = fmaf(__ldg(prm + (11 + 3 * k + ch) * S + i), Y[k], acc);
        acc += 0.5f;
        if (acc < 0.f) flags |= (uint8_t)(1u << ch);
        col[ch] = fmaxf(acc, 0.f);
      }
      const uint32_t rx = (uint32_t)x0 | ((uint32_t)x1 << 16);
      const uint32_t ry = (uint32_t)y0 | ((uint32_t)y1 << 16);
      float4* r4 = rec + 3 * i;
      r4[0] = make_float4(mux, muy, zc, opa);
      r4[1] = make_float4(cA, cB, cC, col[0]);
      r4[2] = make_float4(col[1], col[2], __uint_as_float(rx), __uint_as_float(ry));
    } while (0);
    radius_out[i] = rad;
    tiles_out[i] = ntiles;
    flags_out[i] = flags;
  }
}

// ---------------------------------------------------------------------------
// K8: chain screen-space gradients to parameter gradients (exact derivative of
// k_project, R18), accumulated into grad[F][P_stride].
// ---------------------------------------------------------------------------
template <int DEG>
__global__ void __launch_bounds__(128) k_project_bwd(DevCam cam, int64_t P, int64_t S, const float* __restrict__ prm,
                                                     const float4* __restrict__ rec,
                                                     const int32_t* __restrict__ radius,
                                                     const uint8_t* __restrict__ flags_in,
                                                     const float4* __restrict__ sgrad, float* __restrict__ grad) {
  constexpr int NK = (DEG + 1) * (DEG + 1);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < P; i += stride) {
    if (radius[i] == 0) continue;
    const float4 g0 = sgrad[3 * i], g1 = sgrad[3 * i + 1], g2 = sgrad[3 * i + 2];
    // dmu_x, dmu_y, dA, dB, dC, dopacity, dr, dg, db, dz
    const float gmx = g0.x, gmy = g0.y, gA = g0.z, gB = g0.w, gC = g1.x, gop = g1.y;
    const float gcol[3] = {g1.z, g1.w, g2.x};
    const float gz = g2.y;
    if (gmx == 0.f && gmy == 0.f && gA == 0.f && gB == 0.f && gC == 0.f && gop == 0.f && gcol[0] == 0.f &&
        gcol[1] == 0.f && gcol[2] == 0.f && gz == 0.f)
      continue;  // never composited in this view
    const uint8_t fl = flags_in[i];
    const float* W = cam.R;
    const float px = prm[i], py = prm[S + i], pz = prm[2 * S + i];
    const float xc = W[0] * px + W[1] * py + W[2] * pz + cam.t[0];
    const float yc = W[3] * px + W[4] * py + W[5] * pz + cam.t[1];
    const float zc = W[6] * px + W[7] * py + W[8] * pz + cam.t[2];
    float s[3];
#pragma unroll
    for (int j = 0; j < 3; ++j) s[j] = __expf(prm[(3 + j) * S + i]);
    const float q0 = prm[6 * S + i], q1 = prm[7 * S + i], q2 = prm[8 * S + i], q3 = prm[9 * S + i];
    const float qn = sqrtf(q0 * q0 + q1 * q1 + q2 * q2 + q3 * q3), iqn = 1.f / qn;
    const float w = q0 * iqn, x = q1 * iqn, y = q2 * iqn, z = q3 * iqn;
    float R[3][3];
    R[0][0] = 1.f - 2.f * (y * y + z * z), R[0][1] = 2.f * (x * y - w * z), R[0][2] = 2.f * (x * z + w * y);
    R[1][0] = 2.f * (x * y + w * z), R[1][1] = 1.f - 2.f * (x * x + z * z), R[1][2] = 2.f * (y * z - w * x);
    R[2][0] = 2.f * (x * z - w * y), R[2][1] = 2.f * (y * z + w * x), R[2][2] = 1.f - 2.f * (x * x + y * y);
    float M[3][3], Sig[3][3];
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
      for (int c = 0; c < 3; ++c) M[r][c] = R[r][c] * s[c];
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
      for (int c = 0; c < 3; ++c) Sig[r][c] = M[r][0] * M[c][0] + M[r][1] * M[c][1] + M[r][2] * M[c][2];
    const float iz = 1.f / zc, iz2 = iz * iz;
    const float ux = xc * iz, uy = yc * iz;
    const float limx = 1.3f * ((float)cam.W / (2.f * cam.fx)), limy = 1.3f * ((float)cam.H / (2.f * cam.fy));
    const bool jx = fl & GS_FLAG_JCLAMP_X, jy = fl & GS_FLAG_JCLAMP_Y;
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
    for (int r = 0; r < 2; ++r)
#pragma unroll
      for (int c = 0; c < 3; ++c) TS[r][c] = T[r][0] * Sig[0][c] + T[r][1] * Sig[1][c] + T[r][2] * Sig[2][c];
    const float a = TS[0][0] * T[0][0] + TS[0][1] * T[0][1] + TS[0][2] * T[0][2] + 0.3f;
    const float b = TS[0][0] * T[1][0] + TS[0][1] * T[1][1] + TS[0][2] * T[1][2];
    const float c = TS[1][0] * T[1][0] + TS[1][1] * T[1][1] + TS[1][2] * T[1][2] + 0.3f;
    const float det = a * c - b * b;
    const float id2 = 1.f / (det * det);
    // conic -> Sigma_hat entries (a, b, c)
    const float ga = (-gA * c * c + gB * b * c - gC * b * b) * id2;
    const float gb = (2.f * gA * b * c - gB * (det + 2.f * b * b) + 2.f * gC * a * b) * id2;
    const float gc = (-gA * b * b + gB * a * b - gC * a * a) * id2;
    const float G2[2][2] = {{ga, 0.5f * gb}, {0.5f * gb, gc}};
    // dL/dSigma = T^T G2 T ; dL/dT = 2 G2 T Sigma = 2 G2 TS
    float G2T[2][3];
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
      for (int cc = 0; cc < 3; ++cc) G2T[r][cc] = G2[r][0] * T[0][cc] + G2[r][1] * T[1][cc];
    float gSig[3][3];
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
      for (int cc = 0; cc < 3; ++cc) gSig[r][cc] = T[0][r] * G2T[0][cc] + T[1][r] * G2T[1][cc];
    float gT[2][3];
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
      for (int cc = 0; cc < 3; ++cc) gT[r][cc] = 2.f * (G2[r][0] * TS[0][cc] + G2[r][1] * TS[1][cc]);
    // dL/dJ = dL/dT W^T (entries 00, 02, 11, 12)
    const float gJ00 = gT[0][0] * W[0] + gT[0][1] * W[1] + gT[0][2] * W[2];
    const float gJ02 = gT[0][0] * W[6] + gT[0][1] * W[7] + gT[0][2] * W[8];
    const float gJ11 = gT[1][0] * W[3] + gT[1][1] * W[4] + gT[1][2] * W[5];
    const float gJ12 = gT[1][0] * W[6] + gT[1][1] * W[7] + gT[1][2] * W[8];
    float gx = 0.f, gy = 0.f, gzc = gz;
    gzc += -(gJ00 * cam.fx + gJ11 * cam.fy) * iz2;
    if (!jx) {
      gx += -gJ02 * cam.fx * iz2;
      gzc += gJ02 * 2.f * cam.fx * xc * iz2 * iz;
    } else {
      gzc += gJ02 * cam.fx * uxc * iz2;
    }
    if (!jy) {
      gy += -gJ12 * cam.fy * iz2;
      gzc += gJ12 * 2.f * cam.fy * yc * iz2 * iz;
    } else {
      gzc += gJ12 * cam.fy * uyc * iz2;
    }
    gx += gmx * cam.fx * iz;
    gy += gmy * cam.fy * iz;
    gzc += -(gmx * cam.fx * xc + gmy * cam.fy * yc) * iz2;
    // dL/dp = W^T dL/dp_c
    float gp[3];
#pragma unroll
    for (int cc = 0; cc < 3; ++cc) gp[cc] = W[cc] * gx + W[3 + cc] * gy + W[6 + cc] * gzc;
    // colour
    const float vx = px - cam.ocam[0], vy = py - cam.ocam[1], vz = pz - cam.ocam[2];
    const float vn2 = vx * vx + vy * vy + vz * vz, ivn = rsqrtf(vn2);
    const float dx = vx * ivn, dy = vy * ivn, dz = vz * ivn;
    float Y[NK], GY[NK][3];
    sh_basis<DEG>(dx, dy, dz, Y);
    sh_basis_grad<DEG>(dx, dy, dz, GY);
    float gd[3] = {0.f, 0.f, 0.f};
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) {
      const float gcl = (fl & (1u << ch)) ? 0.f : gcol[ch];
#pragma unroll
      for (int k = 0; k < NK; ++k) {
        float* gptr = grad + (int64_t)(11 + 3 * k + ch) * S + i;
        *gptr += Y[k] * gcl;
        if (k > 0) {
          const float shv = prm[(11 + 3 * k + ch) * S + i] * gcl;
          gd[0] += shv * GY[k][0];
          gd[1] += shv * GY[k][1];
          gd[2] += shv * GY[k][2];
        }
      }
    }
    const float ddot = dx * gd[0] + dy * gd[1] + dz * gd[2];
    gp[0] += (gd[0] - dx * ddot) * ivn;
    gp[1] += (gd[1] - dy * ddot) * ivn;
    gp[2] += (gd[2] - dz * ddot) * ivn;
#pragma unroll
    for (int cc = 0; cc < 3; ++cc) grad[cc * S + i] += gp[cc];
    // Sigma = M M^T -> dL/dM = 2 gSig M; M = R diag(s)
    float gR[3][3];
#pragma unroll
    for (int cc = 0; cc < 3; ++cc) {
      float gs = 0.f;
#pragma unroll
      for (int r = 0; r < 3; ++r) {
        const float gM = 2.f * (gSig[r][0] * M[0][cc] + gSig[r][1] * M[1][cc] + gSig[r][2] * M[2][cc]);
        gs += gM * R[r][cc];
        gR[r][cc] = gM * s[cc];
      }
      grad[(3 + cc) * S + i] += gs * s[cc];
    }
    // R(q_hat) -> q_hat
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
    grad[6 * S + i] += (gw - w * qd) * iqn;
    grad[7 * S + i] += (gqx - x * qd) * iqn;
    grad[8 * S + i] += (gqy - y * qd) * iqn;
    grad[9 * S + i] += (gqz - z * qd) * iqn;
    // opacity
    const float o = 1.f / (1.f + __expf(-prm[10 * S + i]));
    grad[10 * S + i] += gop * o * (1.f - o);
  }
}

}  // namespace

void launch_project(const DevCam& cam, int64_t P, int64_t S, int deg, const float* params, gs_proj out,
                    cudaStream_t s) {
  const int block = 256;
  const int grid = (int)std::min<int64_t>((P + block - 1) / block, (int64_t)sm_count() * 16);
  float4* rec = reinterpret_cast<float4*>(out.rec);
  switch (deg) {
    case 0: k_project<0><<<grid, block, 0, s>>>(cam, P, S, params, rec, out.radius, out.tiles, out.flags); break;
    case 1: k_project<1><<<grid, block, 0, s>>>(cam, P, S, params, rec, out.radius, out.tiles, out.flags); break;
    case 2: k_project<2><<<grid, block, 0, s>>>(cam, P, S, params, rec, out.radius, out.tiles, out.flags); break;
    default: k_project<3><<<grid, block, 0, s>>>(cam, P, S, params, rec, out.radius, out.tiles, out.flags); break;
  }
  count_launch();
}

void launch_project_bwd(const DevCam& cam, int64_t P, int64_t S, int deg, const float* params, gs_proj proj,
                        const float* sgrad, float* grad, cudaStream_t s) {
  const int block = 128;
  const int grid = (int)std::min<int64_t>((P + block - 1) / block, (int64_t)sm_count() * 32);
  const float4* rec = reinterpret_cast<const float4*>(proj.rec);
  const float4* sg = reinterpret_cast<const float4*>(sgrad);
  switch (deg) {
    case 0: k_project_bwd<0><<<grid, block, 0, s>>>(cam, P, S, params, rec, proj.radius, proj.flags, sg, grad); break;
    case 1: k_project_bwd<1><<<grid, block, 0, s>>>(cam, P, S, params, rec, proj.radius, proj.flags, sg, grad); break;
    case 2: k_project_bwd<2><<<grid, block, 0, s>>>(cam, P, S, params, rec, proj.radius, proj.flags, sg, grad); break;
    default: k_project_bwd<3><<<grid, block, 0, s>>>(cam, P, S, params, rec, proj.radius, proj.flags, sg, grad); break;
  }
  count_launch();
}

}  // namespace gsr
