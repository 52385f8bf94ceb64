// oracle/gsref.cpp -- plain, slow, obviously-correct CPU oracle of the GSFusion
// rasterizer hot path (arXiv 2408.12677, §III-A2 Eqs. 1-5, §III-B3 Eqs. 11-12).
//
// TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
// cpu_baseline / --impl reference legs may load this library.  The product path
// (paper_2408_12677_b200/, libgsr.so) never links, imports or calls it, and this
// file shares no code, header, table or constant generator with it.
//
// Build: g++ -O2 -std=c++17 -ffp-contract=off -fopenmp -fPIC -shared (no fast-math), so
// the float ("parity") mode rounds every operation in the order written here.  OpenMP
// only distributes independent loop iterations (tiles, rows, samples, Gaussians); every
// sum is taken in one fixed order, so results do not depend on the thread count.
//
// Every step cites the passage it follows.  Readings R1-R27 are listed in
// DESIGN.md §"Readings"; the ones used here are named inline.
//
// Precision modes (template parameters D = decision precision, S = value
// precision):
//   mode 0  F32   D = S = float   parity reference for forward outputs
//   mode 1  F64   D = S = double  finite-difference reference
//   mode 2  MIXED D = float, S = double: every data-dependent decision
//           (culling, radius, tile rect, clamps, the 1/255 skip, the 1e-4 stop,
//           the 0.99 cap) is taken on fp32 values computed exactly as in mode 0,
//           and every value is carried in fp64.  Used as the gradient parity
//           reference ("both sides take the decision in the same precision").
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <type_traits>
#include <vector>
#ifdef _OPENMP
#include <omp.h>
#endif

namespace {

struct RefCamera {  // marshalled by oracle/gsref.py (not shared with include/gsr.h)
  int32_t width, height;
  float fx, fy, cx, cy;
  float R_cw[9];  // world -> camera rotation W (rotation of T_WC^{-1}), row-major
  float t_cw[3];
  float z_near;
  float bg[3];
};

constexpr int kTile = 16;  // 16x16-pixel tiles (BASELINE.json north_star)

// ---------------------------------------------------------------------------
// activations computed in double and rounded (reading R9)
// ---------------------------------------------------------------------------
inline float act_exp(float x) { return (float)std::exp((double)x); }
inline double act_exp(double x) { return std::exp(x); }
inline float act_sigmoid(float x) { return (float)(1.0 / (1.0 + std::exp(-(double)x))); }
inline double act_sigmoid(double x) { return 1.0 / (1.0 + std::exp(-x)); }

template <class T> inline bool finite(T v) { return std::isfinite(v); }

// ---------------------------------------------------------------------------
// Rn: a value carried in double together with a first-order RUNNING ERROR BOUND
// (Wilkinson's running error analysis; Higham, "Accuracy and Stability of
// Numerical Algorithms", §3.3).  Test infrastructure for the parity tolerance of
// the GPU gradients, not a precision mode of the method: v is computed exactly as
// in the MIXED mode's value track (same double operations, bit-identical), and m
// bounds |fl32(x) - x| / u for an fp32 evaluation of the same expression, u = 2^-24,
// to first order:
//   a +- b : m_a + m_b + |a +- b|
//   acc += t: m_acc + m_t + |t|          (accumulation, e.g. over pixels or views:
//                                          each term charged once, so a sum costs
//                                          sum |terms| whatever the order)
//   a * b  : m_a |b| + |a| m_b + |ab|
//   a / b  : m_a / |b| + |a/b| m_b / |b| + |a/b|
//   sqrt a : m_a / (2 sqrt a) + sqrt a
//   exp a  : e^a (m_a + |a| + 2)          (covers ex2.approx(a log2 e): the scaled
//                                          argument's rounding and 2 ulp)
// Inputs (fp32 parameters, camera, upstream fields) are exact (m = 0).  Decisions
// are never taken on Rn values (the decision track is fp32, as in MIXED).
// ---------------------------------------------------------------------------
struct Rn {
  double v = 0.0, m = 0.0;
  Rn() = default;
  Rn(double x) : v(x), m(0.0) {}  // NOLINT: implicit, exact constant / input
  Rn(double x, double e) : v(x), m(e) {}
  explicit operator double() const { return v; }
  explicit operator int32_t() const { return (int32_t)v; }
  Rn& operator+=(const Rn& t) {
    v += t.v;
    m = std::hypot(m, std::hypot(t.m, v));
    return *this;
  }
};
inline double q3(double a, double b, double c) { return std::sqrt(a * a + b * b + c * c); }
inline Rn operator+(const Rn& a, const Rn& b) { return {a.v + b.v, q3(a.m, b.m, a.v + b.v)}; }
inline Rn operator-(const Rn& a, const Rn& b) { return {a.v - b.v, q3(a.m, b.m, a.v - b.v)}; }
inline Rn operator-(const Rn& a) { return {-a.v, a.m}; }
inline Rn operator*(const Rn& a, const Rn& b) {
  const double p = a.v * b.v;
  return {p, q3(a.m * b.v, a.v * b.m, p)};
}
inline Rn operator/(const Rn& a, const Rn& b) {
  const double q = a.v / b.v;
  return {q, q3(a.m / b.v, q * b.m / b.v, q)};
}
inline bool operator<(const Rn& a, const Rn& b) { return a.v < b.v; }
inline bool operator>(const Rn& a, const Rn& b) { return a.v > b.v; }
inline bool operator<=(const Rn& a, const Rn& b) { return a.v <= b.v; }
inline bool operator>=(const Rn& a, const Rn& b) { return a.v >= b.v; }
inline bool operator==(const Rn& a, const Rn& b) { return a.v == b.v; }
inline Rn sqrt(const Rn& a) {
  const double r = std::sqrt(a.v);
  return {r, std::hypot(r > 0.0 ? a.m / (2.0 * r) : 0.0, r)};
}
inline Rn ceil(const Rn& a) { return {std::ceil(a.v), 0.0}; }
inline Rn floor(const Rn& a) { return {std::floor(a.v), 0.0}; }
inline Rn act_exp(const Rn& a) {
  const double e = std::exp(a.v);
  return {e, e * std::hypot(a.m, std::hypot(a.v, 2.0))};
}
inline Rn act_sigmoid(const Rn& a) {
  const double o = 1.0 / (1.0 + std::exp(-a.v));
  return {o, std::hypot(o * (1.0 - o) * std::hypot(a.m, std::hypot(a.v, 2.0)), 2.0 * o)};
}
inline bool finite(const Rn& a) { return std::isfinite(a.v); }
template <class T> constexpr bool kIsRn = std::is_same_v<T, Rn>;

// ---------------------------------------------------------------------------
// Real spherical harmonics, textbook definition (Condon-Shortley phase), in
// Cartesian polynomial form on the unit sphere:
//   Y_l^m = sqrt(2) K_lm (-1)^m Re((x+iy)^m) P_l^{(m)}(z)      m > 0
//   Y_l^0 = K_l0 P_l(z)
//   Y_l^m = sqrt(2) K_l|m| (-1)^|m| Im((x+iy)^|m|) P_l^{(|m|)}(z) m < 0
// with K_lm = sqrt((2l+1)/(4 pi) (l-m)!/(l+m)!) and P_l^{(m)} the m-th derivative
// of the Legendre polynomial.  Index k = l^2 + l + m.  Pinned by a quadrature
// orthonormality test (tests/test_oracle_pins.py).  The SH degree/basis is not
// fixed by the paper ("spherical harmonics (SH) coefficients"); R13.
// ---------------------------------------------------------------------------
struct ShBasis {
  // Legendre coefficients: leg[l][j] = coefficient of z^j in P_l(z)
  double leg[4][4];
  double K[4][4];
  ShBasis() {
    std::memset(leg, 0, sizeof(leg));
    leg[0][0] = 1.0;
    leg[1][1] = 1.0;
    for (int l = 1; l < 3; ++l) {  // Bonnet: (l+1) P_{l+1} = (2l+1) z P_l - l P_{l-1}
      for (int j = 0; j < 4; ++j) {
        double v = 0.0;
        if (j >= 1) v += (2.0 * l + 1.0) * leg[l][j - 1];
        v -= l * leg[l - 1][j];
        leg[l + 1][j] = v / (l + 1.0);
      }
    }
    for (int l = 0; l < 4; ++l)
      for (int m = 0; m <= l; ++m) {
        double r = 1.0;  // (l-m)!/(l+m)!
        for (int t = l - m + 1; t <= l + m; ++t) r /= t;
        K[l][m] = std::sqrt((2.0 * l + 1.0) / (4.0 * M_PI) * r);
      }
  }
  // value of the n-th derivative of P_l at z
  template <class T> T legendre_deriv(int l, int n, T z) const {
    T acc = T(0);
    for (int j = n; j <= l; ++j) {
      double c = leg[l][j];
      for (int t = 0; t < n; ++t) c *= (j - t);
      T pw = T(1);
      for (int t = 0; t < j - n; ++t) pw = pw * z;
      acc = acc + T(c) * pw;
    }
    return acc;
  }
};
const ShBasis kSh;

// Re / Im of (x + i y)^m
template <class T> void cpow(T x, T y, int m, T& re, T& im) {
  re = T(1);
  im = T(0);
  for (int t = 0; t < m; ++t) {
    T nr = re * x - im * y;
    T ni = re * y + im * x;
    re = nr;
    im = ni;
  }
}

// Y_k(d) for k < (deg+1)^2, and optionally the Cartesian gradient dY_k/d(x,y,z)
template <class T> void sh_eval(int deg, const T d[3], T* Y, T (*dY)[3]) {
  for (int l = 0; l <= deg; ++l) {
    for (int m = -l; m <= l; ++m) {
      const int k = l * l + l + m;
      const int am = m < 0 ? -m : m;
      const T norm = T((am == 0 ? 1.0 : std::sqrt(2.0)) * kSh.K[l][am] * ((am & 1) ? -1.0 : 1.0));
      T re, im, re1 = T(0), im1 = T(0);
      cpow(d[0], d[1], am, re, im);
      if (am > 0) cpow(d[0], d[1], am - 1, re1, im1);
      const T Q = kSh.legendre_deriv(l, am, d[2]);
      const T Qp = kSh.legendre_deriv(l, am + 1, d[2]);
      if (m >= 0) {
        Y[k] = norm * re * Q;
        if (dY) {
          dY[k][0] = norm * T(am) * re1 * Q;
          dY[k][1] = norm * (-T(am)) * im1 * Q;
          dY[k][2] = norm * re * Qp;
        }
      } else {
        Y[k] = norm * im * Q;
        if (dY) {
          dY[k][0] = norm * T(am) * im1 * Q;
          dY[k][1] = norm * T(am) * re1 * Q;
          dY[k][2] = norm * im * Qp;
        }
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Projection of one Gaussian (steps O1-O8, Eqs. 2-5)
// ---------------------------------------------------------------------------
enum : uint8_t {
  FLAG_CLAMP_R = 1, FLAG_CLAMP_G = 2, FLAG_CLAMP_B = 4,
  FLAG_JCLAMP_X = 8, FLAG_JCLAMP_Y = 16, FLAG_CULLED = 128
};

template <class S> struct Proj {
  std::vector<S> mux, muy, z, A, B, C, o, col[3];
  std::vector<int32_t> radius, x0, x1, y0, y1, tiles;
  std::vector<uint8_t> flags;
  explicit Proj(int64_t P)
      : mux(P), muy(P), z(P), A(P), B(P), C(P), o(P), radius(P), x0(P), x1(P), y0(P), y1(P),
        tiles(P), flags(P) {
    for (auto& c : col) c.assign(P, S(0));
  }
};

template <class S> struct ParamView {  // one Gaussian's raw parameters (float storage -> S)
  S p[3], l[3], q[4], logit;
  std::vector<S> sh;  // sh[3k + ch]
};

template <class S>
ParamView<S> load_params(const float* params, int64_t P_stride, int deg, int64_t i) {
  ParamView<S> v;
  for (int j = 0; j < 3; ++j) v.p[j] = S(params[j * P_stride + i]);
  for (int j = 0; j < 3; ++j) v.l[j] = S(params[(3 + j) * P_stride + i]);
  for (int j = 0; j < 4; ++j) v.q[j] = S(params[(6 + j) * P_stride + i]);
  v.logit = S(params[10 * P_stride + i]);
  const int nsh = 3 * (deg + 1) * (deg + 1);
  v.sh.resize(nsh);
  for (int j = 0; j < nsh; ++j) v.sh[j] = S(params[(11 + j) * P_stride + i]);
  return v;
}

// Forward intermediates kept for the backward (O11).
template <class S> struct Fwd {
  S qn, qh[4], R[3][3], s[3], M[3][3], Sig[3][3];
  S pc[3], ux, uy, uxc, uyc, J00, J02, J11, J12, T[2][3];
  S a, b, c, det, A, B, C, mux, muy, o;
  S v[3], vn, d[3], Y[16], col_raw[3];
  bool jclx, jcly, clamp[3];
  bool culled;
  S radius_f;
  int32_t x0, x1, y0, y1;
};

template <class S>
Fwd<S> project_one(const RefCamera& cam, int deg, const ParamView<S>& g) {
  using std::ceil;
  using std::floor;
  using std::sqrt;
  Fwd<S> f{};
  f.culled = true;
  S W[3][3], t[3];
  for (int r = 0; r < 3; ++r) {
    for (int c = 0; c < 3; ++c) W[r][c] = S(cam.R_cw[3 * r + c]);
    t[r] = S(cam.t_cw[r]);
  }
  const S fx = S(cam.fx), fy = S(cam.fy), cx = S(cam.cx), cy = S(cam.cy);

  // O3: p_c = W p + t  (Eq. 4: T_WC^{-1} p_g)
  for (int r = 0; r < 3; ++r) f.pc[r] = ((W[r][0] * g.p[0] + W[r][1] * g.p[1]) + W[r][2] * g.p[2]) + t[r];
  if (!(f.pc[2] > S(cam.z_near))) return f;  // near-plane cull (R6); NaN culls (R23)

  // O1: activations (R3, R4, R5)
  for (int j = 0; j < 3; ++j) f.s[j] = act_exp(g.l[j]);
  f.qn = sqrt(((g.q[0] * g.q[0] + g.q[1] * g.q[1]) + g.q[2] * g.q[2]) + g.q[3] * g.q[3]);
  if (!(f.qn > S(0)) || !finite(f.qn)) return f;
  for (int j = 0; j < 4; ++j) f.qh[j] = g.q[j] / f.qn;
  f.o = act_sigmoid(g.logit);
  const S w = f.qh[0], x = f.qh[1], y = f.qh[2], z = f.qh[3];
  // rotation matrix of a unit quaternion (w, x, y, z), Hamilton convention (R3)
  f.R[0][0] = S(1) - S(2) * (y * y + z * z);
  f.R[0][1] = S(2) * (x * y - w * z);
  f.R[0][2] = S(2) * (x * z + w * y);
  f.R[1][0] = S(2) * (x * y + w * z);
  f.R[1][1] = S(1) - S(2) * (x * x + z * z);
  f.R[1][2] = S(2) * (y * z - w * x);
  f.R[2][0] = S(2) * (x * z - w * y);
  f.R[2][1] = S(2) * (y * z + w * x);
  f.R[2][2] = S(1) - S(2) * (x * x + y * y);

  // O2: Sigma = R S S^T R^T  (Eq. 2), with M = R S
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) f.M[r][c] = f.R[r][c] * f.s[c];
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c)
      f.Sig[r][c] = (f.M[r][0] * f.M[c][0] + f.M[r][1] * f.M[c][1]) + f.M[r][2] * f.M[c][2];

  // O4: mu = pi(p_c)  (Eq. 4), pixel (i,j) at continuous (i,j) (R1)
  f.ux = f.pc[0] / f.pc[2];
  f.uy = f.pc[1] / f.pc[2];
  f.mux = fx * f.ux + cx;
  f.muy = fy * f.uy + cy;

  // O5: Sigma_hat = J W Sigma W^T J^T + 0.3 I  (Eq. 5; R7 clamp, R8 low-pass)
  const S limx = S(1.3) * (S(cam.width) / (S(2) * fx));
  const S limy = S(1.3) * (S(cam.height) / (S(2) * fy));
  f.uxc = std::min(std::max(f.ux, -limx), limx);
  f.uyc = std::min(std::max(f.uy, -limy), limy);
  f.jclx = !(f.ux == f.uxc);
  f.jcly = !(f.uy == f.uyc);
  f.J00 = fx / f.pc[2];
  f.J02 = -(fx * f.uxc) / f.pc[2];
  f.J11 = fy / f.pc[2];
  f.J12 = -(fy * f.uyc) / f.pc[2];
  for (int c = 0; c < 3; ++c) {
    f.T[0][c] = f.J00 * W[0][c] + f.J02 * W[2][c];
    f.T[1][c] = f.J11 * W[1][c] + f.J12 * W[2][c];
  }
  S MT[2][3];
  for (int r = 0; r < 2; ++r)
    for (int c = 0; c < 3; ++c)
      MT[r][c] = (f.T[r][0] * f.Sig[0][c] + f.T[r][1] * f.Sig[1][c]) + f.T[r][2] * f.Sig[2][c];
  f.a = ((MT[0][0] * f.T[0][0] + MT[0][1] * f.T[0][1]) + MT[0][2] * f.T[0][2]) + S(0.3);
  f.b = (MT[0][0] * f.T[1][0] + MT[0][1] * f.T[1][1]) + MT[0][2] * f.T[1][2];
  f.c = ((MT[1][0] * f.T[1][0] + MT[1][1] * f.T[1][1]) + MT[1][2] * f.T[1][2]) + S(0.3);

  // O6: conic = Sigma_hat^{-1} (Eq. 3)
  f.det = f.a * f.c - f.b * f.b;
  if (!(f.det > S(0)) || !finite(f.det)) return f;
  f.A = f.c / f.det;
  f.B = -f.b / f.det;
  f.C = f.a / f.det;
  if (!finite(f.A) || !finite(f.B) || !finite(f.C) || !finite(f.mux) || !finite(f.muy)) return f;

  // O7: 3-sigma radius and tile rectangle (R10, R11)
  const S mid = S(0.5) * (f.a + f.c);
  const S disc = mid * mid - f.det;
  const S lam = mid + sqrt(std::max(disc, S(0)));
  f.radius_f = ceil(S(3) * sqrt(lam));
  S xlo = ceil(f.mux - f.radius_f), xhi = floor(f.mux + f.radius_f);
  S ylo = ceil(f.muy - f.radius_f), yhi = floor(f.muy + f.radius_f);
  xlo = std::max(xlo, S(0));
  ylo = std::max(ylo, S(0));
  xhi = std::min(xhi, S(cam.width - 1));
  yhi = std::min(yhi, S(cam.height - 1));
  if (!(xlo <= xhi) || !(ylo <= yhi)) return f;
  f.x0 = (int32_t)xlo / kTile;
  f.x1 = (int32_t)xhi / kTile + 1;
  f.y0 = (int32_t)ylo / kTile;
  f.y1 = (int32_t)yhi / kTile + 1;

  // O8: view-dependent colour from SH at the mean (R13): +0.5, clamp at 0
  S o_cam[3];
  for (int c = 0; c < 3; ++c) o_cam[c] = -((W[0][c] * t[0] + W[1][c] * t[1]) + W[2][c] * t[2]);
  for (int c = 0; c < 3; ++c) f.v[c] = g.p[c] - o_cam[c];
  f.vn = sqrt((f.v[0] * f.v[0] + f.v[1] * f.v[1]) + f.v[2] * f.v[2]);
  for (int c = 0; c < 3; ++c) f.d[c] = f.v[c] / f.vn;
  sh_eval<S>(deg, f.d, f.Y, nullptr);
  const int nk = (deg + 1) * (deg + 1);
  for (int ch = 0; ch < 3; ++ch) {
    S acc = S(0);
    for (int k = 0; k < nk; ++k) acc = acc + g.sh[3 * k + ch] * f.Y[k];
    f.col_raw[ch] = acc + S(0.5);
    f.clamp[ch] = f.col_raw[ch] < S(0);
  }
  f.culled = false;
  return f;
}

template <class S>
Proj<S> project_all(const RefCamera& cam, int64_t P, int64_t P_stride, int deg, const float* params) {
  Proj<S> pr(P);
#pragma omp parallel for schedule(dynamic, 1024)
  for (int64_t i = 0; i < P; ++i) {
    const Fwd<S> f = project_one<S>(cam, deg, load_params<S>(params, P_stride, deg, i));
    if (f.culled) {
      pr.radius[i] = 0;
      pr.tiles[i] = 0;
      pr.flags[i] = FLAG_CULLED;
      pr.x0[i] = pr.x1[i] = pr.y0[i] = pr.y1[i] = 0;
      continue;
    }
    pr.mux[i] = f.mux;
    pr.muy[i] = f.muy;
    pr.z[i] = f.pc[2];
    pr.A[i] = f.A;
    pr.B[i] = f.B;
    pr.C[i] = f.C;
    pr.o[i] = f.o;
    for (int ch = 0; ch < 3; ++ch) pr.col[ch][i] = f.clamp[ch] ? S(0) : f.col_raw[ch];
    pr.radius[i] = (int32_t)std::min(f.radius_f, S(1 << 30));
    pr.x0[i] = f.x0;
    pr.x1[i] = f.x1;
    pr.y0[i] = f.y0;
    pr.y1[i] = f.y1;
    pr.tiles[i] = (f.x1 - f.x0) * (f.y1 - f.y0);
    pr.flags[i] = (f.clamp[0] ? FLAG_CLAMP_R : 0) | (f.clamp[1] ? FLAG_CLAMP_G : 0) |
                  (f.clamp[2] ? FLAG_CLAMP_B : 0) | (f.jclx ? FLAG_JCLAMP_X : 0) |
                  (f.jcly ? FLAG_JCLAMP_Y : 0);
  }
  return pr;
}

// The fp32 projection (O1-O8) as the raster step's inputs in precision S: the
// stage-wise gradient parity reference (mode 3, STAGE; R42) composites
// exactly the fp32 records the GPU's raster consumes (bit-exact by R9) and carries
// every later value in fp64 (or Rn, with the records as exact inputs).
template <class S> Proj<S> promote(const Proj<float>& pf);

// Rn records for the stage-wise bound: the fp32 values, exact (m = 0) except the SH
// colour, whose bound comes from its own evaluation (the GPU's colour is an
// independent fp32 evaluation of O8, within 1e-6, not bit-exact; R9 covers O1-O7).
Proj<Rn> stage_records(const RefCamera& cam, int64_t P, int64_t P_stride, int deg, const float* params,
                       const Proj<float>& pf) {
  Proj<Rn> p = promote<Rn>(pf);
  const Proj<Rn> full = project_all<Rn>(cam, P, P_stride, deg, params);
  for (int ch = 0; ch < 3; ++ch)
    for (int64_t i = 0; i < P; ++i) p.col[ch][i].m = full.col[ch][i].m;
  return p;
}

template <class S> Proj<S> promote(const Proj<float>& pf) {
  const int64_t P = (int64_t)pf.tiles.size();
  Proj<S> p(P);
  for (int64_t i = 0; i < P; ++i) {
    p.mux[i] = S((double)pf.mux[i]);
    p.muy[i] = S((double)pf.muy[i]);
    p.z[i] = S((double)pf.z[i]);
    p.A[i] = S((double)pf.A[i]);
    p.B[i] = S((double)pf.B[i]);
    p.C[i] = S((double)pf.C[i]);
    p.o[i] = S((double)pf.o[i]);
    for (int ch = 0; ch < 3; ++ch) p.col[ch][i] = S((double)pf.col[ch][i]);
  }
  p.radius = pf.radius;
  p.x0 = pf.x0;
  p.x1 = pf.x1;
  p.y0 = pf.y0;
  p.y1 = pf.y1;
  p.tiles = pf.tiles;
  p.flags = pf.flags;
  return p;
}

// ---------------------------------------------------------------------------
// O9: per-tile depth-sorted lists ("3D Gaussians lying in the current view
// frustum are sorted based on depth in each tile").  Sort key
// (z, index), ties to the lower index (R12).  std::sort is the library step.
// ---------------------------------------------------------------------------
template <class S> struct Key {
  int32_t tile;
  S z;
  int32_t id;
};

template <class S> std::vector<Key<S>> emit_and_sort(const RefCamera& cam, const Proj<S>& pr) {
  const int TX = (cam.width + kTile - 1) / kTile;
  std::vector<Key<S>> keys;
  const int64_t P = (int64_t)pr.tiles.size();
  for (int64_t i = 0; i < P; ++i)
    for (int ty = pr.y0[i]; ty < pr.y1[i]; ++ty)
      for (int tx = pr.x0[i]; tx < pr.x1[i]; ++tx) keys.push_back({ty * TX + tx, pr.z[i], (int32_t)i});
  std::sort(keys.begin(), keys.end(), [](const Key<S>& a, const Key<S>& b) {
    if (a.tile != b.tile) return a.tile < b.tile;
    if (a.z != b.z) return a.z < b.z;
    return a.id < b.id;
  });
  return keys;
}

template <class S> std::vector<std::vector<int32_t>> tile_lists(const RefCamera& cam, const Proj<S>& pr) {
  const int TX = (cam.width + kTile - 1) / kTile, TY = (cam.height + kTile - 1) / kTile;
  std::vector<std::vector<int32_t>> lists((size_t)TX * TY);
  for (const Key<S>& k : emit_and_sort(cam, pr)) lists[k.tile].push_back(k.id);
  return lists;
}

// ---------------------------------------------------------------------------
// O10: front-to-back alpha compositing of one pixel (Eq. 11)
// with cap 0.99, skip alpha < 1/255, stop before T < 1e-4 (north_star; R15-R17,
// R27), depth channel D = sum z alpha T (R17), background T*bg (R26).
// ---------------------------------------------------------------------------
template <class S> struct Entry {
  int32_t id, pos;  // Gaussian index, position in the tile list
  S alpha, G, T, dx, dy;
  bool capped;
};

template <class D, class S> struct PixelResult {
  S C[3], Dep, T;
  int32_t n;
  int64_t blended, evaluated;
  double margin;    // min relative distance of a decision quantity to its threshold
  double margin_u;  // S == Rn only: min |q - threshold| / (u m_q), m_q q's running error bound
  std::vector<Entry<S>> entries;
};

constexpr double kU32 = 5.9604644775390625e-08;  // u = 2^-24, fp32 unit roundoff

// |diff| in units of u m (how many first-order fp32 error bounds separate a decision
// quantity from its threshold); m == 0 means the quantity is exact.
inline double bound_units(double diff, double m) {
  diff = std::fabs(diff);
  if (m > 0.0) return diff / (kU32 * m);
  return diff > 0.0 ? 1e300 : 0.0;
}

template <class T> inline T pixel_power(T A, T B, T C, T dx, T dy) {
  return T(-0.5) * ((A * dx) * dx + (C * dy) * dy) - (B * dx) * dy;
}

template <class D, class S>
PixelResult<D, S> composite_pixel(int px, int py, const std::vector<int32_t>& list, const Proj<D>& pd,
                                  const Proj<S>& ps, const RefCamera& cam, bool keep_entries) {
  PixelResult<D, S> r;
  for (int ch = 0; ch < 3; ++ch) r.C[ch] = S(0);
  r.Dep = S(0);
  r.n = 0;
  r.blended = r.evaluated = 0;
  r.margin = 1e300;
  r.margin_u = 1e300;
  D Td = D(1);
  S Ts = S(1);
  const D inv255 = D(1) / D(255), t_stop = D(1e-4), cap = D(0.99);
  for (size_t pos = 0; pos < list.size(); ++pos) {
    const int32_t i = list[pos];
    r.evaluated++;
    // decision track (precision D)
    const D dxd = pd.mux[i] - D(px), dyd = pd.muy[i] - D(py);
    const D powd = pixel_power(pd.A[i], pd.B[i], pd.C[i], dxd, dyd);
    {
      const double scale = 0.5 * (std::fabs((double)pd.A[i] * dxd * dxd) + std::fabs((double)pd.C[i] * dyd * dyd)) +
                           std::fabs((double)pd.B[i] * dxd * dyd);
      if (scale > 0) r.margin = std::min(r.margin, std::fabs((double)powd) / scale);
    }
    if constexpr (kIsRn<S>) {
      // the same decisions, in units of the value track's running error bounds
      const S pw = pixel_power(ps.A[i], ps.B[i], ps.C[i], ps.mux[i] - S(px), ps.muy[i] - S(py));
      r.margin_u = std::min(r.margin_u, bound_units((double)powd, pw.m));
      if (!(powd > D(0))) {
        const D rawd = pd.o[i] * act_exp(powd);
        const S raw = ps.o[i] * act_exp(pw);
        const bool cp = rawd > cap;
        r.margin_u = std::min(r.margin_u, bound_units((double)rawd - (double)cap, raw.m));
        const S al = cp ? S(cap) : raw;
        const D ald = std::min(cap, rawd);
        if (!cp) r.margin_u = std::min(r.margin_u, bound_units((double)ald - (double)inv255, al.m));
        if (!(ald < inv255)) {
          const S Tn = Ts * (S(1) - al);
          r.margin_u = std::min(r.margin_u, bound_units((double)(Td * (D(1) - ald)) - (double)t_stop, Tn.m));
        }
      }
    }
    if (powd > D(0)) continue;
    const D Gd = act_exp(powd);
    const D raw_d = pd.o[i] * Gd;
    const D ad = std::min(cap, raw_d);
    r.margin = std::min(r.margin, std::fabs((double)ad - (double)inv255) / (double)inv255);
    if (raw_d > cap) r.margin = std::min(r.margin, ((double)raw_d - (double)cap) / (double)cap);
    if (ad < inv255) continue;
    const D Tnd = Td * (D(1) - ad);
    r.margin = std::min(r.margin, std::fabs((double)Tnd - (double)t_stop) / (double)t_stop);
    if (Tnd < t_stop) break;
    // value track (precision S); identical to the decision track when S == D
    const S dxs = ps.mux[i] - S(px), dys = ps.muy[i] - S(py);
    const S pows = pixel_power(ps.A[i], ps.B[i], ps.C[i], dxs, dys);
    const S Gs = act_exp(pows);
    const bool capped = raw_d > cap;
    const S as = capped ? S(cap) : ps.o[i] * Gs;
    const S w = as * Ts;
    for (int ch = 0; ch < 3; ++ch) r.C[ch] = r.C[ch] + ps.col[ch][i] * w;
    r.Dep = r.Dep + ps.z[i] * w;
    if (keep_entries) r.entries.push_back({i, (int32_t)pos, as, Gs, Ts, dxs, dys, capped});
    Ts = Ts * (S(1) - as);
    Td = Tnd;
    r.n = (int32_t)pos + 1;
    r.blended++;
  }
  for (int ch = 0; ch < 3; ++ch) r.C[ch] = r.C[ch] + Ts * S(cam.bg[ch]);
  r.T = Ts;
  return r;
}

uint64_t mix64(uint64_t h, uint64_t v) {
  h ^= v + 0x9e3779b97f4a7c15ULL + (h << 6) + (h >> 2);
  return h;
}

// ---------------------------------------------------------------------------
// O11: exact derivative of O1-O10 ("explicitly derived"), suffix
// form with stored per-entry T_k (not the GPU's division trick); R18 at clamps.
// ---------------------------------------------------------------------------
template <class S> struct ScreenGrad {
  S mux = 0, muy = 0, A = 0, B = 0, C = 0, o = 0, col[3] = {0, 0, 0}, z = 0;
  void add(const ScreenGrad& t) {
    mux += t.mux, muy += t.muy, A += t.A, B += t.B, C += t.C, o += t.o, z += t.z;
    for (int ch = 0; ch < 3; ++ch) col[ch] += t.col[ch];
  }
};

template <class S>
void chain_to_params(const RefCamera& cam, int deg, const ParamView<S>& g, const Fwd<S>& f,
                     const ScreenGrad<S>& sg, S* out /* [F] */) {
  S W[3][3];
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) W[r][c] = S(cam.R_cw[3 * r + c]);
  const S fx = S(cam.fx), fy = S(cam.fy);
  const S zc = f.pc[2];

  // conic (A, B, C) = (c, -b, a)/det  ->  (a, b, c)
  const S det2 = f.det * f.det;
  const S ga = (sg.A * (-f.c * f.c) + sg.B * (f.b * f.c) + sg.C * (-f.b * f.b)) / det2;
  const S gb = (sg.A * (S(2) * f.b * f.c) + sg.B * (-(f.det + S(2) * f.b * f.b)) + sg.C * (S(2) * f.a * f.b)) / det2;
  const S gc = (sg.A * (-f.b * f.b) + sg.B * (f.a * f.b) + sg.C * (-f.a * f.a)) / det2;
  // Sigma_hat = T Sigma T^T: dL/dSigma = T^T G2 T, dL/dT = 2 G2 T Sigma
  const S G2[2][2] = {{ga, gb / S(2)}, {gb / S(2), gc}};
  S gSig[3][3], gT[2][3];
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) {
      S acc = S(0);
      for (int i = 0; i < 2; ++i)
        for (int j = 0; j < 2; ++j) acc += f.T[i][r] * G2[i][j] * f.T[j][c];
      gSig[r][c] = acc;
    }
  for (int i = 0; i < 2; ++i)
    for (int c = 0; c < 3; ++c) {
      S acc = S(0);
      for (int j = 0; j < 2; ++j)
        for (int k = 0; k < 3; ++k) acc += S(2) * G2[i][j] * f.T[j][k] * f.Sig[k][c];
      gT[i][c] = acc;
    }
  // T = J W  ->  dL/dJ = dL/dT W^T (only J00, J02, J11, J12 are non-constant)
  S gJ[2][3];
  for (int i = 0; i < 2; ++i)
    for (int k = 0; k < 3; ++k) {
      S acc = S(0);
      for (int c = 0; c < 3; ++c) acc += gT[i][c] * W[k][c];
      gJ[i][k] = acc;
    }
  // p_c gradient: J(p_c), mu(p_c), depth
  S gpc[3] = {S(0), S(0), S(0)};
  gpc[2] += gJ[0][0] * (-fx / (zc * zc));
  gpc[2] += gJ[1][1] * (-fy / (zc * zc));
  if (!f.jclx) {  // J02 = -fx x / z^2
    gpc[0] += gJ[0][2] * (-fx / (zc * zc));
    gpc[2] += gJ[0][2] * (S(2) * fx * f.pc[0] / (zc * zc * zc));
  } else {  // J02 = -fx kappa / z
    gpc[2] += gJ[0][2] * (fx * f.uxc / (zc * zc));
  }
  if (!f.jcly) {
    gpc[1] += gJ[1][2] * (-fy / (zc * zc));
    gpc[2] += gJ[1][2] * (S(2) * fy * f.pc[1] / (zc * zc * zc));
  } else {
    gpc[2] += gJ[1][2] * (fy * f.uyc / (zc * zc));
  }
  gpc[0] += sg.mux * (fx / zc);
  gpc[2] += sg.mux * (-fx * f.pc[0] / (zc * zc));
  gpc[1] += sg.muy * (fy / zc);
  gpc[2] += sg.muy * (-fy * f.pc[1] / (zc * zc));
  gpc[2] += sg.z;
  // p_c = W p + t  ->  dL/dp = W^T dL/dp_c
  S gp[3];
  for (int c = 0; c < 3; ++c) gp[c] = W[0][c] * gpc[0] + W[1][c] * gpc[1] + W[2][c] * gpc[2];

  // colour: col_ch = max(0, sum_k sh_k,ch Y_k(d) + 0.5), d = v/|v|, v = p - o_cam
  const int nk = (deg + 1) * (deg + 1);
  S Y[16], dY[16][3];
  sh_eval<S>(deg, f.d, Y, dY);
  S gd[3] = {S(0), S(0), S(0)};
  for (int ch = 0; ch < 3; ++ch) {
    if (f.clamp[ch]) {
      for (int k = 0; k < nk; ++k) out[11 + 3 * k + ch] = S(0);
      continue;
    }
    for (int k = 0; k < nk; ++k) {
      out[11 + 3 * k + ch] = Y[k] * sg.col[ch];
      for (int c = 0; c < 3; ++c) gd[c] += sg.col[ch] * g.sh[3 * k + ch] * dY[k][c];
    }
  }
  const S ddot = f.d[0] * gd[0] + f.d[1] * gd[1] + f.d[2] * gd[2];
  for (int c = 0; c < 3; ++c) gp[c] += (gd[c] - f.d[c] * ddot) / f.vn;
  for (int c = 0; c < 3; ++c) out[c] = gp[c];

  // Sigma = M M^T, M = R diag(s): dL/dM = 2 gSig M
  S gM[3][3];
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) {
      S acc = S(0);
      for (int k = 0; k < 3; ++k) acc += S(2) * gSig[r][k] * f.M[k][c];
      gM[r][c] = acc;
    }
  S gR[3][3];
  for (int j = 0; j < 3; ++j) {
    S gs = S(0);
    for (int i = 0; i < 3; ++i) gs += gM[i][j] * f.R[i][j];
    out[3 + j] = gs * f.s[j];  // d s / d l = s
    for (int i = 0; i < 3; ++i) gR[i][j] = gM[i][j] * f.s[j];
  }
  // R(q_hat): partial derivatives of each entry w.r.t. (w, x, y, z)
  const S w = f.qh[0], x = f.qh[1], y = f.qh[2], z = f.qh[3];
  const S dR[3][3][4] = {
      {{0, 0, -4 * y, -4 * z}, {-2 * z, 2 * y, 2 * x, -2 * w}, {2 * y, 2 * z, 2 * w, 2 * x}},
      {{2 * z, 2 * y, 2 * x, 2 * w}, {0, -4 * x, 0, -4 * z}, {-2 * x, -2 * w, 2 * z, 2 * y}},
      {{-2 * y, 2 * z, -2 * w, 2 * x}, {2 * x, 2 * w, 2 * z, 2 * y}, {0, -4 * x, -4 * y, 0}}};
  S gqh[4] = {S(0), S(0), S(0), S(0)};
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      for (int k = 0; k < 4; ++k) gqh[k] += gR[i][j] * dR[i][j][k];
  // q_hat = q/|q|:  dL/dq = (I - q_hat q_hat^T) dL/dq_hat / |q|
  const S qd = gqh[0] * f.qh[0] + gqh[1] * f.qh[1] + gqh[2] * f.qh[2] + gqh[3] * f.qh[3];
  for (int k = 0; k < 4; ++k) out[6 + k] = (gqh[k] - f.qh[k] * qd) / f.qn;
  // opacity: o = sigmoid(logit)
  out[10] = sg.o * f.o * (S(1) - f.o);
}

template <class DT, class ST>
void render_bwd_run(const RefCamera* cam, int64_t P, int64_t P_stride, int deg, const float* params,
                    const float* g_rgb, const float* g_depth, const Proj<DT>& pd, const Proj<ST>& ps,
                    const std::vector<std::vector<int32_t>>& lists, double* grad_out, double* bound_out,
                    double* screen_out, double* screen_bound_out) {
  const int W = cam->width, H = cam->height, TX = (W + kTile - 1) / kTile, TY = (H + kTile - 1) / kTile;
  const int F = 11 + 3 * (deg + 1) * (deg + 1);
  const int NT = TX * TY;
  // Pixels are visited tile by tile (row-major inside the tile); a tile's contributions
  // are summed per position of its list, and the tiles' sums are then added to the
  // Gaussians in tile order: ONE summation order whatever the number of threads
  // (OpenMP over tiles: the CPU baseline on all host cores).
  std::vector<std::vector<ScreenGrad<ST>>> tile_acc((size_t)NT);
#pragma omp parallel for schedule(dynamic, 1)
  for (int t = 0; t < NT; ++t) {
    const auto& list = lists[t];
    std::vector<ScreenGrad<ST>>& acc = tile_acc[(size_t)t];
    const int ox = (t % TX) * kTile, oy = (t / TX) * kTile;
    for (int py = oy; py < std::min(oy + kTile, H); ++py)
      for (int px = ox; px < std::min(ox + kTile, W); ++px) {
        const int64_t pix = (int64_t)py * W + px;
        if (g_rgb[pix] == 0.f && g_rgb[(int64_t)W * H + pix] == 0.f && g_rgb[2 * (int64_t)W * H + pix] == 0.f &&
            (!g_depth || g_depth[pix] == 0.f))
          continue;  // zero upstream: this pixel contributes exactly zero (linearity)
        if (acc.empty()) acc.resize(list.size());
        PixelResult<DT, ST> r = composite_pixel<DT, ST>(px, py, list, pd, ps, *cam, true);
        if constexpr (kIsRn<ST>) {
          // Bound of T_k for ANY evaluation route through this pixel's factors
          // (forward products, or T_final divided back by (1 - alpha_j), j >= k):
          // twice the relative bound of the complete product T_final.
          const double rho = r.T.v != 0.0 ? r.T.m / std::fabs(r.T.v) : 0.0;
          for (auto& e : r.entries) e.T.m = std::max(e.T.m, 2.0 * rho * std::fabs(e.T.v));
        }
        ST gC[3];
        for (int ch = 0; ch < 3; ++ch) gC[ch] = ST(g_rgb[ch * (int64_t)W * H + pix]);
        const ST gD = g_depth ? ST(g_depth[pix]) : ST(0);
        // suffix sums S^C_k = sum_{j>k} c_j a_j T_j + T_final bg,  S^D_k = sum_{j>k} z_j a_j T_j
        const size_t n = r.entries.size();
        std::vector<ST> SC(3 * (n + 1)), SD(n + 1);
        for (int ch = 0; ch < 3; ++ch) SC[3 * n + ch] = r.T * ST(cam->bg[ch]);
        SD[n] = ST(0);
        for (size_t k = n; k-- > 0;) {
          const auto& e = r.entries[k];
          for (int ch = 0; ch < 3; ++ch) SC[3 * k + ch] = SC[3 * (k + 1) + ch] + ps.col[ch][e.id] * e.alpha * e.T;
          SD[k] = SD[k + 1] + ps.z[e.id] * e.alpha * e.T;
        }
        for (size_t k = 0; k < n; ++k) {
          const auto& e = r.entries[k];
          const int32_t i = e.id;
          ScreenGrad<ST>& s = acc[(size_t)e.pos];
          const ST aT = e.alpha * e.T;
          for (int ch = 0; ch < 3; ++ch) s.col[ch] += gC[ch] * aT;
          s.z += gD * aT;
          ST dalpha = ST(0);
          for (int ch = 0; ch < 3; ++ch)
            dalpha += gC[ch] * (ps.col[ch][i] * e.T - SC[3 * (k + 1) + ch] / (ST(1) - e.alpha));
          dalpha += gD * (ps.z[i] * e.T - SD[k + 1] / (ST(1) - e.alpha));
          if (e.capped) continue;  // alpha = 0.99: no derivative w.r.t. o, mu, conic (R18)
          s.o += e.G * dalpha;
          const ST dpow = ps.o[i] * e.G * dalpha;  // d(o exp(power))/d power = o G
          s.mux += dpow * (-(ps.A[i] * e.dx + ps.B[i] * e.dy));
          s.muy += dpow * (-(ps.B[i] * e.dx + ps.C[i] * e.dy));
          s.A += dpow * (ST(-0.5) * e.dx * e.dx);
          s.B += dpow * (-e.dx * e.dy);
          s.C += dpow * (ST(-0.5) * e.dy * e.dy);
        }
      }
  }
  std::vector<ScreenGrad<ST>> sg((size_t)P);
  for (int t = 0; t < NT; ++t)
    for (size_t k = 0; k < tile_acc[(size_t)t].size(); ++k) sg[(size_t)lists[t][k]].add(tile_acc[(size_t)t][k]);
  tile_acc.clear();
#pragma omp parallel for schedule(dynamic, 256)
    for (int64_t i = 0; i < P; ++i) {
      std::vector<ST> out(F);
      for (int r = 0; r < F; ++r) grad_out[r * P + i] = 0.0;
      if (bound_out)
        for (int r = 0; r < F; ++r) bound_out[r * P + i] = 0.0;
      if (screen_out) {
        const ScreenGrad<ST>& s = sg[i];
        const ST v[10] = {s.mux, s.muy, s.A, s.B, s.C, s.o, s.col[0], s.col[1], s.col[2], s.z};
        for (int r = 0; r < 10; ++r) screen_out[r * P + i] = (double)v[r];
        if constexpr (kIsRn<ST>)
          if (screen_bound_out)
            for (int r = 0; r < 10; ++r) screen_bound_out[r * P + i] = v[r].m;
      }
      if (pd.flags[i] & 128) continue;  // culled: exactly zero gradient
      {  // no pixel contributed: the (linear) chain gives exactly zero
        const ScreenGrad<ST>& s = sg[i];
        const ST v[10] = {s.mux, s.muy, s.A, s.B, s.C, s.o, s.col[0], s.col[1], s.col[2], s.z};
        bool any = false;
        for (int r = 0; r < 10; ++r) any = any || (double)v[r] != 0.0;
        if (!any) continue;
      }
      const ParamView<ST> g = load_params<ST>(params, P_stride, deg, i);
      Fwd<ST> f = project_one<ST>(*cam, deg, g);
      if (f.culled) continue;  // value track disagrees with the decision track (flip)
      // decisions (clamps) follow the decision track
      f.jclx = pd.flags[i] & FLAG_JCLAMP_X;
      f.jcly = pd.flags[i] & FLAG_JCLAMP_Y;
      for (int ch = 0; ch < 3; ++ch) f.clamp[ch] = pd.flags[i] & (1 << ch);
      chain_to_params<ST>(*cam, deg, g, f, sg[i], out.data());
      for (int r = 0; r < F; ++r) grad_out[r * P + i] = (double)out[r];
      if constexpr (kIsRn<ST>)
        if (bound_out)
          for (int r = 0; r < F; ++r) bound_out[r * P + i] = out[r].m;
    }
}


}  // namespace

// ===========================================================================
// C entry points (host pointers; return 0 on success, <0 on bad arguments)
// ===========================================================================
extern "C" {

int gsref_version(void) { return 1; }

// OpenMP threads of the oracle's parallel loops (over tiles, rows, samples and
// Gaussians); every result is independent of the count.  n <= 0: the runtime default
// (OMP_NUM_THREADS or all host cores).  Returns the count now in effect.
int gsref_set_threads(int n) {
#ifdef _OPENMP
  if (n > 0) omp_set_num_threads(n);
  return omp_get_max_threads();
#else
  (void)n;
  return 1;
#endif
}

// Real SH values Y_k(d) for k < (deg+1)^2 at n directions d[3n] (double); test hook.
int gsref_sh_basis(int deg, int64_t n, const double* dirs, double* Y, double* dY) {
  if (deg < 0 || deg > 3) return -1;
  const int nk = (deg + 1) * (deg + 1);
  for (int64_t i = 0; i < n; ++i) {
    double y[16], g[16][3];
    sh_eval<double>(deg, dirs + 3 * i, y, g);
    for (int k = 0; k < nk; ++k) {
      Y[i * nk + k] = y[k];
      if (dY)
        for (int c = 0; c < 3; ++c) dY[(i * nk + k) * 3 + c] = g[k][c];
    }
  }
  return 0;
}

// O1-O8.  out_vals: double [10][P] = mu_x, mu_y, z, A, B, C, opacity, r, g, b
// (culled Gaussians: zeros).  rect: int32 [4][P] = x0, x1, y0, y1 (exclusive ends).
// mode: 0 = F32, 1 = F64.  (MIXED == F32 decisions + F64 values: call twice.)
int gsref_project(const RefCamera* cam, int64_t P, int64_t P_stride, int deg, const float* params, int mode,
                  double* out_vals, int32_t* radius, int32_t* rect, int32_t* tiles, uint8_t* flags) {
  if (!cam || P < 0 || P_stride < P || deg < 0 || deg > 3 || (P > 0 && !params)) return -1;
  auto write = [&](const auto& pr) {
    for (int64_t i = 0; i < P; ++i) {
      const double v[10] = {(double)pr.mux[i], (double)pr.muy[i], (double)pr.z[i], (double)pr.A[i],
                            (double)pr.B[i], (double)pr.C[i], (double)pr.o[i], (double)pr.col[0][i],
                            (double)pr.col[1][i], (double)pr.col[2][i]};
      const bool cul = pr.flags[i] & FLAG_CULLED;
      for (int r = 0; r < 10; ++r) out_vals[r * P + i] = cul ? 0.0 : v[r];
      radius[i] = pr.radius[i];
      tiles[i] = pr.tiles[i];
      flags[i] = pr.flags[i];
      rect[0 * P + i] = pr.x0[i];
      rect[1 * P + i] = pr.x1[i];
      rect[2 * P + i] = pr.y0[i];
      rect[3 * P + i] = pr.y1[i];
    }
  };
  if (mode == 0) write(project_all<float>(*cam, P, P_stride, deg, params));
  else if (mode == 1) write(project_all<double>(*cam, P, P_stride, deg, params));
  else return -1;
  return 0;
}

// O9 with fp32 decisions.  Returns K via *num_keys; writes min(K, capacity) ids
// and tile_ranges [NT][2] (start, end) over the full sorted key array.
int gsref_bin_tiles(const RefCamera* cam, int64_t P, int64_t P_stride, int deg, const float* params,
                    int64_t capacity, int32_t* sorted_ids, int32_t* sorted_tiles, int32_t* tile_ranges,
                    int64_t* num_keys) {
  if (!cam || P < 0) return -1;
  const Proj<float> pf = project_all<float>(*cam, P, P_stride, deg, params);
  const std::vector<Key<float>> keys = emit_and_sort(*cam, pf);
  const int NT = ((cam->width + kTile - 1) / kTile) * ((cam->height + kTile - 1) / kTile);
  for (int t = 0; t < NT; ++t) tile_ranges[2 * t] = tile_ranges[2 * t + 1] = 0;
  const int64_t K = (int64_t)keys.size();
  *num_keys = K;
  for (int64_t k = 0; k < K; ++k) {
    if (k < capacity) {
      sorted_ids[k] = keys[k].id;
      if (sorted_tiles) sorted_tiles[k] = keys[k].tile;
    }
    if (k == 0 || keys[k].tile != keys[k - 1].tile) tile_ranges[2 * keys[k].tile] = (int32_t)k;
    if (k == K - 1 || keys[k].tile != keys[k + 1].tile) tile_ranges[2 * keys[k].tile + 1] = (int32_t)(k + 1);
  }
  return 0;
}

// O1-O10 for one view.  rgb [3][H][W], depth/T_final [H][W] (double), n_contrib
// [H][W]; counters blended/evaluated (nullable); margin [H][W] (nullable) = min
// relative distance of any decision to its threshold; signature (nullable) = hash
// of every decision (culls, rects, clamps, per-pixel composited set and stop).
// mode: 0 = F32, 1 = F64, 2 = MIXED (F32 decisions, F64 values).
int gsref_render_fwd(const RefCamera* cam, int64_t P, int64_t P_stride, int deg, const float* params, int mode,
                     double* rgb, double* depth, double* T_final, int32_t* n_contrib, int64_t* blended,
                     int64_t* evaluated, double* margin, uint64_t* signature) {
  if (!cam || P < 0 || P_stride < P || deg < 0 || deg > 3 || mode < 0 || mode > 2) return -1;
  const int W = cam->width, H = cam->height, TX = (W + kTile - 1) / kTile;
  auto run = [&](const auto& pd, const auto& ps) {
    using DT = std::decay_t<decltype(pd.mux[0])>;
    using ST = std::decay_t<decltype(ps.mux[0])>;
    const auto lists = tile_lists(*cam, pd);  // lists follow the decision track
    int64_t nb = 0, ne = 0;
    uint64_t sig = 0;
    for (int64_t i = 0; i < P; ++i) {
      sig = mix64(sig, pd.flags[i]);
      sig = mix64(sig, (uint64_t)pd.radius[i]);
      sig = mix64(sig, ((uint64_t)pd.x0[i] << 48) ^ ((uint64_t)pd.x1[i] << 32) ^ ((uint64_t)pd.y0[i] << 16) ^
                           (uint64_t)pd.y1[i]);
    }
    // every pixel is independent (OpenMP over rows); the signature folds the pixels'
    // decision hashes in pixel order afterwards
    std::vector<uint64_t> pix_sig(signature ? (size_t)W * H : 0);
#pragma omp parallel for schedule(dynamic, 1) reduction(+ : nb, ne)
    for (int py = 0; py < H; ++py)
      for (int px = 0; px < W; ++px) {
        const auto& list = lists[(py / kTile) * TX + px / kTile];
        const PixelResult<DT, ST> r = composite_pixel<DT, ST>(px, py, list, pd, ps, *cam, signature != nullptr);
        const int64_t pix = (int64_t)py * W + px;
        for (int ch = 0; ch < 3; ++ch) rgb[ch * (int64_t)W * H + pix] = (double)r.C[ch];
        depth[pix] = (double)r.Dep;
        T_final[pix] = (double)r.T;
        n_contrib[pix] = r.n;
        if (margin) margin[pix] = r.margin;
        nb += r.blended;
        ne += r.evaluated;
        if (signature) {
          uint64_t h = mix64(0, (uint64_t)r.n);
          for (const auto& e : r.entries) h = mix64(h, ((uint64_t)e.id << 1) | (e.capped ? 1 : 0));
          pix_sig[(size_t)pix] = h;
        }
      }
    for (const uint64_t h : pix_sig) sig = mix64(sig, h);
    if (blended) *blended = nb;
    if (evaluated) *evaluated = ne;
    if (signature) *signature = sig;
  };
  if (mode == 0) {
    const Proj<float> pf = project_all<float>(*cam, P, P_stride, deg, params);
    run(pf, pf);
  } else if (mode == 1) {
    const Proj<double> pd = project_all<double>(*cam, P, P_stride, deg, params);
    run(pd, pd);
  } else {
    const Proj<float> pf = project_all<float>(*cam, P, P_stride, deg, params);
    const Proj<double> pd = project_all<double>(*cam, P, P_stride, deg, params);
    run(pf, pd);
  }
  return 0;
}

// O10 at n selected pixels (px[j], py[j]) only; outputs per sample: rgb [3][n],
// depth/T_final [n] (double), n_contrib [n], margin [n] (nullable).  Tile lists are
// built exactly as in gsref_render_fwd; used for sampled parity at full size.
int gsref_render_pixels(const RefCamera* cam, int64_t P, int64_t P_stride, int deg, const float* params, int mode,
                        int64_t n, const int32_t* px, const int32_t* py, double* rgb, double* depth, double* T_final,
                        int32_t* n_contrib, double* margin) {
  if (!cam || P < 0 || P_stride < P || deg < 0 || deg > 3 || mode < 0 || mode > 2 || n < 0) return -1;
  const int TX = (cam->width + kTile - 1) / kTile;
  auto run = [&](const auto& pd, const auto& ps) {
    using DT = std::decay_t<decltype(pd.mux[0])>;
    using ST = std::decay_t<decltype(ps.mux[0])>;
    const auto lists = tile_lists(*cam, pd);
    for (int64_t j = 0; j < n; ++j)
      if (px[j] < 0 || py[j] < 0 || px[j] >= cam->width || py[j] >= cam->height) return -1;
#pragma omp parallel for schedule(dynamic, 16)
    for (int64_t j = 0; j < n; ++j) {
      const auto& list = lists[(py[j] / kTile) * TX + px[j] / kTile];
      const PixelResult<DT, ST> r = composite_pixel<DT, ST>(px[j], py[j], list, pd, ps, *cam, false);
      for (int ch = 0; ch < 3; ++ch) rgb[ch * n + j] = (double)r.C[ch];
      depth[j] = (double)r.Dep;
      T_final[j] = (double)r.T;
      n_contrib[j] = r.n;
      if (margin) margin[j] = r.margin;
    }
    return 0;
  };
  if (mode == 0) {
    const Proj<float> pf = project_all<float>(*cam, P, P_stride, deg, params);
    return run(pf, pf);
  } else if (mode == 1) {
    const Proj<double> pd = project_all<double>(*cam, P, P_stride, deg, params);
    return run(pd, pd);
  }
  const Proj<float> pf = project_all<float>(*cam, P, P_stride, deg, params);
  const Proj<double> pd = project_all<double>(*cam, P, P_stride, deg, params);
  return run(pf, pd);
}

// O10 + O11 for one view: parameter gradients of L = <g_rgb, C> + <g_depth, D>
// (the vector-Jacobian product the harness feeds in; R19).  grad_out: double
// [F][P] (overwritten, not accumulated); screen_out (nullable): double [10][P] =
// dL/d(mu_x, mu_y, A, B, C, opacity, r, g, b, z).  g_depth may be NULL.
int gsref_render_bwd(const RefCamera* cam, int64_t P, int64_t P_stride, int deg, const float* params, int mode,
                     const float* g_rgb, const float* g_depth, double* grad_out, double* screen_out) {
  if (!cam || P < 0 || P_stride < P || deg < 0 || deg > 3 || mode < 0 || mode > 3 || !g_rgb) return -1;
  if (mode == 0) {
    const Proj<float> pf = project_all<float>(*cam, P, P_stride, deg, params);
    render_bwd_run(cam, P, P_stride, deg, params, g_rgb, g_depth, pf, pf, tile_lists(*cam, pf), grad_out,
                   nullptr, screen_out, nullptr);
  } else if (mode == 3) {
    const Proj<float> pf = project_all<float>(*cam, P, P_stride, deg, params);
    render_bwd_run(cam, P, P_stride, deg, params, g_rgb, g_depth, pf, promote<double>(pf), tile_lists(*cam, pf),
                   grad_out, nullptr, screen_out, nullptr);
  } else if (mode == 2) {
    const Proj<float> pf = project_all<float>(*cam, P, P_stride, deg, params);
    const Proj<double> pd = project_all<double>(*cam, P, P_stride, deg, params);
    render_bwd_run(cam, P, P_stride, deg, params, g_rgb, g_depth, pf, pd, tile_lists(*cam, pf), grad_out,
                   nullptr, screen_out, nullptr);
  } else {
    const Proj<double> pd = project_all<double>(*cam, P, P_stride, deg, params);
    render_bwd_run(cam, P, P_stride, deg, params, g_rgb, g_depth, pd, pd, tile_lists(*cam, pd), grad_out,
                   nullptr, screen_out, nullptr);
  }
  return 0;
}

// MIXED-mode O10 + O11 with running error bounds (struct Rn): grad_out equals
// gsref_render_bwd(mode = MIXED) bit for bit; bound_out [F][P] (double) is the
// first-order bound M of each gradient element in units of u = 2^-24, so an fp32
// evaluation of the same maths is expected within c u M of grad_out (the parity
// tolerance).  screen_out / screen_bound_out (nullable): the same for
// the [10][P] screen-space gradients.
int gsref_render_bwd_bound(const RefCamera* cam, int64_t P, int64_t P_stride, int deg, const float* params,
                           int stage, const float* g_rgb, const float* g_depth, double* grad_out, double* bound_out,
                           double* screen_out, double* screen_bound_out) {
  if (!cam || P < 0 || P_stride < P || deg < 0 || deg > 3 || !g_rgb || !grad_out || !bound_out) return -1;
  const Proj<float> pf = project_all<float>(*cam, P, P_stride, deg, params);
  const Proj<Rn> pr = stage ? stage_records(*cam, P, P_stride, deg, params, pf)
                             : project_all<Rn>(*cam, P, P_stride, deg, params);
  render_bwd_run(cam, P, P_stride, deg, params, g_rgb, g_depth, pf, pr, tile_lists(*cam, pf), grad_out, bound_out,
                 screen_out, screen_bound_out);
  return 0;
}

// Decision margins in units of the running error bound, at n pixels (px[j], py[j]):
// margin_u[j] = min over the pixel's decisions (power > 0, the 0.99 cap, alpha <
// 1/255, T' < 1e-4) of |q_fp32 - threshold| / (u m_q), m_q the bound of q.  A GPU
// decision can differ from the oracle's only where this is below the parity
// constant c (a threshold flip); DESIGN.md §6.
int gsref_margin_bound(const RefCamera* cam, int64_t P, int64_t P_stride, int deg, const float* params, int stage,
                       int64_t n,
                       const int32_t* px, const int32_t* py, double* margin_u) {
  if (!cam || P < 0 || P_stride < P || deg < 0 || deg > 3 || n < 0 || !margin_u) return -1;
  const int TX = (cam->width + kTile - 1) / kTile;
  const Proj<float> pf = project_all<float>(*cam, P, P_stride, deg, params);
  const Proj<Rn> pr = stage ? stage_records(*cam, P, P_stride, deg, params, pf)
                             : project_all<Rn>(*cam, P, P_stride, deg, params);
  const auto lists = tile_lists(*cam, pf);
  for (int64_t j = 0; j < n; ++j)
    if (px[j] < 0 || py[j] < 0 || px[j] >= cam->width || py[j] >= cam->height) return -1;
#pragma omp parallel for schedule(dynamic, 16)
  for (int64_t j = 0; j < n; ++j) {
    const auto& list = lists[(py[j] / kTile) * TX + px[j] / kTile];
    margin_u[j] = composite_pixel<float, Rn>(px[j], py[j], list, pf, pr, *cam, false).margin_u;
  }
  return 0;
}

// O12: Adam (R20), PyTorch convention, per-row learning rate, dense.  fp64 state
// update of fp32 inputs; writes the updated params/m/v (double [F][P]).
int gsref_adam_step(int64_t F, int64_t P, int64_t P_stride, const float* params, const float* grad,
                    const float* m, const float* v, const float* lr_per_row, double beta1, double beta2,
                    double eps, int64_t step, double* params_out, double* m_out, double* v_out) {
  if (P < 0 || F <= 0 || step < 1) return -1;
  const double bc1 = 1.0 - std::pow(beta1, (double)step);
  const double bc2 = 1.0 - std::pow(beta2, (double)step);
  for (int64_t r = 0; r < F; ++r)
    for (int64_t i = 0; i < P; ++i) {
      const int64_t j = r * P_stride + i;
      const double g = grad[j];
      const double mn = beta1 * m[j] + (1.0 - beta1) * g;
      const double vn = beta2 * v[j] + (1.0 - beta2) * g * g;
      const double mhat = mn / bc1, vhat = vn / bc2;
      params_out[r * P + i] = (double)params[j] - (double)lr_per_row[r] * mhat / (std::sqrt(vhat) + eps);
      m_out[r * P + i] = mn;
      v_out[r * P + i] = vn;
    }
  return 0;
}

// Eq. 12 harness (R19): L = mean_{px,ch}|C - C*| + w_d mean_px |D - D*|, sign(0) = 0;
// target samples that are not measurements (non-finite colour, depth <= 0 or
// non-finite: R41, R43) contribute neither loss nor gradient (the means keep npix).
// grads (double) dL/dC [3][H][W], dL/dD [H][W]; returns L via *loss.
int gsref_l1_loss_grad(int64_t npix, const double* rgb, const double* depth, const float* t_rgb,
                       const float* t_depth, double w_depth, double* g_rgb, double* g_depth, double* loss) {
  if (npix <= 0) return -1;
  double L = 0.0;
  const double sc = 1.0 / (3.0 * (double)npix), sd = w_depth / (double)npix;
  for (int64_t j = 0; j < 3 * npix; ++j) {
    if (!std::isfinite(t_rgb[j])) {  // not a measurement (R43): no loss, no gradient
      g_rgb[j] = 0.0;
      continue;
    }
    const double r = rgb[j] - (double)t_rgb[j];
    L += std::fabs(r) * sc;
    g_rgb[j] = (r > 0 ? 1.0 : (r < 0 ? -1.0 : 0.0)) * sc;
  }
  for (int64_t j = 0; j < npix; ++j) {
    if (!(t_depth[j] > 0.f) || !std::isfinite(t_depth[j])) {  // invalid depth (R41, R43)
      g_depth[j] = 0.0;
      continue;
    }
    const double r = depth[j] - (double)t_depth[j];
    L += std::fabs(r) * sd;
    g_depth[j] = (r > 0 ? 1.0 : (r < 0 ? -1.0 : 0.0)) * sd;
  }
  *loss = L;
  return 0;
}

}  // extern "C"
