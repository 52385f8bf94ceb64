// Real spherical-harmonics basis up to degree 3 (Condon-Shortley phase, index
// k = l^2 + l + m), unrolled polynomial forms on the unit sphere, and their Cartesian
// gradients (only the tangential part matters: the direction is normalised).
// Reading R13; the oracle evaluates the textbook definition instead and
// the parity tests tie the two together.
#pragma once

namespace gsr {

constexpr float kC0 = 0.28209479177387814f;
constexpr float kC1 = 0.4886025119029199f;
constexpr float kC2_0 = 1.0925484305920792f, kC2_1 = -1.0925484305920792f, kC2_2 = 0.31539156525252005f,
                kC2_3 = -1.0925484305920792f, kC2_4 = 0.5462742152960396f;
constexpr float kC3_0 = -0.5900435899266435f, kC3_1 = 2.890611442640554f, kC3_2 = -0.4570457994644658f,
                kC3_3 = 0.3731763325901154f, kC3_4 = -0.4570457994644658f, kC3_5 = 1.445305721320277f,
                kC3_6 = -0.5900435899266435f;

// Y_k and dY_k/d(x, y, z) for a compile-time k (the switch folds after unrolling).
__device__ __forceinline__ void sh_term(int k, float x, float y, float z, float& Y, float& gx, float& gy, float& gz) {
  const float xx = x * x, yy = y * y, zz = z * z;
  switch (k) {
    case 0: Y = kC0, gx = gy = gz = 0.f; break;
    case 1: Y = -kC1 * y, gx = 0.f, gy = -kC1, gz = 0.f; break;
    case 2: Y = kC1 * z, gx = 0.f, gy = 0.f, gz = kC1; break;
    case 3: Y = -kC1 * x, gx = -kC1, gy = 0.f, gz = 0.f; break;
    case 4: Y = kC2_0 * x * y, gx = kC2_0 * y, gy = kC2_0 * x, gz = 0.f; break;
    case 5: Y = kC2_1 * y * z, gx = 0.f, gy = kC2_1 * z, gz = kC2_1 * y; break;
    case 6: Y = kC2_2 * (2.f * zz - xx - yy), gx = -2.f * kC2_2 * x, gy = -2.f * kC2_2 * y, gz = 4.f * kC2_2 * z; break;
    case 7: Y = kC2_3 * x * z, gx = kC2_3 * z, gy = 0.f, gz = kC2_3 * x; break;
    case 8: Y = kC2_4 * (xx - yy), gx = 2.f * kC2_4 * x, gy = -2.f * kC2_4 * y, gz = 0.f; break;
    case 9: Y = kC3_0 * y * (3.f * xx - yy), gx = 6.f * kC3_0 * x * y, gy = kC3_0 * (3.f * xx - 3.f * yy), gz = 0.f; break;
    case 10: Y = kC3_1 * x * y * z, gx = kC3_1 * y * z, gy = kC3_1 * x * z, gz = kC3_1 * x * y; break;
    case 11:
      Y = kC3_2 * y * (4.f * zz - xx - yy), gx = -2.f * kC3_2 * x * y, gy = kC3_2 * (4.f * zz - xx - 3.f * yy),
      gz = 8.f * kC3_2 * y * z;
      break;
    case 12:
      Y = kC3_3 * z * (2.f * zz - 3.f * xx - 3.f * yy), gx = -6.f * kC3_3 * x * z, gy = -6.f * kC3_3 * y * z,
      gz = kC3_3 * (6.f * zz - 3.f * xx - 3.f * yy);
      break;
    case 13:
      Y = kC3_4 * x * (4.f * zz - xx - yy), gx = kC3_4 * (4.f * zz - 3.f * xx - yy), gy = -2.f * kC3_4 * x * y,
      gz = 8.f * kC3_4 * x * z;
      break;
    case 14:
      Y = kC3_5 * z * (xx - yy), gx = 2.f * kC3_5 * x * z, gy = -2.f * kC3_5 * y * z, gz = kC3_5 * (xx - yy);
      break;
    default:
      Y = kC3_6 * x * (xx - 3.f * yy), gx = kC3_6 * (3.f * xx - 3.f * yy), gy = -6.f * kC3_6 * x * y, gz = 0.f;
      break;
  }
}

// Y_k only.
__device__ __forceinline__ float sh_value(int k, float x, float y, float z) {
  float Y, gx, gy, gz;
  sh_term(k, x, y, z, Y, gx, gy, gz);
  return Y;
}

}  // namespace gsr
