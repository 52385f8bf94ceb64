// Input frames (gs_decode_rgbd): one sensor RGB-D frame -- 8-bit interleaved RGB and
// 16-bit depth in units of depth_scale metres ("a pair of RGB-D images as
// input"; reading R41) -- into the planar float images of Eq. 12 and
// Eqs. 6 / 10.  An HBM-streaming kernel: 5 B read and 16 B written per pixel.  The host
// ships the frame in its 5-B/px sensor form instead of 16-B/px floats, so the per-step
// host -> device traffic of Trainer.step_host drops 3.2x.
#include "gsr_internal.cuh"

namespace gsr {
namespace {

__device__ __forceinline__ float u8f(uint32_t w, int byte) { return __fdiv_rn((float)((w >> (8 * byte)) & 0xffu), 255.f); }

// 4 pixels per thread: 12 B of RGB (3 aligned words), 8 B of depth, one float4 per plane.
__global__ void __launch_bounds__(256) k_decode_rgbd4(int64_t n4, int64_t npix, const uint32_t* __restrict__ rgb,
                                                      const uint2* __restrict__ depth, float scale,
                                                      float4* __restrict__ out_rgb, float4* __restrict__ out_d) {
  const int64_t plane4 = npix / 4;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n4; q += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t w0 = rgb[3 * q], w1 = rgb[3 * q + 1], w2 = rgb[3 * q + 2];
    const uint2 d = depth[q];
    // bytes b0..b11 = R0 G0 B0 R1 | G1 B1 R2 G2 | B2 R3 G3 B3
    out_rgb[q] = make_float4(u8f(w0, 0), u8f(w0, 3), u8f(w1, 2), u8f(w2, 1));
    out_rgb[plane4 + q] = make_float4(u8f(w0, 1), u8f(w1, 0), u8f(w1, 3), u8f(w2, 2));
    out_rgb[2 * plane4 + q] = make_float4(u8f(w0, 2), u8f(w1, 1), u8f(w2, 0), u8f(w2, 3));
    out_d[q] = make_float4(__fmul_rn((float)(d.x & 0xffffu), scale), __fmul_rn((float)(d.x >> 16), scale),
                           __fmul_rn((float)(d.y & 0xffffu), scale), __fmul_rn((float)(d.y >> 16), scale));
  }
}

__global__ void __launch_bounds__(256) k_decode_rgbd1(int64_t npix, const uint8_t* __restrict__ rgb,
                                                      const uint16_t* __restrict__ depth, float scale,
                                                      float* __restrict__ out_rgb, float* __restrict__ out_d) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < npix; i += (int64_t)gridDim.x * blockDim.x) {
#pragma unroll
    for (int c = 0; c < 3; ++c) out_rgb[c * npix + i] = __fdiv_rn((float)rgb[3 * i + c], 255.f);
    out_d[i] = __fmul_rn((float)depth[i], scale);
  }
}

bool aligned(const void* p, uintptr_t a) { return (reinterpret_cast<uintptr_t>(p) & (a - 1)) == 0; }

}  // namespace

void launch_decode_rgbd(int64_t npix, const uint8_t* rgb, const uint16_t* depth, float scale, float* out_rgb,
                        float* out_d, cudaStream_t s) {
  const int64_t cap = (int64_t)sm_count() * 8;
  if (npix % 4 == 0 && aligned(rgb, 4) && aligned(depth, 8) && aligned(out_rgb, 16) && aligned(out_d, 16)) {
    const int64_t n4 = npix / 4;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((n4 + 255) / 256, cap));
    k_decode_rgbd4<<<grid, 256, 0, s>>>(n4, npix, reinterpret_cast<const uint32_t*>(rgb),
                                        reinterpret_cast<const uint2*>(depth), scale,
                                        reinterpret_cast<float4*>(out_rgb), reinterpret_cast<float4*>(out_d));
  } else {
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((npix + 255) / 256, cap));
    k_decode_rgbd1<<<grid, 256, 0, s>>>(npix, rgb, depth, scale, out_rgb, out_d);
  }
  count_launch();
}

}  // namespace gsr
