// Visibility-sparse gradient exchange: the
// union of the ranks' visible sets, its ordered compaction, and the gather / scatter
// of the gradient columns it names.  All HBM-streaming; the collective itself (an
// all-reduce of the packed columns) is NCCL's, issued by the caller between gather
// and scatter.
#include "gsr_internal.cuh"

namespace gsr {
namespace {

constexpr int kVisPtrs = 32;
struct FlagPtrs {
  const uint8_t* p[kVisPtrs];
};

__global__ void __launch_bounds__(256) k_vis_union(FlagPtrs fp, int n, int64_t P, int accumulate,
                                                   uint8_t* __restrict__ visible) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < P; i += (int64_t)gridDim.x * blockDim.x) {
    uint32_t vis = accumulate ? visible[i] : 0u;
    for (int v = 0; v < n; ++v) vis |= (fp.p[v][i] & GS_FLAG_CULLED) ? 0u : 1u;
    visible[i] = (uint8_t)(vis ? 1u : 0u);
  }
}

constexpr int kCpThreads = 256, kCpItems = 16, kCpTile = kCpThreads * kCpItems;

// per tile of 4096 entries: the count of nonzero entries
__global__ void __launch_bounds__(kCpThreads) k_cp_count(const uint8_t* __restrict__ visible, int64_t P,
                                                         uint32_t* __restrict__ tile_cnt) {
  __shared__ uint32_t s_w[kCpThreads / 32];
  const int64_t base = (int64_t)blockIdx.x * kCpTile + (int64_t)threadIdx.x * kCpItems;
  uint32_t c = 0;
#pragma unroll
  for (int k = 0; k < kCpItems; ++k) c += (base + k < P && visible[base + k]) ? 1u : 0u;
  c = __reduce_add_sync(kFull, c);
  if ((threadIdx.x & 31) == 0) s_w[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t t = 0;
    for (int w = 0; w < kCpThreads / 32; ++w) t += s_w[w];
    tile_cnt[blockIdx.x] = t;
  }
}

// one CTA: exclusive scan of the tile counts in place; *count = total
__global__ void __launch_bounds__(1024) k_cp_scan(uint32_t* __restrict__ tile_cnt, int64_t ntiles,
                                                  long long* __restrict__ count) {
  __shared__ uint32_t s_w[32];
  __shared__ uint32_t s_carry;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) s_carry = 0;
  __syncthreads();
  for (int64_t b0 = 0; b0 < ntiles; b0 += 1024) {
    const int64_t i = b0 + threadIdx.x;
    const uint32_t v = i < ntiles ? tile_cnt[i] : 0u;
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(kFull, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) s_w[warp] = x;
    __syncthreads();
    uint32_t wpre = 0, tot = 0;
    for (int w = 0; w < 32; ++w) {
      const uint32_t t = s_w[w];
      wpre += (w < warp) ? t : 0u;
      tot += t;
    }
    const uint32_t carry = s_carry;
    if (i < ntiles) tile_cnt[i] = carry + wpre + x - v;
    __syncthreads();
    if (threadIdx.x == 0) s_carry = carry + tot;
    __syncthreads();
  }
  if (threadIdx.x == 0) *count = (long long)s_carry;
}

// per tile: ordered positions (block-local exclusive scan + the tile's offset)
__global__ void __launch_bounds__(kCpThreads) k_cp_write(const uint8_t* __restrict__ visible, int64_t P,
                                                         const uint32_t* __restrict__ tile_off,
                                                         int32_t* __restrict__ idx) {
  __shared__ uint32_t s_w[kCpThreads / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t base = (int64_t)blockIdx.x * kCpTile + (int64_t)threadIdx.x * kCpItems;
  uint32_t bits = 0;
#pragma unroll
  for (int k = 0; k < kCpItems; ++k) bits |= (base + k < P && visible[base + k]) ? (1u << k) : 0u;
  const uint32_t c = __popc(bits);
  uint32_t x = c;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(kFull, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_w[warp] = x;
  __syncthreads();
  uint32_t wpre = 0;
  for (int w = 0; w < warp; ++w) wpre += s_w[w];
  uint32_t pos = tile_off[blockIdx.x] + wpre + x - c;
#pragma unroll
  for (int k = 0; k < kCpItems; ++k)
    if (bits >> k & 1u) idx[pos++] = (int32_t)(base + k);
}

__global__ void __launch_bounds__(256) k_gather_cols(const float* __restrict__ full, int64_t F, int64_t S,
                                                     const int32_t* __restrict__ idx, int64_t M,
                                                     float* __restrict__ packed) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < M; j += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = idx[j];
    GSR_CHECK(c >= 0 && c < S);
    for (int64_t r = 0; r < F; ++r) packed[r * M + j] = full[r * S + c];
  }
}

__global__ void __launch_bounds__(256) k_scatter_cols(const float* __restrict__ packed, int64_t F, int64_t S,
                                                      const int32_t* __restrict__ idx, int64_t M,
                                                      float* __restrict__ full) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < M; j += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = idx[j];
    GSR_CHECK(c >= 0 && c < S);
    for (int64_t r = 0; r < F; ++r) full[r * S + c] = packed[r * M + j];
  }
}

int grid_for(int64_t n, int per_sm) {
  return (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, (int64_t)sm_count() * per_sm));
}

}  // namespace

size_t compact_workspace(int64_t P) { return (size_t)((P + kCpTile - 1) / kCpTile + 1) * 4; }

void launch_vis_union(int n_views, const uint8_t* const* flags, int64_t P, bool accumulate, uint8_t* visible,
                      cudaStream_t s) {
  if (n_views == 0) {
    cudaMemsetAsync(visible, 0, (size_t)P, s);
    return;
  }
  for (int v0 = 0; v0 < n_views; v0 += kVisPtrs) {
    FlagPtrs fp{};
    const int n = std::min(kVisPtrs, n_views - v0);
    for (int v = 0; v < n; ++v) fp.p[v] = flags[v0 + v];
    k_vis_union<<<grid_for(P, 8), 256, 0, s>>>(fp, n, P, (v0 > 0 || accumulate) ? 1 : 0, visible);
    count_launch();
  }
}

void launch_compact_index(const uint8_t* visible, int64_t P, uint32_t* tile_cnt, int32_t* idx, int64_t* count,
                          cudaStream_t s) {
  const int64_t ntiles = (P + kCpTile - 1) / kCpTile;
  if (ntiles > 0) {
    k_cp_count<<<(int)ntiles, kCpThreads, 0, s>>>(visible, P, tile_cnt);
    count_launch();
  }
  k_cp_scan<<<1, 1024, 0, s>>>(tile_cnt, ntiles, reinterpret_cast<long long*>(count));
  count_launch();
  if (ntiles > 0) {
    k_cp_write<<<(int)ntiles, kCpThreads, 0, s>>>(visible, P, tile_cnt, idx);
    count_launch();
  }
}

void launch_gather_cols(const float* full, int64_t F, int64_t S, const int32_t* idx, int64_t M, float* packed,
                        cudaStream_t s) {
  if (M <= 0 || F <= 0) return;
  k_gather_cols<<<grid_for(M, 8), 256, 0, s>>>(full, F, S, idx, M, packed);
  count_launch();
}

void launch_scatter_cols(const float* packed, int64_t F, int64_t S, const int32_t* idx, int64_t M, float* full,
                         cudaStream_t s) {
  if (M <= 0 || F <= 0) return;
  k_scatter_cols<<<grid_for(M, 8), 256, 0, s>>>(packed, F, S, idx, M, full);
  count_launch();
}

}  // namespace gsr
