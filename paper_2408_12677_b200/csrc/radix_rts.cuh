// Reduce-then-scan LSD radix pass (8-bit digit at `shift`): the alternative to the
// decoupled look-back (onesweep) pass in binning.cu, without inter-CTA waiting.
//   k_rs_hist    per-partition digit counts -> table[digit][partition]
//   k_rs_scan    one CTA per digit: exclusive scan over partitions + the digit's
//                global offset (from the histogram fused into the producing kernel)
//   k_rs_scatter stable in-partition ranking (warp __match_any_sync multisplit),
//                shared-memory staging in block-sorted order, per-digit coalesced writes
// Used when many partitions are in flight at once: measured on B200,
// a look-back pass over ~1400 partitions with ~450 resident CTAs spends most of its
// time walking predecessor chains in the first wave.
#pragma once

namespace gsr {
namespace rts {

constexpr int kThreads = 256, kWarps = kThreads / 32;

template <typename KeyT, int ITEMS>
__global__ void __launch_bounds__(kThreads) k_rs_hist(const KeyT* __restrict__ kin, const unsigned long long* n_ptr,
                                                     int64_t cap, int shift, uint32_t* __restrict__ table,
                                                     int64_t parts_max) {
  constexpr int TILE = kThreads * ITEMS;
  __shared__ uint32_t s_h[kWarps][256];
  int64_t n = (int64_t)*n_ptr;
  if (n > cap) n = 0;
  const int64_t part = blockIdx.x;
  if (part * TILE >= n) return;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  uint32_t lt;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(lt));
#pragma unroll
  for (int w = 0; w < kWarps; ++w) s_h[w][t] = 0;
  __syncthreads();
  const int64_t base = part * TILE + warp * (ITEMS * 32);
  uint32_t key[ITEMS];
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    const int64_t idx = base + i * 32 + lane;
    key[i] = idx < n ? (uint32_t)kin[idx] : 0u;
  }
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    const bool valid = base + i * 32 + lane < n;
    const uint32_t d = valid ? ((key[i] >> shift) & 255u) : (256u + lane);
    const uint32_t peers = digit_peers(d & 255u, valid);
    if (valid && (peers & lt) == 0) s_h[warp][d] += __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  uint32_t c = 0;
#pragma unroll
  for (int w = 0; w < kWarps; ++w) c += s_h[w][t];
  table[(int64_t)t * parts_max + part] = c;
}

// One CTA per digit.  ghist: global counts of this pass's digits (all keys).
__global__ void __launch_bounds__(kThreads) k_rs_scan(uint32_t* __restrict__ table, int64_t parts_max,
                                                     const unsigned long long* n_ptr, int64_t cap, int tile,
                                                     const uint32_t* __restrict__ ghist) {
  __shared__ uint32_t s_warp[kWarps];
  int64_t n = (int64_t)*n_ptr;
  if (n > cap) n = 0;
  const int64_t num_parts = (n + tile - 1) / tile;
  if (num_parts == 0) return;
  const int d = blockIdx.x, t = threadIdx.x, lane = t & 31, warp = t >> 5;
  // this digit's global offset: sum of the counts of the smaller digits
  uint32_t v = t < d ? ghist[t] : 0u;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if (lane == 0) s_warp[warp] = v;
  __syncthreads();
  uint32_t carry = 0;
#pragma unroll
  for (int w = 0; w < kWarps; ++w) carry += s_warp[w];
  __syncthreads();
  uint32_t* row = table + (int64_t)d * parts_max;
  constexpr int kItems = 8;
  for (int64_t c0 = 0; c0 < num_parts; c0 += kThreads * kItems) {
    uint32_t x[kItems];
    uint32_t sum = 0;
#pragma unroll
    for (int i = 0; i < kItems; ++i) {
      const int64_t p = c0 + t * kItems + i;
      x[i] = p < num_parts ? row[p] : 0u;
      sum += x[i];
    }
    // block exclusive scan of the per-thread sums
    uint32_t incl = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) s_warp[warp] = incl;
    __syncthreads();
    uint32_t wpre = 0, tot = 0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) {
      const uint32_t s = s_warp[w];
      wpre += w < warp ? s : 0u;
      tot += s;
    }
    __syncthreads();
    uint32_t run = carry + wpre + incl - sum;
#pragma unroll
    for (int i = 0; i < kItems; ++i) {
      const int64_t p = c0 + t * kItems + i;
      if (p < num_parts) row[p] = run;
      run += x[i];
    }
    carry += tot;
  }
}

template <typename KeyT, int ITEMS>
__global__ void __launch_bounds__(kThreads, 3) k_rs_scatter(const KeyT* __restrict__ kin,
                                                           const uint32_t* __restrict__ vin, KeyT* __restrict__ kout,
                                                           uint32_t* __restrict__ vout,
                                                           const unsigned long long* n_ptr, int64_t cap,
                                                           const uint32_t* __restrict__ table, int64_t parts_max,
                                                           int shift) {
  constexpr int TILE = kThreads * ITEMS;
  __shared__ uint32_t s_keys[TILE];
  __shared__ uint32_t s_vals[TILE];
  __shared__ uint32_t s_whist[kWarps][256];
  __shared__ uint32_t s_gbase[256], s_bexcl[256];
  __shared__ uint32_t s_warp[kWarps];
  int64_t n = (int64_t)*n_ptr;
  if (n > cap) n = 0;
  const int64_t part = blockIdx.x;
  if (part * TILE >= n) return;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  uint32_t lt;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(lt));
#pragma unroll
  for (int w = 0; w < kWarps; ++w) s_whist[w][t] = 0;
  s_gbase[t] = table[(int64_t)t * parts_max + part];
  __syncthreads();
  const int64_t base = part * TILE + warp * (ITEMS * 32);
  uint32_t key[ITEMS], rank[ITEMS];
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    const int64_t idx = base + i * 32 + lane;
    key[i] = idx < n ? (uint32_t)kin[idx] : 0u;
  }
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    const bool valid = base + i * 32 + lane < n;
    const uint32_t d = valid ? ((key[i] >> shift) & 255u) : (256u + lane);
    const uint32_t peers = digit_peers(d & 255u, valid);
    const uint32_t r = __popc(peers & lt);
    uint32_t b = 0;
    if (valid) b = s_whist[warp][d];
    __syncwarp();
    if (valid && r == 0) s_whist[warp][d] = b + __popc(peers);
    __syncwarp();
    rank[i] = valid ? (b + r) : 0xffffffffu;
  }
  __syncthreads();
  // per digit t: exclusive over warps, block count, block-local exclusive offset
  uint32_t cnt = 0;
#pragma unroll
  for (int w = 0; w < kWarps; ++w) {
    const uint32_t c = s_whist[w][t];
    s_whist[w][t] = cnt;
    cnt += c;
  }
  {
    uint32_t incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) s_warp[warp] = incl;
    __syncthreads();
    uint32_t wpre = 0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) wpre += w < warp ? s_warp[w] : 0u;
    s_bexcl[t] = wpre + incl - cnt;
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    if (rank[i] != 0xffffffffu) {
      const uint32_t d = (key[i] >> shift) & 255u;
      const uint32_t pos = s_bexcl[d] + s_whist[warp][d] + rank[i];
      s_keys[pos] = key[i];
      s_vals[pos] = vin[base + i * 32 + lane];
    }
  }
  __syncthreads();
  const int64_t rem = n - part * TILE;
  const int nv = (int)(rem < TILE ? rem : TILE);
  for (int j = t; j < nv; j += kThreads) {
    const uint32_t k = s_keys[j];
    const uint32_t d = (k >> shift) & 255u;
    const uint32_t dst = s_gbase[d] + (uint32_t)j - s_bexcl[d];
    kout[dst] = (KeyT)k;
    vout[dst] = s_vals[j];
  }
}

// One reduce-then-scan pass; table: >= 256 * parts_max uint32 of scratch.
template <typename KeyT, int ITEMS>
void radix_pass(const KeyT* kin, const uint32_t* vin, KeyT* kout, uint32_t* vout, const unsigned long long* n_ptr,
                int64_t cap, const uint32_t* ghist, uint32_t* table, int64_t parts_max, int shift, cudaStream_t s) {
  constexpr int TILE = kThreads * ITEMS;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((cap + TILE - 1) / TILE, parts_max));
  k_rs_hist<KeyT, ITEMS><<<grid, kThreads, 0, s>>>(kin, n_ptr, cap, shift, table, parts_max);
  k_rs_scan<<<256, kThreads, 0, s>>>(table, parts_max, n_ptr, cap, TILE, ghist);
  k_rs_scatter<KeyT, ITEMS><<<grid, kThreads, 0, s>>>(kin, vin, kout, vout, n_ptr, cap, table, parts_max, shift);
  count_launch(3);
}

}  // namespace rts
}  // namespace gsr
