// K2-K5: tile binning and per-tile depth ordering (readings R11, R12).
//
// Design: instead of sorting K duplicated 64-bit
// (tile << 32 | depth) keys (6 LSD passes over K), we
//   1. compact the visible Gaussians in index order (single-pass chained scan),
//   2. sort their fp32 depths (4 onesweep passes over V << K items; LSD radix is
//      stable, so equal depths keep index order = the R12 tie-break),
//   3. emit one 16-bit tile key per touched tile in depth order (offsets from a
//      second chained scan), and
//   4. stably sort those keys by tile id (1-2 onesweep passes, 8-bit digits).
// The result is exactly the (tile, depth, index) order of the oracle's sort, with
// ~32 B moved per key instead of ~150 B.  All counts stay on the device: grids are
// sized from host-known bounds (P, key capacity) and surplus CTAs exit, so the
// whole call is graph-capturable when num_keys_host == NULL.
//
// Onesweep pass (Merrill & Garland style, written from scratch): each CTA takes a
// 4096-key partition from an atomic counter, ranks digits per warp with
// __match_any_sync (stable: warp-striped items processed in order), publishes its
// per-digit counts, resolves its global offsets by decoupled look-back over the
// preceding partitions, stages keys in shared memory in block-sorted order and
// writes them out as per-digit coalesced runs.
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "gsr_internal.cuh"
#include "radix_rts.cuh"

namespace gsr {
namespace {

#ifndef GSR_SCAN_ITEMS
#define GSR_SCAN_ITEMS 8
#endif
constexpr int kScanThreads = 256, kScanItems = GSR_SCAN_ITEMS, kScanTile = kScanThreads * kScanItems;
constexpr int kRsThreads = 256, kRsWarps = kRsThreads / 32;
#ifndef GSR_EMIT_PER_SM
#define GSR_EMIT_PER_SM 4  // k_emit CTAs per SM (persistent, 2048 keys per iteration)
#endif
// Depth passes: 4 keys per thread (1024 per partition) for scenes below 512K
// Gaussians (one view per step, latency-bound: more partitions finish sooner), 16 (4096)
// above (views in flight: fewer, longer CTAs churn fewer SM slots against the render
// kernels; scannetpp 6.01 -> 5.96 ms/step): a P heuristic, depth_items_big().
constexpr int kRsItemsKeys = 16, kRsItemsDepth = 4, kRsItemsDepthBig = 16;  // items per thread
constexpr int kRsTileKeys = kRsThreads * kRsItemsKeys, kRsTileDepth = kRsThreads * kRsItemsDepth;
constexpr uint32_t kLbAgg = 1u << 30, kLbInc = 2u << 30, kLbMask = (1u << 30) - 1;
constexpr unsigned long long kScAgg = 1ull << 62, kScInc = 2ull << 62, kScMask = (1ull << 62) - 1;

struct Counters {
  uint32_t part[8];  // 0 compaction scan, 1 offset scan, 2-5 depth passes, 6-7 tile passes
  unsigned long long V, K;
  unsigned long long pad[4];
};

__device__ __forceinline__ unsigned long long ld_vol(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.volatile.global.u64 %0, [%1];" : "=l"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ void st_vol(unsigned long long* p, unsigned long long v) {
  asm volatile("st.volatile.global.u64 [%0], %1;" ::"l"(p), "l"(v));
}
__device__ __forceinline__ uint32_t ld_vol(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.volatile.global.u32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ void st_vol(uint32_t* p, uint32_t v) {
  asm volatile("st.volatile.global.u32 [%0], %1;" ::"l"(p), "r"(v));
}
__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// Exclusive scan over a 256-thread block; `total` receives the block sum.
template <typename T>
__device__ __forceinline__ T block_excl_scan256(T v, T* s_warp /*[8]*/, T& total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  T x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const T y = __shfl_up_sync(kFull, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_warp[warp] = x;
  __syncthreads();
  T wpre = 0;
  total = 0;
#pragma unroll
  for (int w = 0; w < 8; ++w) {
    const T t = s_warp[w];
    if (w < warp) wpre += t;
    total += t;
  }
  __syncthreads();
  return wpre + x - v;
}

// Decoupled look-back for the chained scans, run by one whole warp: publishes this
// partition's aggregate, then examines 32 predecessors per round trip (lane l reads
// partition part - 1 - l - 32 r), adds every aggregate up to and including the
// nearest inclusive prefix, and spins only while a needed predecessor has not
// published yet.  Returns the exclusive prefix (all lanes) and publishes the
// inclusive one.
__device__ __forceinline__ unsigned long long warp_lookback(unsigned long long* lookback, int64_t part,
                                                            unsigned long long total) {
  const int lane = threadIdx.x & 31;
  if (part == 0) {
    if (lane == 0) st_vol(&lookback[0], kScInc | total);
    return 0ull;
  }
  if (lane == 0) st_vol(&lookback[part], kScAgg | total);
  unsigned long long prefix = 0;
  int64_t p = part - 1;
  while (true) {
    const int64_t q = p - lane;
    const unsigned long long v = q >= 0 ? ld_vol(&lookback[q]) : kScInc;  // before partition 0: prefix 0
    const uint32_t inc = __ballot_sync(kFull, (v >> 62) == 2);
    const uint32_t ready = __ballot_sync(kFull, (v >> 62) != 0);
    const uint32_t need = inc ? ((inc & (0u - inc)) << 1) - 1u : kFull;  // lanes up to the nearest inclusive
    if ((ready & need) != need) continue;                                  // someone needed is not ready
    unsigned long long x = (lane < 32 && ((need >> lane) & 1u)) ? (v & kScMask) : 0ull;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(kFull, x, o);
    prefix += x;
    if (inc) break;
    p -= 32;
  }
  if (lane == 0) st_vol(&lookback[part], kScInc | (prefix + total));
  return prefix;
}

// ---------------------------------------------------------------------------
// K2a: order-preserving compaction of the visible set (tiles > 0), fused with the
// 4 x 256-bin histograms of the depth-key bytes for the depth sort.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kScanThreads) k_compact(int64_t P, const int32_t* __restrict__ tiles,
                                                          const float* __restrict__ rec, Counters* ctr,
                                                          unsigned long long* lookback, uint32_t* __restrict__ dkeys,
                                                          uint32_t* __restrict__ dvals, uint32_t* __restrict__ ghist) {
  __shared__ uint32_t s_part;
  __shared__ unsigned long long s_warp[8];
  __shared__ unsigned long long s_prefix;
  __shared__ uint32_t s_hist[4][256];
  for (int t = threadIdx.x; t < 4 * 256; t += kScanThreads) (&s_hist[0][0])[t] = 0;
  if (threadIdx.x == 0) s_part = atomicAdd(&ctr->part[0], 1u);
  __syncthreads();
  const uint32_t part = s_part;
  const int64_t num_parts = (P + kScanTile - 1) / kScanTile;
  const int64_t base = (int64_t)part * kScanTile + (int64_t)threadIdx.x * kScanItems;
  uint32_t flag = 0;
  unsigned long long cnt = 0;
  uint32_t zk[kScanItems];  // depth keys of the visible items, gathered before the scan so
                            // their latency overlaps the scan and the look-back
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    const int64_t i = base + k;
    const bool vis = i < P && tiles[i] > 0;
    flag |= (vis ? 1u : 0u) << k;
    cnt += vis;
    zk[k] = vis ? __float_as_uint(rec[12 * i + 2]) : 0u;  // z > z_near > 0: bits order = value order
  }
  unsigned long long total;
  const unsigned long long excl = block_excl_scan256<unsigned long long>(cnt, s_warp, total);
  if (threadIdx.x < 32) {
    const unsigned long long prefix = warp_lookback(lookback, part, total);
    if (threadIdx.x == 0) {
      s_prefix = prefix;
      if ((int64_t)part == num_parts - 1) ctr->V = prefix + total;
    }
  }
  __syncthreads();
  unsigned long long pos = s_prefix + excl;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    if (flag >> k & 1) {
      const int64_t i = base + k;
      const uint32_t key = zk[k];
      dkeys[pos] = key;
      dvals[pos] = (uint32_t)i;
      atomicAdd(&s_hist[0][key & 255], 1u);
      atomicAdd(&s_hist[1][(key >> 8) & 255], 1u);
      atomicAdd(&s_hist[2][(key >> 16) & 255], 1u);
      atomicAdd(&s_hist[3][key >> 24], 1u);
      ++pos;
    }
  }
  __syncthreads();
  for (int t = threadIdx.x; t < 4 * 256; t += kScanThreads) {
    const uint32_t c = (&s_hist[0][0])[t];
    if (c) atomicAdd(&ghist[t], c);
  }
}

// ---------------------------------------------------------------------------
// K2b: exclusive scan of tiles_touched in depth order -> key offsets, and K.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kScanThreads) k_offsets(const int32_t* __restrict__ tiles,
                                                          const uint32_t* __restrict__ sorted_gid, Counters* ctr,
                                                          unsigned long long* lookback, uint32_t* __restrict__ offs,
                                                          long long* num_keys_dev) {
  __shared__ uint32_t s_part;
  __shared__ unsigned long long s_warp[8];
  __shared__ unsigned long long s_prefix;
  const int64_t V = (int64_t)ctr->V;
  const int64_t num_parts = (V + kScanTile - 1) / kScanTile;
  if (threadIdx.x == 0) s_part = atomicAdd(&ctr->part[1], 1u);
  __syncthreads();
  const uint32_t part = s_part;
  if ((int64_t)part >= num_parts) return;
  const int64_t base = (int64_t)part * kScanTile + (int64_t)threadIdx.x * kScanItems;
  uint32_t c[kScanItems];
  unsigned long long sum = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    const int64_t s = base + k;
    c[k] = s < V ? (uint32_t)tiles[sorted_gid[s]] : 0u;
    sum += c[k];
  }
  unsigned long long total;
  const unsigned long long excl = block_excl_scan256<unsigned long long>(sum, s_warp, total);
  if (threadIdx.x < 32) {
    const unsigned long long prefix = warp_lookback(lookback, part, total);
    if (threadIdx.x == 0) {
      s_prefix = prefix;
      if ((int64_t)part == num_parts - 1) {
        ctr->K = prefix + total;
        if (num_keys_dev) *num_keys_dev = (long long)(prefix + total);
      }
    }
  }
  __syncthreads();
  unsigned long long run = s_prefix + excl;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    const int64_t s = base + k;
    if (s < V) offs[s] = (uint32_t)run;
    run += c[k];
  }
}

// ---------------------------------------------------------------------------
// K3: emit one 16-bit tile key per touched tile, in depth order, with a
// load-balanced (merge-path) expansion: CTA b owns output keys [2048 b, 2048 b +
// 2048), finds the Gaussians spanning them by a 32-ary search over the key
// offsets, stages their offsets / ids / rects in shared memory, and each thread
// writes 8 consecutive keys with 16-B vector stores.  Work per thread is constant
// whatever the footprint distribution (one Gaussian can touch > 6000 tiles).
// Fused: the 2 x 256-bin histograms of the tile-key bytes for the tile sort.
// ---------------------------------------------------------------------------
constexpr int kEmThreads = 256, kEmItems = 8, kEmTile = kEmThreads * kEmItems;

// largest s in [0, V) with offs[s] <= k (offs strictly increasing, offs[0] = 0)
__device__ __forceinline__ int64_t warp_search(const uint32_t* __restrict__ offs, int64_t V, uint32_t k, int lane) {
  int64_t lo = 0, hi = V;  // offs[lo] <= k < offs[hi] (offs[V] := +inf)
  while (hi - lo > 1) {
    const int64_t step = (hi - lo + 31) / 32;
    const int64_t p = lo + step * (lane + 1);
    const bool le = p < hi && offs[p] <= k;
    const int c = __popc(__ballot_sync(kFull, le));
    lo = lo + step * c;
    hi = min(hi, lo + step);
  }
  return lo;
}

// kHist: also the 2 x 256-bin tile-key histograms (needed by the radix tile passes only)
template <bool kHist>
__global__ void __launch_bounds__(kEmThreads) k_emit(const uint32_t* __restrict__ sorted_gid,
                                                     const uint32_t* __restrict__ offs, const float* __restrict__ rec,
                                                     int TX, const Counters* __restrict__ ctr, int64_t cap,
                                                     uint16_t* __restrict__ tkeys, uint32_t* __restrict__ tvals,
                                                     uint32_t* __restrict__ ghist /* [2][256] */) {
  __shared__ uint32_t s_off[kEmTile + 1];
  __shared__ uint32_t s_gid[kEmTile];
  __shared__ uint32_t s_rx[kEmTile], s_ry[kEmTile];
  __shared__ uint32_t s_hist[2][256];
  __shared__ int64_t s_lo[2];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  for (int i = t; i < 512; i += kEmThreads) (&s_hist[0][0])[i] = 0;
  const int64_t V = (int64_t)ctr->V, K = (int64_t)ctr->K;
  const int64_t nblk = K <= cap ? (K + kEmTile - 1) / kEmTile : 0;
  for (int64_t blk = blockIdx.x; blk < nblk; blk += gridDim.x) {
    const int64_t k0 = blk * kEmTile, k1 = min(K, k0 + kEmTile);
    if (warp < 2) {
      const int64_t s = warp_search(offs, V, (uint32_t)(warp == 0 ? k0 : k1 - 1), lane);
      if (lane == 0) s_lo[warp] = s;
    }
    __syncthreads();
    const int64_t slo = s_lo[0];
    const int ns = (int)(s_lo[1] - slo + 1);
    for (int j = t; j < ns; j += kEmThreads) {
      const uint32_t g = sorted_gid[slo + j];
      s_off[j] = offs[slo + j];
      s_gid[j] = g;
      const uint2 r = *reinterpret_cast<const uint2*>(rec + 12 * (int64_t)g + 10);
      s_rx[j] = r.x;
      s_ry[j] = r.y;
    }
    if (t == 0) s_off[ns] = (slo + ns < V) ? offs[slo + ns] : (uint32_t)K;
    __syncthreads();
    const int64_t kb = k0 + (int64_t)t * kEmItems;
    if (kb < k1) {
      // locate the Gaussian of key kb in the staged offsets
      int lo = 0, hi = ns;
      while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (s_off[mid] <= (uint32_t)kb) lo = mid; else hi = mid;
      }
      int j = lo;
      uint32_t next = s_off[j + 1];
      int x0 = s_rx[j] & 0xffff, w = (int)(s_rx[j] >> 16) - x0, y0 = s_ry[j] & 0xffff;
      int local = (int)(kb - s_off[j]);
      int row = local / w, col = local - row * w;
      uint32_t gid = s_gid[j];
      uint16_t kk[kEmItems];
      uint32_t vv[kEmItems];
      uint32_t hb_run = 0xffffffffu, hb_cnt = 0;
      const int nk = (int)((k1 - kb) < kEmItems ? (k1 - kb) : kEmItems);
#pragma unroll
      for (int q = 0; q < kEmItems; ++q) {
        if (q < nk) {
          if ((uint32_t)(kb + q) >= next) {
            ++j;
            GSR_CHECK(j < ns);
            next = s_off[j + 1];
            x0 = s_rx[j] & 0xffff, w = (int)(s_rx[j] >> 16) - x0, y0 = s_ry[j] & 0xffff;
            gid = s_gid[j];
            row = 0, col = 0;
          }
          const uint32_t tile = (uint32_t)((y0 + row) * TX + x0 + col);
          GSR_CHECK(w > 0 && col < w && x0 + col < TX && tile < 65536u && (int64_t)(kb + q) < cap);
          kk[q] = (uint16_t)tile;
          vv[q] = gid;
          if (kHist) {
            atomicAdd(&s_hist[0][tile & 255], 1u);
            const uint32_t hb = tile >> 8;
            if (hb != hb_run) {
              if (kHist && hb_cnt) atomicAdd(&s_hist[1][hb_run], hb_cnt);
              hb_run = hb, hb_cnt = 0;
            }
            ++hb_cnt;
          }
          if (++col == w) col = 0, ++row;
        }
      }
      if (kHist && hb_cnt) atomicAdd(&s_hist[1][hb_run], hb_cnt);
      if (nk == kEmItems) {
        uint4 k4;
        k4.x = kk[0] | ((uint32_t)kk[1] << 16);
        k4.y = kk[2] | ((uint32_t)kk[3] << 16);
        k4.z = kk[4] | ((uint32_t)kk[5] << 16);
        k4.w = kk[6] | ((uint32_t)kk[7] << 16);
        *reinterpret_cast<uint4*>(tkeys + kb) = k4;
        reinterpret_cast<uint4*>(tvals + kb)[0] = make_uint4(vv[0], vv[1], vv[2], vv[3]);
        reinterpret_cast<uint4*>(tvals + kb)[1] = make_uint4(vv[4], vv[5], vv[6], vv[7]);
      } else {
#pragma unroll
        for (int q = 0; q < kEmItems; ++q)
          if (q < nk) tkeys[kb + q] = kk[q], tvals[kb + q] = vv[q];
      }
    }
    __syncthreads();
  }
  if (kHist) {
    __syncthreads();
    for (int i = t; i < 512; i += kEmThreads) {
      const uint32_t c = (&s_hist[0][0])[i];
      if (c) atomicAdd(&ghist[i], c);
    }
  }
}

// ---------------------------------------------------------------------------
// K4: one onesweep LSD pass (8-bit digit at `shift`) over n = *n_ptr items
// (n := 0 if n > cap).  Persistent CTAs pull 4096-item partitions in order.
// ---------------------------------------------------------------------------
#ifndef GSR_LB_WIN
#define GSR_LB_WIN 16
#endif
constexpr int kLbWin = GSR_LB_WIN;
template <typename KeyT, int ITEMS>
__global__ void __launch_bounds__(kRsThreads, 3) k_onesweep(const KeyT* __restrict__ kin, const uint32_t* __restrict__ vin,
                                                            KeyT* __restrict__ kout, uint32_t* __restrict__ vout,
                                                            const unsigned long long* n_ptr, int64_t cap,
                                                            const uint32_t* __restrict__ ghist, uint32_t* lookback,
                                                            uint32_t* part_ctr, int shift) {
  constexpr int TILE = kRsThreads * ITEMS;
  __shared__ uint32_t s_keys[TILE];
  __shared__ uint32_t s_vals[TILE];
  __shared__ uint32_t s_whist[kRsWarps][256];
  __shared__ uint32_t s_gpref[256], s_gbase[256], s_bexcl[256];
  __shared__ uint32_t s_scan[8];
  __shared__ uint32_t s_part;
  int64_t n = (int64_t)*n_ptr;
  if (n > cap) n = 0;
  const int64_t num_parts = (n + TILE - 1) / TILE;
  // CTAs past the partition count (the grid is sized from P, the pass sorts V <= P
  // items) leave before touching anything: ids are claimed in order, so the first
  // num_parts CTAs take them all
  if ((int64_t)blockIdx.x >= num_parts) return;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const uint32_t g_t = ghist[t];  // in flight with the claim and the key loads
  bool first = true;
  const uint32_t lt = lanemask_lt();
  for (;;) {
    if (t == 0) s_part = atomicAdd(part_ctr, 1u);
#pragma unroll
    for (int w = 0; w < kRsWarps; ++w) s_whist[w][t] = 0;
    __syncthreads();
    const uint32_t part = s_part;
    if ((int64_t)part >= num_parts) break;
    const int64_t base = (int64_t)part * TILE + warp * (ITEMS * 32);
    uint32_t key[ITEMS], rank[ITEMS], val[ITEMS];
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {  // values with the keys: no load after the look-back
      const int64_t idx = base + i * 32 + lane;
      key[i] = idx < n ? (uint32_t)kin[idx] : 0u;
      val[i] = idx < n ? vin[idx] : 0u;
    }
    if (first) {  // global digit offsets (exclusive scan of the pass histogram)
      uint32_t tot;
      s_gpref[t] = block_excl_scan256<uint32_t>(g_t, s_scan, tot);
      first = false;
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
    // per digit t: exclusive over warps and the partition count; publish it early
    uint32_t cnt = 0;
#pragma unroll
    for (int w = 0; w < kRsWarps; ++w) {
      const uint32_t c = s_whist[w][t];
      s_whist[w][t] = cnt;
      cnt += c;
    }
    uint32_t* lb = lookback + (int64_t)part * 256 + t;
    st_vol(lb, (part == 0 ? kLbInc : kLbAgg) | cnt);
    uint32_t tot;
    s_bexcl[t] = block_excl_scan256<uint32_t>(cnt, s_scan, tot);
    // decoupled look-back over a window of kLbWin predecessors per round trip (the
    // partitions publish their aggregates at about the same time, so a wide window
    // cuts the round trips of the last partition from ~parts/4 to ~parts/16)
    uint32_t excl = 0;
    for (int64_t p = (int64_t)part - 1; p >= 0;) {
      uint32_t v[kLbWin];
#pragma unroll
      for (int k = 0; k < kLbWin; ++k) v[k] = (p - k >= 0) ? ld_vol(lookback + (p - k) * 256 + t) : kLbInc;
      int k = 0;
      bool done = false;
#pragma unroll
      for (; k < kLbWin; ++k) {
        const uint32_t f = v[k] >> 30;
        if (f == 0) break;
        excl += v[k] & kLbMask;
        if (f == 2) {
          done = true;
          break;
        }
      }
      if (done) break;
      p -= k;
    }
    if (part != 0) st_vol(lb, kLbInc | (excl + cnt));
    s_gbase[t] = s_gpref[t] + excl;
    __syncthreads();
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
      if (rank[i] != 0xffffffffu) {
        const uint32_t d = (key[i] >> shift) & 255u;
        const uint32_t pos = s_bexcl[d] + s_whist[warp][d] + rank[i];
        s_keys[pos] = key[i];
        s_vals[pos] = val[i];
      }
    }
    __syncthreads();
    const int64_t rem = n - (int64_t)part * TILE;
    const int nv = (int)(rem < TILE ? rem : TILE);
    for (int j = t; j < nv; j += kRsThreads) {
      const uint32_t k = s_keys[j];
      const uint32_t d = (k >> shift) & 255u;
      const uint32_t dst = s_gbase[d] + (uint32_t)j - s_bexcl[d];
      kout[dst] = (KeyT)k;
      vout[dst] = s_vals[j];
    }
    __syncthreads();
  }
}

// K5: [start, end) of every tile from the sorted tile keys.
__global__ void k_ranges(const uint16_t* __restrict__ skeys, const Counters* __restrict__ ctr, int64_t cap,
                         int2* __restrict__ ranges) {
  int64_t n = (int64_t)ctr->K;
  if (n > cap) return;
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t t = skeys[k];
    if (k == 0 || skeys[k - 1] != t) ranges[t].x = (int)k;
    if (k == n - 1 || skeys[k + 1] != t) ranges[t].y = (int)(k + 1);
  }
}

// ---------------------------------------------------------------------------
// K4' (default when the per-tile counters fit in shared memory): stable bucket
// placement of the depth-ordered tile keys by tile id, replacing the two 8-bit radix
// passes.  The K keys are cut into C equal chunks (one CTA each, 8 warps, each warp
// a contiguous sub-chunk):
//   k_tcount:   per chunk and tile, the key count           -> chist[c][t]
//   k_tscan:    per tile, exclusive prefix over the chunks plus the tile's start (the
//               tile totals chained by look-back)  -> chist[c][t], tile_ranges
//   k_tscatter: per chunk: per-warp tile counts, their prefix over the
//               warps, then each warp walks its keys in order and places key k of
//               tile t at  start(t) + chist[c][t] + (warp prefix) + (earlier keys of
//               t in this warp), ranking equal tiles within 32 keys by bit-sliced
//               ballots.  Keys of a tile thus keep their depth order: the output is
//               the same stable sort, in ~3 passes of 2-6 B/key and no look-back.
// ---------------------------------------------------------------------------
constexpr int kBkThreads = 256, kBkWarps = kBkThreads / 32;
// k_tscatter runs W = 8 warps (sub-chunks) per chunk (GSR_TSC_WARPS=4: 4, A/B only).
constexpr int kBkMaxChunks = 512;  // chist capacity (workspace); C = min(this, SMs x CTAs/SM)

constexpr int kBkBatch = 256;  // keys per staged batch of a warp (32 lanes x 8 keys)
// Chunk c = keys [c chunk, (c + 1) chunk), cut into 8 warp sub-chunks; chunk and
// sub-chunk sizes are multiples of kBkBatch, so every sub-chunk starts 16-B aligned in
// the key (u16) and value (u32) arrays (vector loads, cp.async staging).
__device__ __forceinline__ void chunk_bounds(int64_t K, int C, int W, int c, int w, int64_t& a, int64_t& b) {
  const int64_t q = (int64_t)W * kBkBatch;
  const int64_t chunk = ((K + C - 1) / C + q - 1) / q * q;
  const int64_t k0 = min(K, (int64_t)c * chunk), k1 = min(K, k0 + chunk);
  const int64_t sub = chunk / W;
  a = min(k1, k0 + (int64_t)w * sub);
  b = min(k1, a + sub);
}

// Count the tile keys [a, b) (a % 8 == 0) into packed 16-bit (pk16) or 32-bit counters:
// one 16-B load (8 keys) per thread and step; key 0xffff marks past-the-end.
template <bool kPk16>
__device__ __forceinline__ void count_keys(const uint16_t* __restrict__ tkeys, int64_t a, int64_t b, int tid,
                                           int nthreads, uint32_t* cnt) {
  constexpr int U = 4;  // 16-B loads in flight per thread
  for (int64_t kb = a + 8 * (int64_t)tid; kb < b; kb += 8 * (int64_t)nthreads * U) {
    uint4 q[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t k = kb + 8 * (int64_t)nthreads * u;
      q[u] = k < b ? *reinterpret_cast<const uint4*>(tkeys + k) : make_uint4(~0u, ~0u, ~0u, ~0u);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t k = kb + 8 * (int64_t)nthreads * u;
      const uint32_t w[4] = {q[u].x, q[u].y, q[u].z, q[u].w};
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const uint32_t t = (w[e >> 1] >> (16 * (e & 1))) & 0xffffu;
        if (k + e < b) {
          if (kPk16)
            atomicAdd(cnt + (t >> 1), 1u << (16 * (t & 1)));
          else
            atomicAdd(cnt + t, 1u);
        }
      }
    }
  }
}

__device__ __forceinline__ void cp_async16_bin(void* smem, const void* gmem) {
  const uint32_t sa = (uint32_t)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gmem) : "memory");
}

// k_tcount runs 32 warps per CTA (one CTA per chunk): 4x the loads in flight of an
// 8-warp CTA (12 -> 7.5 us per scannetpp view).
constexpr int kTcThreads = 1024;

__global__ void __launch_bounds__(kTcThreads) k_tcount(const uint16_t* __restrict__ tkeys,
                                                       const Counters* __restrict__ ctr, int64_t cap, int NT, int C,
                                                       int W, uint32_t* __restrict__ chist) {
  extern __shared__ uint32_t s_cnt[];  // [NT]
  for (int t = threadIdx.x; t < NT; t += kTcThreads) s_cnt[t] = 0;
  __syncthreads();
  int64_t K = (int64_t)ctr->K;
  if (K > cap) K = 0;
  int64_t a, b;
  chunk_bounds(K, C, W, blockIdx.x, 0, a, b);
  const int64_t k0 = a;
  chunk_bounds(K, C, W, blockIdx.x, W - 1, a, b);
  const int64_t k1 = b;
  count_keys<false>(tkeys, k0, k1, threadIdx.x, kTcThreads, s_cnt);
  __syncthreads();
  uint32_t* out = chist + (int64_t)blockIdx.x * ((NT + 3) & ~3);  // rows padded to 16 B
  for (int t = threadIdx.x; t < NT; t += kTcThreads) out[t] = s_cnt[t];
}

// CTA = 32 tiles x 8 warps; warp w scans chunks [w Cw, (w+1) Cw) of its lane's tile.
// The CTAs take their 32 tiles in launch order (partition counter) and chain the tile
// totals by decoupled look-back, so every chist[c][t] leaves as the global position of
// chunk c's first key of tile t (tile start + keys of t in earlier chunks), and
// tile_ranges are written here once.
__global__ void __launch_bounds__(kBkThreads) k_tscan(uint32_t* __restrict__ chist, int NT, int C,
                                                      Counters* __restrict__ ctr,
                                                      unsigned long long* __restrict__ lookback,
                                                      int2* __restrict__ ranges) {
  __shared__ uint32_t s_part[kBkWarps][32];
  __shared__ uint32_t s_blk;
  __shared__ unsigned long long s_prefix;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) s_blk = atomicAdd(&ctr->part[6], 1u);
  __syncthreads();
  const int blk = (int)s_blk;
  const int t = blk * 32 + lane;
  const int NS = (NT + 3) & ~3;  // chist row stride
  const int Cw = (C + kBkWarps - 1) / kBkWarps;
  const int c0 = min(C, warp * Cw), c1 = min(C, c0 + Cw);
  uint32_t s = 0;
  if (t < NT)
    for (int c = c0; c < c1; ++c) s += chist[(int64_t)c * NS + t];
  s_part[warp][lane] = s;
  __syncthreads();
  uint32_t run = 0, all = 0;
#pragma unroll
  for (int w = 0; w < kBkWarps; ++w) {
    const uint32_t v = s_part[w][lane];
    run += (w < warp) ? v : 0u;
    all += v;
  }
  // tile starts: exclusive scan of the 32 tile totals, plus the preceding CTAs' keys
  uint32_t incl = all;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(kFull, incl, o);
    if (lane >= o) incl += y;
  }
  if (warp == 0) {
    const unsigned long long pre = warp_lookback(lookback, blk, (unsigned long long)__shfl_sync(kFull, incl, 31));
    if (lane == 0) s_prefix = pre;
  }
  __syncthreads();
  const uint32_t start = (uint32_t)s_prefix + incl - all;
  if (t < NT) {
    run += start;
    for (int c = c0; c < c1; ++c) {
      uint32_t* p = chist + (int64_t)c * NS + t;
      const uint32_t v = *p;
      *p = run;
      run += v;
    }
    if (warp == 0) ranges[t] = make_int2((int)start, (int)(start + all));
  }
}

// Lanes of the warp holding the same tile id (bits: id width); invalid lanes match nobody.
__device__ __forceinline__ uint32_t tile_peers(uint32_t t, bool valid, int bits) {
  uint32_t peers = __ballot_sync(kFull, valid);
  for (int b = 0; b < bits; ++b) {
    const uint32_t m = __ballot_sync(kFull, (t >> b) & 1u);
    peers &= ((t >> b) & 1u) ? m : ~m;
  }
  return peers;
}

template <int kTsWarps>
__global__ void __launch_bounds__(32 * kTsWarps) k_tscatter(const uint16_t* __restrict__ tkeys,
                                                         const uint32_t* __restrict__ tvals,
                                                         const Counters* __restrict__ ctr, int64_t cap, int NT, int C,
                                                         int tile_bits, const uint32_t* __restrict__ chist,
                                                         int32_t* __restrict__ out, int own_bits) {
  extern __shared__ __align__(16) uint32_t s_dyn[];
  // dynamic layout (tscatter_layout): s_base [NT] u32 | s_w [8][NTp] u16 | stage [8][2] x
  // (256 u16 keys, 256 u32 values) | own [8][2^own_bits] u8
  // tables carry 32 dummy tiles NT + lane for the lanes past the end of the last group
  // (branch-free fast path; their counters are never read back)
  uint32_t* s_base = s_dyn;                                // [NT + 32] global position of this chunk's first key of t
  const int NTx = NT + 32;
  const int NTp = (NTx + 1) & ~1;                          // even row stride: 4-B aligned rows
  const size_t off_w = ((size_t)NTx * 4 + 15) & ~size_t(15);
  const size_t off_stage = (off_w + (size_t)NTp * kTsWarps * 2 + 15) & ~size_t(15);
  const size_t off_own = off_stage + (size_t)kTsWarps * 2 * kBkBatch * 6;
  char* s_bytes = reinterpret_cast<char*>(s_dyn);
  uint16_t* s_w = reinterpret_cast<uint16_t*>(s_bytes + off_w);  // [8][NTp] per-warp count, then running offset
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int64_t K = (int64_t)ctr->K;
  if (K > cap) return;  // chist is all zero then: tile_ranges (k_tscan) are empty
  // this chunk's row of global positions (k_tscan) -> s_base: all 16-B pieces in flight
  // at once (cp.async) instead of one L2 round trip per loop iteration
  const uint32_t* ch = chist + (int64_t)blockIdx.x * ((NT + 3) & ~3);
  for (int i = threadIdx.x; i < (NT + 3) / 4; i += (32 * kTsWarps)) cp_async16_bin(s_base + 4 * i, ch + 4 * i);
  asm volatile("cp.async.commit_group;" ::: "memory");
  for (int i = threadIdx.x; i < NTp * kTsWarps / 2; i += (32 * kTsWarps)) reinterpret_cast<uint32_t*>(s_w)[i] = 0;
  int64_t a, b;
  chunk_bounds(K, C, kTsWarps, blockIdx.x, warp, a, b);
  uint16_t* my = s_w + (int64_t)warp * NTp;
  // per-warp tile -> lane arbitration slots (hashed by the low own_bits of the tile id)
  uint8_t* own = reinterpret_cast<uint8_t*>(s_bytes + off_own) + ((int64_t)warp << own_bits);
  const uint32_t omask = (1u << own_bits) - 1u;
  uint16_t* stk = reinterpret_cast<uint16_t*>(s_bytes + off_stage + (size_t)warp * 2 * kBkBatch * 6);  // [2][256]
  uint32_t* stv = reinterpret_cast<uint32_t*>(stk + 2 * kBkBatch);                                     // [2][256]
  // stage batch [kb, kb + 256) of this warp's keys and values into buffer sb (cp.async;
  // a 16-B piece starting past b is skipped, the keys past b are masked when read)
  auto stage = [&](int64_t kb, int sb) {
    const int64_t k = kb + 8 * lane;
    if (k < b) {
      cp_async16_bin(stk + sb * kBkBatch + 8 * lane, tkeys + k);
      cp_async16_bin(stv + sb * kBkBatch + 8 * lane, tvals + k);
      cp_async16_bin(stv + sb * kBkBatch + 8 * lane + 4, tvals + k + 4);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  __syncthreads();          // s_w zeroed, s_base loaded
  if (a < b) stage(a, 0);   // in flight during the counting pass
  // per-warp counts: packed 16-bit increments on 32-bit words (a chunk has < 2^16 keys)
  count_keys<true>(tkeys, a, b, lane, 32, reinterpret_cast<uint32_t*>(my));
  __syncthreads();
  for (int t = threadIdx.x; t < NT; t += (32 * kTsWarps)) {
    uint32_t run = 0;
#pragma unroll
    for (int w = 0; w < kTsWarps; ++w) {
      const uint32_t v = s_w[w * NTp + t];
      s_w[w * NTp + t] = (uint16_t)run;
      run += v;
    }
  }
  __syncthreads();
  const uint32_t lt = lanemask_lt();
  int sb = 0;
  for (int64_t kb = a; kb < b; kb += kBkBatch, sb ^= 1) {
    if (kb + kBkBatch < b) stage(kb + kBkBatch, sb ^ 1);  // next batch in flight
    else asm volatile("cp.async.commit_group;" ::: "memory");
    asm volatile("cp.async.wait_group 1;" ::: "memory");
    __syncwarp();
    const int rem = (int)min((int64_t)kBkBatch, b - kb);  // keys of this batch
#pragma unroll
    for (int g = 0; g < kBkBatch / 32; ++g) {
      if (32 * g >= rem) break;  // warp-uniform
      const bool valid = 32 * g + lane < rem;
      const uint32_t t = valid ? (uint32_t)stk[sb * kBkBatch + 32 * g + lane] : (uint32_t)NT + lane;
      const uint32_t id = stv[sb * kBkBatch + 32 * g + lane];
      // Fast path: every lane writes its lane id into its tile's slot; if every lane
      // reads its own id back, the group's tiles are distinct (rank 0, count 1 each) --
      // the common case, since a group spans ~2 Gaussians whose keys are distinct tiles.
      // Otherwise (a repeated tile or a hash collision) the exact ballot ranking below.
      own[t & omask] = (uint8_t)lane;
      __syncwarp();
      if (__all_sync(kFull, own[t & omask] == (uint8_t)lane)) {
        const uint32_t run = my[t];
        my[t] = (uint16_t)(run + 1u);
        GSR_CHECK(!valid || (t < (uint32_t)NT && (int64_t)s_base[t] + run < K));
        if (valid) out[s_base[t] + run] = (int32_t)id;
        continue;
      }
      const uint32_t peers = tile_peers(t, valid, tile_bits);
      const uint32_t r = __popc(peers & lt);
      uint32_t run = 0;
      if (valid) run = my[t];
      __syncwarp();
      if (valid && r == 0) my[t] = (uint16_t)(run + __popc(peers));
      __syncwarp();
      GSR_CHECK(!valid || (t < (uint32_t)NT && (int64_t)s_base[t] + run + r < K));
      if (valid) out[s_base[t] + run + r] = (int32_t)id;
    }
    __syncwarp();  // buffer sb is restaged two batches from now
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
}

// Shared memory of k_tscatter for NT tiles; bucket placement is used when it fits.
constexpr size_t kSmemOptIn = 227 * 1024 - 1024;  // dynamic opt-in (static smem of the kernels < 1 KB)
size_t tscatter_smem_base(int NT, int W) {
  const size_t off_w = ((size_t)(NT + 32) * 4 + 15) & ~size_t(15);
  const size_t off_stage = (off_w + (size_t)((NT + 33) & ~1) * W * 2 + 15) & ~size_t(15);
  return off_stage + (size_t)W * 2 * kBkBatch * 6;
}
// arbitration slots per warp: 2^own_bits, the most (<= 4096) that still fit (0: none fit)
int tscatter_own_bits(int NT, int W) {
  int bits = 12;
  while (bits >= 10 && tscatter_smem_base(NT, W) + ((size_t)W << bits) > kSmemOptIn) --bits;
  return bits >= 10 ? bits : 0;
}
size_t tscatter_smem(int NT, int W) { return tscatter_smem_base(NT, W) + ((size_t)W << tscatter_own_bits(NT, W)); }
// warps per tscatter CTA: 8 if it fits with >= 1024 slots per warp, else 0 (radix tile
// passes).  GSR_TSC_WARPS=4 forces 4 warps where they fit -- measured slower than 8
// (scannetpp) and than the radix passes (config 4: bin 340 vs 288 us/view).
int tscatter_warps(int NT) {
  const char* e = std::getenv("GSR_TSC_WARPS");
  if (e && std::strcmp(e, "4") == 0) return tscatter_own_bits(NT, 4) ? 4 : 0;
  return tscatter_own_bits(NT, 8) ? 8 : 0;
}

// ---------------------------------------------------------------------------
// K4'' (GSR_TILE_SORT=lsd; measured slower, kept for A/B): the stable tile placement as two LSD passes over the bytes of the
// 16-bit tile id (low byte, then high byte; one pass if NT <= 256), each pass three
// short, light kernels with no look-back chain and no persistent CTAs, so that they
// interleave with the render kernels of the views in flight instead of holding whole
// SMs (k_tscatter's 218 KB of shared memory, the onesweep passes' register file):
//   k_dcount:   per chunk of kDcTile keys, the 256-bin histogram of the pass's byte,
//               stored bin-major: dch[b][c]
//   k_dscan:    one CTA per bin: exclusive scan of dch[b][.] over the chunks (in
//               place) and the bin's total -> dtot[b]
//   k_dscatter: per chunk: stable warp-multisplit ranks (the chunk's keys in order),
//               block-sorted staging in shared memory, and coalesced per-bin runs to
//               start(b) + dch[b][c] + (rank within the chunk), start(b) = exclusive
//               scan of dtot, recomputed by every CTA (256 values).
// Keys enter in depth order; each pass is stable, so the output is the (tile, depth,
// index) order (R12), bit-identical to the other placements.
// ---------------------------------------------------------------------------
constexpr int kDcItems = 8, kDcTile = kRsThreads * kDcItems;  // 2048 keys per chunk

__global__ void __launch_bounds__(kRsThreads) k_dcount(const uint16_t* __restrict__ keys,
                                                       const Counters* __restrict__ ctr, int64_t cap, int shift,
                                                       int64_t cstride, uint32_t* __restrict__ dch) {
  __shared__ uint32_t s_h[256];
  int64_t K = (int64_t)ctr->K;
  if (K > cap) K = 0;
  const int64_t k0 = (int64_t)blockIdx.x * kDcTile;
  if (k0 >= K) return;
  const int t = threadIdx.x;
  s_h[t] = 0;
  __syncthreads();
  const int64_t kb = k0 + 8 * (int64_t)t;  // 8 keys (16 B) per thread
  if (kb < K) {
    if (kb + 8 <= K) {
      const uint4 q = *reinterpret_cast<const uint4*>(keys + kb);
      const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
      for (int e = 0; e < 8; ++e) atomicAdd(&s_h[(((w[e >> 1] >> (16 * (e & 1))) & 0xffffu) >> shift) & 255u], 1u);
    } else {
      for (int64_t k = kb; k < K; ++k) atomicAdd(&s_h[(keys[k] >> shift) & 255u], 1u);
    }
  }
  __syncthreads();
  dch[(int64_t)t * cstride + blockIdx.x] = s_h[t];
}

__global__ void __launch_bounds__(kRsThreads) k_dscan(const Counters* __restrict__ ctr, int64_t cap, int64_t cstride,
                                                      uint32_t* __restrict__ dch, uint32_t* __restrict__ dtot) {
  __shared__ uint32_t s_scan[8];
  int64_t K = (int64_t)ctr->K;
  if (K > cap) K = 0;
  const int64_t C = (K + kDcTile - 1) / kDcTile;
  uint32_t* row = dch + (int64_t)blockIdx.x * cstride;
  uint32_t carry = 0;
  for (int64_t c0 = 0; c0 < C; c0 += kRsThreads * 4) {
    uint32_t v[4], sum = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int64_t c = c0 + 4 * (int64_t)threadIdx.x + i;
      v[i] = c < C ? row[c] : 0u;
      sum += v[i];
    }
    uint32_t tot;
    uint32_t run = carry + block_excl_scan256<uint32_t>(sum, s_scan, tot);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int64_t c = c0 + 4 * (int64_t)threadIdx.x + i;
      if (c < C) row[c] = run;
      run += v[i];
    }
    carry += tot;
  }
  if (threadIdx.x == 0) dtot[blockIdx.x] = carry;
}

template <typename KeyOutT>
__global__ void __launch_bounds__(kRsThreads) k_dscatter(const uint16_t* __restrict__ kin,
                                                         const uint32_t* __restrict__ vin,
                                                         KeyOutT* __restrict__ kout, uint32_t* __restrict__ vout,
                                                         const Counters* __restrict__ ctr, int64_t cap, int shift,
                                                         int64_t cstride, const uint32_t* __restrict__ dch,
                                                         const uint32_t* __restrict__ dtot) {
  __shared__ uint16_t s_keys[kDcTile];
  __shared__ uint32_t s_vals[kDcTile];
  __shared__ uint32_t s_whist[kRsWarps][256];
  __shared__ uint32_t s_gbase[256], s_bexcl[256];
  __shared__ uint32_t s_scan[8];
  int64_t K = (int64_t)ctr->K;
  if (K > cap) K = 0;
  const int64_t k0 = (int64_t)blockIdx.x * kDcTile;
  if (k0 >= K) return;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
#pragma unroll
  for (int w = 0; w < kRsWarps; ++w) s_whist[w][t] = 0;
  {
    uint32_t tot;  // bin starts: exclusive scan of the bin totals, plus this chunk's offset
    s_gbase[t] = block_excl_scan256<uint32_t>(dtot[t], s_scan, tot) + dch[(int64_t)t * cstride + blockIdx.x];
  }
  const int64_t base = k0 + warp * (kDcItems * 32);  // this warp's sub-chunk, keys in order
  uint32_t key[kDcItems], rank[kDcItems];
  const uint32_t lt = lanemask_lt();
#pragma unroll
  for (int i = 0; i < kDcItems; ++i) {
    const int64_t idx = base + i * 32 + lane;
    key[i] = idx < K ? (uint32_t)kin[idx] : 0u;
  }
  __syncthreads();  // s_whist zeroed
#pragma unroll
  for (int i = 0; i < kDcItems; ++i) {
    const bool valid = base + i * 32 + lane < K;
    const uint32_t d = (key[i] >> shift) & 255u;
    const uint32_t peers = digit_peers(d, valid);
    const uint32_t r = __popc(peers & lt);
    uint32_t b = 0;
    if (valid) b = s_whist[warp][d];
    __syncwarp();
    if (valid && r == 0) s_whist[warp][d] = b + __popc(peers);
    __syncwarp();
    rank[i] = valid ? (b + r) : 0xffffffffu;
  }
  __syncthreads();
  uint32_t cnt = 0;  // per digit t: exclusive over the warps, then over the digits
#pragma unroll
  for (int w = 0; w < kRsWarps; ++w) {
    const uint32_t c = s_whist[w][t];
    s_whist[w][t] = cnt;
    cnt += c;
  }
  {
    uint32_t tot;
    s_bexcl[t] = block_excl_scan256<uint32_t>(cnt, s_scan, tot);
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < kDcItems; ++i) {
    if (rank[i] != 0xffffffffu) {
      const uint32_t d = (key[i] >> shift) & 255u;
      const uint32_t pos = s_bexcl[d] + s_whist[warp][d] + rank[i];
      s_keys[pos] = (uint16_t)key[i];
      s_vals[pos] = vin[base + i * 32 + lane];
    }
  }
  __syncthreads();
  const int64_t rem = K - k0;
  const int nv = (int)(rem < kDcTile ? rem : kDcTile);
  for (int j = t; j < nv; j += kRsThreads) {
    const uint32_t k = s_keys[j];
    const uint32_t d = (k >> shift) & 255u;
    const uint32_t dst = s_gbase[d] + (uint32_t)j - s_bexcl[d];
    if (kout) kout[dst] = (KeyOutT)k;
    vout[dst] = s_vals[j];
  }
}

struct Layout {
  size_t ctr, ghist, lb_scan0, lb_scan1, lb_depth, lb_tile, zero_end;
  size_t dk0, dk1, dv0, dv1, offs, tk0, tk1, tv0, tv1, chist, dch, dtot, total;
  int64_t depth_parts, tile_parts, dc_stride;
};

size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

Layout make_layout(int64_t P, int64_t cap, int NT) {
  Layout L{};
  size_t o = 0;
  auto take = [&](size_t bytes) {
    const size_t at = o;
    o = align256(o + bytes);
    return at;
  };
  const int64_t scan_parts = (P + kScanTile - 1) / kScanTile + 1;
  L.depth_parts = (P + kRsTileDepth - 1) / kRsTileDepth + 1;
  L.tile_parts = (cap + kRsTileKeys - 1) / kRsTileKeys + 1;
  L.ctr = take(sizeof(Counters));
  L.ghist = take(6 * 256 * sizeof(uint32_t));
  L.lb_scan0 = take(scan_parts * 8);
  L.lb_scan1 = take(scan_parts * 8);
  L.lb_depth = take(4 * L.depth_parts * 256 * sizeof(uint32_t));
  // tile passes' look-back (radix mode) or k_tscan's tile-total chain (bucket mode)
  L.lb_tile = take(std::max<size_t>(2 * L.tile_parts * 256 * sizeof(uint32_t), ((size_t)NT / 32 + 2) * 8));
  L.zero_end = o;
  L.dk0 = take(P * 4);
  L.dk1 = take(P * 4);
  L.dv0 = take(P * 4);
  L.dv1 = take(P * 4);
  L.offs = take(P * 4);
  L.tk0 = take(cap * 2);
  L.tk1 = take(cap * 2);
  L.tv0 = take(cap * 4);
  L.tv1 = take(cap * 4);
  L.chist = take((size_t)kBkMaxChunks * ((NT + 3) & ~3) * 4);
  L.dc_stride = (cap + kDcTile - 1) / kDcTile + 1;
  L.dch = take((size_t)256 * L.dc_stride * 4);
  L.dtot = take(256 * 4);
  L.total = o;
  return L;
}

// Tile placement: "bucket" (K4', default when its shared memory fits), "radix" (two
// onesweep / reduce-then-scan 8-bit passes, GSR_TILE_SORT=radix) or "lsd" (K4'',
// GSR_TILE_SORT=lsd).  scannetpp step (r02 A/B): bucket 6.02, lsd 6.35, radix 6.41 ms
// (lsd: 2 x (dcount 8 + dscan 5 + dscatter 37) + ranges 12 us per view serialised).
int tile_sort_mode() {
  static const int mode = [] {
    const char* e = std::getenv("GSR_TILE_SORT");
    if (e && std::strcmp(e, "radix") == 0) return 0;
    if (e && std::strcmp(e, "lsd") == 0) return 2;
    return 1;
  }();
  return mode;
}
bool use_bucket(int NT) { return tile_sort_mode() == 1 && tscatter_warps(NT) > 0; }

}  // namespace

// Radix pass implementation: decoupled look-back onesweep (default) or
// reduce-then-scan (GSR_SORT=rts).  Both produce identical output; onesweep measured
// faster end to end on B200 (profiles/r01/sort_ab.txt).
bool use_rts() {
  const char* e = std::getenv("GSR_SORT");
  return e && std::strcmp(e, "rts") == 0;
}

// Depth-pass partition size (see kRsItemsDepthBig): a P heuristic (P >= 512K stands in
// for "several views in flight", true of every workload that large in bench.py);
// GSR_DEPTH_ITEMS=4|16 overrides it, any other value is reported once and ignored.
bool depth_items_big(int64_t P) {
  static const int forced = [] {
    const char* e = std::getenv("GSR_DEPTH_ITEMS");
    if (!e) return 0;
    if (std::strcmp(e, "4") == 0) return 4;
    if (std::strcmp(e, "16") == 0) return 16;
    std::fprintf(stderr, "gsr: GSR_DEPTH_ITEMS=%s ignored (accepted: 4, 16)\n", e);
    return 0;
  }();
  return forced ? forced == 16 : P >= ((int64_t)1 << 19);
}

#ifdef GSR_BOUNDS_CHECK
__global__ void k_check_lists(int NT, int64_t P, const int32_t* __restrict__ ids, const int2* __restrict__ ranges) {
  int32_t kmax = 0;
  for (int t = 0; t < NT; ++t) kmax = max(kmax, ranges[t].y);  // every thread: K = the largest end
  const int lane = threadIdx.x & 31;
  for (int t = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5); t < NT; t += (int)((gridDim.x * blockDim.x) >> 5)) {
    const int2 rg = ranges[t];
    GSR_CHECK(rg.x >= 0 && rg.x <= rg.y && rg.y <= kmax);
    for (int k = rg.x + lane; k < rg.y; k += 32) GSR_CHECK(ids[k] >= 0 && (int64_t)ids[k] < P);
  }
}
void launch_check_lists(int NT, int64_t P, const int32_t* ids, const int32_t* ranges, cudaStream_t s) {
  k_check_lists<<<std::max(1, std::min(NT / 8 + 1, 4 * sm_count())), 256, 0, s>>>(NT, P, ids,
                                                                                 reinterpret_cast<const int2*>(ranges));
}
#else
void launch_check_lists(int, int64_t, const int32_t*, const int32_t*, cudaStream_t) {}
#endif

size_t bin_workspace_bytes(int64_t P, int64_t cap, int num_tiles) { return make_layout(P, cap, num_tiles).total; }

gs_status finish_bin(const void* ctr, int64_t cap, int64_t* num_keys_host, cudaStream_t s);

gs_status launch_bin_tiles(const DevCam& cam, int64_t P, gs_proj proj, void* ws, size_t ws_bytes, int64_t cap,
                           int32_t* sorted_ids, int32_t* tile_ranges, int64_t* num_keys_dev, int64_t* num_keys_host,
                           cudaStream_t s) {
  const int NT = cam.TX * cam.TY;
  const Layout L = make_layout(P, cap, NT);
  if (ws_bytes < L.total) {
    set_error("gs_bin_tiles: workspace %zu B < required %zu B", ws_bytes, L.total);
    return GS_ERR_ARG;
  }
  char* w = static_cast<char*>(ws);
  Counters* ctr = reinterpret_cast<Counters*>(w + L.ctr);
  uint32_t* ghist = reinterpret_cast<uint32_t*>(w + L.ghist);
  if (cudaMemsetAsync(w, 0, L.zero_end, s) != cudaSuccess || cudaMemsetAsync(tile_ranges, 0, (size_t)NT * 8, s) != cudaSuccess)
    return check_launch("gs_bin_tiles memset");
  if (P == 0) {
    if (num_keys_dev && cudaMemsetAsync(num_keys_dev, 0, 8, s) != cudaSuccess) return check_launch("memset");
    if (num_keys_host) *num_keys_host = 0;
    return GS_OK;
  }
  uint32_t* dk0 = reinterpret_cast<uint32_t*>(w + L.dk0);
  uint32_t* dk1 = reinterpret_cast<uint32_t*>(w + L.dk1);
  uint32_t* dv0 = reinterpret_cast<uint32_t*>(w + L.dv0);
  uint32_t* dv1 = reinterpret_cast<uint32_t*>(w + L.dv1);
  uint32_t* offs = reinterpret_cast<uint32_t*>(w + L.offs);
  uint16_t* tk0 = reinterpret_cast<uint16_t*>(w + L.tk0);
  uint16_t* tk1 = reinterpret_cast<uint16_t*>(w + L.tk1);
  uint32_t* tv0 = reinterpret_cast<uint32_t*>(w + L.tv0);
  uint32_t* tv1 = reinterpret_cast<uint32_t*>(w + L.tv1);
  uint32_t* lbd = reinterpret_cast<uint32_t*>(w + L.lb_depth);
  uint32_t* lbt = reinterpret_cast<uint32_t*>(w + L.lb_tile);
  const int nsm = sm_count();

  const int scan_grid = (int)((P + kScanTile - 1) / kScanTile);
  k_compact<<<scan_grid, kScanThreads, 0, s>>>(P, proj.tiles, proj.rec, ctr,
                                               reinterpret_cast<unsigned long long*>(w + L.lb_scan0), dk0, dv0, ghist);
  count_launch();
  // depth sort: 4 passes, result back in (dk0, dv0)
  const int rs_grid_d = (int)std::min<int64_t>((P + kRsTileDepth - 1) / kRsTileDepth, (int64_t)nsm * 3);
  uint32_t* kin = dk0;
  uint32_t* vin = dv0;
  uint32_t* kout = dk1;
  uint32_t* vout = dv1;
  const bool rts_mode = use_rts();
  const bool big = depth_items_big(P);
  const int rs_grid_big =
      (int)std::min<int64_t>((P + kRsThreads * kRsItemsDepthBig - 1) / (kRsThreads * kRsItemsDepthBig), (int64_t)nsm * 3);
  for (int pass = 0; pass < 4; ++pass) {
    uint32_t* lb = lbd + (int64_t)pass * L.depth_parts * 256;  // sized for the smaller partitions
    if (rts_mode) {
      rts::radix_pass<uint32_t, kRsItemsDepth>(kin, vin, kout, vout, &ctr->V, P, ghist + pass * 256, lb, L.depth_parts,
                                               8 * pass, s);
    } else if (big) {
      k_onesweep<uint32_t, kRsItemsDepthBig><<<std::max(rs_grid_big, 1), kRsThreads, 0, s>>>(
          kin, vin, kout, vout, &ctr->V, P, ghist + pass * 256, lb, &ctr->part[2 + pass], 8 * pass);
      count_launch();
    } else {
      k_onesweep<uint32_t, kRsItemsDepth><<<rs_grid_d, kRsThreads, 0, s>>>(kin, vin, kout, vout, &ctr->V, P,
                                                                           ghist + pass * 256, lb,
                                                                           &ctr->part[2 + pass], 8 * pass);
      count_launch();
    }
    std::swap(kin, kout);
    std::swap(vin, vout);
  }
  // kin/vin now hold the depth-sorted (z bits, gid)
  k_offsets<<<scan_grid, kScanThreads, 0, s>>>(proj.tiles, vin, ctr,
                                               reinterpret_cast<unsigned long long*>(w + L.lb_scan1), offs,
                                               reinterpret_cast<long long*>(num_keys_dev));
  count_launch();
  const int emit_grid = (int)std::min<int64_t>((cap + kEmTile - 1) / kEmTile, (int64_t)nsm * GSR_EMIT_PER_SM);
  const bool bucket = use_bucket(NT);
  if (bucket || tile_sort_mode() == 2)
    k_emit<false><<<std::max(emit_grid, 1), kEmThreads, 0, s>>>(vin, offs, proj.rec, cam.TX, ctr, cap, tk0, tv0,
                                                                ghist + 4 * 256);
  else
    k_emit<true><<<std::max(emit_grid, 1), kEmThreads, 0, s>>>(vin, offs, proj.rec, cam.TX, ctr, cap, tk0, tv0,
                                                               ghist + 4 * 256);
  count_launch();
  if (tile_sort_mode() == 2) {
    uint32_t* dch = reinterpret_cast<uint32_t*>(w + L.dch);
    uint32_t* dtot = reinterpret_cast<uint32_t*>(w + L.dtot);
    const int cgrid = (int)std::max<int64_t>(1, (cap + kDcTile - 1) / kDcTile);
    auto lsd_pass = [&](const uint16_t* ki, const uint32_t* vi, uint16_t* ko, uint32_t* vo, int shift) {
      k_dcount<<<cgrid, kRsThreads, 0, s>>>(ki, ctr, cap, shift, L.dc_stride, dch);
      k_dscan<<<256, kRsThreads, 0, s>>>(ctr, cap, L.dc_stride, dch, dtot);
      k_dscatter<uint16_t><<<cgrid, kRsThreads, 0, s>>>(ki, vi, ko, vo, ctr, cap, shift, L.dc_stride, dch, dtot);
      count_launch(3);
    };
    const uint16_t* final_keys;
    uint32_t* ids_out = reinterpret_cast<uint32_t*>(sorted_ids);
    if (NT <= 256) {
      lsd_pass(tk0, tv0, tk1, ids_out, 0);
      final_keys = tk1;
    } else {
      lsd_pass(tk0, tv0, tk1, tv1, 0);
      lsd_pass(tk1, tv1, tk0, ids_out, 8);
      final_keys = tk0;
    }
    const int rg_grid = (int)std::min<int64_t>((cap + 255) / 256, (int64_t)nsm * 8);
    k_ranges<<<std::max(rg_grid, 1), 256, 0, s>>>(final_keys, ctr, cap, reinterpret_cast<int2*>(tile_ranges));
    count_launch();
    return finish_bin(ctr, cap, num_keys_host, s);
  }
  if (bucket) {
    // chunks: a multiple of the SMs (CTAs resident per SM by shared memory), each < 2^16 keys
    const int W = tscatter_warps(NT);
    const size_t smem = tscatter_smem(NT, W);
    const int per_sm = (int)std::max<size_t>(1, std::min<size_t>(4, kSmemOptIn / (smem + 1024)));
    const int64_t need = (cap + 63000 - 1) / 63000;  // chunks (rounded up to 2048 keys) stay < 2^16 keys
    const int C = (int)std::max<int64_t>(std::min<int64_t>((int64_t)nsm * per_sm, kBkMaxChunks), need);
    if (C <= kBkMaxChunks) {
      uint32_t* chist = reinterpret_cast<uint32_t*>(w + L.chist);
      int2* rng = reinterpret_cast<int2*>(tile_ranges);
      int tile_bits = 1;
      while ((1 << tile_bits) < NT) ++tile_bits;
      static bool attr_set = false;  // opt-in shared memory above 48 KB (once per process)
      if (!attr_set) {
        if (cudaFuncSetAttribute(k_tscatter<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemOptIn) !=
                cudaSuccess ||
            cudaFuncSetAttribute(k_tscatter<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemOptIn) !=
                cudaSuccess ||
            cudaFuncSetAttribute(k_tcount, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemOptIn) != cudaSuccess)
          return check_launch("gs_bin_tiles smem opt-in");
        attr_set = true;
      }
      k_tcount<<<C, kTcThreads, (size_t)NT * 4, s>>>(tk0, ctr, cap, NT, C, W, chist);
      k_tscan<<<(NT + 31) / 32, kBkThreads, 0, s>>>(chist, NT, C, ctr, reinterpret_cast<unsigned long long*>(lbt),
                                                    rng);
      if (W == 8)
        k_tscatter<8><<<C, 256, smem, s>>>(tk0, tv0, ctr, cap, NT, C, tile_bits, chist, sorted_ids,
                                           tscatter_own_bits(NT, 8));
      else
        k_tscatter<4><<<C, 128, smem, s>>>(tk0, tv0, ctr, cap, NT, C, tile_bits, chist, sorted_ids,
                                           tscatter_own_bits(NT, 4));
      count_launch(3);
      return finish_bin(ctr, cap, num_keys_host, s);
    }
  }
  const int rs_grid_t = (int)std::max<int64_t>(1, std::min<int64_t>((cap + kRsTileKeys - 1) / kRsTileKeys, (int64_t)nsm * 3));
  const uint16_t* final_keys;
  uint32_t* lbt1 = lbt + (int64_t)L.tile_parts * 256;
  uint32_t* ids_out = reinterpret_cast<uint32_t*>(sorted_ids);
  auto tile_pass = [&](const uint16_t* ki, const uint32_t* vi, uint16_t* ko, uint32_t* vo, int pass) {
    uint32_t* lb = pass == 0 ? lbt : lbt1;
    if (rts_mode) {
      rts::radix_pass<uint16_t, kRsItemsKeys>(ki, vi, ko, vo, &ctr->K, cap, ghist + (4 + pass) * 256, lb,
                                              L.tile_parts, 8 * pass, s);
    } else {
      k_onesweep<uint16_t, kRsItemsKeys><<<rs_grid_t, kRsThreads, 0, s>>>(ki, vi, ko, vo, &ctr->K, cap,
                                                                          ghist + (4 + pass) * 256, lb,
                                                                          &ctr->part[6 + pass], 8 * pass);
      count_launch();
    }
  };
  if (NT <= 256) {
    tile_pass(tk0, tv0, tk1, ids_out, 0);
    final_keys = tk1;
  } else {
    tile_pass(tk0, tv0, tk1, tv1, 0);
    tile_pass(tk1, tv1, tk0, ids_out, 1);
    final_keys = tk0;
  }
  const int rg_grid = (int)std::min<int64_t>((cap + 255) / 256, (int64_t)nsm * 8);
  k_ranges<<<std::max(rg_grid, 1), 256, 0, s>>>(final_keys, ctr, cap, reinterpret_cast<int2*>(tile_ranges));
  count_launch();
  return finish_bin(ctr, cap, num_keys_host, s);
}

gs_status finish_bin(const void* ctr_v, int64_t cap, int64_t* num_keys_host, cudaStream_t s) {
  const Counters* ctr = static_cast<const Counters*>(ctr_v);
  gs_status st = check_launch("gs_bin_tiles");
  if (st != GS_OK) return st;
  if (num_keys_host) {
    unsigned long long K = 0;
    if (cudaMemcpyAsync(&K, &ctr->K, 8, cudaMemcpyDeviceToHost, s) != cudaSuccess || cudaStreamSynchronize(s) != cudaSuccess)
      return check_launch("gs_bin_tiles readback");
    *num_keys_host = (int64_t)K;
    if ((int64_t)K > cap) {
      set_error("gs_bin_tiles: %lld keys exceed key_capacity %lld", (long long)K, (long long)cap);
      return GS_ERR_CAPACITY;
    }
  }
  return GS_OK;
}


// ---------------------------------------------------------------------------
// gs_spatial_order: permute the Gaussian store into Morton (Z-curve) order of the
// means (10 bits per axis inside the means' bounding box).  A setup-time layout
// transform: per-view SoA reads of the visible subset then touch contiguous
// sectors instead of every sector of every row.  Reuses the onesweep passes.
// ---------------------------------------------------------------------------
namespace {

__device__ __forceinline__ uint32_t f2ord(float f) {  // order-preserving float -> uint
  const uint32_t u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float ord2f(uint32_t u) {
  return __uint_as_float((u & 0x80000000u) ? (u & 0x7fffffffu) : ~u);
}
__device__ __forceinline__ uint32_t spread10(uint32_t v) {  // 10 bits -> every third bit
  v &= 0x3ffu;
  v = (v | (v << 16)) & 0x030000ffu;
  v = (v | (v << 8)) & 0x0300f00fu;
  v = (v | (v << 4)) & 0x030c30c3u;
  v = (v | (v << 2)) & 0x09249249u;
  return v;
}

struct OrderCtr {
  uint32_t bmin[3], bmax[3];
  uint32_t part[4];
  unsigned long long n;
};

__global__ void __launch_bounds__(256) k_bbox(int64_t P, int64_t S, const float* __restrict__ prm, OrderCtr* ctr) {
  if (blockIdx.x == 0 && threadIdx.x == 0) ctr->n = (unsigned long long)P;
  uint32_t mn[3] = {0xffffffffu, 0xffffffffu, 0xffffffffu}, mx[3] = {0u, 0u, 0u};
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < P; i += (int64_t)gridDim.x * blockDim.x) {
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const float v = prm[a * S + i];
      if (isfinite(v)) {
        const uint32_t o = f2ord(v);
        mn[a] = min(mn[a], o);
        mx[a] = max(mx[a], o);
      }
    }
  }
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    mn[a] = __reduce_min_sync(kFull, mn[a]);
    mx[a] = __reduce_max_sync(kFull, mx[a]);
    if ((threadIdx.x & 31) == 0) {
      atomicMin(&ctr->bmin[a], mn[a]);
      atomicMax(&ctr->bmax[a], mx[a]);
    }
  }
}

__global__ void __launch_bounds__(256) k_morton(int64_t P, int64_t S, const float* __restrict__ prm,
                                                const OrderCtr* __restrict__ ctr, uint32_t* __restrict__ keys,
                                                uint32_t* __restrict__ vals, uint32_t* __restrict__ ghist) {
  __shared__ uint32_t s_hist[4][256];
  for (int t = threadIdx.x; t < 1024; t += 256) (&s_hist[0][0])[t] = 0;
  __syncthreads();
  float lo[3], sc[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    lo[a] = ord2f(ctr->bmin[a]);
    const float ext = ord2f(ctr->bmax[a]) - lo[a];
    sc[a] = ext > 0.f ? 1023.99f / ext : 0.f;
  }
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < P; i += (int64_t)gridDim.x * blockDim.x) {
    uint32_t code = 0;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const float v = prm[a * S + i];
      const float q = isfinite(v) ? fminf(fmaxf((v - lo[a]) * sc[a], 0.f), 1023.f) : 1023.f;
      code |= spread10((uint32_t)q) << a;
    }
    keys[i] = code;
    vals[i] = (uint32_t)i;
    atomicAdd(&s_hist[0][code & 255], 1u);
    atomicAdd(&s_hist[1][(code >> 8) & 255], 1u);
    atomicAdd(&s_hist[2][(code >> 16) & 255], 1u);
    atomicAdd(&s_hist[3][code >> 24], 1u);
  }
  __syncthreads();
  for (int t = threadIdx.x; t < 1024; t += 256) {
    const uint32_t c = (&s_hist[0][0])[t];
    if (c) atomicAdd(&ghist[t], c);
  }
}

// params_out[r][j] = params_in[r][perm[j]] for j < P; padding columns zeroed.
__global__ void __launch_bounds__(256) k_gather_rows(int64_t F, int64_t P, int64_t S, const float* __restrict__ in,
                                                     const uint32_t* __restrict__ perm, float* __restrict__ out) {
  const int64_t n = F * S;
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = k / S, j = k - r * S;
    out[k] = j < P ? in[r * S + perm[j]] : 0.f;
  }
}

struct OrderLayout {
  size_t ctr, ghist, lb, zero_end, k0, k1, v0, v1, total;
  int64_t parts;
};

OrderLayout order_layout(int64_t P) {
  OrderLayout L{};
  size_t o = 0;
  auto take = [&](size_t bytes) {
    const size_t at = o;
    o = align256(o + bytes);
    return at;
  };
  L.parts = (P + kRsTileDepth - 1) / kRsTileDepth + 1;
  L.ctr = take(sizeof(OrderCtr));
  L.ghist = take(4 * 256 * sizeof(uint32_t));
  L.lb = take(4 * L.parts * 256 * sizeof(uint32_t));
  L.zero_end = o;
  L.k0 = take(P * 4);
  L.k1 = take(P * 4);
  L.v0 = take(P * 4);
  L.v1 = take(P * 4);
  L.total = o;
  return L;
}

}  // namespace

size_t spatial_order_workspace_bytes(int64_t P) { return order_layout(P).total; }

gs_status launch_spatial_order(int64_t F, int64_t P, int64_t S, const float* params_in, float* params_out,
                               int32_t* perm, void* ws, size_t ws_bytes, cudaStream_t s) {
  const OrderLayout L = order_layout(P);
  if (ws_bytes < L.total) {
    set_error("gs_spatial_order: workspace %zu B < required %zu B", ws_bytes, L.total);
    return GS_ERR_ARG;
  }
  char* w = static_cast<char*>(ws);
  OrderCtr* ctr = reinterpret_cast<OrderCtr*>(w + L.ctr);
  uint32_t* ghist = reinterpret_cast<uint32_t*>(w + L.ghist);
  if (cudaMemsetAsync(w, 0, L.zero_end, s) != cudaSuccess) return check_launch("gs_spatial_order memset");
  if (cudaMemsetAsync(ctr->bmin, 0xff, sizeof(ctr->bmin), s) != cudaSuccess)  // bmax, part = 0 from above
    return check_launch("gs_spatial_order init");
  const int nsm = sm_count();
  const int grid = (int)std::min<int64_t>((P + 255) / 256, (int64_t)nsm * 8);
  uint32_t* kin = reinterpret_cast<uint32_t*>(w + L.k0);
  uint32_t* kout = reinterpret_cast<uint32_t*>(w + L.k1);
  uint32_t* vin = reinterpret_cast<uint32_t*>(w + L.v0);
  uint32_t* vout = reinterpret_cast<uint32_t*>(w + L.v1);
  k_bbox<<<grid, 256, 0, s>>>(P, S, params_in, ctr);
  k_morton<<<grid, 256, 0, s>>>(P, S, params_in, ctr, kin, vin, ghist);
  count_launch(2);
  const int rs_grid = (int)std::min<int64_t>((P + kRsTileDepth - 1) / kRsTileDepth, (int64_t)nsm * 3);
  for (int pass = 0; pass < 4; ++pass) {  // stable: equal codes keep index order
    k_onesweep<uint32_t, kRsItemsDepth><<<rs_grid, kRsThreads, 0, s>>>(
        kin, vin, kout, vout, &ctr->n, P, ghist + pass * 256, reinterpret_cast<uint32_t*>(w + L.lb) + (int64_t)pass * L.parts * 256,
        &ctr->part[pass], 8 * pass);
    count_launch();
    std::swap(kin, kout);
    std::swap(vin, vout);
  }
  k_gather_rows<<<(int)std::min<int64_t>((F * S + 255) / 256, (int64_t)nsm * 16), 256, 0, s>>>(F, P, S, params_in, vin,
                                                                                               params_out);
  count_launch();
  if (perm && cudaMemcpyAsync(perm, vin, (size_t)P * 4, cudaMemcpyDeviceToDevice, s) != cudaSuccess)
    return check_launch("gs_spatial_order perm");
  return check_launch("gs_spatial_order");
}

// ---------------------------------------------------------------------------
// Tile work order (gs_tile_order): the render kernels run one warp per tile and
// per-tile work is very uneven (list lengths: mean 580, p99 ~2200 at config 3), so
// a tile list sorted by decreasing length makes the block scheduler start the
// longest tiles first (longest-processing-time-first) and fill the tail with the
// short ones.  One CTA: counting sort of the NT tiles by min(length, 4095) / 4,
// descending, in shared memory; the order inside a bucket is arbitrary (results
// do not depend on it).
// ---------------------------------------------------------------------------
namespace {
constexpr int kOrdBuckets = 1024, kOrdThreads = 1024;
__global__ void __launch_bounds__(kOrdThreads) k_tile_order(const int2* __restrict__ ranges, int NT,
                                                             int32_t* __restrict__ order) {
  __shared__ uint32_t s_cnt[kOrdBuckets];
  __shared__ uint32_t s_wsum[kOrdThreads / 32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  s_cnt[tid] = 0;
  __syncthreads();
  auto bucket = [&](int t) {
    const int2 r = ranges[t];
    const int len = min(max(r.y - r.x, 0), 4095);
    return kOrdBuckets - 1 - (len >> 2);  // descending length
  };
  for (int t = tid; t < NT; t += kOrdThreads) atomicAdd(&s_cnt[bucket(t)], 1u);
  __syncthreads();
  // exclusive scan of the 1024 bucket counts (one per thread)
  const uint32_t v = s_cnt[tid];
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(kFull, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_wsum[warp] = x;
  __syncthreads();
  if (warp == 0) {
    const uint32_t w = s_wsum[lane];
    uint32_t z = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(kFull, z, o);
      if (lane >= o) z += y;
    }
    s_wsum[lane] = z - w;
  }
  __syncthreads();
  s_cnt[tid] = s_wsum[warp] + x - v;
  __syncthreads();
  for (int t = tid; t < NT; t += kOrdThreads) order[atomicAdd(&s_cnt[bucket(t)], 1u)] = t;
}
}  // namespace

void launch_tile_order(int NT, const int32_t* tile_ranges, int32_t* order, cudaStream_t s) {
  k_tile_order<<<1, kOrdThreads, 0, s>>>(reinterpret_cast<const int2*>(tile_ranges), NT, order);
  count_launch();
}

}  // namespace gsr
