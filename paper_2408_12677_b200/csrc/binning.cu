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
#include "gsr_internal.cuh"

namespace gsr {
namespace {

constexpr int kScanThreads = 256, kScanItems = 8, kScanTile = kScanThreads * kScanItems;
constexpr int kRsThreads = 256, kRsWarps = kRsThreads / 32, kRsItems = 16, kRsTile = kRsThreads * kRsItems;
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
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    const int64_t i = base + k;
    const bool vis = i < P && tiles[i] > 0;
    flag |= (vis ? 1u : 0u) << k;
    cnt += vis;
  }
  unsigned long long total;
  const unsigned long long excl = block_excl_scan256<unsigned long long>(cnt, s_warp, total);
  if (threadIdx.x == 0) {
    unsigned long long prefix = 0;
    if (part == 0) {
      st_vol(&lookback[0], kScInc | total);
    } else {
      st_vol(&lookback[part], kScAgg | total);
      for (int64_t p = part - 1; p >= 0;) {
        const unsigned long long v = ld_vol(&lookback[p]);
        if ((v >> 62) == 0) continue;
        prefix += v & kScMask;
        if ((v >> 62) == 2) break;
        --p;
      }
      st_vol(&lookback[part], kScInc | (prefix + total));
    }
    s_prefix = prefix;
    if ((int64_t)part == num_parts - 1) ctr->V = prefix + total;
  }
  __syncthreads();
  unsigned long long pos = s_prefix + excl;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    if (flag >> k & 1) {
      const int64_t i = base + k;
      const uint32_t key = __float_as_uint(rec[12 * i + 2]);  // z > z_near > 0: bits order = value order
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
  if (threadIdx.x == 0) {
    unsigned long long prefix = 0;
    if (part == 0) {
      st_vol(&lookback[0], kScInc | total);
    } else {
      st_vol(&lookback[part], kScAgg | total);
      for (int64_t p = part - 1; p >= 0;) {
        const unsigned long long v = ld_vol(&lookback[p]);
        if ((v >> 62) == 0) continue;
        prefix += v & kScMask;
        if ((v >> 62) == 2) break;
        --p;
      }
      st_vol(&lookback[part], kScInc | (prefix + total));
    }
    s_prefix = prefix;
    if ((int64_t)part == num_parts - 1) {
      ctr->K = prefix + total;
      if (num_keys_dev) *num_keys_dev = (long long)(prefix + total);
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
// K3: emit one 16-bit tile key per touched tile, in depth order; fused 2 x 256-bin
// histograms of the tile-key bytes.  One warp broadcasts 32 Gaussians at a time
// and strides its lanes over each footprint (coalesced writes for any size).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_emit(const uint32_t* __restrict__ sorted_gid,
                                              const uint32_t* __restrict__ offs, const float* __restrict__ rec,
                                              int TX, const Counters* __restrict__ ctr, int64_t cap,
                                              uint16_t* __restrict__ tkeys, uint32_t* __restrict__ tvals,
                                              uint32_t* __restrict__ ghist /* [2][256] */) {
  __shared__ uint32_t s_hist[2][256];
  for (int t = threadIdx.x; t < 512; t += 256) (&s_hist[0][0])[t] = 0;
  __syncthreads();
  const int64_t V = (int64_t)ctr->V;
  const bool ok = (int64_t)ctr->K <= cap;
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  if (ok) {
    for (int64_t chunk = gw; chunk * 32 < V; chunk += nw) {
      const int64_t s = chunk * 32 + lane;
      uint32_t gid = 0, off = 0, rx = 0, ry = 0;
      if (s < V) {
        gid = sorted_gid[s];
        off = offs[s];
        const float2 r = *reinterpret_cast<const float2*>(rec + 12 * (int64_t)gid + 10);
        rx = __float_as_uint(r.x);
        ry = __float_as_uint(r.y);
      }
      const int nvalid = (int)((V - chunk * 32) < 32 ? (V - chunk * 32) : 32);
      for (int k = 0; k < nvalid; ++k) {
        const uint32_t g = __shfl_sync(kFull, gid, k);
        const uint32_t o = __shfl_sync(kFull, off, k);
        const uint32_t xr = __shfl_sync(kFull, rx, k), yr = __shfl_sync(kFull, ry, k);
        const int x0 = xr & 0xffff, x1 = xr >> 16, y0 = yr & 0xffff, y1 = yr >> 16;
        const int w = x1 - x0, cnt = w * (y1 - y0);
        for (int j0 = 0; j0 < cnt; j0 += 32) {
          const int j = j0 + lane;
          const bool act = j < cnt;
          uint32_t tile = 0;
          if (act) {
            const int dyq = j / w;
            tile = (uint32_t)((y0 + dyq) * TX + x0 + (j - dyq * w));
            tkeys[o + j] = (uint16_t)tile;
            tvals[o + j] = g;
            atomicAdd(&s_hist[0][tile & 255], 1u);
          }
          // high byte: warp-aggregated (a footprint row shares it)
          const uint32_t hb = act ? (tile >> 8) : 0xffffffffu;
          const uint32_t peers = __match_any_sync(kFull, hb);
          if (act && (peers & lanemask_lt()) == 0) atomicAdd(&s_hist[1][hb], (uint32_t)__popc(peers));
        }
      }
    }
  }
  __syncthreads();
  for (int t = threadIdx.x; t < 512; t += 256) {
    const uint32_t c = (&s_hist[0][0])[t];
    if (c) atomicAdd(&ghist[t], c);
  }
}

// ---------------------------------------------------------------------------
// K4: one onesweep LSD pass (8-bit digit at `shift`) over n = *n_ptr items
// (n := 0 if n > cap).  Persistent CTAs pull 4096-item partitions in order.
// ---------------------------------------------------------------------------
template <typename KeyT>
__global__ void __launch_bounds__(kRsThreads) k_onesweep(const KeyT* __restrict__ kin, const uint32_t* __restrict__ vin,
                                                         KeyT* __restrict__ kout, uint32_t* __restrict__ vout,
                                                         const unsigned long long* n_ptr, int64_t cap,
                                                         const uint32_t* __restrict__ ghist, uint32_t* lookback,
                                                         uint32_t* part_ctr, int shift) {
  __shared__ uint32_t s_keys[kRsTile];
  __shared__ uint32_t s_vals[kRsTile];
  __shared__ uint32_t s_whist[kRsWarps][256];
  __shared__ uint32_t s_gpref[256], s_gbase[256], s_bexcl[256];
  __shared__ uint32_t s_scan[8];
  __shared__ uint32_t s_part;
  int64_t n = (int64_t)*n_ptr;
  if (n > cap) n = 0;
  const int64_t num_parts = (n + kRsTile - 1) / kRsTile;
  if (num_parts == 0) return;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  {
    uint32_t tot;
    s_gpref[t] = block_excl_scan256<uint32_t>(ghist[t], s_scan, tot);
  }
  const uint32_t lt = lanemask_lt();
  for (;;) {
    if (t == 0) s_part = atomicAdd(part_ctr, 1u);
#pragma unroll
    for (int w = 0; w < kRsWarps; ++w) s_whist[w][t] = 0;
    __syncthreads();
    const uint32_t part = s_part;
    if ((int64_t)part >= num_parts) break;
    const int64_t base = (int64_t)part * kRsTile + warp * (kRsItems * 32);
    uint32_t key[kRsItems], val[kRsItems], rank[kRsItems];
#pragma unroll
    for (int i = 0; i < kRsItems; ++i) {
      const int64_t idx = base + i * 32 + lane;
      const bool valid = idx < n;
      key[i] = valid ? (uint32_t)kin[idx] : 0u;
      val[i] = valid ? vin[idx] : 0u;
      const uint32_t d = valid ? ((key[i] >> shift) & 255u) : (256u + lane);
      const uint32_t peers = __match_any_sync(kFull, d);
      const uint32_t r = __popc(peers & lt);
      uint32_t b = 0;
      if (valid) b = s_whist[warp][d];
      __syncwarp();
      if (valid && r == 0) s_whist[warp][d] = b + __popc(peers);
      __syncwarp();
      rank[i] = valid ? (b + r) : 0xffffffffu;
    }
    __syncthreads();
    // per digit: exclusive over warps, partition count
    uint32_t cnt = 0;
#pragma unroll
    for (int w = 0; w < kRsWarps; ++w) {
      const uint32_t c = s_whist[w][t];
      s_whist[w][t] = cnt;
      cnt += c;
    }
    uint32_t tot;
    s_bexcl[t] = block_excl_scan256<uint32_t>(cnt, s_scan, tot);
    uint32_t* lb = lookback + (int64_t)part * 256 + t;
    uint32_t excl = 0;
    if (part == 0) {
      st_vol(lb, kLbInc | cnt);
    } else {
      st_vol(lb, kLbAgg | cnt);
      for (int64_t p = (int64_t)part - 1; p >= 0;) {
        const uint32_t v = ld_vol(lookback + p * 256 + t);
        const uint32_t f = v >> 30;
        if (f == 0) continue;
        excl += v & kLbMask;
        if (f == 2) break;
        --p;
      }
      st_vol(lb, kLbInc | (excl + cnt));
    }
    s_gbase[t] = s_gpref[t] + excl;
    __syncthreads();
#pragma unroll
    for (int i = 0; i < kRsItems; ++i) {
      if (rank[i] != 0xffffffffu) {
        const uint32_t d = (key[i] >> shift) & 255u;
        const uint32_t pos = s_bexcl[d] + s_whist[warp][d] + rank[i];
        s_keys[pos] = key[i];
        s_vals[pos] = val[i];
      }
    }
    __syncthreads();
    const int64_t rem = n - (int64_t)part * kRsTile;
    const int nv = (int)(rem < kRsTile ? rem : kRsTile);
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

struct Layout {
  size_t ctr, ghist, lb_scan0, lb_scan1, lb_depth, lb_tile, zero_end;
  size_t dk0, dk1, dv0, dv1, offs, tk0, tk1, tv0, tv1, total;
  int64_t depth_parts, tile_parts;
};

size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

Layout make_layout(int64_t P, int64_t cap) {
  Layout L{};
  size_t o = 0;
  auto take = [&](size_t bytes) {
    const size_t at = o;
    o = align256(o + bytes);
    return at;
  };
  const int64_t scan_parts = (P + kScanTile - 1) / kScanTile + 1;
  L.depth_parts = (P + kRsTile - 1) / kRsTile + 1;
  L.tile_parts = (cap + kRsTile - 1) / kRsTile + 1;
  L.ctr = take(sizeof(Counters));
  L.ghist = take(6 * 256 * sizeof(uint32_t));
  L.lb_scan0 = take(scan_parts * 8);
  L.lb_scan1 = take(scan_parts * 8);
  L.lb_depth = take(4 * L.depth_parts * 256 * sizeof(uint32_t));
  L.lb_tile = take(2 * L.tile_parts * 256 * sizeof(uint32_t));
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
  L.total = o;
  return L;
}

}  // namespace

size_t bin_workspace_bytes(int64_t P, int64_t cap, int /*num_tiles*/) { return make_layout(P, cap).total; }

gs_status launch_bin_tiles(const DevCam& cam, int64_t P, gs_proj proj, void* ws, size_t ws_bytes, int64_t cap,
                           int32_t* sorted_ids, int32_t* tile_ranges, int64_t* num_keys_dev, int64_t* num_keys_host,
                           cudaStream_t s) {
  const Layout L = make_layout(P, cap);
  if (ws_bytes < L.total) {
    set_error("gs_bin_tiles: workspace %zu B < required %zu B", ws_bytes, L.total);
    return GS_ERR_ARG;
  }
  char* w = static_cast<char*>(ws);
  Counters* ctr = reinterpret_cast<Counters*>(w + L.ctr);
  uint32_t* ghist = reinterpret_cast<uint32_t*>(w + L.ghist);
  const int NT = cam.TX * cam.TY;
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
  const int rs_grid_d = (int)std::min<int64_t>((P + kRsTile - 1) / kRsTile, (int64_t)nsm * 4);
  uint32_t* kin = dk0;
  uint32_t* vin = dv0;
  uint32_t* kout = dk1;
  uint32_t* vout = dv1;
  for (int pass = 0; pass < 4; ++pass) {
    k_onesweep<uint32_t><<<rs_grid_d, kRsThreads, 0, s>>>(kin, vin, kout, vout, &ctr->V, P, ghist + pass * 256,
                                                           lbd + (int64_t)pass * L.depth_parts * 256,
                                                           &ctr->part[2 + pass], 8 * pass);
    count_launch();
    std::swap(kin, kout);
    std::swap(vin, vout);
  }
  // kin/vin now hold the depth-sorted (z bits, gid)
  k_offsets<<<scan_grid, kScanThreads, 0, s>>>(proj.tiles, vin, ctr,
                                               reinterpret_cast<unsigned long long*>(w + L.lb_scan1), offs,
                                               reinterpret_cast<long long*>(num_keys_dev));
  count_launch();
  const int emit_grid = (int)std::min<int64_t>((P + 255) / 256, (int64_t)nsm * 8);
  k_emit<<<emit_grid, 256, 0, s>>>(vin, offs, proj.rec, cam.TX, ctr, cap, tk0, tv0, ghist + 4 * 256);
  count_launch();
  const int rs_grid_t = (int)std::min<int64_t>((cap + kRsTile - 1) / kRsTile, (int64_t)nsm * 4);
  const uint16_t* final_keys;
  if (NT <= 256) {
    k_onesweep<uint16_t><<<rs_grid_t, kRsThreads, 0, s>>>(tk0, tv0, tk1, reinterpret_cast<uint32_t*>(sorted_ids),
                                                           &ctr->K, cap, ghist + 4 * 256, lbt, &ctr->part[6], 0);
    count_launch();
    final_keys = tk1;
  } else {
    k_onesweep<uint16_t><<<rs_grid_t, kRsThreads, 0, s>>>(tk0, tv0, tk1, tv1, &ctr->K, cap, ghist + 4 * 256, lbt,
                                                           &ctr->part[6], 0);
    count_launch();
    k_onesweep<uint16_t><<<rs_grid_t, kRsThreads, 0, s>>>(tk1, tv1, tk0, reinterpret_cast<uint32_t*>(sorted_ids),
                                                           &ctr->K, cap, ghist + 5 * 256,
                                                           lbt + (int64_t)L.tile_parts * 256, &ctr->part[7], 8);
    count_launch();
    final_keys = tk0;
  }
  const int rg_grid = (int)std::min<int64_t>((cap + 255) / 256, (int64_t)nsm * 8);
  k_ranges<<<std::max(rg_grid, 1), 256, 0, s>>>(final_keys, ctr, cap, reinterpret_cast<int2*>(tile_ranges));
  count_launch();
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

}  // namespace gsr
