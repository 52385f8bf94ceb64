// Morton keys and the open-addressing block hash of the TSDF grid (NEXT-3), shared by
// the fusion kernels (tsdf.cu) and the seeding gate (seed.cu): one definition of the
// key layout and the probe sequence.
#pragma once

#include "gsr_internal.cuh"

namespace gsr {
namespace tsdfhash {

__device__ __forceinline__ uint64_t spread3(uint32_t x) {  // 21 bits -> every third bit
  uint64_t v = x & 0x1fffffu;
  v = (v | (v << 32)) & 0x1f00000000ffffull;
  v = (v | (v << 16)) & 0x1f0000ff0000ffull;
  v = (v | (v << 8)) & 0x100f00f00f00f00full;
  v = (v | (v << 4)) & 0x10c30c30c30c30c3ull;
  v = (v | (v << 2)) & 0x1249249249249249ull;
  return v;
}
__device__ __forceinline__ uint32_t compact3(uint64_t v) {
  v &= 0x1249249249249249ull;
  v = (v | (v >> 2)) & 0x10c30c30c30c30c3ull;
  v = (v | (v >> 4)) & 0x100f00f00f00f00full;
  v = (v | (v >> 8)) & 0x1f0000ff0000ffull;
  v = (v | (v >> 16)) & 0x1f00000000ffffull;
  v = (v | (v >> 32)) & 0x1fffffull;
  return (uint32_t)v;
}
__device__ __forceinline__ uint64_t morton3(uint32_t x, uint32_t y, uint32_t z) {
  return spread3(x) | (spread3(y) << 1) | (spread3(z) << 2);
}
__device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x ^= x >> 33;
  x *= 0xff51afd7ed558ccdull;
  x ^= x >> 33;
  x *= 0xc4ceb9fe1a85ec53ull;
  return x ^ (x >> 33);
}

// Pool index of a block key, -1 if not allocated.
__device__ __forceinline__ int64_t find_block(const gs_tsdf_volume& vol, uint64_t key) {
  const uint64_t mask = (uint64_t)vol.table_cap - 1;
  uint64_t h = mix64(key) & mask;
  for (int64_t probe = 0; probe < vol.table_cap; ++probe, h = (h + 1) & mask) {
    const uint64_t k = vol.keys[h];
    if (k == key) return vol.slots[h];
    if (k == GS_TSDF_EMPTY_KEY) return -1;
  }
  return -1;
}

// Insert a block key; returns 1 if this call created the block.
__device__ __forceinline__ int insert_block(const gs_tsdf_volume& vol, uint64_t key) {
  const uint64_t mask = (uint64_t)vol.table_cap - 1;
  uint64_t h = mix64(key) & mask;
  for (int64_t probe = 0; probe < vol.table_cap; ++probe, h = (h + 1) & mask) {
    uint64_t k = vol.keys[h];
    if (k == key) return 0;
    if (k == GS_TSDF_EMPTY_KEY) {
      k = atomicCAS(reinterpret_cast<unsigned long long*>(vol.keys + h), (unsigned long long)GS_TSDF_EMPTY_KEY,
                    (unsigned long long)key);
      if (k == GS_TSDF_EMPTY_KEY) {
        const long long idx = atomicAdd(reinterpret_cast<unsigned long long*>(vol.num_blocks), 1ull);
        vol.slots[h] = (int32_t)(idx < (long long)INT32_MAX ? idx : (long long)INT32_MAX);
        if (idx < vol.block_cap) vol.pool_keys[idx] = key;
        return 1;
      }
      if (k == key) return 0;
    }
  }
  // table full: poison the block counter so that the overflow is visible (> block_cap)
  atomicAdd(reinterpret_cast<unsigned long long*>(vol.num_blocks), (unsigned long long)vol.block_cap + 1ull);
  return 0;
}

}  // namespace tsdfhash
}  // namespace gsr
