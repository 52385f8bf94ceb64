// NEXT-3: TSDF band allocation and integration (PAPER.md:80-82
// §III-A1, §III-B1, Eqs. 6-9) -- a second HBM-bound data-parallel
// workload, upstream of the Gaussian initialisation gate.
//
// B200 design: the octree of 8^3-voxel blocks becomes a flat open-addressing hash table
// keyed by the block's Morton code (the tree is only "a spatial index"),
// a block pool of SoA voxel arrays (tsdf, weight: 2 KB + 2 KB per block, contiguous
// per block so a CTA streams a block with coalesced 16-B accesses), and two kernels:
//  * k_tsdf_alloc: one thread per pixel marches its line of sight through the
//    +-eps band and inserts the blocks of its samples (atomicCAS on the key slot,
//    atomicAdd on the pool counter for a new block); consecutive samples in the same
//    block are inserted once;
//  * k_tsdf_integrate: persistent CTAs walk the pool, one block per iteration, 4
//    voxels per thread; each voxel is projected, reads its depth sample and applies
//    Eqs. 6-9 in place.  HBM-bound: 16 B of voxel state per voxel (read + write).
// The voxel chain uses explicitly rounded fp32 intrinsics in a fixed order (as the
// projection does, reading R9) so that block sets, tsdf and weights are bit-identical
// to the CPU oracle (oracle/tsdf_ref.cpp).
#include "gsr_internal.cuh"
#include "tsdf_hash.cuh"

namespace gsr {
namespace {
using namespace tsdfhash;

#define TM(a, b) __fmul_rn((a), (b))
#define TA(a, b) __fadd_rn((a), (b))
#define TS(a, b) __fsub_rn((a), (b))
#define TD(a, b) __fdiv_rn((a), (b))

constexpr int kVoxBits = 21;  // per axis in the 63-bit Morton code
constexpr int kIntThreads = 128;

struct TsdfDev {
  float vs, inv_vs, eps, wmax, step;
  int org[3];
};

// Two phases per ray so that the warp stays converged: the sample loop only records the
// distinct blocks its samples fall in (consecutive samples mostly share a block; a
// per-lane list of up to kRayBlocks), and the insertion loop -- Morton code, hash probe,
// CAS -- runs once per recorded block with the lanes in step.
constexpr int kRayBlocks = 8;

__global__ void __launch_bounds__(256) k_tsdf_alloc(TsdfDev tp, gs_tsdf_volume vol, DevCam cam,
                                                     const float* __restrict__ depth,
                                                     unsigned long long* __restrict__ new_blocks) {
  const int64_t npix = (int64_t)cam.W * cam.H;
  uint32_t created = 0;
  int nb = 0;
  int bl[kRayBlocks][3];
  auto flush = [&]() {
    const int n_max = __reduce_max_sync(__activemask(), nb);
    for (int q = 0; q < n_max; ++q)
      if (q < nb) created += insert_block(vol, morton3((uint32_t)bl[q][0], (uint32_t)bl[q][1], (uint32_t)bl[q][2]));
    nb = 0;
  };
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < npix; p += (int64_t)gridDim.x * blockDim.x) {
    const float d = depth[p];
    const int i = (int)(p % cam.W), j = (int)(p / cam.W);
    const float rx = TD(TS((float)i, cam.cx), cam.fx), ry = TD(TS((float)j, cam.cy), cam.fy);
    const float z0 = TS(d, tp.eps), z1 = TA(d, tp.eps);
    const int n = d > 0.f ? (int)ceilf(TD(TS(z1, z0), tp.step)) : -1;
    // the pixel's line of sight in the world: p(z) = o + z dw, dw = R^T (rx, ry, 1),
    // o = the camera centre (R34: per-pixel direction, two operations per sample axis)
    float dw[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) dw[a] = TA(TA(TM(cam.R[a], rx), TM(cam.R[3 + a], ry)), cam.R[6 + a]);
    int lb0 = -1, lb1 = -1, lb2 = -1;  // block of the previous sample
    for (int k = 0; k <= n; ++k) {
      const float z = (k == n) ? z1 : TA(z0, TM((float)k, tp.step));
      int b[3];
      bool ok = true;
#pragma unroll
      for (int a = 0; a < 3; ++a) {  // voxel = floor(p * (1 / voxel_size)) + origin (R34)
        const float pw = TA(TM(z, dw[a]), cam.ocam[a]);
        const float vv = TA(floorf(TM(pw, tp.inv_vs)), (float)tp.org[a]);
        ok = ok && (vv >= 0.f) && (vv < (float)(1 << kVoxBits));
        b[a] = ok ? ((int)vv >> 3) : 0;
      }
      if (!ok || (b[0] == lb0 && b[1] == lb1 && b[2] == lb2)) continue;
      lb0 = b[0], lb1 = b[1], lb2 = b[2];
      if (nb == kRayBlocks) flush();  // rare: a long band through many blocks
      bl[nb][0] = b[0], bl[nb][1] = b[1], bl[nb][2] = b[2];
      ++nb;
    }
    flush();
  }
  if (new_blocks) {
    const uint32_t tot = __reduce_add_sync(kFull, created);
    if ((threadIdx.x & 31) == 0 && tot) atomicAdd(new_blocks, (unsigned long long)tot);
  }
}

__global__ void __launch_bounds__(kIntThreads) k_tsdf_integrate(TsdfDev tp, gs_tsdf_volume vol, DevCam cam,
                                                                const float* __restrict__ depth,
                                                                unsigned long long* __restrict__ updated) {
  const int64_t nb = *vol.num_blocks < vol.block_cap ? *vol.num_blocks : vol.block_cap;
  uint32_t cnt = 0;
  for (int64_t blk = blockIdx.x; blk < nb; blk += gridDim.x) {
    const uint64_t key = vol.pool_keys[blk];
    const int bx = (int)compact3(key), by = (int)compact3(key >> 1), bz = (int)compact3(key >> 2);
    float* ts = vol.tsdf + blk * 512;
    float* ws = vol.weight + blk * 512;
#pragma unroll
    for (int k = 0; k < 512 / kIntThreads; ++k) {
      const int l = threadIdx.x + k * kIntThreads;
      const int v[3] = {bx * 8 + (l & 7), by * 8 + ((l >> 3) & 7), bz * 8 + (l >> 6)};
      float pw[3];
#pragma unroll
      for (int a = 0; a < 3; ++a) pw[a] = TM(TA((float)(v[a] - tp.org[a]), 0.5f), tp.vs);
      const float* R = cam.R;
      const float x = TA(TA(TA(TM(R[0], pw[0]), TM(R[1], pw[1])), TM(R[2], pw[2])), cam.t[0]);
      const float y = TA(TA(TA(TM(R[3], pw[0]), TM(R[4], pw[1])), TM(R[5], pw[2])), cam.t[1]);
      const float z = TA(TA(TA(TM(R[6], pw[0]), TM(R[7], pw[1])), TM(R[8], pw[2])), cam.t[2]);
      if (!(z > 0.f)) continue;
      const float u = TA(TM(cam.fx, TD(x, z)), cam.cx), w = TA(TM(cam.fy, TD(y, z)), cam.cy);
      const float fu = floorf(TA(u, 0.5f)), fw = floorf(TA(w, 0.5f));  // nearest pixel (R1)
      if (!(fu >= 0.f && fu < (float)cam.W && fw >= 0.f && fw < (float)cam.H)) continue;
      const float d = depth[(int64_t)fw * cam.W + (int64_t)fu];
      if (!(d > 0.f)) continue;
      const float sdf = TS(d, z);  // Eq. 6
      if (sdf < -tp.eps) continue;  // far behind the surface (R35)
      const float q = TD(sdf, tp.eps);
      const float tsdf = sdf > 0.f ? fminf(1.f, q) : fmaxf(-1.f, q);  // Eq. 7
      const float wp = ws[l], tpv = ts[l];
      const float wk = fminf(tp.wmax, TA(wp, 1.f));  // Eq. 8
      ts[l] = TD(TA(TM(tpv, wp), TM(tsdf, wk)), TA(wp, wk));  // Eq. 9
      ws[l] = wk;
      ++cnt;
    }
  }
  if (updated) {
    const uint32_t tot = __reduce_add_sync(kFull, cnt);
    if ((threadIdx.x & 31) == 0 && tot) atomicAdd(updated, (unsigned long long)tot);
  }
}

__global__ void k_tsdf_fill_keys(uint64_t* keys, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    keys[i] = GS_TSDF_EMPTY_KEY;
}

TsdfDev make_tsdf(const gs_tsdf_params& p) {
  TsdfDev t{};
  t.vs = p.voxel_size, t.eps = p.trunc, t.wmax = p.w_max, t.step = p.step;
  t.inv_vs = 1.0f / p.voxel_size;  // fp32 reciprocal, as the oracle (R34)
  for (int a = 0; a < 3; ++a) t.org[a] = p.origin[a];
  return t;
}

gs_status check_tsdf(const gs_tsdf_params* p, const gs_tsdf_volume& v, const char* fn) {
  if (p && !(p->voxel_size > 0.f && p->trunc >= p->voxel_size && p->w_max >= 1.f && p->step > 0.f &&
             p->step <= p->voxel_size)) {
    set_error("%s: invalid parameters (voxel %g, eps %g, w_max %g, step %g)", fn, (double)p->voxel_size,
              (double)p->trunc, (double)p->w_max, (double)p->step);
    return GS_ERR_ARG;
  }
  if (!v.keys || !v.slots || !v.pool_keys || !v.tsdf || !v.weight || !v.num_blocks || v.table_cap <= 0 ||
      (v.table_cap & (v.table_cap - 1)) || v.block_cap <= 0 || v.block_cap > INT32_MAX) {
    set_error("%s: invalid volume (NULL buffer, table_cap not a power of two, or capacities)", fn);
    return GS_ERR_ARG;
  }
  if (!aligned16(v.tsdf) || !aligned16(v.weight)) {
    set_error("%s: tsdf / weight not 16-byte aligned", fn);
    return GS_ERR_ALIGN;
  }
  return GS_OK;
}

}  // namespace
}  // namespace gsr

using namespace gsr;

extern "C" {

gs_status gs_tsdf_reset(gs_tsdf_volume vol, void* stream) {
  if (const gs_status st = check_tsdf(nullptr, vol, "gs_tsdf_reset")) return st;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  k_tsdf_fill_keys<<<sm_count() * 8, 256, 0, s>>>(vol.keys, vol.table_cap);
  count_launch();
  if (cudaMemsetAsync(vol.tsdf, 0, (size_t)vol.block_cap * 512 * 4, s) != cudaSuccess ||
      cudaMemsetAsync(vol.weight, 0, (size_t)vol.block_cap * 512 * 4, s) != cudaSuccess ||
      cudaMemsetAsync(vol.num_blocks, 0, 8, s) != cudaSuccess)
    return check_launch("gs_tsdf_reset memset");
  return check_launch("gs_tsdf_reset");
}

gs_status gs_tsdf_allocate(const gs_tsdf_params* prm, gs_tsdf_volume vol, const gs_camera* cam, const float* depth,
                           int64_t* new_blocks, void* stream) {
  if (!prm || !cam || !depth) {
    set_error("gs_tsdf_allocate: NULL argument");
    return GS_ERR_ARG;
  }
  if (const gs_status st = check_tsdf(prm, vol, "gs_tsdf_allocate")) return st;
  if (cam->width <= 0 || cam->height <= 0 || !(cam->fx > 0.f) || !(cam->fy > 0.f)) {
    set_error("gs_tsdf_allocate: invalid camera");
    return GS_ERR_ARG;
  }
  const DevCam dc = make_devcam(*cam);
  const int64_t npix = (int64_t)cam->width * cam->height;
  const int grid = (int)std::min<int64_t>((npix + 255) / 256, (int64_t)sm_count() * 16);
  k_tsdf_alloc<<<std::max(grid, 1), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      make_tsdf(*prm), vol, dc, depth, reinterpret_cast<unsigned long long*>(new_blocks));
  count_launch();
  return check_launch("gs_tsdf_allocate");
}

gs_status gs_tsdf_integrate(const gs_tsdf_params* prm, gs_tsdf_volume vol, const gs_camera* cam, const float* depth,
                            int64_t* updated, void* stream) {
  if (!prm || !cam || !depth) {
    set_error("gs_tsdf_integrate: NULL argument");
    return GS_ERR_ARG;
  }
  if (const gs_status st = check_tsdf(prm, vol, "gs_tsdf_integrate")) return st;
  if (cam->width <= 0 || cam->height <= 0 || !(cam->fx > 0.f) || !(cam->fy > 0.f)) {
    set_error("gs_tsdf_integrate: invalid camera");
    return GS_ERR_ARG;
  }
  const int grid = (int)std::min<int64_t>(vol.block_cap, (int64_t)sm_count() * 16);
  k_tsdf_integrate<<<std::max(grid, 1), kIntThreads, 0, static_cast<cudaStream_t>(stream)>>>(
      make_tsdf(*prm), vol, make_devcam(*cam), depth, reinterpret_cast<unsigned long long*>(updated));
  count_launch();
  return check_launch("gs_tsdf_integrate");
}

}  // extern "C"
