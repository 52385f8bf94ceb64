// NEXT-4: quadtree seeding and weight-gated Gaussian initialisation
// (§III-B2, Eq. 10), on the GPU.
//
// Quadtree (readings R37-R39): a cell (x, y, w, h) is split into NW (x, y,
// w/2, h/2), NE, SW, SE (floor halves) when w > min_cell, h > min_cell and its contrast
// max(L) - min(L) > threshold, L = 0.299 R + 0.587 G + 0.114 B.  Because the split
// points depend only on the geometry, every pixel lies in a fixed cell at every level:
// node (l, c) with Z-index c = 4 c_parent + child.  B200 design (no recursion):
//   k_qt_leafmax: each pixel descends to depth D (virtual child 0 below cells that cannot
//     split) and folds L into that cell's min / max (float bits of L >= 0 compare as
//     integers: atomicMin / atomicMax);
//   k_qt_reduce:  levels D-1 .. 0, each cell's min / max from its four children;
//   k_qt_split:   levels 0 .. D-1, split = parent split && splittable && contrast > thr;
//   k_qt_emit:    one CTA scans the depth-D index space in order; a leaf (l, c) sits at
//     its first depth-D index c 4^(D-l), so the scan lists the leaves in depth-first
//     (NW, NE, SW, SE) order without sorting.
// Seeding (Eq. 10): per leaf, back-project the centre pixel with its depth, look up the
// voxel containing the point in the TSDF hash; if its weight is exactly 1 (first
// observed in this frame, fused before seeding) append a Gaussian: mean p_q, identity
// rotation, isotropic scale = back-projected centre-to-corner length, opacity 0.5, SH
// DC from the pixel colour, higher SH 0.  Appends keep leaf order (block scan).
#include <cmath>
#include <vector>

#include "gsr_internal.cuh"
#include "tsdf_hash.cuh"

namespace gsr {
namespace {
using namespace tsdfhash;

#define QM(a, b) __fmul_rn((a), (b))
#define QA(a, b) __fadd_rn((a), (b))
#define QS(a, b) __fsub_rn((a), (b))
#define QD(a, b) __fdiv_rn((a), (b))

struct QtGeom {
  int W, H, min_cell, D;
};

__device__ __forceinline__ bool splittable(int w, int h, int mc) { return w > mc && h > mc; }

// Geometry of node (l, c): descend from the root along c's base-4 digits.
__device__ __forceinline__ void node_rect(const QtGeom& g, int l, uint32_t c, int& x, int& y, int& w, int& h) {
  x = 0, y = 0, w = g.W, h = g.H;
  for (int k = l - 1; k >= 0; --k) {
    const int ch = (c >> (2 * k)) & 3;
    const int hw = w / 2, hh = h / 2;
    if (ch & 1) x += hw, w -= hw; else w = hw;
    if (ch & 2) y += hh, h -= hh; else h = hh;
  }
}

__device__ __forceinline__ float luminance(const float* rgb, int64_t npix, int64_t p) {
  return QA(QA(QM(0.299f, rgb[p]), QM(0.587f, rgb[npix + p])), QM(0.114f, rgb[2 * npix + p]));
}

__global__ void __launch_bounds__(256) k_qt_leafmax(QtGeom g, const float* __restrict__ rgb, uint32_t* __restrict__ mn,
                                                     uint32_t* __restrict__ mx) {
  const int64_t npix = (int64_t)g.W * g.H;
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < npix; p += (int64_t)gridDim.x * blockDim.x) {
    uint32_t c = 0, lb = 0;
    {
      const int px = (int)(p % g.W), py = (int)(p / g.W);
      int x = 0, y = 0, w = g.W, h = g.H;
      for (int l = 0; l < g.D; ++l) {
        int ch = 0;
        if (splittable(w, h, g.min_cell)) {
          const int hw = w / 2, hh = h / 2;
          if (px >= x + hw) ch |= 1, x += hw, w -= hw; else w = hw;
          if (py >= y + hh) ch |= 2, y += hh, h -= hh; else h = hh;
        }
        c = c * 4 + ch;
      }
      lb = __float_as_uint(fmaxf(luminance(rgb, npix, p), 0.f));
    }
    atomicMin(mn + c, lb);
    atomicMax(mx + c, lb);
  }
}

__global__ void k_qt_reduce(uint32_t* __restrict__ mn_l, uint32_t* __restrict__ mx_l,
                            const uint32_t* __restrict__ mn_c, const uint32_t* __restrict__ mx_c, int64_t n) {
  for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < n; c += (int64_t)gridDim.x * blockDim.x) {
    uint32_t lo = 0xffffffffu, hi = 0u;
#pragma unroll
    for (int k = 0; k < 4; ++k) lo = min(lo, mn_c[4 * c + k]), hi = max(hi, mx_c[4 * c + k]);
    mn_l[c] = lo;
    mx_l[c] = hi;
  }
}

// split flags of level l (parent flags of level l - 1; the root's parent "splits")
__global__ void k_qt_split(QtGeom g, int l, const uint32_t* __restrict__ mn, const uint32_t* __restrict__ mx,
                           const uint8_t* __restrict__ split_parent, uint8_t* __restrict__ split, float thr,
                           int64_t n) {
  for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < n; c += (int64_t)gridDim.x * blockDim.x) {
    uint8_t s = 0;
    if (l == 0 || split_parent[c >> 2]) {
      int x, y, w, h;
      node_rect(g, l, (uint32_t)c, x, y, w, h);
      const float contrast = QS(__uint_as_float(mx[c]), __uint_as_float(mn[c]));
      s = (splittable(w, h, g.min_cell) && contrast > thr) ? 1 : 2;  // 1 split, 2 leaf, 0 not a node
    }
    split[c] = s;
  }
}

// One CTA: depth-D indices in order; index s starts a leaf at the coarsest level l
// whose node c = s >> 2 (D - l) is a leaf and s is its first descendant.
__global__ void __launch_bounds__(1024) k_qt_emit(QtGeom g, const uint8_t* const* __restrict__ split_lv,
                                                   int32_t* __restrict__ leaves, int64_t cap,
                                                   int64_t* __restrict__ num_leaves) {
  __shared__ int s_wsum[32];
  __shared__ int64_t s_base;
  if (threadIdx.x == 0) s_base = 0;
  __syncthreads();
  const int64_t nD = (int64_t)1 << (2 * g.D);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int64_t s0 = 0; s0 < nD; s0 += 1024) {
    const int64_t s = s0 + threadIdx.x;
    int lvl = -1;
    if (s < nD) {
      for (int l = 0; l <= g.D; ++l) {
        const int sh = 2 * (g.D - l);
        const int64_t c = s >> sh;
        const uint8_t f = split_lv[l][c];
        if (f == 2) {
          if ((c << sh) == s) lvl = l;
          break;
        }
        if (f != 1) break;
      }
    }
    const int flag = lvl >= 0;
    const uint32_t bal = __ballot_sync(kFull, flag);
    if (lane == 0) s_wsum[warp] = __popc(bal);
    __syncthreads();
    int pre = 0, tot = 0;
    for (int k = 0; k < 32; ++k) {
      const int v = s_wsum[k];
      pre += k < warp ? v : 0;
      tot += v;
    }
    const int64_t pos = s_base + pre + __popc(bal & ((1u << lane) - 1u));
    if (flag && pos < cap) {
      int x, y, w, h;
      node_rect(g, lvl, (uint32_t)(s >> (2 * (g.D - lvl))), x, y, w, h);
      reinterpret_cast<int4*>(leaves)[pos] = make_int4(x, y, w, h);
    }
    __syncthreads();
    if (threadIdx.x == 0) s_base += tot;
    __syncthreads();
  }
  if (threadIdx.x == 0) *num_leaves = s_base;
}

// ---------------------------------------------------------------- seeding
struct SeedCtx {
  float vs, inv_vs;
  int org[3];
  int64_t P0, S, cap;
  int F;
};

// One CTA: leaves in order; gate, ordered append (block scan), parameter writes.
__global__ void __launch_bounds__(1024) k_seed(SeedCtx sc, gs_tsdf_volume vol, DevCam cam,
                                                const float* __restrict__ depth, const float* __restrict__ rgb,
                                                const int32_t* __restrict__ leaves,
                                                const int64_t* __restrict__ num_leaves, float* __restrict__ params,
                                                int64_t* __restrict__ num_new) {
  __shared__ int s_wsum[32];
  __shared__ int64_t s_base;
  if (threadIdx.x == 0) s_base = 0;
  __syncthreads();
  const int64_t nl = *num_leaves;
  const int64_t npix = (int64_t)cam.W * cam.H;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int64_t q0 = 0; q0 < nl; q0 += 1024) {
    const int64_t q = q0 + threadIdx.x;
    bool take = false;
    float pw[3] = {0.f, 0.f, 0.f}, scale = 0.f, col[3] = {0.f, 0.f, 0.f};
    if (q < nl) {
      const int4 lf = reinterpret_cast<const int4*>(leaves)[q];
      const int u = lf.x + lf.z / 2, v = lf.y + lf.w / 2;  // centre pixel (R38)
      const int64_t pp = (int64_t)v * cam.W + u;
      GSR_CHECK(u >= 0 && u < cam.W && v >= 0 && v < cam.H);
      const float d = depth[pp];
      if (d > 0.f) {
        // Eq. 10: p_q = T_WC pi^-1(u_q, D[u_q])
        const float rx = QD(QS((float)u, cam.cx), cam.fx), ry = QD(QS((float)v, cam.cy), cam.fy);
        const float pc[3] = {QM(rx, d), QM(ry, d), d};
        float qv[3];
#pragma unroll
        for (int r = 0; r < 3; ++r) qv[r] = QS(pc[r], cam.t[r]);
        int vox[3];
        bool ok = true;
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          pw[a] = QA(QA(QM(cam.R[a], qv[0]), QM(cam.R[3 + a], qv[1])), QM(cam.R[6 + a], qv[2]));
          const float vv = QA(floorf(QM(pw[a], sc.inv_vs)), (float)sc.org[a]);
          ok = ok && vv >= 0.f && vv < 2097152.f;
          vox[a] = ok ? (int)vv : 0;
        }
        if (ok) {
          const uint64_t key = spread3((uint32_t)(vox[0] >> 3)) | (spread3((uint32_t)(vox[1] >> 3)) << 1) |
                               (spread3((uint32_t)(vox[2] >> 3)) << 2);
          const int64_t blk = find_block(vol, key);
          if (blk >= 0 && blk < vol.block_cap) {
            const int loc = (vox[0] & 7) + 8 * (vox[1] & 7) + 64 * (vox[2] & 7);
            take = vol.weight[blk * 512 + loc] == 1.f;  // newly observed voxel
          }
        }
        if (take) {
          // isotropic scale: centre-to-corner length back-projected at the centre depth (R39)
          const float cx0 = QM(QD(QS((float)lf.x, cam.cx), cam.fx), d), cy0 = QM(QD(QS((float)lf.y, cam.cy), cam.fy), d);
          const float dx = QS(pc[0], cx0), dy = QS(pc[1], cy0);
          scale = __fsqrt_rn(QA(QM(dx, dx), QM(dy, dy)));
#pragma unroll
          for (int ch = 0; ch < 3; ++ch) col[ch] = rgb[ch * npix + pp];
          take = scale > 0.f;
        }
      }
    }
    const uint32_t bal = __ballot_sync(kFull, take);
    if (lane == 0) s_wsum[warp] = __popc(bal);
    __syncthreads();
    int pre = 0, tot = 0;
    for (int k = 0; k < 32; ++k) {
      const int vv = s_wsum[k];
      pre += k < warp ? vv : 0;
      tot += vv;
    }
    const int64_t i = sc.P0 + s_base + pre + __popc(bal & ((1u << lane) - 1u));
    if (take && i < sc.cap) {
      const int64_t S = sc.S;
      params[i] = pw[0], params[S + i] = pw[1], params[2 * S + i] = pw[2];
      const float ls = (float)log((double)scale);  // activations in double (R9)
      params[3 * S + i] = ls, params[4 * S + i] = ls, params[5 * S + i] = ls;
      params[6 * S + i] = 1.f, params[7 * S + i] = 0.f, params[8 * S + i] = 0.f, params[9 * S + i] = 0.f;
      params[10 * S + i] = 0.f;  // opacity 0.5
#pragma unroll
      for (int ch = 0; ch < 3; ++ch) params[(11 + ch) * S + i] = QD(QS(col[ch], 0.5f), 0.28209479177387814f);
      for (int r = 14; r < sc.F; ++r) params[(int64_t)r * S + i] = 0.f;
    }
    __syncthreads();
    if (threadIdx.x == 0) s_base += tot;
    __syncthreads();
  }
  if (threadIdx.x == 0) *num_new = s_base;
}

}  // namespace

int quadtree_depth(int W, int H, int min_cell) {
  // deepest level at which some cell can still split, + 1 (cells at one level differ by
  // at most one pixel per dimension, so the distinct (w, h) pairs are few)
  std::vector<std::pair<int, int>> cur = {{W, H}};
  int D = 0;
  while (true) {
    std::vector<std::pair<int, int>> nxt;
    for (auto [w, h] : cur)
      if (w > min_cell && h > min_cell)
        for (int cw : {w / 2, w - w / 2})
          for (int ch : {h / 2, h - h / 2}) nxt.push_back({cw, ch});
    if (nxt.empty()) return D;
    std::sort(nxt.begin(), nxt.end());
    nxt.erase(std::unique(nxt.begin(), nxt.end()), nxt.end());
    cur.swap(nxt);
    ++D;
  }
}

}  // namespace gsr

using namespace gsr;

extern "C" {

size_t gs_quadtree_workspace(int32_t width, int32_t height, int32_t min_cell) {
  if (width <= 0 || height <= 0 || min_cell < 1) return 0;
  const int D = quadtree_depth(width, height, min_cell);
  size_t cells = 0;
  for (int l = 0; l <= D; ++l) cells += (size_t)1 << (2 * l);
  return cells * 9 + 64 * (D + 2) + 256;  // min, max (u32) + split (u8) per node, level pointers
}

gs_status gs_quadtree(int32_t width, int32_t height, const float* rgb, float threshold, int32_t min_cell, void* ws,
                      size_t ws_bytes, int32_t* leaves, int64_t leaf_capacity, int64_t* num_leaves, void* stream) {
  if (width <= 0 || height <= 0 || !rgb || !ws || !leaves || !num_leaves || min_cell < 2 || !(threshold > 0.f) ||
      leaf_capacity < 0) {
    set_error("gs_quadtree: invalid arguments");
    return GS_ERR_ARG;
  }
  if (ws_bytes < gs_quadtree_workspace(width, height, min_cell)) {
    set_error("gs_quadtree: workspace too small");
    return GS_ERR_ARG;
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  QtGeom g{width, height, min_cell, quadtree_depth(width, height, min_cell)};
  // layout: level pointer table (device), then per level min, max, split
  char* w = static_cast<char*>(ws);
  const uint8_t** lvptr_dev = reinterpret_cast<const uint8_t**>(w);
  char* o = w + 64 * ((8 * (g.D + 2) + 63) / 64);
  std::vector<uint32_t*> mn(g.D + 1), mx(g.D + 1);
  std::vector<uint8_t*> sp(g.D + 1);
  for (int l = 0; l <= g.D; ++l) {
    const size_t n = (size_t)1 << (2 * l);
    mn[l] = reinterpret_cast<uint32_t*>(o), o += 4 * n;
    mx[l] = reinterpret_cast<uint32_t*>(o), o += 4 * n;
  }
  for (int l = 0; l <= g.D; ++l) sp[l] = reinterpret_cast<uint8_t*>(o), o += ((size_t)1 << (2 * l));
  const size_t nD = (size_t)1 << (2 * g.D);
  if (cudaMemsetAsync(mn[g.D], 0xff, 4 * nD, s) != cudaSuccess || cudaMemsetAsync(mx[g.D], 0, 4 * nD, s) != cudaSuccess ||
      cudaMemcpyAsync(lvptr_dev, sp.data(), sizeof(uint8_t*) * (g.D + 1), cudaMemcpyHostToDevice, s) != cudaSuccess)
    return check_launch("gs_quadtree memset");
  const int64_t npix = (int64_t)width * height;
  const int nsm = sm_count();
  k_qt_leafmax<<<(int)std::min<int64_t>((npix + 255) / 256, (int64_t)nsm * 8), 256, 0, s>>>(g, rgb, mn[g.D], mx[g.D]);
  for (int l = g.D - 1; l >= 0; --l) {
    const int64_t n = (int64_t)1 << (2 * l);
    k_qt_reduce<<<(int)std::min<int64_t>((n + 255) / 256, (int64_t)nsm * 8), 256, 0, s>>>(mn[l], mx[l], mn[l + 1],
                                                                                         mx[l + 1], n);
  }
  for (int l = 0; l < g.D; ++l) {
    const int64_t n = (int64_t)1 << (2 * l);
    k_qt_split<<<(int)std::min<int64_t>((n + 255) / 256, (int64_t)nsm * 8), 256, 0, s>>>(
        g, l, mn[l], mx[l], l > 0 ? sp[l - 1] : nullptr, sp[l], threshold, n);
  }
  // depth-D nodes are leaves whenever their parent split
  {
    const int64_t n = (int64_t)nD;
    k_qt_split<<<(int)std::min<int64_t>((n + 255) / 256, (int64_t)nsm * 8), 256, 0, s>>>(
        g, g.D, mn[g.D], mx[g.D], g.D > 0 ? sp[g.D - 1] : nullptr, sp[g.D], 3.4e38f, n);
  }
  k_qt_emit<<<1, 1024, 0, s>>>(g, lvptr_dev, leaves, leaf_capacity, num_leaves);
  count_launch(2 + 2 * g.D + 1);
  return check_launch("gs_quadtree");
}

gs_status gs_seed_gaussians(const gs_camera* cam, const gs_tsdf_params* prm, gs_tsdf_volume vol, const float* depth,
                            const float* rgb, const int32_t* leaves, const int64_t* num_leaves, const gs_scene* scene,
                            float* params, int64_t* num_new, void* stream) {
  if (!cam || !prm || !depth || !rgb || !leaves || !num_leaves || !scene || !params || !num_new || scene->P < 0 ||
      scene->P_stride < scene->P || scene->sh_degree < 0 || scene->sh_degree > GS_MAX_SH_DEGREE) {
    set_error("gs_seed_gaussians: invalid arguments");
    return GS_ERR_ARG;
  }
  SeedCtx sc{};
  sc.vs = prm->voxel_size, sc.inv_vs = 1.0f / prm->voxel_size;
  for (int a = 0; a < 3; ++a) sc.org[a] = prm->origin[a];
  sc.P0 = scene->P, sc.S = scene->P_stride, sc.cap = scene->P_stride;
  sc.F = 11 + 3 * (scene->sh_degree + 1) * (scene->sh_degree + 1);
  k_seed<<<1, 1024, 0, static_cast<cudaStream_t>(stream)>>>(sc, vol, make_devcam(*cam), depth, rgb, leaves, num_leaves,
                                                             params, num_new);
  count_launch();
  return check_launch("gs_seed_gaussians");
}

}  // extern "C"
