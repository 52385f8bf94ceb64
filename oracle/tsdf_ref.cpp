// CPU ORACLE of GSFusion's TSDF fusion -- TEST INFRASTRUCTURE ONLY (SURVEY.md §8(f)
// NEXT-3).  Only tests/ and bench.py's CPU legs may load it; the product never does.
//
// Plain definition, written from the paper, independent of the CUDA path
// (paper_2408_12677_b200/csrc/tsdf.cu):
//  * the grid (§III-A1): single-resolution voxels holding (tsdf,
//    weight) in 8^3-voxel blocks identified by the Morton code of their integer block
//    coordinates ("interleaved bits from the 3D coordinates form a unique identifier");
//    here a std::map from that code to the block (the octree is only an index);
//  * band allocation: "a ray is marched along the line of sight for each
//    pixel, and voxel blocks are allocated only if they fall into the specified eps
//    band around the depth measurement" -- samples at z = d - eps + k step, k = 0..n,
//    n = ceil(2 eps / step), the last one at z = d + eps, world point o + z R^T (rx, ry, 1)
//    (readings R33, R34);
//  * integration, Eqs. 6-9, per voxel of every allocated block:
//      sdf = D[pi(T^-1 p_v)] - z_v                  (Eq. 6; nearest pixel, R1)
//      tsdf = min(1, sdf/eps) if sdf > 0 else max(-1, sdf/eps)      (Eq. 7)
//      w_k = min(w_max, w_{k-1} + 1)                                (Eq. 8)
//      tsdf_k = (tsdf_{k-1} w_{k-1} + tsdf w_k) / (w_{k-1} + w_k)   (Eq. 9, as written)
//    skipping voxels behind the camera, off the image, on invalid depth, or with
//    sdf < -eps (R35).
// Arithmetic: fp32, one operation per statement in the order written, compiled with
// -ffp-contract=off (reading R9) -- the parity tests compare the GPU bit for bit.
#include <cmath>
#include <cstdint>
#include <map>
#include <vector>

namespace {

struct Params {
  float voxel_size, trunc, w_max, step;
  int32_t origin[3];
};
struct Camera {
  int32_t width, height;
  float fx, fy, cx, cy;
  float R_cw[9], t_cw[3];
  float z_near;
  float bg[3];
};
struct Block {
  float tsdf[512];
  float weight[512];
};
struct Volume {
  Params p;
  std::map<uint64_t, Block> blocks;
};

// Morton code: bit i of x, y, z goes to bit 3i, 3i+1, 3i+2 (21 bits per axis).
uint64_t morton(uint32_t x, uint32_t y, uint32_t z) {
  uint64_t m = 0;
  for (int i = 0; i < 21; ++i) {
    m |= (uint64_t)((x >> i) & 1u) << (3 * i);
    m |= (uint64_t)((y >> i) & 1u) << (3 * i + 1);
    m |= (uint64_t)((z >> i) & 1u) << (3 * i + 2);
  }
  return m;
}
void unmorton(uint64_t m, uint32_t& x, uint32_t& y, uint32_t& z) {
  x = y = z = 0;
  for (int i = 0; i < 21; ++i) {
    x |= (uint32_t)((m >> (3 * i)) & 1u) << i;
    y |= (uint32_t)((m >> (3 * i + 1)) & 1u) << i;
    z |= (uint32_t)((m >> (3 * i + 2)) & 1u) << i;
  }
}

}  // namespace

extern "C" {

uint64_t ref_morton(uint32_t x, uint32_t y, uint32_t z) { return morton(x, y, z); }
void ref_unmorton(uint64_t m, uint32_t* xyz) { unmorton(m, xyz[0], xyz[1], xyz[2]); }

void* ref_tsdf_new(const Params* p) {
  Volume* v = new Volume();
  v->p = *p;
  return v;
}
void ref_tsdf_free(void* h) { delete static_cast<Volume*>(h); }
int64_t ref_tsdf_num_blocks(void* h) { return (int64_t) static_cast<Volume*>(h)->blocks.size(); }

// Band allocation; returns the number of blocks created.
int64_t ref_tsdf_allocate(void* h, const Camera* c, const float* depth) {
  Volume& V = *static_cast<Volume*>(h);
  const Params& P = V.p;
  int64_t created = 0;
  const float inv_vs = 1.0f / P.voxel_size;  // voxel of a sample: floor(p * (1 / voxel_size)) (R34)
  for (int j = 0; j < c->height; ++j) {
    for (int i = 0; i < c->width; ++i) {
      const float d = depth[(int64_t)j * c->width + i];
      if (!(d > 0.f)) continue;
      // line of sight of pixel (i, j): camera point (rx z, ry z, z)
      const float rx = ((float)i - c->cx) / c->fx;
      const float ry = ((float)j - c->cy) / c->fy;
      const float z0 = d - P.trunc;
      const float z1 = d + P.trunc;
      const int n = (int)std::ceil((z1 - z0) / P.step);
      // the same line in the world: p(z) = o + z dw with dw = R^T (rx, ry, 1) and the
      // camera centre o = -R^T t (double, rounded; reading R34)
      float dw[3], o[3];
      for (int a = 0; a < 3; ++a) {
        const float m0 = c->R_cw[a] * rx;
        const float m1 = c->R_cw[3 + a] * ry;
        const float s01 = m0 + m1;
        dw[a] = s01 + c->R_cw[6 + a];
        double acc = 0.0;
        for (int r = 0; r < 3; ++r) acc += (double)c->R_cw[3 * r + a] * (double)c->t_cw[r];
        o[a] = (float)(-acc);
      }
      for (int k = 0; k <= n; ++k) {
        float z;
        if (k == n) {
          z = z1;
        } else {
          const float dz = (float)k * P.step;
          z = z0 + dz;
        }
        int64_t blk[3];
        bool inside = true;
        for (int a = 0; a < 3; ++a) {
          const float zd = z * dw[a];
          const float pw = zd + o[a];
          const float cell = std::floor(pw * inv_vs);
          const float vox = cell + (float)P.origin[a];
          if (!(vox >= 0.f && vox < 2097152.f)) inside = false;
          blk[a] = inside ? ((int64_t)vox / 8) : 0;
        }
        if (!inside) continue;
        const uint64_t key = morton((uint32_t)blk[0], (uint32_t)blk[1], (uint32_t)blk[2]);
        if (V.blocks.find(key) == V.blocks.end()) {
          Block b;
          for (int l = 0; l < 512; ++l) b.tsdf[l] = 0.f, b.weight[l] = 0.f;
          V.blocks.emplace(key, b);
          ++created;
        }
      }
    }
  }
  return created;
}

// Integration, Eqs. 6-9; returns the number of voxels updated.
int64_t ref_tsdf_integrate(void* h, const Camera* c, const float* depth) {
  Volume& V = *static_cast<Volume*>(h);
  const Params& P = V.p;
  int64_t updated = 0;
  for (auto& kv : V.blocks) {
    uint32_t b[3];
    unmorton(kv.first, b[0], b[1], b[2]);
    Block& B = kv.second;
    for (int lz = 0; lz < 8; ++lz)
      for (int ly = 0; ly < 8; ++ly)
        for (int lx = 0; lx < 8; ++lx) {
          const int l = lx + 8 * ly + 64 * lz;
          const int vox[3] = {(int)b[0] * 8 + lx, (int)b[1] * 8 + ly, (int)b[2] * 8 + lz};
          float p[3];  // voxel centre (v - origin + 0.5) voxel_size
          for (int a = 0; a < 3; ++a) {
            const float cell = (float)(vox[a] - P.origin[a]) + 0.5f;
            p[a] = cell * P.voxel_size;
          }
          float pc[3];  // p_c = W p + t  (T_WC^-1)
          for (int r = 0; r < 3; ++r) {
            const float m0 = c->R_cw[3 * r] * p[0];
            const float m1 = c->R_cw[3 * r + 1] * p[1];
            const float m2 = c->R_cw[3 * r + 2] * p[2];
            const float s = (m0 + m1) + m2;
            pc[r] = s + c->t_cw[r];
          }
          const float zc = pc[2];
          if (!(zc > 0.f)) continue;
          const float u = c->fx * (pc[0] / zc) + c->cx;
          const float w = c->fy * (pc[1] / zc) + c->cy;
          const float pu = std::floor(u + 0.5f);
          const float pv = std::floor(w + 0.5f);
          if (!(pu >= 0.f && pu < (float)c->width && pv >= 0.f && pv < (float)c->height)) continue;
          const float d = depth[(int64_t)pv * c->width + (int64_t)pu];
          if (!(d > 0.f)) continue;
          const float sdf = d - zc;  // Eq. 6
          if (sdf < -P.trunc) continue;
          const float ratio = sdf / P.trunc;
          float tsdf;  // Eq. 7
          if (sdf > 0.f)
            tsdf = ratio < 1.f ? ratio : 1.f;
          else
            tsdf = ratio > -1.f ? ratio : -1.f;
          const float w_prev = B.weight[l];
          const float w_inc = w_prev + 1.f;
          const float w_k = w_inc < P.w_max ? w_inc : P.w_max;  // Eq. 8
          const float num0 = B.tsdf[l] * w_prev;
          const float num1 = tsdf * w_k;
          const float num = num0 + num1;
          const float den = w_prev + w_k;
          B.tsdf[l] = num / den;  // Eq. 9
          B.weight[l] = w_k;
          ++updated;
        }
  }
  return updated;
}

// Blocks in increasing key order: keys[n], tsdf[n][512], weight[n][512].
void ref_tsdf_dump(void* h, uint64_t* keys, float* tsdf, float* weight) {
  Volume& V = *static_cast<Volume*>(h);
  int64_t n = 0;
  for (auto& kv : V.blocks) {
    keys[n] = kv.first;
    for (int l = 0; l < 512; ++l) tsdf[n * 512 + l] = kv.second.tsdf[l], weight[n * 512 + l] = kv.second.weight[l];
    ++n;
  }
}

}  // extern "C"
