// Keyframe-scheduled online optimisation plan, host code.
//
// GSFusion optimises the map online with a keyframe list (§III-B3
// "Online Optimization"; settings PAPER.md:174):
//   * a frame is a keyframe when its number of newly initialised Gaussians exceeds
//     a threshold (50), and keyframes are kept in a list;
//   * keyframes get m iterations on themselves, non-keyframes n, and a non-keyframe
//     spends the remaining (m - n) on "the first (m - n) keyframes after shuffling"
//     the list (random keyframe optimisation against forgetting);
//   * "offline optimization over the keyframe list after scanning" for a number of
//     global iterations (10).
// Readings (R28-R31): threshold test is strict (>); with store_all_frames
// (the paper's ScanNet++ setting, "all frames are stored in the keyframe list") every
// frame joins the list but the m / n split still follows the threshold; the current
// frame joins the list before the draw and is excluded from its own draw; one global
// iteration = one pass over the list in a freshly shuffled order.  Shuffles are
// Fisher-Yates driven by splitmix64(seed, stream, counter), a counter-based generator
// the CPU reference (oracle/schedule.py) implements independently.
//
// The plan is a flat list of iterations (view index, frame index or -1 for the
// global passes); every iteration is then one fwd + bwd + Adam step of the GPU path
// (pipeline.KeyframeOptimizer).  Pure integer host logic: bit-exact against the oracle.
#include <algorithm>
#include <cstdint>
#include <vector>

#include "gsr.h"

namespace {

uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

// Uniform integer in [0, n) from draw `c` of stream `s` (n > 0; modulo bias < 2^-40
// for the list sizes used, and identical on both sides by construction).
uint64_t draw(uint64_t seed, uint64_t s, uint64_t c, uint64_t n) {
  return splitmix64(seed ^ splitmix64((s << 32) ^ c)) % n;
}

// Fisher-Yates shuffle of v with stream s.
void shuffle(std::vector<int32_t>& v, uint64_t seed, uint64_t s) {
  for (int64_t i = (int64_t)v.size() - 1; i > 0; --i) {
    const int64_t j = (int64_t)draw(seed, s, (uint64_t)i, (uint64_t)(i + 1));
    std::swap(v[i], v[j]);
  }
}

}  // namespace

extern "C" gs_status gs_keyframe_schedule(const gs_kf_params* prm, int64_t n_frames, const int64_t* new_prims,
                                          int32_t* iter_view, int32_t* iter_frame, int64_t capacity,
                                          int64_t* n_iters, uint8_t* is_keyframe) {
  if (!prm || !n_iters || n_frames < 0 || (n_frames > 0 && !new_prims) || prm->m < 0 || prm->n < 0 ||
      prm->n > prm->m || prm->global_iters < 0 || capacity < 0)
    return GS_ERR_ARG;
  std::vector<int32_t> kf;   // the keyframe list, in insertion order
  std::vector<int32_t> plan_v, plan_f;
  for (int64_t t = 0; t < n_frames; ++t) {
    const bool key = new_prims[t] > prm->threshold;
    if (is_keyframe) is_keyframe[t] = key ? 1 : 0;
    if (key || prm->store_all_frames) kf.push_back((int32_t)t);
    const int own = key ? prm->m : prm->n;
    for (int k = 0; k < own; ++k) plan_v.push_back((int32_t)t), plan_f.push_back((int32_t)t);
    if (!key && prm->m > prm->n) {
      std::vector<int32_t> pool;
      for (int32_t f : kf)
        if (f != (int32_t)t) pool.push_back(f);
      shuffle(pool, prm->seed, (uint64_t)t);
      const int64_t take = std::min<int64_t>((int64_t)(prm->m - prm->n), (int64_t)pool.size());
      for (int64_t k = 0; k < take; ++k) plan_v.push_back(pool[k]), plan_f.push_back((int32_t)t);
    }
  }
  for (int g = 0; g < prm->global_iters; ++g) {
    std::vector<int32_t> order = kf;
    shuffle(order, prm->seed, (uint64_t)(n_frames + g));
    for (int32_t f : order) plan_v.push_back(f), plan_f.push_back(-1);
  }
  *n_iters = (int64_t)plan_v.size();
  if ((int64_t)plan_v.size() > capacity) return GS_ERR_CAPACITY;
  if (!plan_v.empty() && (!iter_view || !iter_frame)) return GS_ERR_ARG;
  for (size_t i = 0; i < plan_v.size(); ++i) iter_view[i] = plan_v[i], iter_frame[i] = plan_f[i];
  return GS_OK;
}
