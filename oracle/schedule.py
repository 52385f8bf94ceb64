"""Oracle of the keyframe-scheduled online optimisation plan -- TEST INFRASTRUCTURE.

Only tests/ (and bench.py's reference legs) may import this module.  It is the
plain definition of GSFusion's online optimisation strategy, written from the paper
and independent of the product's C++ scheduler (paper_2408_12677_b200/csrc/
schedule.cpp); the two share only the documented counter-based generator (R31),
each implementing it separately.

PAPER.md:149 (§III-B3 "Online Optimization"):
  "we select a keyframe and add it to the list once the number of new primitives
   is greater than a certain threshold.  Keyframes and non-keyframes will undergo m
   and n iterations of optimization, respectively. [...] reserving some resources to
   randomly selected keyframes from the maintained list (i.e., the first (m-n)
   keyframes after shuffling). [...] our system also supports offline optimization
   over the keyframe list after scanning."
PAPER.md:174 (Implementation details): keyframe threshold 50, 10 global iterations;
Replica m = 5, n = 3 (+2 random); ScanNet++ m = 10, n = 1 (+9 random), "all frames
are stored in the keyframe list".

Readings: R28 strict ">" threshold; R29 store_all_frames puts every
frame in the list, the m/n split still follows the threshold; R30 the current frame
joins the list before the draw and is not drawn for itself; one global iteration =
one pass over the list in a freshly shuffled order; R31 shuffles are Fisher-Yates
with j = splitmix64(seed XOR splitmix64((stream << 32) XOR i)) mod (i + 1), stream =
frame index for a frame's draw and n_frames + g for global pass g.
"""
from __future__ import annotations

MASK = (1 << 64) - 1


def splitmix64(x: int) -> int:
    """Steele, Lea & Flood's SplitMix64 finaliser (the R31 generator)."""
    x = (x + 0x9E3779B97F4A7C15) & MASK
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & MASK
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & MASK
    return x ^ (x >> 31)


def shuffled(items, seed: int, stream: int):
    """Fisher-Yates (Durstenfeld) from the last position down, R31 draws."""
    a = list(items)
    for i in range(len(a) - 1, 0, -1):
        j = splitmix64((seed ^ splitmix64(((stream << 32) ^ i) & MASK)) & MASK) % (i + 1)
        a[i], a[j] = a[j], a[i]
    return a


def keyframe_schedule(new_prims, threshold=50, m=5, n=3, global_iters=10, store_all_frames=False, seed=0):
    """Returns (plan, is_keyframe): plan = list of (view, frame) iterations, frame = -1
    for the passes after scanning; is_keyframe = list of bools per frame."""
    keyframes = []
    plan = []
    is_kf = []
    for t, count in enumerate(new_prims):
        key = count > threshold                      # "greater than a certain threshold"
        is_kf.append(key)
        if key or store_all_frames:
            keyframes.append(t)                      # "add it to the list"
        own = m if key else n                        # "m and n iterations, respectively"
        plan += [(t, t)] * own
        if not key:                                  # "the first (m-n) keyframes after shuffling"
            pool = [f for f in keyframes if f != t]
            for f in shuffled(pool, seed, t)[:max(m - n, 0)]:
                plan.append((f, t))
    for g in range(global_iters):                    # "offline optimization over the keyframe list"
        for f in shuffled(keyframes, seed, len(new_prims) + g):
            plan.append((f, -1))
    return plan, is_kf
