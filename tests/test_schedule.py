"""Keyframe-scheduled optimisation plan.

-m "not gpu": the oracle (oracle/schedule.py) pinned against what the paper and the
generator's published definition fix, and the product's host scheduler
(gs_keyframe_schedule in libgsr.so, C++) bit-exact against the oracle."""
import collections
import itertools

import numpy as np
import pytest

import scenegen
from oracle import schedule as ref


# ----------------------------------------------------------------------------- oracle pins
def test_splitmix64_published_first_output():
    # SplitMix64 (Steele, Lea & Flood 2014) seeded with 0: first output 0xE220A8397B1DCDAF
    assert ref.splitmix64(0) == 0xE220A8397B1DCDAF


def test_shuffle_is_a_uniform_permutation():
    counts = collections.Counter(tuple(ref.shuffled(range(4), s, 7)) for s in range(24000))
    assert len(counts) == 24  # every permutation of 4 items occurs
    exp = 24000 / 24
    chi2 = sum((c - exp) ** 2 / exp for c in counts.values())
    assert chi2 < 60  # 23 dof: p ~ 1e-4 at 52


def _closed_form_len(new, thr, m, n, G, store_all):
    kf, total = [], 0
    for t, c in enumerate(new):
        key = c > thr
        if key or store_all:
            kf.append(t)
        total += m if key else n + min(m - n, len([f for f in kf if f != t]))
    return total + G * len(kf), kf


@pytest.mark.parametrize("setting", [dict(m=5, n=3, store_all_frames=False),    # Replica
                                     dict(m=10, n=1, store_all_frames=True),    # ScanNet++
                                     dict(m=4, n=4, store_all_frames=False)])
def test_plan_counts_and_structure(setting):
    new = scenegen.new_primitive_counts(60, seed=1)
    plan, is_kf = ref.keyframe_schedule(new, threshold=50, global_iters=10, seed=5, **setting)
    m, n, store = setting["m"], setting["n"], setting["store_all_frames"]
    total, kf = _closed_form_len(new, 50, m, n, 10, store)
    assert len(plan) == total
    assert is_kf == [c > 50 for c in new]
    by_frame = collections.defaultdict(list)
    for v, f in plan:
        by_frame[f].append(v)
    for t in range(len(new)):
        views = by_frame[t]
        own = m if is_kf[t] else n
        assert views[:own] == [t] * own
        extra = views[own:]
        assert len(set(extra)) == len(extra)                       # distinct keyframes
        assert all(f in kf and f <= t and f != t for f in extra)  # from the list, not itself
        if is_kf[t]:
            assert not extra
    glob = by_frame[-1]
    for g in range(10):  # each global pass is a permutation of the keyframe list
        assert sorted(glob[g * len(kf):(g + 1) * len(kf)]) == kf


def test_plan_threshold_is_strict_and_all_keyframes_case():
    plan, is_kf = ref.keyframe_schedule([50, 51, 0], threshold=50, m=5, n=3, global_iters=0)
    assert is_kf == [False, True, False]
    assert plan == [(0, 0)] * 3 + [(1, 1)] * 5 + [(2, 2)] * 3 + [(1, 2)]  # frame 0 had no keyframe to draw
    plan, _ = ref.keyframe_schedule([100] * 4, m=5, n=3, global_iters=2, seed=3)
    assert len(plan) == 4 * 5 + 2 * 4


# ----------------------------------------------------------------------------- product vs oracle
@pytest.fixture(scope="module")
def lib():
    from paper_2408_12677_b200 import _build, gsr
    _build.build()
    return gsr.load()


@pytest.mark.parametrize("T,thr,m,n,G,store,seed", [(0, 50, 5, 3, 10, False, 0), (1, 50, 5, 3, 10, False, 0),
                                                    (100, 50, 5, 3, 10, False, 0), (100, 50, 10, 1, 10, True, 1),
                                                    (37, 200, 6, 2, 3, False, 9), (80, 50, 3, 3, 1, True, 2)])
def test_scheduler_bitexact_vs_oracle(lib, T, thr, m, n, G, store, seed):
    new = scenegen.new_primitive_counts(T, seed=seed)
    views, frames, kf = lib.keyframe_schedule(new, thr, m, n, G, store, seed)
    plan, is_kf = ref.keyframe_schedule(list(new), thr, m, n, G, store, seed)
    assert list(zip(views.tolist(), frames.tolist())) == plan
    assert kf.tolist() == is_kf


def test_scheduler_rejects_bad_parameters(lib):
    from paper_2408_12677_b200 import gsr
    with pytest.raises(gsr.GsError):
        lib.keyframe_schedule([10, 20], m=2, n=3)
