"""Pins of the parity machinery the GPU gradient tests rest on (-m "not gpu"):

* the STAGE reference (the stage-wise gradient reference, R42) and the
  running error bounds M (oracle/gsref.cpp, struct Rn);
* the decision margins that classify threshold flips (relative, and in units of
  the bound);
* gsref_render_pixels against gsref_render_fwd.

The bound is pinned against something other than itself: the oracle's own plain
fp32 evaluation (mode F32, every operation rounded to float in the written order)
must lie within C_PIN * u * M of the fp64 value of the same maths on every element,
and every pixel whose fp32 and fp64 decisions differ must be flagged by the
bound-unit margin.  The relative margin is recomputed by brute force in numpy.
"""
import numpy as np
import pytest

import scenegen
from threshold_scenes import near_skip_scene

U = 2.0 ** -24
C_PIN = 4.0      # fp32 evaluation vs bound (observed max 1.7 on small)
C_FLIP = 8.0     # the GPU tests' flip / tolerance constant


def _scenes():
    out = [("tiny", scenegen.make("tiny").scene, scenegen.make("tiny").cameras[0])]
    for seed in range(6):
        deg = (0, 1, 3)[seed % 3]
        sc, cam = scenegen.random_small_scene(300 + seed, 6 + 3 * seed, deg)
        cam.bg = (0.3, 0.2, 0.1)
        out.append((f"rand{seed}", sc, cam))
    return out


SCENES = _scenes()
IDS = [s[0] for s in SCENES]


@pytest.mark.parametrize("name,scene,cam", SCENES, ids=IDS)
def test_bound_mode_values_are_the_reference_values(oracle, name, scene, cam):
    """render_bwd_bound's values are bit-identical to render_bwd(STAGE) (stage=True)
    and to render_bwd(MIXED) (stage=False): the bound is carried alongside, it never
    changes a value."""
    g_rgb, g_d = scenegen.upstream_fields(4, cam.width, cam.height)
    st, sst = oracle.render_bwd(cam, scene, g_rgb, g_d, mode=oracle.STAGE)
    mx, _ = oracle.render_bwd(cam, scene, g_rgb, g_d, mode=oracle.MIXED)
    b = oracle.render_bwd_bound(cam, scene, g_rgb, g_d, stage=True)
    np.testing.assert_array_equal(b["grad"], st)
    np.testing.assert_array_equal(b["screen"], sst)
    b2 = oracle.render_bwd_bound(cam, scene, g_rgb, g_d, stage=False)
    np.testing.assert_array_equal(b2["grad"], mx)
    assert np.all(b["bound"] >= 0) and np.all(np.isfinite(b["bound"]))


@pytest.mark.parametrize("name,scene,cam", SCENES + [("small", scenegen.make("small").scene,
                                                        scenegen.make("small").cameras[0])], ids=IDS + ["small"])
def test_bound_covers_fp32_evaluation(oracle, name, scene, cam):
    """|F32 - STAGE| <= C_PIN u M on every gradient element and every screen-space
    gradient: the running bound covers a real fp32 evaluation of the same maths
    (decisions are fp32 on both sides, records identical)."""
    g_rgb, g_d = scenegen.upstream_fields(5, cam.width, cam.height)
    b = oracle.render_bwd_bound(cam, scene, g_rgb, g_d)
    f32, s32 = oracle.render_bwd(cam, scene, g_rgb, g_d, mode=oracle.F32)
    d = np.abs(f32 - b["grad"])
    ratio = d / np.maximum(U * b["bound"], 1e-300)
    assert np.all((d == 0) | (ratio <= C_PIN)), f"max ratio {ratio.max():.2f}"
    ds = np.abs(s32 - b["screen"])
    rs = ds / np.maximum(U * b["screen_bound"], 1e-300)
    assert np.all((ds == 0) | (rs <= C_PIN)), f"screen max ratio {rs.max():.2f}"


def test_bound_is_not_vacuous(oracle):
    """The bound relaxes the north_star tolerance only where the element is genuinely
    ill-conditioned: on the small config C_FLIP u M exceeds 1e-3 |g| for a small
    minority of the significant elements, and the median bound is < 1e-4 |g|."""
    w = scenegen.make("small")
    cam = w.cameras[0]
    g_rgb, g_d = scenegen.upstream_fields(1, cam.width, cam.height)
    b = oracle.render_bwd_bound(cam, w.scene, g_rgb, g_d)
    g, M = b["grad"], b["bound"]
    sig = np.abs(g) > 1e-6
    rel = C_FLIP * U * M[sig] / np.abs(g[sig])
    assert np.median(rel) < 1e-4
    assert (rel > 1e-3).mean() < 0.1


@pytest.mark.parametrize("name,scene,cam", SCENES[:4], ids=IDS[:4])
def test_relative_margin_brute_force(oracle, name, scene, cam):
    """The oracle's relative decision margin (min over a pixel's power > 0, cap, 1/255
    and T' < 1e-4 decisions of the relative distance to the threshold) against a
    numpy float64 recomputation from the oracle's fp32 records and per-pixel lists."""
    pr = oracle.project(cam, scene, oracle.F32)
    f = oracle.render_fwd(cam, scene, oracle.F32, want_margin=True)
    vis = np.nonzero(pr["radius"] > 0)[0]
    rect = pr["rect"]
    checked = 0
    for py in range(cam.height):
        for px in range(cam.width):
            tx, ty = px // 16, py // 16
            lst = [i for i in vis if rect[0, i] <= tx < rect[1, i] and rect[2, i] <= ty < rect[3, i]]
            lst.sort(key=lambda i: (np.float32(pr["z"][i]), i))
            T, best = 1.0, np.inf
            for i in lst:
                dx, dy = pr["mu_x"][i] - px, pr["mu_y"][i] - py
                A, B, C = pr["conic_A"][i], pr["conic_B"][i], pr["conic_C"][i]
                pw = -0.5 * (A * dx * dx + C * dy * dy) - B * dx * dy
                scale = 0.5 * (abs(A * dx * dx) + abs(C * dy * dy)) + abs(B * dx * dy)
                if scale > 0:
                    best = min(best, abs(pw) / scale)
                if pw > 0:
                    continue
                raw = pr["opacity"][i] * np.exp(pw)
                a = min(0.99, raw)
                best = min(best, abs(a - 1 / 255) * 255)
                if raw > 0.99:
                    best = min(best, (raw - 0.99) / 0.99)
                if a < 1 / 255:
                    continue
                Tn = T * (1 - a)
                best = min(best, abs(Tn - 1e-4) / 1e-4)
                if Tn < 1e-4:
                    break
                T = Tn
            got = f["margin"][py, px]
            if np.isinf(best):
                assert got >= 1e299
            else:
                # fp32 decision track vs float64 recomputation: a few ulp of the quantity
                assert abs(got - best) <= 1e-5 * best + 2e-6, (px, py, got, best)
            checked += 1
    assert checked == cam.width * cam.height


@pytest.mark.parametrize("seed", range(4))
def test_flips_between_precisions_are_flagged(oracle, seed):
    """Every pixel whose fp32 and fp64 oracle decisions differ (n_contrib) has a
    bound-unit margin below C_FLIP: on scenes built with decisions ON the 1/255
    threshold (tests/threshold_scenes.py) such flips exist, and the margin flags them
    while flagging only a small minority of all pixels."""
    scene, cam, pix = near_skip_scene(seed)
    a = oracle.render_fwd(cam, scene, oracle.F32)
    b = oracle.render_fwd(cam, scene, oracle.F64)
    mu = oracle.margin_bound(cam, scene, stage=False)
    differ = a["n_contrib"] != b["n_contrib"]
    assert differ.sum() >= 1, "the scene should produce fp32/fp64 decision flips"
    assert np.all(mu[differ] < C_FLIP), mu[differ]
    for px, py in pix:  # every tuned pixel is flagged, with both precisions' margins small
        assert mu[py, px] < C_FLIP
    assert (mu < C_FLIP).mean() < 0.01


def test_margin_flags_nothing_on_generic_scenes(oracle):
    """On the tiny / small configs the fp32 and fp64 decisions agree everywhere and the
    bound-unit margin flags < 0.1% of the pixels (it is not vacuous)."""
    for name in ("tiny", "small"):
        w = scenegen.make(name)
        cam, scene = w.cameras[0], w.scene
        a = oracle.render_fwd(cam, scene, oracle.F32)
        b = oracle.render_fwd(cam, scene, oracle.F64)
        np.testing.assert_array_equal(a["n_contrib"], b["n_contrib"])
        assert (oracle.margin_bound(cam, scene) < C_FLIP).mean() < 1e-3


@pytest.mark.parametrize("mode", ["F32", "MIXED"])
def test_render_pixels_equals_render_fwd(oracle, mode):
    """gsref_render_pixels (sampled parity at full size) gives exactly
    gsref_render_fwd's values, n_contrib and margin at the same pixels."""
    w = scenegen.make("small")
    cam, scene = w.cameras[0], w.scene
    m = getattr(oracle, mode)
    full = oracle.render_fwd(cam, scene, m, want_margin=True)
    rng = np.random.default_rng(9)
    px = rng.integers(0, cam.width, 500)
    py = rng.integers(0, cam.height, 500)
    s = oracle.render_pixels(cam, scene, px, py, m)
    np.testing.assert_array_equal(s["rgb"], full["rgb"][:, py, px])
    np.testing.assert_array_equal(s["depth"], full["depth"][py, px])
    np.testing.assert_array_equal(s["T_final"], full["T_final"][py, px])
    np.testing.assert_array_equal(s["n_contrib"], full["n_contrib"][py, px])
    np.testing.assert_array_equal(s["margin"], full["margin"][py, px])
    mu_full = oracle.margin_bound(cam, scene)
    np.testing.assert_array_equal(oracle.margin_bound(cam, scene, px, py), mu_full[py, px])


def test_oracle_results_independent_of_thread_count(oracle):
    """The oracle's OpenMP loops distribute independent iterations only and take every
    sum in one fixed order: 1 thread and all host threads give bit-identical outputs
    (forward, MIXED / STAGE gradients, bounds, margins)."""
    w = scenegen.make("small")
    cam, scene = w.cameras[0], w.scene
    g_rgb, g_d = scenegen.upstream_fields(2, cam.width, cam.height)
    outs = []
    n_all = oracle.set_threads(0)
    for n in (1, max(n_all, 2)):
        oracle.set_threads(n)
        f = oracle.render_fwd(cam, scene, oracle.F32, want_margin=True, want_signature=True)
        gm, sm = oracle.render_bwd(cam, scene, g_rgb, g_d, mode=oracle.MIXED)
        b = oracle.render_bwd_bound(cam, scene, g_rgb, g_d)
        mu = oracle.margin_bound(cam, scene)
        outs.append([f["rgb"], f["depth"], f["margin"], np.array([f["signature"], f["blended"]]), gm, sm, b["grad"],
                     b["bound"], mu])
    oracle.set_threads(n_all)
    for a, c in zip(*outs):
        np.testing.assert_array_equal(a, c)
