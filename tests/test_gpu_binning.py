"""Both radix-pass implementations of gs_bin_tiles (reduce-then-scan, the default,
and decoupled look-back onesweep, GSR_SORT=onesweep) give the oracle's exact
(tile, depth, index) order (-m gpu)."""
import os

import numpy as np
import pytest
import torch

import scenegen
from oracle import gsref

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_2408_12677_b200 import gsr
    from gpu_helpers import gpu_bin, gpu_project


@pytest.mark.parametrize("impl", ["onesweep", "rts"])
@pytest.mark.parametrize("name", ["small", "replica"])
def test_sort_impls_bitexact(impl, name):
    lib = gsr.load()
    kw = {"num_views": 1} if name == "replica" else {}
    w = scenegen.make(name, **kw)
    cam, scene = w.cameras[0], w.scene
    old = os.environ.get("GSR_SORT")
    os.environ["GSR_SORT"] = impl
    try:
        proj, _, _ = gpu_project(lib, cam, scene)
        out = gpu_bin(lib, cam, scene, proj)
    finally:
        if old is None:
            del os.environ["GSR_SORT"]
        else:
            os.environ["GSR_SORT"] = old
    ref = gsref.bin_tiles(cam, scene)
    assert out["K"] == ref["K"]
    np.testing.assert_array_equal(out["sorted_ids"][:out["K"]].cpu().numpy(), ref["sorted_ids"])
    np.testing.assert_array_equal(out["ranges"].cpu().numpy(), ref["tile_ranges"])
