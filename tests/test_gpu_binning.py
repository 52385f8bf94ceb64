"""Every placement implementation of gs_bin_tiles gives the oracle's exact (tile,
depth, index) order (-m gpu): the default bucket placement by tile (k_tcount /
k_tscan / k_tstart / k_tscatter), and the two 8-bit radix passes (GSR_TILE_SORT=radix)
with decoupled look-back onesweep (default) or reduce-then-scan (GSR_SORT=rts)."""
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


IMPLS = {"bucket": {}, "radix-onesweep": {"GSR_TILE_SORT": "radix"},
         "radix-rts": {"GSR_TILE_SORT": "radix", "GSR_SORT": "rts"}}


@pytest.mark.parametrize("impl", list(IMPLS))
@pytest.mark.parametrize("name", ["tiny", "small", "replica", "scannetpp"])
def test_sort_impls_bitexact(impl, name):
    lib = gsr.load()
    kw = {"num_views": 1} if name in ("replica", "scannetpp") else {}
    w = scenegen.make(name, **kw)
    cam, scene = w.cameras[0], w.scene
    old = {k: os.environ.get(k) for k in ("GSR_TILE_SORT", "GSR_SORT")}
    for k in old:
        os.environ.pop(k, None)
    os.environ.update(IMPLS[impl])
    try:
        proj, _, _ = gpu_project(lib, cam, scene)
        out = gpu_bin(lib, cam, scene, proj)
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    ref = gsref.bin_tiles(cam, scene)
    assert out["K"] == ref["K"]
    np.testing.assert_array_equal(out["sorted_ids"][:out["K"]].cpu().numpy(), ref["sorted_ids"])
    np.testing.assert_array_equal(out["ranges"].cpu().numpy(), ref["tile_ranges"])
