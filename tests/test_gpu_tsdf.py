"""GPU TSDF fusion (gs_tsdf_allocate / gs_tsdf_integrate, NEXT-3) against the CPU oracle
(oracle/tsdf_ref.cpp) on identical synthetic depth frames (-m gpu): allocated block set,
every voxel's tsdf and weight, and the new-block / updated-voxel counts, bit for bit."""
import numpy as np
import pytest
import torch

import scenegen
from oracle import tsdf as T

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_2408_12677_b200 import gsr, pipeline
    DEV = torch.device("cuda:0")


@pytest.fixture(scope="module")
def lib():
    return gsr.load()


def _compare(vol_gpu, vol_ref):
    kg, tg, wg = vol_gpu.blocks()
    kr, tr, wr = vol_ref.dump()
    assert np.array_equal(kg, kr), f"block sets differ: {len(kg)} vs {len(kr)}"
    assert np.array_equal(wg, wr)
    assert np.array_equal(tg, tr)


def _run(lib, cams, depths, voxel=0.02, w_max=100.0, block_cap=1 << 16):
    vg = pipeline.TsdfVolume(lib, DEV, block_cap, voxel_size=voxel, w_max=w_max)
    vr = T.Volume(T.params(voxel, 6 * voxel, w_max))
    for cam, d in zip(cams, depths):
        vg.new_blocks.zero_()
        vg.updated.zero_()
        vg.integrate_frame(cam, torch.from_numpy(d).to(DEV))
        torch.cuda.synchronize()
        n_new = vr.allocate(cam, d)
        n_upd = vr.integrate(cam, d)
        assert int(vg.new_blocks.item()) == n_new
        assert int(vg.updated.item()) == n_upd
        _compare(vg, vr)
    return vg, vr


def test_tsdf_small_room_sequence_bitexact(lib):
    w = scenegen.make("replica", num_views=6)
    cams = [scenegen.camera_from_forward(160, 90, 80.0, 79.5, 44.5, -c.R_cw.T @ c.t_cw, c.R_cw[2]) for c in w.cameras]
    depths = [scenegen.render_depth(w.faces, c, noise_sigma=0.003, dropout=0.02, seed=k) for k, c in enumerate(cams)]
    vg, vr = _run(lib, cams, depths, voxel=0.02, w_max=4.0)  # w_max reached by re-seen voxels
    _, _, ws = vr.dump()
    assert ws.max() >= 2.0


def test_tsdf_plane_and_idempotent_allocation(lib):
    cam = scenegen.identity_camera(64, 48, 50.0, 31.5, 23.5)
    d = scenegen.render_depth(scenegen.plane_faces(1.1), cam)
    vg, vr = _run(lib, [cam, cam], [d, d], voxel=0.01)
    assert int(vg.new_blocks.item()) == 0  # second frame: nothing new


def test_tsdf_full_size_replica_frames(lib):
    """Full 1200x680 replica frames at 1 cm voxels (the bench's setting), 2 frames."""
    w = scenegen.make("replica", num_views=2)
    depths = [scenegen.render_depth(w.faces, c, noise_sigma=0.002, seed=k) for k, c in enumerate(w.cameras)]
    _run(lib, w.cameras, depths, voxel=0.01, block_cap=1 << 18)


def test_tsdf_capacity_overflow_visible(lib):
    cam = scenegen.identity_camera(64, 48, 50.0, 31.5, 23.5)
    d = scenegen.render_depth(scenegen.plane_faces(1.1), cam)
    vg = pipeline.TsdfVolume(lib, DEV, 4, voxel_size=0.01)
    vg.integrate_frame(cam, torch.from_numpy(d).to(DEV))
    torch.cuda.synchronize()
    assert int(vg.num_blocks.item()) > 4
    with pytest.raises(gsr.GsError):
        vg.blocks()
