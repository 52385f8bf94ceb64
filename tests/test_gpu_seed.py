"""GPU quadtree seeding (gs_quadtree, gs_seed_gaussians; NEXT-4) against the oracle
(oracle/seed.py + oracle/tsdf_ref.cpp) on the same frames (-m gpu): the leaf list
(order included) and every initialised parameter, bit for bit, over a sequence in
which the TSDF gate admits fewer Gaussians as the room gets observed."""
import numpy as np
import pytest
import torch

import scenegen
from oracle import seed as Q
from oracle import tsdf as T

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_2408_12677_b200 import gsr, pipeline
    DEV = torch.device("cuda:0")


@pytest.fixture(scope="module")
def lib():
    return gsr.load()


def _frame_rgb(depth, k):
    """A synthetic colour frame: smooth shading with depth edges (contrast for the quadtree)."""
    H, W = depth.shape
    yy, xx = np.mgrid[0:H, 0:W]
    base = np.stack([0.5 + 0.4 * np.sin(xx / 17.0 + k), 0.5 + 0.4 * np.cos(yy / 13.0), np.clip(depth / 5.0, 0, 1)])
    return np.clip(base, 0, 1).astype(np.float32)


@pytest.mark.parametrize("W,H,min_cell", [(160, 90, 2), (97, 61, 4)])
def test_quadtree_leaves_bitexact(lib, W, H, min_cell):
    rng = np.random.default_rng(W)
    rgb = np.clip(rng.normal(0.5, 0.2, (3, H, W)).cumsum(axis=1) / 8, 0, 1).astype(np.float32)
    sd = pipeline.Seeder(lib, W, H, DEV, threshold=0.1, min_cell=min_cell)
    for thr in (0.3, 0.1, 0.02):
        sd.threshold = thr
        sd.leaves_of(torch.from_numpy(rgb).to(DEV))
        torch.cuda.synchronize()
        n = int(sd.num_leaves.item())
        got = [tuple(r) for r in sd.leaves[:n].cpu().numpy().tolist()]
        assert got == Q.quadtree(rgb, thr, min_cell)


def test_seed_sequence_bitexact(lib):
    w = scenegen.make("replica", num_views=5)
    cams = [scenegen.camera_from_forward(160, 90, 80.0, 79.5, 44.5, -c.R_cw.T @ c.t_cw, c.R_cw[2]) for c in w.cameras]
    vs = 0.02
    vg = pipeline.TsdfVolume(lib, DEV, 1 << 16, voxel_size=vs)
    vr = T.Volume(T.params(vs, 6 * vs, 100.0))
    model = pipeline.empty_model(20000, 1, DEV)
    sd = pipeline.Seeder(lib, 160, 90, DEV, threshold=0.1, min_cell=2)
    counts = []
    for k, cam in enumerate(cams + cams[:1]):  # the first view again at the end: nothing new
        depth = scenegen.render_depth(w.faces, cam, noise_sigma=0.002, seed=k)
        rgb = _frame_rgb(depth, k)
        dg, cg = torch.from_numpy(depth).to(DEV), torch.from_numpy(rgb).to(DEV)
        vg.integrate_frame(cam, dg)
        vr.allocate(cam, depth)
        vr.integrate(cam, depth)
        P0 = model.P
        n = sd.seed_frame(cam, dg, cg, vg, model)
        keys, _, ws = vr.dump()
        ref = Q.seed(Q.quadtree(rgb, 0.1, 2), cam, depth, rgb, keys, ws, vs, vr.p.origin, 1)
        assert n == ref.shape[1]
        got = model.params[:, P0:model.P].cpu().numpy()
        np.testing.assert_array_equal(got, ref)
        counts.append(n)
    assert counts[0] > 0 and counts[-1] < counts[0] // 4  # revisited view: mostly already observed


def test_online_mapper_grows_and_fits(lib):
    """The whole incremental loop (TSDF fusion -> seeding -> keyframe-scheduled steps ->
    global passes) on a small room: the map grows from nothing, new-Gaussian counts drop
    as the room gets observed, and the colour loss of the mapped views decreases."""
    w = scenegen.make("replica", num_views=8)
    cams = [scenegen.camera_from_forward(160, 90, 80.0, 79.5, 44.5, -c.R_cw.T @ c.t_cw, c.R_cw[2]) for c in w.cameras]
    cams.append(cams[0])  # revisit the first view at the end
    gt = pipeline.GaussianModel(w.scene, DEV)
    cap = pipeline.default_capacity(pipeline.measure_keys(lib, gt, cams, DEV))
    rgbs = [t[0] for t in pipeline.render_targets(lib, gt, cams, DEV, cap)]  # stand-in for the sensor's colour
    om = pipeline.OnlineMapper(lib, cams, DEV, capacity=60000, sh_degree=0, key_capacity=1 << 21, voxel_size=0.02,
                               block_cap=1 << 16, min_cell=2, m=5, n=3, global_iters=3)
    for t, cam in enumerate(cams):
        depth = torch.from_numpy(scenegen.render_depth(w.faces, cam, noise_sigma=0.002, seed=t)).to(DEV)
        om.add_frame(t, rgbs[t].contiguous(), depth)
    P_online = om.model.P
    tr = om.trainer

    def loss():
        tot = 0.0
        for t in range(len(cams)):
            pipeline.render(lib, om.model, cams[t], tr.buf)
            tot += float((tr.buf.rgb - rgbs[t]).abs().mean())
        return tot
    before = loss()
    om.finish()
    torch.cuda.synchronize()
    tr.check_capacity()
    assert P_online > 1000 and om.model.P == P_online == sum(om.counts)
    assert om.counts[-1] < om.counts[0] // 4  # the revisited view adds little (weight gate)
    assert om.iterations == om.model.step_count > 0
    assert loss() < before
