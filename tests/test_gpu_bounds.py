"""The bounds-checked build (libgsr_check.so, -DGSR_BOUNDS_CHECK) in place of
compute-sanitizer, which is closed on the GPU pool (-m gpu).

libgsr_check.so adds device asserts where kernels scatter through computed indices
(k_emit's key -> tile, k_tscatter's list position, the exchange's column indices, the
seeding's centre pixel) and validates, at every render entry point, the lists it is
given (each id in [0, P), 0 <= start <= end <= K).  A failed check prints its condition
and traps.  Each run is a subprocess with CUDA_LAUNCH_BLOCKING=1 (a trap poisons the
CUDA context):
* tools/kernel_smoke.py (every kernel family, ragged views, graphs) runs clean;
* the full-size binning tests (every config, both tile placements) run clean;
* a deliberately corrupted list (one id = P) is caught: the run fails with the check's
  message, so the checks are live.
"""
import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHECK_LIB = os.path.join(ROOT, "paper_2408_12677_b200", "libgsr_check.so")


def _run(args, timeout=900):
    if not os.path.exists(CHECK_LIB):
        pytest.fail("libgsr_check.so missing: run __graft_entry__.build()")
    env = dict(os.environ, GSR_LIB="libgsr_check.so", CUDA_LAUNCH_BLOCKING="1")
    return subprocess.run([sys.executable, *args], cwd=ROOT, env=env, capture_output=True, text=True,
                          timeout=timeout)


def test_kernel_smoke_bounds_checked():
    r = _run(["tools/kernel_smoke.py"])
    out = r.stdout + r.stderr
    assert r.returncode == 0 and "kernel smoke ok" in out, out[-3000:]
    assert "GSR_CHECK failed" not in out
    assert "libgsr_check.so" in out  # the script reports the library it loaded


def test_binning_suite_bounds_checked():
    r = _run(["-m", "pytest", "-x", "-q", "-p", "no:cacheprovider", "tests/test_gpu_binning.py"], timeout=1800)
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-3000:]
    assert "GSR_CHECK failed" not in out


_BAD = r'''
import sys
sys.path.insert(0, "tests")
import torch, scenegen
from paper_2408_12677_b200 import gsr
from gpu_helpers import DEV, gpu_project, gpu_bin
lib = gsr.load()
assert lib.path.endswith("libgsr_check.so"), lib.path
w = scenegen.make("small")
cam, scene = w.cameras[0], w.scene
proj, t, _ = gpu_project(lib, cam, scene)
b = gpu_bin(lib, cam, scene, proj)
ids = b["sorted_ids"].clone()
ids[b["K"] // 2] = scene.P  # one id past the end
H, W = cam.height, cam.width
out = [torch.empty((3, H, W), device=DEV), torch.empty((H, W), device=DEV), torch.empty((H, W), device=DEV),
       torch.empty((H, W), dtype=torch.int32, device=DEV)]
try:
    lib.render_fwd(gsr.camera(cam), gsr.scene_desc(scene.P, scene.P_stride, scene.sh_degree), proj, ids, b["ranges"],
                   *out)
    torch.cuda.synchronize()
except Exception as ex:
    print("raised", type(ex).__name__, ex)
    sys.exit(3)
print("not caught")
'''


def test_bounds_check_catches_corrupt_list():
    r = _run(["-c", _BAD], timeout=600)
    out = r.stdout + r.stderr
    assert r.returncode != 0 and "not caught" not in out, out[-3000:]
    assert "GSR_CHECK failed" in out and "ids[k]" in out, out[-3000:]
