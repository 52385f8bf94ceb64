"""bench.py's JSON line carries every key of the driver's contract (small config, a
few steps), for the GPU arm and the reference (CPU oracle) arm."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*args):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                         timeout=900, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    return json.loads(out.stdout.strip().splitlines()[-1])


def test_gpu_arm_line():
    d = _run("--config", "small", "--steps", "3", "--warmup", "3")
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e", "gpu_launches", "clocks"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3 and d["value"] > 0
    assert d["config"]["workload"] == "small"
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in d["roofline"], k
    for k in ("value", "unit", "cores", "kind", "sample"):
        assert k in d["cpu_baseline"], k
    for k in ("value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step"):
        assert k in d["e2e"], k
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] > 0
    assert "sm_mhz" in d["clocks"] and "reasons" in d["clocks"]


def test_reference_arm_line():
    d = _run("--impl", "reference", "--config", "tiny", "--steps", "1", "--warmup", "1")
    assert d["impl"] == "reference" and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["value"] == d["value"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]


def test_gpus_flag_launches_ranks_or_refuses():
    """`bench.py --gpus 2` without torchrun: two ranks when two GPUs are visible (one
    rank-0 line with n_gpus = 2), else exit 2 with a message -- never a silent 1-GPU
    number reported as 2."""
    import torch
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--config", "small", "--steps", "2",
           "--warmup", "3", "--no-cpu-baseline", "--no-naive"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    if torch.cuda.device_count() < 2:
        assert out.returncode == 2 and "GPU(s) visible" in out.stderr
    else:
        assert out.returncode == 0, out.stderr[-2000:]
        d = json.loads(out.stdout.strip().splitlines()[-1])
        assert d["n_gpus"] == 2


def test_distributed_flow_at_world_one():
    """The N > 1 bench flow (process group, the default exchange with its fallbacks and
    self-test, graph capture of the exchange, host-streamed e2e) through torchrun at
    world size 1 (GSR_FORCE_DIST=1) on the batched config."""
    env = dict(os.environ, GSR_FORCE_DIST="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=1", "--master-addr",
           "127.0.0.1", "--master-port=29561", os.path.join(ROOT, "bench.py"), "--gpus", "1", "--steps", "2",
           "--warmup", "3", "--no-cpu-baseline", "--no-naive"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=1200, cwd=ROOT, env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    d = json.loads(out.stdout.strip().splitlines()[-1])
    assert d["config"]["workload"] == "scannetpp" and d["value"] > 0 and d["e2e"]["value"] > 0
    assert "views/dp1" in d["config"]["parallelism"]
    assert any(x in d["config"]["parallelism"] for x in ("nvls", "peer", "sharded"))
