"""B200-native GSFusion rasterizer hot path (arXiv 2408.12677).

The product is the C-ABI library ``libgsr.so`` (include/gsr.h, CUDA for sm_100a);
``gsr`` is its ctypes binding and ``pipeline`` the host orchestration of one
fwd + bwd + Adam iteration.  Importing this package never loads the CPU oracle.
"""
import os

# A step keeps 8 render streams, 8 binning streams, a copy stream and a readback stream
# in flight; with the driver's default of 8 hardware work queues several of them share a
# queue and serialise falsely (config 4 host-streamed: 92 ms/step, 80.4 ms with 32,
# tools/e2e_diag4.py).  Read when the CUDA context is created, so it only takes effect
# if this package is imported before torch first touches the GPU (bench.py sets it too).
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

from . import gsr  # noqa: F401,E402

__all__ = ["gsr", "pipeline", "load"]


def load(exact: bool = False):
    """Load libgsr.so (or the GSR_EXACT_EXP debug build); raises if it was not built."""
    return gsr.load(exact)
