"""B200-native GSFusion rasterizer hot path (arXiv 2408.12677).

The product is the C-ABI library ``libgsr.so`` (include/gsr.h, CUDA for sm_100a);
``gsr`` is its ctypes binding and ``pipeline`` the host orchestration of one
fwd + bwd + Adam iteration.  Importing this package never loads the CPU oracle.
"""
from . import gsr  # noqa: F401

__all__ = ["gsr", "pipeline", "load"]


def load(exact: bool = False):
    """Load libgsr.so (or the GSR_EXACT_EXP debug build); raises if it was not built."""
    return gsr.load(exact)
