"""B200-native ScaleSim invocation-distance memory planner (arXiv 2601.21473).

The planner runs in libscalesim.so (hand-written sm_100a CUDA behind the C ABI of
include/scalesim.h); this package is the thin Python binding (ctypes) plus the in-tree
build.  PyTorch supplies device / pinned memory, streams and process groups only.
"""
from . import _lib  # noqa: F401
from ._lib import ScaleSimError  # noqa: F401


def __getattr__(name):
    if name == "Planner":
        from .planner import Planner
        return Planner
    raise AttributeError(name)
