"""paper_2307_12119_b200 — B200-native Green's-function thermal solver.

The product is the C-ABI shared library ``libgreentherm_b200.so`` built from
``csrc/`` (sm_100a CUDA kernels + C++ host layer). It exports the reference's
49 ``gt_*`` entry points (``include/greentherm.h``) and a batched, device-
resident extension (``include/greentherm_b200.h``). This package is the thin
Python mirror of that interface (ctypes), used by the tests and ``bench.py``;
it does no arithmetic of its own and has no CPU fallback: if the library is
missing, :func:`lib` raises.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

from .api import (  # noqa: F401
    GT_FP32,
    GT_FP64,
    BatchOpts,
    DeviceGreens,
    GreensArrays,
    GtError,
    SampleStats,
    bind,
    lib,
    library_path,
)

__all__ = ["lib", "bind", "library_path", "GreensArrays", "DeviceGreens", "BatchOpts", "SampleStats",
           "GtError", "GT_FP32", "GT_FP64"]
