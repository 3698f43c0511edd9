"""paper_2605_09735_b200 — B200-native KV-RM decode-step path (kvrail-b200).

The product is two in-tree shared libraries built from ``csrc/``:
``lib/libkvr_cuda.so`` (sm_100a kernels, C-ABI ``include/kvr_cuda.h``) and
``lib/libkvrail.so`` (host C++ pager / transport / driver, C-ABI
``include/kvrail_c.h``). This package only binds them (``kvrail.py``).
"""
from .kvrail import (  # noqa: F401
    ArenaStats, Device, Driver, Geometry, KvrailError, Pager, PagerConfig, StepRecord,
    WorkCounters, api, device_count, native_lib, reduce, stage,
)

__all__ = ["ArenaStats", "Device", "Driver", "Geometry", "KvrailError", "Pager", "PagerConfig",
           "StepRecord", "WorkCounters", "api", "device_count", "native_lib", "reduce", "stage"]
