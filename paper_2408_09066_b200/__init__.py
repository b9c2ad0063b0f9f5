"""B200-native (sm_100a) VSA-OGM hot path: encode/bundle -> decode -> local entropy.

See include/vsaogm.h for the C ABI and DESIGN.md for the design.  The Python
surface is the thin binding in ``vsaogm.py`` plus the multi-GPU sharding
helpers in ``parallel.py``.
"""
from .vsaogm import (BF16, F16, IO_SLOTS, KERNELS, Mapper, VsaogmError, load, strerror, test_gemm)  # noqa: F401

__all__ = ["Mapper", "VsaogmError", "F16", "BF16", "IO_SLOTS", "KERNELS", "load", "strerror", "test_gemm"]
