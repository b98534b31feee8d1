"""B200-native DCP head of F2C (arXiv 2105.10375).

Thin Python binding over the C ABI of ``libf2c_dcp.so`` (``include/f2c_dcp.h``):
argument marshalling only -- every step of the hot path runs in the library's
CUDA kernels.  PyTorch provides device memory, streams and process groups.
There is no CPU fallback: constructing a head without the built library or
without an sm_100 device raises.
"""
from .dcp import (BF16, F32, PHI_MAX, PHI_MEAN, PHI_SUM, DCPError, DCPHead, gnet_ema, lib_path,
                  load_library, nccl_unique_id)

__all__ = ["BF16", "F32", "PHI_MAX", "PHI_MEAN", "PHI_SUM", "DCPError", "DCPHead", "gnet_ema", "lib_path", "load_library",
           "nccl_unique_id"]
