"""B200-native (sm_100a) FlashSparse hot path: CSR -> ME-BCRS conversion,
SpMM and SDDMM with the 8x1 swap-and-transpose strategy.

The product is the C-ABI shared library ``libtcsparse_b200.so`` (sources in
``csrc/``, header ``include/tcs/tcs.h``, C++ drop-in adapter
``include/tcsparse/gpu.hpp``).  ``tcsparse`` is its Python front end on
torch CUDA tensors and ``distributed`` the row-window sharding layer.
"""
from . import _abi  # noqa: F401

__all__ = ["tcsparse", "distributed", "graphs"]
