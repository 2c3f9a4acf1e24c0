"""B200-native exact triangle counting (arXiv 1706.05151 capabilities).

The product is libtrigraph_b200.so (CUDA sm_100a kernels behind the C ABI in
include/trigraph_b200.h).  ``trigraph`` mirrors the reference
``trigraph`` C++ API in Python; ``distributed`` is the one-process-per-GPU
driver (torch.distributed over NCCL).
"""
from . import trigraph  # noqa: F401  (raises if the library is not built)
from ._lib import lib as _lib_handle

_lib_handle()
