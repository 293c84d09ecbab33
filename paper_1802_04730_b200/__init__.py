"""tc-b200 — a B200-native (sm_100a) execution path for the Tensor
Comprehensions benchmark operators of arXiv 1802.04730.

The product is the C ABI shared library libtcb.so (include/tcb.h): a C++
runtime (TC front end, shape inference, operator recognition, MappingOptions,
TCCACHE-compatible compilation cache, GPU genetic autotuner) over
hand-written CUDA kernels. This package is its Python mirror of the paper's
ExecutionEngine API.
"""
from ._lib import TcError, lib  # noqa: F401  (raises ImportError if libtcb.so is not built)
from .engine import (ExecutionEngine, cache_deserialize, cache_load, cache_purge, cache_save,  # noqa: F401
                     cache_entries, cache_serialize, cache_set_history, cache_size, device_info, fill_uniform,
                     measure_peaks, options_baseline, options_digest, options_normalize, options_validate, tensor_file_read,
                     tensor_file_write, version)

__all__ = [
    "ExecutionEngine", "TcError", "cache_load", "cache_save", "cache_size", "cache_purge",
    "cache_set_history", "cache_serialize", "cache_deserialize", "fill_uniform",
    "options_baseline", "options_digest", "options_normalize", "options_validate", "version",
    "device_info", "measure_peaks", "tensor_file_read", "tensor_file_write", "cache_entries",
]
