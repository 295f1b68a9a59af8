"""B200-native GCN training hot path of Morphling (arXiv 2512.01678).

The compute lives in `lib/libmorphling.so` (CUDA, sm_100a) behind the C-ABI of
include/morphling.h; `_lib` is its ctypes binding and `api` a thin object layer.
Importing this package fails if the shared library has not been built — there is
no CPU fallback.
"""
from . import _lib  # noqa: F401  (raises ImportError when the library is missing)
from .api import (Comm, Features, GCN, Graph, Plan, device_view, optimizer, pad_width,  # noqa: F401
                  partition_1d, partition_components, partition_greedy, partition_hierarchical, partition_stats,
                  relabel, stream_ptr, use_torch_allocator)

__all__ = ["Comm", "Features", "GCN", "Graph", "Plan", "device_view", "optimizer", "pad_width", "partition_1d",
           "partition_components", "partition_greedy", "partition_hierarchical", "partition_stats", "relabel",
           "stream_ptr", "use_torch_allocator"]
