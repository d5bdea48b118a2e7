"""B200-native (sm_100a) edge-partition-scheduled irregular kernels of arXiv 1605.02043.

The product is libepg.so (C ABI in include/epg.h); `epg` is its thin ctypes binding.
"""
from . import epg  # noqa: F401  (raises ImportError if libepg.so is missing)
from .epg import Context, Plan, Layout, Report, EpgError, partition_host, num_parts  # noqa: F401
