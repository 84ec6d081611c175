"""B200-native CachePrune hot path: token-granular, privacy-masked KV reuse.

C-ABI library: libcacheprune.so (include/cacheprune.h).  This package is the
thin Python binding (api.py) plus the build helper (build.py).  It never
imports oracle/ and has no CPU fallback.
"""
from .api import (DeviceBatch, Hits, IndexConfig, KVIndex, KVIndexView, PagedKV, annotate_spans, hash_prefix, policy_spans,  # noqa: F401
                  kernel_launch_count, score_deviation, score_kv_deviation)
from . import _lib  # noqa: F401
