"""ctypes declarations of libcacheprune.so (include/cacheprune.h).  Marshalling only.

The product path has no fallback: importing this module without the built
library raises immediately (build it with `python -c "import __graft_entry__ as g; g.build()"`).
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libcacheprune.so")

CP_OK, CP_ERR_INVALID_ARG, CP_ERR_SENSITIVE_SPAN, CP_ERR_SPAN_TOO_SHORT = 0, -1, -2, -3
CP_ERR_CAPACITY, CP_ERR_CUDA, CP_ERR_UNSUPPORTED = -4, -5, -6
CP_FP32, CP_BF16 = 0, 1
CP_ROPE_NEOX, CP_ROPE_GPTJ = 0, 1
CP_MATCH_NO_TOUCH, CP_MATCH_FIXED_CHUNK, CP_MATCH_PREFIX_ONLY = 1, 2, 4
CP_POLICY_FIXED_CHUNK, CP_POLICY_PREFIX_ONLY = 1, 2
CP_ZERO_RECOMPUTE, CP_ZERO_UNCOVERED, CP_SKIP_LINKED, CP_REUSE_WORKLIST, CP_SKIP_RECOMPUTE = 1, 2, 4, 8, 16
CP_SCORE_INTER_INTRA, CP_SCORE_KVDEV = 0, 1
CP_STORED, CP_SUPERSEDED, CP_DUPLICATE, CP_DROPPED_CONTAINED, CP_DEFERRED_PINNED = 0, 1, 2, 3, 4
CP_WS_COUNT = 4

i32, i64, u64, vp = C.c_int32, C.c_int64, C.c_uint64, C.c_void_p
P_i32, P_i64, P_u64, P_u8, P_u32 = C.POINTER(i32), C.POINTER(i64), C.POINTER(u64), C.POINTER(C.c_uint8), C.POINTER(C.c_uint32)


class CpConfig(C.Structure):
    _fields_ = [("window_len", i32), ("block_size", i32), ("hash_seed", u64),
                ("num_layers", i32), ("num_kv_heads", i32), ("head_dim", i32),
                ("layer_offset", i32), ("head_offset", i32), ("dtype", i32), ("rope_style", i32),
                ("rope_theta", C.c_double), ("pool_capacity_tokens", i64), ("max_entries", i32),
                ("max_span_len", i32), ("max_req_tokens", i32), ("max_batch_reqs", i32),
                ("max_batch_tokens", i64), ("max_spans_per_insert", i32), ("max_sessions", i32)]


class CpBatch(C.Structure):
    _fields_ = [("num_reqs", i32), ("total_tokens", i64), ("tokens", vp), ("offsets", vp), ("mask", vp),
                ("max_req_len", i32), ("session", vp)]


class CpPagedKV(C.Structure):
    _fields_ = [("k_layers_h", C.POINTER(vp)), ("v_layers_h", C.POINTER(vp)), ("block_tables", vp),
                ("max_blocks_per_req", i32)]


class CpHits(C.Structure):
    _fields_ = [("max_hits", i32), ("num_hits", vp), ("req_hit_offsets", vp), ("hit_req", vp),
                ("hit_entry", vp), ("hit_slot", vp), ("hit_dst", vp), ("hit_len", vp), ("hit_delta", vp),
                ("plan", vp), ("req_covered", vp), ("req_recompute", vp), ("req_candidates", vp)]


class CpSnapshot(C.Structure):
    _fields_ = [("num_live", i32), ("next_id", i32), ("live_tokens", i64), ("fifo_count", i32), ("error", i32),
                ("id", vp), ("len", vp), ("origin_pos", vp), ("prefix_hash", vp), ("full_hash", vp),
                ("last_used", vp), ("digest", vp), ("pages", vp), ("tokens", vp), ("recompute", vp), ("fifo", vp),
                ("pin", vp), ("owner", vp)]


EXPORTS = {
    "cp_index_workspace": (i32, [C.POINTER(CpConfig), C.POINTER(C.c_size_t)]),
    "cp_pool_num_pages": (i64, [C.POINTER(CpConfig)]),
    "cp_max_pages_per_entry": (i32, [C.POINTER(CpConfig)]),
    "cp_index_create": (i32, [C.POINTER(CpConfig), C.POINTER(vp), vp, C.POINTER(vp)]),
    "cp_index_destroy": (i32, [vp]),
    "cp_index_create_view": (i32, [vp, i32, i32, i32, i32, vp, vp, C.POINTER(vp)]),
    "cp_index_copy_in": (i32, [vp, C.POINTER(CpBatch), C.POINTER(CpPagedKV), i32, vp]),
    "cp_index_insert": (i32, [vp, C.POINTER(CpBatch), C.POINTER(CpPagedKV), i32, vp, vp, vp, vp, vp, u64,
                              vp, vp, vp]),
    "cp_index_insert_prepare": (i32, [vp, C.POINTER(CpBatch), C.POINTER(CpPagedKV), i32, vp, vp, vp, vp, vp, u64,
                                      vp, vp, vp]),
    "cp_index_insert_commit": (i32, [vp, C.POINTER(CpBatch), C.POINTER(CpPagedKV), i32, vp, vp, vp, vp, vp, u64,
                                     vp, vp, vp]),
    "cp_index_insert_commit_rects": (i32, [vp, i32, C.POINTER(vp), C.POINTER(CpBatch), C.POINTER(CpPagedKV), i32,
                                           vp, vp, vp, vp, vp, u64, vp, vp, vp]),
    "cp_match_spans": (i32, [vp, C.POINTER(CpBatch), u64, i32, C.POINTER(CpHits), vp]),
    "cp_gather_rerotate": (i32, [vp, C.POINTER(CpBatch), C.POINTER(CpHits), C.POINTER(CpPagedKV), i32, vp]),
    "cp_gather_rerotate_rects": (i32, [vp, i32, C.POINTER(vp), C.POINTER(CpBatch), C.POINTER(CpHits),
                                       C.POINTER(CpPagedKV), i32, vp]),
    "cp_score_deviation": (i32, [i32, C.POINTER(vp), P_i32, P_i32, P_i32, P_i32, i32, i32, i32, i32,
                                 vp, P_i64, vp, P_i64, vp]),
    "cp_score_kv_deviation": (i32, [i32, P_i32, P_i32, P_i32, vp, vp, vp, i32, vp, vp, vp, i32, i32, i32, i32,
                                    i32, i32, i32, vp, P_i64, vp, P_i64, vp]),
    "cp_link_blocks": (i32, [vp, C.POINTER(CpBatch), C.POINTER(CpHits), vp, i32, vp]),
    "cp_pin_links": (i32, [vp, vp, i64, i32, vp]),
    "cp_index_set_clock": (i32, [vp, vp]),
    "cp_index_l2_persist": (i32, [vp, vp, C.c_float]),
    "cp_index_insert_session": (i32, [vp, C.POINTER(CpBatch), C.POINTER(CpPagedKV), u64, vp, vp, vp]),
    "cp_hash_prefix": (i32, [C.POINTER(CpBatch), u64, vp, vp]),
    "cp_policy_spans": (i32, [C.POINTER(CpBatch), i32, i32, i32, i32, vp, vp, vp, vp, vp, vp]),
    "cp_index_snapshot": (i32, [vp, C.POINTER(CpSnapshot), vp]),
    "cp_index_last_error": (i32, [vp, vp]),
    "cp_index_hash_base": (u64, [vp]),
    "cp_index_commit_stats": (i32, [vp, P_i32, vp]),
    "cp_index_match_work": (i32, [vp, P_u64, i32, vp]),
    "cp_kernel_launch_count": (u64, []),
    "cp_set_gather_variant": (i32, [i32]),
    "cp_set_score_variant": (i32, [i32]),
    "cp_copy_diag": (i32, [vp, vp, i64, i32, vp]),
    "cp_annotate_workspace": (C.c_size_t, [i32, P_i32, i32]),
    "cp_annotate_spans": (i32, [i32, C.POINTER(vp), P_i32, P_i32, C.POINTER(vp), i32, i32, vp, C.c_size_t,
                                vp, vp, vp, vp, vp]),
    "cp_status_string": (C.c_char_p, [i32]),
    "cp_build_info": (C.c_char_p, []),
}

_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"libcacheprune.so not built ({LIB_PATH}); run __graft_entry__.build() -- "
                               "there is no CPU fallback")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in EXPORTS.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        # provenance: the library must be the build of THESE sources (build.py source_hash)
        from .build import source_hash
        info = L.cp_build_info().decode()
        if f"cp-src-sha256={source_hash()}" not in info and os.environ.get("CP_DIAGNOSTIC_BUILD") != "1":
            raise RuntimeError(f"libcacheprune.so was built from other sources ({info}); run __graft_entry__.build()")
        _lib = L
    return _lib


class CacheHitError(RuntimeError):
    pass


def check(rc: int, what: str = ""):
    if rc != CP_OK:
        msg = lib().cp_status_string(rc).decode()
        raise CacheHitError(f"{what}: {msg} ({rc})")
    return rc
