"""C-ABI checks that need no GPU: the library builds, loads, and exports every symbol include/*.h
declares; host-side argument validation returns synchronously (no device calls)."""
import ctypes as C
import os
import re


ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    names = set()
    for fn in os.listdir(os.path.join(ROOT, "include")):
        if fn.endswith(".h"):
            src = open(os.path.join(ROOT, "include", fn)).read()
            src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
            for m in re.finditer(r"\b(?:cp_status|int64_t|int32_t|uint64_t|size_t|const char\*)\s+(cp_\w+)\s*\(", src):
                names.add(m.group(1))
    return names


def test_library_exports_every_declared_symbol():
    import __graft_entry__ as g
    g.build()
    from paper_2605_23640_b200 import _lib as L
    lib = L.lib()
    names = declared_functions()
    assert {"cp_index_insert", "cp_match_spans", "cp_gather_rerotate", "cp_score_deviation",
            "cp_annotate_spans", "cp_annotate_workspace"} <= names
    for n in sorted(names):
        assert hasattr(lib, n), n
        assert n in L.EXPORTS, f"binding does not declare {n}"


def test_library_is_the_build_of_these_sources():
    """Build provenance: the loaded library carries the SHA-256 of the current sources and flags."""
    import __graft_entry__ as g
    g.build()
    from paper_2605_23640_b200 import _lib as L
    from paper_2605_23640_b200.build import built_hash, source_hash
    h = source_hash()
    assert re.fullmatch(r"[0-9a-f]{64}", h)
    assert built_hash() == h
    assert L.lib().cp_build_info().decode() == f"cp-src-sha256={h} arch=sm_100a"


def test_host_side_validation_without_gpu():
    from paper_2605_23640_b200 import _lib as L
    lib = L.lib()
    cfg = L.CpConfig(128, 16, 42, 32, 8, 128, 0, 0, L.CP_BF16, L.CP_ROPE_NEOX, 500000.0, 400000, 4096, 2048,
                     2048, 256, 400000, 512)
    sizes = (C.c_size_t * 4)()
    assert lib.cp_index_workspace(C.byref(cfg), sizes) == 0
    assert all(s > 0 and s % 256 == 0 for s in sizes)
    pages = lib.cp_pool_num_pages(C.byref(cfg))
    assert pages == (400000 + 2048 + 15) // 16 + (400000 + 127) // 128 + 1
    bad = L.CpConfig(*[getattr(cfg, f) for f, _ in L.CpConfig._fields_])
    bad.block_size = 32
    assert lib.cp_index_workspace(C.byref(bad), sizes) == L.CP_ERR_INVALID_ARG
    bad.block_size = 16; bad.head_dim = 100        # (d/2) not a multiple of the 8-wide bf16 vector
    assert lib.cp_index_workspace(C.byref(bad), sizes) == L.CP_ERR_INVALID_ARG
    bad.head_dim = 128; bad.max_span_len = 25600   # k_ins_scan's 8 B/token prefix array would exceed 200 KB smem
    assert lib.cp_index_workspace(C.byref(bad), sizes) == L.CP_ERR_INVALID_ARG
    bad.max_span_len = 25599; bad.max_entries = 4096
    assert lib.cp_index_workspace(C.byref(bad), sizes) == 0
    bad.max_span_len = 2048; bad.window_len = 2; bad.max_req_tokens = 20000   # long-request matcher scratch needs w >= 3
    assert lib.cp_index_workspace(C.byref(bad), sizes) == L.CP_ERR_INVALID_ARG
    bad.window_len = 3
    assert lib.cp_index_workspace(C.byref(bad), sizes) == 0
    bad.window_len = 2; bad.max_req_tokens = 10240                 # shared-memory matcher: any w
    assert lib.cp_index_workspace(C.byref(bad), sizes) == 0
    # score: KVDEV mode is not built; bad rho rejected -- both before any device call
    assert lib.cp_score_deviation(0, None, None, None, None, None, 1, 4, L.CP_SCORE_KVDEV, 1, None, None, None,
                                  None, None) == L.CP_ERR_UNSUPPORTED
    assert lib.cp_score_deviation(1, None, None, None, None, None, 5, 4, 0, 1, None, None, None, None,
                                  None) == L.CP_ERR_INVALID_ARG
    # one-launch rectangles gather: no index, too many views, a views list missing -- before any device call
    kv = (L.CpPagedKV * 2)()
    assert lib.cp_gather_rerotate_rects(None, 0, None, None, None, kv, 0, None) == L.CP_ERR_INVALID_ARG
    assert lib.cp_gather_rerotate_rects(None, 4, None, None, None, kv, 0, None) == L.CP_ERR_INVALID_ARG
    assert lib.cp_gather_rerotate_rects(None, -1, None, None, None, kv, 0, None) == L.CP_ERR_INVALID_ARG
    assert lib.cp_gather_rerotate_rects(None, 1, None, None, None, kv, 0, None) == L.CP_ERR_INVALID_ARG
    assert lib.cp_index_insert_commit_rects(None, 4, None, None, kv, 1, None, None, None, None, None, 1, None, None,
                                            None) == L.CP_ERR_INVALID_ARG
    assert lib.cp_index_insert_commit_rects(None, 0, None, None, None, 1, None, None, None, None, None, 1, None, None,
                                            None) == L.CP_ERR_INVALID_ARG
    # KV deviation (NEXT-4): bad rho, a row that is not a whole number of 16-B vectors
    args = lambda rn, H, d: (1, None, None, None, None, None, None, 1, None, None, None, 1, H, d, L.CP_BF16, rn, 20,
                             16, None, None, None, None, None)
    assert lib.cp_score_kv_deviation(*args(21, 8, 128)) == L.CP_ERR_INVALID_ARG
    assert lib.cp_score_kv_deviation(*args(3, 1, 3)) == L.CP_ERR_INVALID_ARG
    assert lib.cp_index_insert(None, None, None, 0, None, None, None, None, None, 0, None, None,
                               None) == L.CP_ERR_INVALID_ARG
    # annotator: n * heads must stay inside the int64 domain of its 2^-40 sums (n * heads < 2^22)
    dummy = (C.c_void_p * 1)(C.c_void_p(16))
    outs = [C.c_void_p(16)] * 4
    for n, h, want in [((1 << 20), 4, L.CP_ERR_INVALID_ARG), ((1 << 21), 1, L.CP_ERR_INVALID_ARG)]:
        rc = lib.cp_annotate_spans(1, dummy, (C.c_int32 * 1)(n), (C.c_int32 * 1)(h), dummy, 128, 8,
                                   C.c_void_p(16), C.c_size_t(2 ** 63), *outs, None)
        assert rc == want, (n, h, rc)
    assert lib.cp_status_string(-2) == b"CP_ERR_SENSITIVE_SPAN"


def test_product_package_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2605_23640_b200")
    for dirpath, _, files in os.walk(pkg):
        for fn in files:
            if fn.endswith((".py", ".cu", ".cuh", ".h")):
                src = open(os.path.join(dirpath, fn)).read()
                assert not re.search(r"^\s*(import|from)\s+oracle|liboracle|cp_oracle|#include .*oracle", src, re.M), fn
