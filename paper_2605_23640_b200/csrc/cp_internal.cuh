// cp_internal.cuh -- private declarations of libcacheprune (not part of the C-ABI).
//
// Device layout of an index (all inside caller-owned workspaces, see cp_index_workspace):
//   POOL_K / POOL_V : [L][P][16][H][d] dtype             (pool pages, per layer)
//   META            : DevHeader + slot-indexed entry table + page-indexed token/bit store
//                     + free-page FIFO + free-slot stack + prefix hash table + power table
//   SCRATCH         : per-call temporaries of match / gather / insert (union)
#pragma once
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>
#include <atomic>
#include "../../include/cacheprune.h"

#define CP_PMOD ((((uint64_t)1) << 61) - 1)
#define CP_EMPTY_KEY (~0ULL)
#define CP_TOMB_KEY (~0ULL - 1ULL)
#define CP_BLOCK 16
#define CP_MAX_LAYERS 128
#define CP_GATHER_CHUNK 32          // tokens per gather work item
#define CP_MATCH_SMEM_TOKENS 10240  // requests up to this length keep the matcher's arrays in shared memory
#define CP_MAX_MATCH_TOKENS (1 << 20) // longer ones (cfg.max_req_tokens > CP_MATCH_SMEM_TOKENS) use scratch
#define CP_NO_ERR_KEY (~0ULL)

// slot states
#define CP_SLOT_FREE 0
#define CP_SLOT_LIVE 1

struct __align__(32) HEntry {        // open-addressing multi-value table entry (32 B)
    unsigned long long key;          // prefix hash; CP_EMPTY_KEY / CP_TOMB_KEY are never valid hashes (< p)
    unsigned long long full;         // full-length hash of the entry (the O(1) pre-check needs no extra load)
    int32_t slot;                    // pool slot (or batch span index for the insert's batch table)
    int32_t len;                     // entry length
    unsigned long long pad;
};
static_assert(sizeof(HEntry) == 32, "HEntry must be 32 B");

struct DevHeader {                   // first 256 B of META
    int32_t error;                   // sticky cp_status (0 = none)
    int32_t next_id;
    int32_t num_live;
    int32_t fifo_head;
    int32_t fifo_count;
    int32_t slot_free_top;           // number of entries on the free-slot stack
    uint32_t match_done;             // last-block ticket of the matcher
    int32_t table_used;              // live + tombstone entries in the prefix table
    long long live_tokens;
    unsigned long long first_err;    // insert validation: min((span << 32) | code index)
    int32_t rebuild;                 // prefix table needs a rebuild
    int32_t n_cand;                  // insert: candidate relations found
    int32_t n_copy;                  // insert: entries to copy in
    int32_t n_removed;               // insert: slots removed this call
    int32_t n_chunks;                // gather/copy: work chunks
    int32_t n_new_live;
    int32_t n_cand0;                 // insert: candidates of the first scan phase
    int32_t n_need;                  // insert: spans that need the old-entry haystack scan
    unsigned long long gather_next;  // gather/copy: next work item (dynamic scheduling), reset by k_rows_prep
    int32_t commits_parallel;        // insert commits applied by the parallel path (diagnostics)
    int32_t commits_serial;          // ... and by the sequential path
    int32_t commit_why;              // OR of the reasons the sequential path was taken (k_ins_commit bits)
    int32_t n_unc;                   // gather: uncovered positions listed for CP_ZERO_UNCOVERED
    unsigned long long match_work[4];   // matcher work counters (cp_index_match_work)
    int32_t pin_neg;                 // cp_pin_links: a count went negative (undone)
    uint32_t pin_epoch;              // cp_pin_links calls so far (a prepared LRU list is stale after one)
    int32_t pad[28];
};
static_assert(sizeof(DevHeader) == 256, "DevHeader must be 256 B");

struct Rec16 { unsigned long long full; int32_t len; int32_t id; };   // bucket record (16 B)

// candidate relation found by the insert scans: needle's tokens occur in haystack at offset
struct Cand {
    int32_t hay;      // >= 0: pool slot;  < 0: new span (-1 - j)
    int32_t needle;   // >= 0: pool slot;  < 0: new span (-1 - j)
    int32_t off;
    int32_t ok;       // set by verification
};

// Host-side identity of the gather / copy-in work list now in SCRATCH (chunk list, row table, cos/sin),
// shared by an index and its pool views: a view's gather or copy-in may reuse it (CP_REUSE_WORKLIST)
// instead of rebuilding it, because the row table holds token-row indices, not geometry-dependent offsets.
struct WorkKey {
    int valid = 0;
    int dir = 0;
    const void* p[9] = {};      // count, req, slot, dst, len, delta, req_off, plan, block_tables
    int64_t cap = 0;
    int32_t max_blocks = 0, skip_linked = 0;
    bool same(const WorkKey& o) const {
        if (!valid || !o.valid || dir != o.dir || cap != o.cap || max_blocks != o.max_blocks || skip_linked != o.skip_linked)
            return false;
        for (int i = 0; i < 9; ++i) if (p[i] != o.p[i]) return false;
        return true;
    }
};

struct cp_index {
    cp_config cfg;
    int64_t P;           // physical pages
    int32_t MP;          // max pages per entry
    char* match_g = nullptr;   // matcher arrays in global scratch (only when max_req_tokens > CP_MATCH_SMEM_TOKENS)
    int insert_prepared = 0;   // cp_index_insert_prepare issued, commit pending (host-side guard)
    int is_view = 0;           // a pool view (cp_index_create_view): own geometry + pool, the base's META/SCRATCH
    WorkKey* wk = nullptr;     // owned by the base, shared by its views
    const unsigned long long* clock = nullptr;         // cp_index_set_clock (device logical time)
    cudaStream_t side = nullptr;                       // the insert's SHA-256 digests run here, beside the copy-in
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;  // (owned by the base)
    cudaEvent_t ev_pfork = nullptr, ev_pjoin = nullptr;  // the prepare's LRU branch on `side` (owned by the base)
    int32_t S;           // slots
    int64_t T;           // prefix-table entries (pow2)
    int32_t logT;
    uint64_t B, Bw;      // base and B^w
    int32_t elem;        // bytes per element
    // workspaces
    char* pool_k; char* pool_v; char* meta; char* scratch;
    size_t ws[CP_WS_COUNT];
    // META arrays
    DevHeader* hdr;
    int32_t* slot_id; int32_t* slot_len; int32_t* slot_origin; uint8_t* slot_state;
    unsigned long long* slot_prefix; unsigned long long* slot_full; unsigned long long* slot_last;
    uint8_t* slot_digest; int32_t* slot_pages; int32_t* fifo; int32_t* slot_stack;
    int32_t* page_tokens; uint16_t* page_bits; HEntry* htab; unsigned long long* pw;
    int32_t* slot_pin; int32_t* page_owner;          // R#32: linked-page pins per slot, owning slot per page
    int32_t* slot_owner; int32_t* session_slot;      // R#33: owner session per slot, private slot per session
    // SCRATCH (match)
    int64_t HS;          // sparse hit capacity
    int32_t *sp_entry, *sp_slot, *sp_dst, *sp_len, *sp_delta, *req_cnt;
    // SCRATCH (gather / copy-in work lists)
    int64_t CH;          // chunk capacity
    int32_t *chunk_hit, *chunk_t0, *hit_coff;
    int64_t* unc_list;   // [max_batch_tokens] uncovered positions (CP_ZERO_UNCOVERED)
    long long *row_src, *row_dst;   // [CH * CP_GATHER_CHUNK] element offsets; row_dst carries the plan code in bits 62-63
    float2* hit_cs;      // [hits][d/2] cos/sin
    int64_t CS_HITS;     // hits capacity of hit_cs
    // SCRATCH (insert)
    int32_t MS;          // max spans
    int64_t MAXC;        // candidate capacity
    int64_t BT; int32_t logBT;
    unsigned long long *span_pre, *span_full;
    HEntry* btab;
    Cand* cand;
    int32_t *rel_off, *rel_rec;    // CSR per span of relation records (other << 2 | kind)
    int32_t *new_slot, *removed, *rm_pos, *cp_req, *cp_slot, *cp_dst, *cp_len, *cp_delta, *out_tmp;
    int32_t* eq_old;     // [MS] span has an equal live pool entry
    HEntry* dtab;        // unique table keyed by full hash -> smallest span index (batch dedup)
    int32_t* span_rep;   // [MS] representative (smallest equal span) of each span
    char* fscr;          // parallel-apply scratch of the commit
    char* lru_scr;       // LRU candidate list prepared by cp_index_insert_prepare (k_lru_*)
    size_t meta_bytes = 0;   // size of META (cp_index_l2_persist)
    int32_t* rel_cur;    // relation CSR fill cursors (k_ins_rel_*)
    Rec16* precs;        // [MS] bucket records of the batch prefix table
};

// ---- launch bookkeeping -------------------------------------------------------------------
extern std::atomic<unsigned long long> g_cp_launches;
// SM count of the current device (grids are sized in multiples of it; 148 on B200)
inline int cp_sm_count() {
    static int n = 0;
    if (!n) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n <= 0) n = 148;
    }
    return n;
}
#define CP_COUNT_LAUNCH() (g_cp_launches.fetch_add(1, std::memory_order_relaxed))
#define CP_CUDA_CHECK(x) do { cudaError_t _e = (x); if (_e != cudaSuccess) return CP_ERR_CUDA; } while (0)

// ---- host launchers shared across translation units ---------------------------------------
// Copy or gather rows between a paged cache and the pool. dir 0: pool -> paged (gather, rotate by
// delta, plan codes honoured); dir 1: paged -> pool (copy-in, no rotation).  The hit-like list
// (req, slot, dst, len, delta) and its count live in device memory.
cp_status cp_launch_rows(cp_index* x, int dir, const int32_t* d_count, const int32_t* l_req,
                         const int32_t* l_slot, const int32_t* l_dst, const int32_t* l_len,
                         const int32_t* l_delta, int64_t list_cap, const int64_t* req_off,
                         const uint8_t* plan, const cp_paged_kv* kv, int32_t flags, cudaStream_t st,
                         int32_t nviews = 0, cp_index* const* views = nullptr, const cp_paged_kv* view_kvs = nullptr);
inline void cp_invalidate_worklist(cp_index* x) { if (x && x->wk) x->wk->valid = 0; }

// ---- device helpers ---------------------------------------------------------------------------
__device__ __forceinline__ uint64_t cp_mulmod(uint64_t a, uint64_t b) {
    // a, b < p = 2^61-1.  a*b = hi*2^64 + lo, 2^64 = 8 * 2^61 = 8 (mod p).
    uint64_t lo = a * b;
    uint64_t hi = __umul64hi(a, b);
    uint64_t r = (lo & CP_PMOD) + (lo >> 61) + (hi << 3);
    r = (r & CP_PMOD) + (r >> 61);
    return r >= CP_PMOD ? r - CP_PMOD : r;
}
__device__ __forceinline__ uint64_t cp_addmod(uint64_t a, uint64_t b) {
    uint64_t r = a + b;
    return r >= CP_PMOD ? r - CP_PMOD : r;
}
__device__ __forceinline__ uint64_t cp_submod(uint64_t a, uint64_t b) {
    return a >= b ? a - b : a + CP_PMOD - b;
}
__device__ __forceinline__ uint64_t cp_tokval(int32_t t) { return (uint64_t)(int64_t)t + 1ULL; }

// substring hash of positions [k, k+m) from a prefix array h[0..n]
__device__ __forceinline__ uint64_t cp_subhash(const uint64_t* h, int k, int m, uint64_t Bm) {
    return cp_submod(h[k + m], cp_mulmod(h[k], Bm));
}

__device__ __forceinline__ uint32_t cp_hpos(uint64_t key, int logT) {
    return (uint32_t)((key * 0x9E3779B97F4A7C15ULL) >> (64 - logT));
}

// Block-wide prefix hashes h[0..n] of tokens tok(i), i < n, into shared memory `sh` (n+1 values).
// Parallel scan of (hash, B^len) pairs: (h1,p1) o (h2,p2) = (h1*p2 + h2, p1*p2).  `wtmp` must hold
// 2 * (NT/32) u64 in shared memory.  Ends with __syncthreads().
template <int NT, typename F>
__device__ void cp_block_prefix_hash(F tok, int n, uint64_t B, uint64_t* sh, uint64_t* wtmp) {
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int c = (n + NT - 1) / NT;
    const int c0 = min(n, tid * c), c1 = min(n, c0 + c);
    uint64_t hh = 0, pp = 1;
    for (int i = c0; i < c1; ++i) { hh = cp_addmod(cp_mulmod(hh, B), cp_tokval(tok(i))); pp = cp_mulmod(pp, B); }
    // warp inclusive scan
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        uint64_t h2 = __shfl_up_sync(0xffffffffu, hh, off);
        uint64_t p2 = __shfl_up_sync(0xffffffffu, pp, off);
        if (lane >= off) { hh = cp_addmod(cp_mulmod(h2, pp), hh); pp = cp_mulmod(p2, pp); }
    }
    if (lane == 31) { wtmp[2 * wid] = hh; wtmp[2 * wid + 1] = pp; }
    __syncthreads();
    if (wid == 0) {
        constexpr int NW = NT / 32;
        uint64_t wh = lane < NW ? wtmp[2 * lane] : 0, wp = lane < NW ? wtmp[2 * lane + 1] : 1;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            uint64_t h2 = __shfl_up_sync(0xffffffffu, wh, off);
            uint64_t p2 = __shfl_up_sync(0xffffffffu, wp, off);
            if (lane >= off) { wh = cp_addmod(cp_mulmod(h2, wp), wh); wp = cp_mulmod(p2, wp); }
        }
        // exclusive
        uint64_t eh = __shfl_up_sync(0xffffffffu, wh, 1), ep = __shfl_up_sync(0xffffffffu, wp, 1);
        if (lane == 0) { eh = 0; ep = 1; }
        if (lane < NW) { wtmp[2 * lane] = eh; wtmp[2 * lane + 1] = ep; }
    }
    __syncthreads();
    // thread exclusive prefix = warp_excl o lane_excl
    uint64_t lh = __shfl_up_sync(0xffffffffu, hh, 1), lp = __shfl_up_sync(0xffffffffu, pp, 1);
    if (lane == 0) { lh = 0; lp = 1; }
    uint64_t weh = wtmp[2 * wid];
    uint64_t start = cp_addmod(cp_mulmod(weh, lp), lh);
    (void)lp;
    uint64_t cur = start;
    if (tid == 0) sh[0] = 0;
    for (int i = c0; i < c1; ++i) { cur = cp_addmod(cp_mulmod(cur, B), cp_tokval(tok(i))); sh[i + 1] = cur; }
    __syncthreads();
}


// ---- unique-key tables (find-or-insert: contention only on the first insert of a key) -----------

__device__ __forceinline__ HEntry* cp_find_or_insert(HEntry* tab, uint32_t mask, int logT, uint64_t key) {
    uint32_t pos = (uint32_t)((key * 0x9E3779B97F4A7C15ULL) >> (64 - logT));
    while (true) {
        const unsigned long long k = *((volatile unsigned long long*)&tab[pos].key);
        if (k == key) return &tab[pos];
        if (k == CP_EMPTY_KEY) {
            const unsigned long long prev = atomicCAS(&tab[pos].key, CP_EMPTY_KEY, (unsigned long long)key);
            if (prev == CP_EMPTY_KEY || prev == key) return &tab[pos];
        }
        pos = (pos + 1) & mask;
    }
}
__device__ __forceinline__ const HEntry* cp_find_unique(const HEntry* tab, uint32_t mask, int logT, uint64_t key) {
    uint32_t pos = (uint32_t)((key * 0x9E3779B97F4A7C15ULL) >> (64 - logT));
    while (true) {
        const unsigned long long k = tab[pos].key;
        if (k == key) return &tab[pos];
        if (k == CP_EMPTY_KEY) return nullptr;
        pos = (pos + 1) & mask;
    }
}

// Warp-level probe of a bucketed multi-value table (unique keys -> [offset, count) into `recs`):
// each lane finds its bucket; small buckets are walked per lane, large ones (hundreds of spans
// sharing one system-prompt window) by the whole warp, 32 records per step.
// on_match(owner_lane, full, len, id) is invoked by the lane that loaded the record.
template <typename F>
__device__ __forceinline__ void cp_warp_bucket_probe(const HEntry* tab, uint32_t mask, int logT, const Rec16* recs,
                                                     uint64_t key, bool active, F on_match) {
    const int lane = threadIdx.x & 31;
    int off = 0, cnt = 0;
    if (active) {
        const HEntry* e = cp_find_unique(tab, mask, logT, key);
        if (e) { off = e->slot; cnt = e->len; }
    }
    if (cnt <= 4) for (int i = 0; i < cnt; ++i) { const Rec16 r = recs[off + i]; on_match(lane, r.full, r.len, r.id); }
    unsigned pend = __ballot_sync(0xffffffffu, cnt > 4);
    while (pend) {
        const int owner = __ffs(pend) - 1;
        pend &= pend - 1;
        const int o = __shfl_sync(0xffffffffu, off, owner), c = __shfl_sync(0xffffffffu, cnt, owner);
        for (int b = 0; b < c; b += 32)
            if (b + lane < c) { const Rec16 r = recs[o + b + lane]; on_match(owner, r.full, r.len, r.id); }
    }
}

// ---- hash-table probing ----------------------------------------------------------------------
__device__ __forceinline__ HEntry cp_ld_entry(const HEntry* p) {
    const ulonglong4 v = *reinterpret_cast<const ulonglong4*>(p);
    HEntry e;
    e.key = v.x; e.full = v.y; e.slot = (int32_t)(v.z & 0xffffffffu); e.len = (int32_t)(v.z >> 32); e.pad = 0;
    return e;
}
__device__ __forceinline__ HEntry cp_ldg_entry(const HEntry* p) {
    const ulonglong2 a = __ldg(reinterpret_cast<const ulonglong2*>(p));
    const ulonglong2 b = __ldg(reinterpret_cast<const ulonglong2*>(p) + 1);
    HEntry e;
    e.key = a.x; e.full = a.y; e.slot = (int32_t)(b.x & 0xffffffffu); e.len = (int32_t)(b.x >> 32); e.pad = 0;
    return e;
}

// Warp-level multi-value probe.  Every lane may carry one key (`active`).  Short chains are
// walked per lane (up to kShort slots); lanes whose chain is longer (e.g. the hundreds of stored
// segments that share one system-prompt window) are then served one at a time by the whole warp,
// 32 consecutive entries per step with __ballot_sync.  on_match(owner_lane, entry) is invoked by
// the lane that loaded a matching entry, in no particular order.  All 32 lanes must call it.
template <bool LDG, typename F>
__device__ __forceinline__ void cp_warp_probe(const HEntry* tab, uint32_t mask, int logT, uint64_t key,
                                              bool active, F on_match) {
    constexpr int kShort = 4;
    const int lane = threadIdx.x & 31;
    uint32_t pos = active ? cp_hpos(key, logT) : 0;
    bool done = !active;
    for (int s = 0; s < kShort && !done; ++s) {
        const HEntry e = LDG ? cp_ldg_entry(tab + pos) : cp_ld_entry(tab + pos);
        if (e.key == CP_EMPTY_KEY) { done = true; break; }
        if (e.key == key) on_match(lane, e);
        pos = (pos + 1) & mask;
    }
    unsigned pend = __ballot_sync(0xffffffffu, !done);
    while (pend) {
        const int owner = __ffs(pend) - 1;
        pend &= pend - 1;
        const uint64_t k = __shfl_sync(0xffffffffu, key, owner);
        uint32_t p0 = __shfl_sync(0xffffffffu, pos, owner);
        while (true) {
            const uint32_t p = (p0 + lane) & mask;
            const HEntry e = LDG ? cp_ldg_entry(tab + p) : cp_ld_entry(tab + p);
            const unsigned empt = __ballot_sync(0xffffffffu, e.key == CP_EMPTY_KEY);
            const int lim = empt ? __ffs(empt) - 1 : 32;
            if (lane < lim && e.key == k) on_match(owner, e);
            if (empt) break;
            p0 = (p0 + 32) & mask;
        }
    }
}

// Warp-cooperative insert of one entry (all lanes call with the same arguments): claims the first
// EMPTY (or TOMB when allow_tomb) slot of the probe sequence with atomicCAS on the key.
// Returns true (on every lane) if an EMPTY slot (not a tombstone) was consumed.
__device__ __forceinline__ bool cp_warp_insert(HEntry* tab, uint32_t mask, int logT, const HEntry& val,
                                               bool allow_tomb) {
    const int lane = threadIdx.x & 31;
    uint32_t p0 = cp_hpos(val.key, logT);
    while (true) {
        const uint32_t p = (p0 + lane) & mask;
        const unsigned long long k = *((volatile unsigned long long*)&tab[p].key);
        unsigned cand = __ballot_sync(0xffffffffu, k == CP_EMPTY_KEY || (allow_tomb && k == CP_TOMB_KEY));
        // always the FIRST free slot of the probe sequence: linear probing stops at the first EMPTY,
        // so an entry placed after an EMPTY of its own sequence would be unreachable
        while (cand) {
            const int l = __ffs(cand) - 1;
            int won = 0, was_empty = 0;
            if (lane == l) {
                const unsigned long long prev = atomicCAS(&tab[p].key, k, val.key);
                if (prev == k) {
                    tab[p].full = val.full; tab[p].slot = val.slot; tab[p].len = val.len;
                    won = 1; was_empty = (k == CP_EMPTY_KEY);
                }
            }
            won = __shfl_sync(0xffffffffu, won, l);
            if (won) return __shfl_sync(0xffffffffu, was_empty, l);
            cand &= cand - 1;           // lost the race: that slot is taken now, the next free one is first
        }
        p0 = (p0 + 32) & mask;
    }
}

__device__ __forceinline__ bool cp_err_set(const DevHeader* hdr) {
    return *((volatile const int32_t*)&hdr->error) != 0;
}
__device__ __forceinline__ void cp_raise(DevHeader* hdr, int32_t code) {
    atomicCAS(&hdr->error, 0, code);
}
