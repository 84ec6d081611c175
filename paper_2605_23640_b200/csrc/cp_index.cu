// cp_index.cu -- index lifecycle and cp_index_insert (§4.3.5 KV Pool).
//
// Insert pipeline (one call, stream ordered; the sequential semantics of DESIGN.md R#20-22 are
// reproduced exactly: spans are applied in input order):
//   k_ins_validate  warp per span: range / length / budget / mask checks (no side effects on error)
//   k_ins_hash      warp per span: prefix (first w) and full polynomial hashes; batch prefix table
//   k_ins_scan      CTA per haystack (new span or live entry): rolling windows probe the batch table
//                   and (for new spans) the pool's prefix table -> containment candidates
//   k_ins_verify    warp per candidate: exact token comparison
//   k_ins_commit    one CTA: Duplicate -> Contained -> Supersede -> store -> LRU evict, in order
//   k_ins_delete / k_ins_publish  table tombstones / inserts, token + bit store, SHA-256 digests
//   copy-in         cp_launch_rows(dir = 1): writer paged KV -> pool pages (no rotation)
#include "cp_internal.cuh"
#include <algorithm>
#include <climits>
#include <cstdlib>
#include <cstring>
#include <vector>

std::atomic<unsigned long long> g_cp_launches{0};

namespace {

constexpr int kValThreads = 256;
constexpr int kScanThreads = 256;
constexpr int kCommitThreads = 1024;
constexpr int kCommitRecCap = 8192;
constexpr int kLruK = 4096;            // prepared LRU candidates (the commit's list capacity, candK <= this)
constexpr int kLruBins = 2048;         // 11-bit radix digits; at most 3 passes (compact keys <= 33 bits)

int64_t next_pow2(int64_t v) { int64_t p = 1; while (p < v) p <<= 1; return p; }
int ilog2(int64_t v) { int l = 0; while ((1LL << l) < v) ++l; return l; }
size_t al(size_t v) { return (v + 255) & ~(size_t)255; }

uint64_t host_splitmix64(uint64_t x) {
    uint64_t z = x + 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
uint64_t host_mulmod(uint64_t a, uint64_t b) {
    unsigned __int128 x = (unsigned __int128)a * b;
    uint64_t lo = (uint64_t)x & CP_PMOD, hi = (uint64_t)(x >> 61);
    uint64_t r = lo + hi;
    r = (r & CP_PMOD) + (r >> 61);
    return r >= CP_PMOD ? r - CP_PMOD : r;
}

struct Layout {
    int64_t P; int32_t MP, S; int64_t T; int logT;
    int64_t HS, CH, CS_HITS; int32_t MS; int64_t MAXC, BT; int logBT;
    size_t meta_off[20]; size_t meta_size;
    size_t scr_off[40]; size_t scr_size;
};

bool valid_cfg(const cp_config* c) {
    if (!c) return false;
    if (c->window_len < 1 || c->block_size != CP_BLOCK) return false;
    if (c->num_layers < 1 || c->num_layers > CP_MAX_LAYERS || c->num_kv_heads < 1 || c->head_dim < 2) return false;
    if (c->dtype != CP_FP32 && c->dtype != CP_BF16) return false;
    const int vec = c->dtype == CP_FP32 ? 4 : 8;
    if (c->rope_style == CP_ROPE_NEOX) { if ((c->head_dim / 2) % vec != 0 || c->head_dim % 2) return false; }
    else if (c->rope_style == CP_ROPE_GPTJ) { if (c->head_dim % (2 * vec) != 0) return false; }
    else return false;
    if (c->head_dim > 512) return false;
    if (c->pool_capacity_tokens < c->window_len) return false;
    if (c->max_entries < 1 || c->max_entries > 131072) return false;
    // k_ins_scan keeps a span's prefix hashes (8 B per token) in <= 200 KB of shared memory
    if (c->max_span_len < c->window_len || c->max_span_len > 200 * 1024 / 8 - 1) return false;
    if (c->max_req_tokens < 1 || c->max_req_tokens > CP_MAX_MATCH_TOKENS) return false;
    // long requests keep the matcher arrays in 24 B/token of scratch: 20 n + 12 (n/w + 1) + 8 fits only for w >= 3
    if (c->max_req_tokens > CP_MATCH_SMEM_TOKENS && c->window_len < 3) return false;
    if (c->max_batch_reqs < 1 || c->max_batch_tokens < 1 || c->max_spans_per_insert < 1) return false;
    if (c->max_sessions < 0 || c->max_sessions > (1 << 20)) return false;
    if (c->max_spans_per_insert > 16384) return false;
    if (!(c->rope_theta > 0)) return false;
    return true;
}

void compute_layout(const cp_config* c, Layout* L) {
    L->P = cp_pool_num_pages(c);
    L->MP = cp_max_pages_per_entry(c);
    L->S = c->max_entries;
    L->T = next_pow2(std::max<int64_t>(64, 4LL * L->S));
    L->logT = ilog2(L->T);
    const int64_t S = L->S, P = L->P, MP = L->MP;
    size_t o = 0, i = 0;
    auto put = [&](size_t bytes) { L->meta_off[i++] = o; o += al(bytes); };
    put(sizeof(DevHeader));                  // 0 hdr
    put(4 * S); put(4 * S); put(4 * S); put(1 * S);          // 1 id 2 len 3 origin 4 state
    put(8 * S); put(8 * S); put(8 * S);                      // 5 prefix 6 full 7 last
    put(32 * S);                                             // 8 digest
    put(4 * S * MP);                                         // 9 pages
    put(4 * P);                                              // 10 fifo
    put(4 * S);                                              // 11 slot stack
    put(4 * CP_BLOCK * P);                                   // 12 page tokens
    put(2 * P);                                              // 13 page bits
    put(sizeof(HEntry) * L->T);                              // 14 htab
    put(8 * (size_t)(c->max_span_len + 1));                  // 15 pow table
    put(4 * S);                                              // 16 slot pins (R#32)
    put(4 * P);                                              // 17 page owner slot
    put(4 * S);                                              // 18 slot owner: 0 shared, s session (R#33)
    put(4 * ((size_t)c->max_sessions + 1));                  // 19 session -> its private slot
    L->meta_size = o;
    // scratch
    L->HS = c->max_batch_tokens / c->window_len + c->max_batch_reqs + 1;
    L->MS = c->max_spans_per_insert;
    L->CH = c->max_batch_tokens / CP_GATHER_CHUNK + std::max<int64_t>(L->HS, L->MS) + 1;
    L->CS_HITS = std::max<int64_t>(L->HS, L->MS);
    L->MAXC = 16LL * L->MS + 4096;
    L->BT = next_pow2(std::max<int64_t>(64, 4LL * L->MS));
    L->logBT = ilog2(L->BT);
    o = 0; i = 0;
    auto sput = [&](size_t bytes) { L->scr_off[i++] = o; o += al(bytes); };
    for (int k = 0; k < 5; ++k) sput(4 * L->HS);             // 0-4 sp_entry sp_slot sp_dst sp_len sp_delta
    sput(4 * (size_t)c->max_batch_reqs);                     // 5 req_cnt
    sput(4 * L->CH); sput(4 * L->CH);                        // 6 chunk_hit 7 chunk_t0
    sput(sizeof(float2) * L->CS_HITS * (size_t)(c->head_dim / 2));   // 8 hit_cs
    sput(8 * (size_t)L->MS); sput(8 * (size_t)L->MS);        // 9 span_pre 10 span_full
    sput(sizeof(HEntry) * L->BT);                            // 11 btab
    sput(sizeof(Cand) * L->MAXC);                            // 12 cand
    sput(4 * (size_t)(L->MS + 1));                           // 13 rel_off
    sput(8 * (size_t)(2 * L->MAXC));                         // 14 rel_rec (int2)
    sput(4 * (size_t)L->MS);                                 // 15 new_slot
    sput(4 * (size_t)(S + L->MS));                           // 16 removed
    for (int k = 0; k < 5; ++k) sput(4 * (size_t)L->MS);     // 17-21 cp_req cp_slot cp_dst cp_len cp_delta
    sput(4 * (size_t)L->MS);                                 // 22 out_tmp
    sput(8 * (size_t)L->CH * CP_GATHER_CHUNK);               // 23 row_src
    sput(8 * (size_t)L->CH * CP_GATHER_CHUNK);               // 24 row_dst
    sput(4 * (size_t)L->MS);                                 // 25 eq_old
    sput(sizeof(HEntry) * L->BT);                            // 26 dtab
    sput(4 * (size_t)L->MS);                                 // 27 span_rep
    sput(sizeof(Rec16) * (size_t)L->MS);                     // 28 precs
    sput(4 * (size_t)(S + L->MS));                           // 29 rm_pos (FIFO tail position per removal)
    // 30 matcher arrays for long requests: request r at 24 * offsets[r] + 64 * r (cp_match.cu)
    sput(c->max_req_tokens > CP_MATCH_SMEM_TOKENS ? 24 * (size_t)c->max_batch_tokens + 64 * (size_t)c->max_batch_reqs + 64 : 16);
    // 31 parallel-apply scratch: 12 int32 + 1 int64 arrays of MS + 1, 4 int32 arrays of S, 4 int32 + 1 int64 of 4097
    sput(4 * (size_t)(L->MS + 1) * 12 + 8 * (size_t)(L->MS + 1) + 4 * (size_t)S * 4 + 4 * 4097 * 4 + 8 * 4097 + 64);
    sput(4 * (size_t)(std::max<int64_t>(L->HS, L->MS) + 1));                 // 32 hit_coff (gather / copy-in)
    sput(8 * (size_t)c->max_batch_tokens);                                   // 33 unc_list (CP_ZERO_UNCOVERED)
    // 34 prepared LRU list (k_lru_*): header, per-slot key snapshot, 3 x 2048-bin histograms, list /
    // rank / sorted of kLruK candidates
    sput(64 + 8 * (size_t)S + 4 * 3 * kLruBins + 8 * kLruK + 4 * kLruK + 8 * kLruK + 64);
    sput(4 * (size_t)(L->MS + 1));                                           // 35 rel_cur (relation CSR fill cursors)
    L->scr_size = o;
}

// ------------------------------------------------------------------------------------------
// kernels: initialisation
// ------------------------------------------------------------------------------------------
__global__ void k_init(DevHeader* hdr, int32_t* slot_id, uint8_t* slot_state, int32_t* fifo, int32_t* slot_stack,
                       HEntry* htab, int64_t P, int32_t S, int64_t T, int32_t* slot_pin, int32_t* page_owner,
                       int32_t* slot_owner, int32_t* session_slot, int32_t nsess) {
    const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x, nt = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = tid; i < P; i += nt) { fifo[i] = (int32_t)i; page_owner[i] = -1; }   // FIFO: ascending (R#22)
    for (int64_t i = tid; i < S; i += nt) {
        slot_id[i] = -1; slot_state[i] = CP_SLOT_FREE; slot_stack[i] = S - 1 - (int32_t)i; slot_pin[i] = 0;
        slot_owner[i] = 0;
    }
    for (int64_t i = tid; i <= nsess; i += nt) session_slot[i] = -1;
    for (int64_t i = tid; i < T; i += nt) { htab[i].key = CP_EMPTY_KEY; htab[i].full = 0; htab[i].slot = -1; htab[i].len = 0; }
    if (tid == 0) {
        hdr->error = 0; hdr->next_id = 0; hdr->num_live = 0; hdr->fifo_head = 0; hdr->fifo_count = (int32_t)P;
        hdr->slot_free_top = S; hdr->match_done = 0; hdr->table_used = 0; hdr->live_tokens = 0;
        hdr->first_err = CP_NO_ERR_KEY; hdr->rebuild = 0; hdr->n_cand = 0; hdr->n_copy = 0; hdr->n_removed = 0;
        hdr->n_chunks = 0; hdr->n_new_live = 0; hdr->commits_parallel = 0; hdr->commits_serial = 0; hdr->commit_why = 0; hdr->pin_neg = 0;
        for (int i = 0; i < 4; ++i) hdr->match_work[i] = 0;
    }
}

// ------------------------------------------------------------------------------------------
// kernels: insert
// ------------------------------------------------------------------------------------------
// LRU candidate list prepared beside match + gather (k_lru_*, cp_index_insert_prepare): the K smallest
// (last_used, id) keys of the live unpinned entries of a snapshot, sorted
struct LruHdr {
    unsigned long long minl, maxl;   // last_used range of the snapshot's evictable entries
    unsigned idmin, idmax;           // their id range
    int valid;                       // 1: the list below is usable by the commit that follows
    int count;                       // entries with compact key <= the K-th smallest (<= K)
    int all;                         // fewer evictable entries than K: all of them are listed
    uint32_t pin_epoch;              // hdr->pin_epoch at the snapshot
};

struct InsArgs {
    DevHeader* hdr;
    const int32_t* tokens; const int64_t* offsets; const uint8_t* mask; int32_t num_reqs;
    int32_t S; const int32_t* span_req; const int32_t* span_begin; const int32_t* span_len;
    const uint32_t* bits; const int64_t* bits_off;
    uint64_t t; int32_t w; uint64_t B; int64_t capacity; int32_t max_span_len;
    int32_t* out_id; int32_t* out_oc;
    // index
    int32_t nslots; int64_t P; int32_t MP;
    int32_t* slot_id; int32_t* slot_len; int32_t* slot_origin; uint8_t* slot_state;
    unsigned long long* slot_prefix; unsigned long long* slot_full; unsigned long long* slot_last;
    uint8_t* slot_digest; int32_t* slot_pages; int32_t* fifo; int32_t* slot_stack;
    int32_t* page_tokens; uint16_t* page_bits; HEntry* htab; int logT; int64_t T; const unsigned long long* pw;
    const int32_t* slot_pin; int32_t* page_owner;     // R#32 pins, page -> owning slot
    int32_t* slot_owner;                              // R#33: 0 shared, s = private entry of session s
    const int32_t* session; int32_t* session_slot; int32_t max_sessions;   // cp_index_insert_session
    // scratch
    unsigned long long* span_pre; unsigned long long* span_full; HEntry* btab; int logBT; int64_t BT;
    Cand* cand; int64_t MAXC; int32_t* rel_off; int2* rel_rec; int32_t* new_slot; int32_t* removed; int32_t* rm_pos;
    int32_t* cp_req; int32_t* cp_slot; int32_t* cp_dst; int32_t* cp_len; int32_t* cp_delta; int32_t* out_tmp;
    int32_t* eq_old; HEntry* dtab; int32_t* span_rep; Rec16* precs;
    int64_t CH;             // copy-in chunk capacity (scratch)
    int32_t max_blocks;     // writer block-table width
    // parallel-apply scratch (k_ins_commit fast path): per span / per store [MS + 1], per slot [nslots],
    // per filtered LRU candidate [candK + 1]
    int32_t *f_last, *f_kind, *f_target, *f_supcnt, *f_suptok, *f_suppg, *f_sidx;
    int32_t *f_sj, *f_pgpref, *f_rmpref, *f_suppgpref, *f_vk;
    long long* f_netpref;
    int32_t *f_refs, *f_evpos, *f_maxpos, *f_supby;
    int32_t *f_vslot, *f_vlen, *f_vcpg, *f_vfc;
    long long* f_vcum;
    int32_t force_serial;   // CP_COMMIT_SERIAL=1: skip the parallel apply (A/B measurement, tests)
    const unsigned long long* clock;   // cp_index_set_clock: logical time read on the device (else t)
    int32_t candK;          // LRU candidate list size in the commit's shared memory (power of two, or 0)
    LruHdr* lru; unsigned long long* lru_key; unsigned* lru_hist; unsigned long long* lru_list;
    unsigned* lru_rank; unsigned long long* lru_sorted;
    int32_t* rel_cur;       // relation CSR fill cursors (k_ins_rel_*)
    int32_t rec_cap;        // relation records cached in the commit's shared memory
};

// error codes are ordered per span: range -> too short -> capacity -> sensitive (same order as the oracle)
__device__ __forceinline__ int32_t code_of(int k) {
    return k == 0 ? CP_ERR_INVALID_ARG : k == 1 ? CP_ERR_SPAN_TOO_SHORT : k == 2 ? CP_ERR_CAPACITY : CP_ERR_SENSITIVE_SPAN;
}

__global__ void k_ins_validate(InsArgs a) {
    const int lane = threadIdx.x & 31;
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int nwarps = (gridDim.x * blockDim.x) >> 5;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        a.hdr->n_cand = 0; a.hdr->n_copy = 0; a.hdr->n_removed = 0; a.hdr->n_new_live = 0;
        a.hdr->n_cand0 = 0; a.hdr->n_need = 0;
    }
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < a.S; j += gridDim.x * blockDim.x) a.eq_old[j] = 0;
    {   // the commit's relation-CSR counts and parallel-apply scratch (filled by k_ins_rep / k_ins_verify /
        // k_ins_rel_fill below; the commit's one CTA used to build them)
        const int g = blockIdx.x * blockDim.x + threadIdx.x, ng = gridDim.x * blockDim.x;
        for (int j = g; j <= a.S; j += ng) a.rel_off[j] = 0;
        for (int j = g; j < a.S; j += ng) { a.f_last[j] = -1; a.f_sidx[j] = 0; }
        for (int i = g; i < a.nslots; i += ng) { a.f_refs[i] = 0; a.f_evpos[i] = INT_MAX; a.f_maxpos[i] = -1; a.f_supby[i] = -1; }
    }
    // clear the batch prefix table
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < a.BT; i += (int64_t)gridDim.x * blockDim.x) {
        a.btab[i].key = CP_EMPTY_KEY; a.btab[i].slot = 0; a.btab[i].len = 0; a.btab[i].full = 0;      // prefix buckets
        a.dtab[i].key = CP_EMPTY_KEY; a.dtab[i].slot = 0x7fffffff; a.dtab[i].len = 0; a.dtab[i].full = 0;
    }
    if (cp_err_set(a.hdr)) return;
    for (int s = warp; s < a.S; s += nwarps) {
        const int r = a.span_req[s];
        int bad = -1;
        if (r < 0 || r >= a.num_reqs) bad = 0;
        int64_t b = a.span_begin[s], m = a.span_len[s], n = 0;
        if (bad < 0) {
            n = a.offsets[r + 1] - a.offsets[r];
            if (b < 0 || m < 0 || b + m > n) bad = 0;
            else if (m < a.w) bad = 1;
            else if (m > a.capacity || m > a.max_span_len) bad = 2;
            else if (((b + m - 1) >> 4) >= a.max_blocks) bad = 0;   // writer block table too narrow for the copy-in
        }
        if (bad < 0) {
            const uint8_t* mk = a.mask + a.offsets[r] + b;
            int any = 0;
            for (int64_t k = lane; k < m; k += 32) any |= mk[k];
            if (__any_sync(0xffffffffu, any)) bad = 3;
        }
        if (bad >= 0 && lane == 0) atomicMin(&a.hdr->first_err, ((unsigned long long)s << 32) | (unsigned)bad);
    }
    if (blockIdx.x == 0 && threadIdx.x == 0 && a.hdr->slot_free_top < a.S)
        atomicMin(&a.hdr->first_err, ((unsigned long long)0x7FFFFFFF << 32) | 2u);
}

// warp per span: prefix hash (first w tokens) and full hash; insert into the batch prefix table
__global__ void k_ins_hash(InsArgs a) {
    const int lane = threadIdx.x & 31;
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int nwarps = (gridDim.x * blockDim.x) >> 5;
    if (cp_err_set(a.hdr) || a.hdr->first_err != CP_NO_ERR_KEY) return;
    for (int s = warp; s < a.S; s += nwarps) {
        const int32_t* tau = a.tokens + a.offsets[a.span_req[s]] + a.span_begin[s];
        const int m = a.span_len[s];
        // lane folds a contiguous chunk; combine with B^(tokens after the chunk)
        auto fold = [&](int len) -> uint64_t {
            const int c = (len + 31) / 32;
            const int c0 = min(len, lane * c), c1 = min(len, c0 + c);
            uint64_t h = 0;
            for (int i = c0; i < c1; ++i) h = cp_addmod(cp_mulmod(h, a.B), cp_tokval(tau[i]));
            uint64_t v = cp_mulmod(h, a.pw[len - c1]);
#pragma unroll
            for (int off = 16; off; off >>= 1) v = cp_addmod(v, __shfl_xor_sync(0xffffffffu, v, off));
            return v;
        };
        const uint64_t pre = fold(a.w), full = fold(m);
        if (lane == 0) {
            a.span_pre[s] = pre; a.span_full[s] = full;
            HEntry* e = cp_find_or_insert(a.dtab, (uint32_t)(a.BT - 1), a.logBT, full);   // batch dedup
            atomicMin(&e->slot, s);
        }
    }
}

// token fetch helpers (forward)
__device__ __forceinline__ const int32_t* span_tokens_f(const InsArgs& a, int j) {
    return a.tokens + a.offsets[a.span_req[j]] + a.span_begin[j];
}

// warp per span: representative = smallest span with identical tokens (verified); representatives
// are counted into their prefix bucket
__global__ void k_ins_rep(InsArgs a) {
    const int lane = threadIdx.x & 31;
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int nwarps = (gridDim.x * blockDim.x) >> 5;
    if (cp_err_set(a.hdr) || a.hdr->first_err != CP_NO_ERR_KEY) return;
    for (int s = warp; s < a.S; s += nwarps) {
        const HEntry* e = cp_find_unique(a.dtab, (uint32_t)(a.BT - 1), a.logBT, a.span_full[s]);
        int r = e ? e->slot : s;
        if (r != s) {
            bool same = a.span_len[r] == a.span_len[s] && a.span_pre[r] == a.span_pre[s];
            if (same) {
                const int32_t* x = span_tokens_f(a, s);
                const int32_t* y = span_tokens_f(a, r);
                int bad = 0;
                for (int t = lane; t < a.span_len[s]; t += 32) bad |= x[t] != y[t];
                same = !__any_sync(0xffffffffu, bad);
            }
            if (!same) r = s;                       // full-hash collision: keep the span on its own
        }
        if (lane == 0) {
            a.span_rep[s] = r;
            atomicMax(&a.f_last[r], s);                   // the content's last span (parallel apply)
            if (r == s) {
                HEntry* b = cp_find_or_insert(a.btab, (uint32_t)(a.BT - 1), a.logBT, a.span_pre[s]);
                atomicAdd(&b->len, 1);
            }
        }
    }
}

// one block: bucket offsets = exclusive scan of the counts over the prefix table; a thread owns a
// contiguous run of BT/1024 buckets (one block scan instead of BT/1024 rounds of them)
__global__ void __launch_bounds__(1024) k_ins_bucket_offsets(InsArgs a) {
    __shared__ int s_w[33];
    if (cp_err_set(a.hdr) || a.hdr->first_err != CP_NO_ERR_KEY) return;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int64_t c = (a.BT + 1023) / 1024;
    const int64_t c0 = tid * c < a.BT ? tid * c : a.BT, c1 = c0 + c < a.BT ? c0 + c : a.BT;
    int loc = 0;
    for (int64_t i = c0; i < c1; ++i) if (a.btab[i].key != CP_EMPTY_KEY) loc += a.btab[i].len;
    int inc = loc;
    for (int o = 1; o < 32; o <<= 1) { const int y = __shfl_up_sync(0xffffffffu, inc, o); if (lane >= o) inc += y; }
    if (lane == 31) s_w[wid] = inc;
    __syncthreads();
    if (wid == 0) {
        int x = s_w[lane], xi = x;
        for (int o = 1; o < 32; o <<= 1) { const int y = __shfl_up_sync(0xffffffffu, xi, o); if (lane >= o) xi += y; }
        s_w[lane] = xi - x;
    }
    __syncthreads();
    int run = s_w[wid] + inc - loc;
    for (int64_t i = c0; i < c1; ++i) {
        if (a.btab[i].key == CP_EMPTY_KEY) continue;
        const int v = a.btab[i].len;
        if (v > 0) { a.btab[i].slot = run; a.btab[i].full = (unsigned long long)run; }   // offset, fill cursor
        run += v;
    }
}

// thread per representative: scatter into its prefix bucket
__global__ void k_ins_bucket_fill(InsArgs a) {
    if (cp_err_set(a.hdr) || a.hdr->first_err != CP_NO_ERR_KEY) return;
    for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < a.S; s += gridDim.x * blockDim.x) {
        if (a.span_rep[s] != s) continue;
        HEntry* b = const_cast<HEntry*>(cp_find_unique(a.btab, (uint32_t)(a.BT - 1), a.logBT, a.span_pre[s]));
        const unsigned long long pos = atomicAdd(&b->full, 1ULL);
        Rec16 r; r.full = a.span_full[s]; r.len = a.span_len[s]; r.id = s;
        a.precs[pos] = r;
    }
}

// token fetch helpers
__device__ __forceinline__ int32_t slot_token(const InsArgs& a, int slot, int t) {
    const int page = a.slot_pages[(int64_t)slot * a.MP + (t >> 4)];
    return a.page_tokens[(int64_t)page * CP_BLOCK + (t & 15)];
}
__device__ __forceinline__ const int32_t* span_tokens(const InsArgs& a, int j) {
    return a.tokens + a.offsets[a.span_req[j]] + a.span_begin[j];
}

__device__ __forceinline__ void push_cand(const InsArgs& a, int hay, int needle, int off) {
    int i = atomicAdd(&a.hdr->n_cand, 1);
    if (i < a.MAXC) { a.cand[i].hay = hay; a.cand[i].needle = needle; a.cand[i].off = off; a.cand[i].ok = 0; }
    else cp_raise(a.hdr, CP_ERR_CAPACITY);
}

// phase 0: items = new spans as haystacks (needles: other new spans via the batch table, live
//          entries via the pool table)
// phase 1: items = live slots as haystacks (needles: new spans WITHOUT an equal live entry, via
//          btab2).  A span equal to a live entry cannot be strictly inside another live entry (the
//          pool is containment-free), so those spans need no old-haystack scan.
__global__ void __launch_bounds__(kScanThreads) k_ins_scan(InsArgs a, int phase) {
    extern __shared__ uint64_t sm[];
    __shared__ uint64_t wtmp[2 * (kScanThreads / 32)];
    if (cp_err_set(a.hdr) || a.hdr->first_err != CP_NO_ERR_KEY) return;
    if (phase == 1 && a.hdr->n_need == 0) return;
    const int64_t items = phase == 0 ? (int64_t)a.S : (int64_t)a.nslots;
    for (int64_t it = blockIdx.x; it < items; it += gridDim.x) {
        const bool is_new = phase == 0;
        const int id = (int)it;
        int m;
        if (is_new) {
            if (a.span_rep[id] != id) continue;               // duplicates inherit their representative's relations
            m = a.span_len[id];
        } else {
            if (a.slot_state[id] != CP_SLOT_LIVE || a.slot_owner[id] != 0) continue;   // private: no relations (R#33)
            m = a.slot_len[id];
        }
        if (is_new) {
            const int32_t* tau = span_tokens(a, id);
            cp_block_prefix_hash<kScanThreads>([&](int i) { return tau[i]; }, m, a.B, sm, wtmp);
        } else {
            cp_block_prefix_hash<kScanThreads>([&](int i) { return slot_token(a, id, i); }, m, a.B, sm, wtmp);
        }
        const uint64_t Bw = a.pw[a.w];
        const int nwin = m - a.w + 1;
        const int wbase = threadIdx.x & ~31;
        for (int base = 0; base < nwin; base += blockDim.x) {
            const int o = base + threadIdx.x;
            const bool act = o < nwin;
            const uint64_t W = act ? cp_subhash(sm, o, a.w, Bw) : 0;
            // needles among the batch's representatives (bucketed prefix table)
            cp_warp_bucket_probe(a.btab, (uint32_t)(a.BT - 1), a.logBT, a.precs, W, act,
                                 [&](int owner, unsigned long long full, int mj, int j) {
                const int oo = base + wbase + owner;
                if (is_new && j == id) return;
                if (!is_new && a.eq_old[j]) return;           // equal to a live entry: cannot be strictly inside one
                if (oo + mj <= m && cp_subhash(sm, oo, mj, a.pw[mj]) == full)
                    push_cand(a, is_new ? -1 - id : id, -1 - j, oo);
            });
            // needles among live pool entries (new-span haystacks only)
            if (is_new)
                cp_warp_probe<false>(a.htab, (uint32_t)(a.T - 1), a.logT, W, act, [&](int owner, const HEntry& e) {
                    const int oo = base + wbase + owner;
                    const int me = e.len;
                    if (oo + me <= m && cp_subhash(sm, oo, me, a.pw[me]) == e.full) push_cand(a, -1 - id, e.slot, oo);
                });
        }
        __syncthreads();
    }
}

// after the phase-0 verification: flag spans that equal a live entry, then build btab2 from the rest
__global__ void k_ins_flag_eq(InsArgs a) {
    if (cp_err_set(a.hdr) || a.hdr->first_err != CP_NO_ERR_KEY) return;
    const int nc = min((int64_t)a.hdr->n_cand, a.MAXC);
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < nc; c += gridDim.x * blockDim.x) {
        const Cand cd = a.cand[c];
        if (cd.ok && cd.hay < 0 && cd.needle >= 0 && a.slot_len[cd.needle] == a.span_len[-1 - cd.hay])
            a.eq_old[-1 - cd.hay] = 1;
    }
}
__global__ void k_ins_count_need(InsArgs a) {
    if (cp_err_set(a.hdr) || a.hdr->first_err != CP_NO_ERR_KEY) return;
    if (blockIdx.x == 0 && threadIdx.x == 0) a.hdr->n_cand0 = min((int64_t)a.hdr->n_cand, a.MAXC);
    int need = 0;
    for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < a.S; s += gridDim.x * blockDim.x)
        need += (a.span_rep[s] == s && !a.eq_old[s]);
    for (int o = 16; o; o >>= 1) need += __shfl_xor_sync(0xffffffffu, need, o);
    if ((threadIdx.x & 31) == 0 && need) atomicAdd(&a.hdr->n_need, need);
}

// warp per candidate: exact token comparison of needle vs haystack[off, off + len(needle))
__global__ void k_ins_verify(InsArgs a, int from_phase1) {
    const int lane = threadIdx.x & 31;
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int nwarps = (gridDim.x * blockDim.x) >> 5;
    if (cp_err_set(a.hdr) || a.hdr->first_err != CP_NO_ERR_KEY) return;
    const int nc = min((int64_t)a.hdr->n_cand, a.MAXC);
    const int c0 = from_phase1 ? a.hdr->n_cand0 : 0;
    constexpr int U = 8;                      // tokens per lane in flight (256 per warp step)
    for (int c = c0 + warp; c < nc; c += nwarps) {
        const Cand cd = a.cand[c];
        const int nm = cd.needle < 0 ? a.span_len[-1 - cd.needle] : a.slot_len[cd.needle];
        const int32_t* xs = cd.needle < 0 ? span_tokens(a, -1 - cd.needle) : nullptr;
        const int32_t* ys = cd.hay < 0 ? span_tokens(a, -1 - cd.hay) + cd.off : nullptr;
        int bad = 0;
        for (int t0 = 0; t0 < nm && !__any_sync(0xffffffffu, bad); t0 += 32 * U) {
            int32_t x[U], y[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int t = t0 + 32 * u + lane;
                x[u] = t < nm ? (xs ? xs[t] : slot_token(a, cd.needle, t)) : 0;
                y[u] = t < nm ? (ys ? ys[t] : slot_token(a, cd.hay, cd.off + t)) : 0;
            }
#pragma unroll
            for (int u = 0; u < U; ++u) bad |= (x[u] != y[u]);
        }
        bad = __any_sync(0xffffffffu, bad);
        if (lane == 0) {
            a.cand[c].ok = !bad;
            if (!bad) {                               // relation-CSR counts per new span
                if (cd.needle < 0) atomicAdd(&a.rel_off[-1 - cd.needle], 1);
                if (cd.hay < 0) atomicAdd(&a.rel_off[-1 - cd.hay], 1);
            }
        }
    }
}

enum { REL_EQ = 0, REL_CONTAINER = 1, REL_CONTAINED = 2 };
constexpr int kMaxSupersede = 1024;
constexpr int kStackCache = 2048;          // free-slot stack entries cached in shared memory
constexpr int kFifoCache = 4096;           // free-page FIFO head entries cached in shared memory

struct CommitSmem {                  // byte offsets of the dynamic shared-memory carve-up
    size_t snew, srep, soff, seq, slen, sfpos, ckey, cslot, clen, srec, fixed, total;
    __host__ __device__ CommitSmem(int nslots, int S, int K, int rec_cap) {
        snew = ((size_t)nslots + 15) & ~(size_t)15;
        srep = snew + 4 * (size_t)S;
        soff = srep + 4 * (size_t)S;
        seq = soff + 4 * ((size_t)S + 1);                   // per group: last entry known equal to it
        slen = seq + 4 * (size_t)S;                         // span lengths
        sfpos = slen + 4 * (size_t)S;                       // deferred stores: FIFO position of their pages
        ckey = (sfpos + 4 * (size_t)S + 15) & ~(size_t)15;   // LRU candidates: (last_used - min) << 32 | id
        cslot = ckey + 8 * (size_t)K;
        clen = cslot + 4 * (size_t)K;
        srec = (clen + 4 * (size_t)K + 15) & ~(size_t)15;  // relation records (rec_cap of them)
        fixed = srec;
        total = srec + 8 * (size_t)rec_cap;
    }
};

// block-wide exclusive scan of v[0..n) in shared memory (in place); returns the total
template <int NT>
__device__ int block_excl_scan(int32_t* v, int n, int32_t* wsum) {
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int c = (n + NT - 1) / NT, c0 = min(n, tid * c), c1 = min(n, c0 + c);
    int loc = 0;
    for (int i = c0; i < c1; ++i) loc += v[i];
    int inc = loc;
    for (int off = 1; off < 32; off <<= 1) { int y = __shfl_up_sync(0xffffffffu, inc, off); if (lane >= off) inc += y; }
    if (lane == 31) wsum[wid] = inc;
    __syncthreads();
    if (wid == 0) {
        int x = lane < NT / 32 ? wsum[lane] : 0, xi = x;
        for (int off = 1; off < 32; off <<= 1) { int y = __shfl_up_sync(0xffffffffu, xi, off); if (lane >= off) xi += y; }
        if (lane < NT / 32) wsum[lane] = xi - x;
        if (lane == 31) wsum[NT / 32] = xi;
    }
    __syncthreads();
    int run = wsum[wid] + inc - loc;
    for (int i = c0; i < c1; ++i) { int t = v[i]; v[i] = run; run += t; }
    const int total = wsum[NT / 32];
    __syncthreads();
    return total;
}

// block-wide exclusive scan of 64-bit values (in place); returns the total
template <int NT>
__device__ long long block_excl_scan64(long long* v, int n, long long* wsum) {
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int c = (n + NT - 1) / NT, c0 = min(n, tid * c), c1 = min(n, c0 + c);
    long long loc = 0;
    for (int i = c0; i < c1; ++i) loc += v[i];
    long long inc = loc;
    for (int off = 1; off < 32; off <<= 1) { long long y = __shfl_up_sync(0xffffffffu, inc, off); if (lane >= off) inc += y; }
    if (lane == 31) wsum[wid] = inc;
    __syncthreads();
    if (wid == 0) {
        long long x = lane < NT / 32 ? wsum[lane] : 0, xi = x;
        for (int off = 1; off < 32; off <<= 1) { long long y = __shfl_up_sync(0xffffffffu, xi, off); if (lane >= off) xi += y; }
        if (lane < NT / 32) wsum[lane] = xi - x;
        if (lane == 31) wsum[NT / 32] = xi;
    }
    __syncthreads();
    long long run = wsum[wid] + inc - loc;
    for (int i = c0; i < c1; ++i) { long long t = v[i]; v[i] = run; run += t; }
    const long long total = wsum[NT / 32];
    __syncthreads();
    return total;
}

// block-wide inclusive max-scan of v[0..n) (in place)
template <int NT>
__device__ void block_incl_maxscan(int32_t* v, int n, int32_t* wsum) {
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int c = (n + NT - 1) / NT, c0 = min(n, tid * c), c1 = min(n, c0 + c);
    int loc = INT_MIN;
    for (int i = c0; i < c1; ++i) loc = max(loc, v[i]);
    int inc = loc;
    for (int off = 1; off < 32; off <<= 1) { int y = __shfl_up_sync(0xffffffffu, inc, off); if (lane >= off) inc = max(inc, y); }
    if (lane == 31) wsum[wid] = inc;
    __syncthreads();
    if (wid == 0) {
        int x = lane < NT / 32 ? wsum[lane] : INT_MIN, xi = x;
        for (int off = 1; off < 32; off <<= 1) { int y = __shfl_up_sync(0xffffffffu, xi, off); if (lane >= off) xi = max(xi, y); }
        const int ex = __shfl_up_sync(0xffffffffu, xi, 1);
        if (lane < NT / 32) wsum[lane] = lane == 0 ? INT_MIN : ex;
    }
    __syncthreads();
    const int lex = __shfl_up_sync(0xffffffffu, inc, 1);
    int run = max(wsum[wid], lane == 0 ? INT_MIN : lex);
    for (int i = c0; i < c1; ++i) { run = max(run, v[i]); v[i] = run; }
    __syncthreads();
}

constexpr int kFastSup = 8;               // parallel apply: most live segments one stored span supersedes

#ifdef CP_COMMIT_PROF
// diagnostic build only: [0..5] phase timestamps, [6..11] cycles per path, [12..15] counts
__device__ unsigned long long g_commit_prof[16];
#define PROF_T(i) do { if (tid == 0) g_commit_prof[i] += clock64() - t_phase; if (tid == 0) t_phase = clock64(); } while (0)
#define PROF_ACC(i, c) do { g_commit_prof[i] += clock64() - (c); } while (0)
#define PROF_CNT(i, n) do { g_commit_prof[i] += (n); } while (0)
#else
#define PROF_T(i) do {} while (0)
#define PROF_ACC(i, c) do {} while (0)
#define PROF_CNT(i, n) do {} while (0)
#endif

// One CTA applies the spans in input order (exact sequential semantics of R#20-22).
// sflag bit 0: live; bit 1: stored by this call.
// ---- relation CSR of the commit, finished at the end of the prepare: k_ins_verify counted the verified
//      relations per new span; one CTA scans the counts and places the records (they depend only on the
//      verified candidates and on lengths, none of which change before the commit)
__global__ void __launch_bounds__(1024) k_ins_rel_fill(InsArgs a) {
    __shared__ int32_t s_w[1024 / 32 + 1];
    if (cp_err_set(a.hdr) || a.hdr->first_err != CP_NO_ERR_KEY) return;   // the commit aborts
    block_excl_scan<1024>(a.rel_off, a.S + 1, s_w);             // rel_off[S] = the record count
    for (int j = threadIdx.x; j <= a.S; j += blockDim.x) a.rel_cur[j] = a.rel_off[j];
    __syncthreads();
    const int nc = (int)min((int64_t)a.hdr->n_cand, a.MAXC);     // more: the commit aborts (CP_ERR_CAPACITY)
    auto len_of = [&](int code) { return code < 0 ? a.span_len[-1 - code] : a.slot_len[code]; };
    for (int c = threadIdx.x; c < nc; c += blockDim.x) {
        const Cand cd = a.cand[c];
        if (!cd.ok) continue;
        const bool eq = len_of(cd.needle) == len_of(cd.hay);
        if (cd.needle < 0) {       // the new span (needle) occurs inside hay
            const int p = atomicAdd(&a.rel_cur[-1 - cd.needle], 1);
            a.rel_rec[p] = make_int2(cd.hay, eq ? REL_EQ : REL_CONTAINER);
        }
        if (cd.hay < 0) {          // the new span (hay) contains needle
            const int p = atomicAdd(&a.rel_cur[-1 - cd.hay], 1);
            a.rel_rec[p] = make_int2(cd.needle, eq ? REL_EQ : REL_CONTAINED);
        }
    }
}

// ---- LRU candidate list, prepared beside match + gather (cp_index_insert_prepare, R#21) ----
// The commit evicts in (last_used, id) order.  Instead of selecting the K smallest keys with one CTA
// inside the commit (a radix select over the slot table and a K-element sort: ~135 us per evicting
// config-5 batch), the prepare snapshots the evictable keys and selects + sorts them with the whole
// grid: 11-bit MSB digits of the compact key ((last - minl) << idb | (id - idmin), <= 33 bits), a global
// histogram per digit, then a rank-by-count sort.  The snapshot may precede this step's match, whose
// touches only RAISE keys: the commit pops an entry only if its last_used still equals the listed one,
// so the entries it accepts are exactly the smallest current keys below the list's threshold, in order
// (an entry whose key rose is skipped; a pin since the snapshot, or a non-monotone clock, discards the
// list and the commit selects in-kernel as before).
struct LruGeom {
    unsigned long long minl; unsigned idmin; int idb, kb, digits;
    __device__ bool load(const LruHdr* h) {
        if (!h->valid || h->minl > h->maxl || h->maxl - h->minl >= (1ULL << 32)) return false;
        minl = h->minl; idmin = h->idmin;
        idb = 32 - __clz((int)(h->idmax - h->idmin) | 1);
        kb = idb + (64 - __clzll((long long)((h->maxl - h->minl) | 1)));
        digits = (kb + 10) / 11;
        return kb <= 33;
    }
    __device__ int hi(int p) const { return kb - 11 * p; }
    __device__ int lo(int p) const { return max(0, kb - 11 * (p + 1)); }
    __device__ unsigned long long ckey(unsigned long long last, int id) const {
        return ((last - minl) << idb) | (unsigned long long)((unsigned)id - idmin);
    }
};

// digits 0..upto-1 of the K-th smallest compact key, from the global histograms (every CTA computes the
// same result; 256 threads); all = 1 when there are no more than K evictable entries
__device__ void lru_select(const InsArgs& a, const LruGeom& g, int upto, unsigned long long& prefix, int& all) {
    __shared__ int s_w[8], s_bin, s_rem, s_tot;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    int rem = a.candK;
    prefix = 0; all = 0;
    for (int p = 0; p < upto; ++p) {
        const unsigned* hist = a.lru_hist + p * kLruBins;
        const int nb = 1 << (g.hi(p) - g.lo(p));
        int own = 0;
        for (int b = tid * 8; b < min(nb, tid * 8 + 8); ++b) own += hist[b];
        int inc = own;
        for (int o = 1; o < 32; o <<= 1) { const int y = __shfl_up_sync(0xffffffffu, inc, o); if (lane >= o) inc += y; }
        if (lane == 31) s_w[wid] = inc;
        __syncthreads();
        int base = 0;
        for (int w = 0; w < wid; ++w) base += s_w[w];
        if (tid == 255) s_tot = base + inc;
        const int excl = base + inc - own;
        if (own > 0 && excl < rem && rem <= excl + own) {
            int c = excl;
            for (int b = tid * 8; b < min(nb, tid * 8 + 8); ++b) {
                if (c + (int)hist[b] >= rem) { s_bin = b; s_rem = rem - c; break; }
                c += hist[b];
            }
        }
        __syncthreads();
        if (p == 0 && s_tot <= a.candK) { all = 1; __syncthreads(); return; }
        prefix = (prefix << (g.hi(p) - g.lo(p))) | (unsigned long long)s_bin;
        rem = s_rem;
        __syncthreads();
    }
}

__global__ void __launch_bounds__(1024) k_lru_init(InsArgs a) {
    __shared__ unsigned long long s_sum;
    __shared__ int s_valid;
    if (threadIdx.x == 0) s_sum = 0;
    __syncthreads();
    unsigned long long sum = 0;
    for (int j = threadIdx.x; j < a.S; j += blockDim.x) sum += (unsigned long long)max(0, a.span_len[j]);
    for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    if ((threadIdx.x & 31) == 0 && sum) atomicAdd(&s_sum, sum);
    __syncthreads();
    if (threadIdx.x == 0) {
        LruHdr* h = a.lru;
        h->minl = ~0ULL; h->maxl = 0; h->idmin = 0xffffffffu; h->idmax = 0; h->count = 0; h->all = 0;
        h->pin_epoch = a.hdr->pin_epoch;
        // only when this call may evict (the commit's own test is tighter: spans after its duplicates)
        s_valid = (a.candK > 0 && a.candK <= kLruK && !cp_err_set(a.hdr) &&
                   a.hdr->live_tokens + (long long)s_sum > a.capacity) ? 1 : 0;
        h->valid = s_valid;
    }
    __syncthreads();
    if (!s_valid) return;                      // steady state without eviction: nothing else to do
    for (int i = threadIdx.x; i < 3 * kLruBins; i += blockDim.x) a.lru_hist[i] = 0;
    for (int i = threadIdx.x; i < kLruK; i += blockDim.x) a.lru_rank[i] = 0;
}

__global__ void __launch_bounds__(256) k_lru_snap(InsArgs a) {
    if (!a.lru->valid) return;
    unsigned long long mn = ~0ULL, mx = 0;
    unsigned imn = 0xffffffffu, imx = 0;
    for (int sl = blockIdx.x * blockDim.x + threadIdx.x; sl < a.nslots; sl += gridDim.x * blockDim.x) {
        unsigned long long k = ~0ULL;
        if (a.slot_state[sl] == CP_SLOT_LIVE && a.slot_pin[sl] == 0) {
            k = a.slot_last[sl];
            const unsigned id = (unsigned)a.slot_id[sl];
            mn = k < mn ? k : mn; mx = k > mx ? k : mx; imn = id < imn ? id : imn; imx = id > imx ? id : imx;
        }
        a.lru_key[sl] = k;
    }
    for (int o = 16; o; o >>= 1) {
        const unsigned long long a2 = __shfl_xor_sync(0xffffffffu, mn, o), b2 = __shfl_xor_sync(0xffffffffu, mx, o);
        const unsigned c2 = __shfl_xor_sync(0xffffffffu, imn, o), d2 = __shfl_xor_sync(0xffffffffu, imx, o);
        mn = a2 < mn ? a2 : mn; mx = b2 > mx ? b2 : mx; imn = c2 < imn ? c2 : imn; imx = d2 > imx ? d2 : imx;
    }
    if ((threadIdx.x & 31) == 0 && mn <= mx) {
        atomicMin(&a.lru->minl, mn); atomicMax(&a.lru->maxl, mx);
        atomicMin(&a.lru->idmin, imn); atomicMax(&a.lru->idmax, imx);
    }
}

__global__ void __launch_bounds__(256) k_lru_hist(InsArgs a, int p) {
    __shared__ unsigned s_h[kLruBins];
    LruGeom g;
    if (!g.load(a.lru)) { if (p == 0 && blockIdx.x == 0 && threadIdx.x == 0) a.lru->valid = 0; return; }
    if (p >= g.digits) return;
    unsigned long long prefix; int all;
    lru_select(a, g, p, prefix, all);
    if (all) return;
    const int hi = g.hi(p), lo = g.lo(p);
    const unsigned long long bmask = (1ULL << (hi - lo)) - 1;
    for (int b = threadIdx.x; b < kLruBins; b += blockDim.x) s_h[b] = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    for (int s0 = (blockIdx.x * blockDim.x + threadIdx.x) & ~31; s0 < a.nslots; s0 += gridDim.x * blockDim.x) {
        const int sl = s0 + lane;                              // warp-uniform trip count
        int bin = -1;
        if (sl < a.nslots) {
            const unsigned long long k = a.lru_key[sl];
            if (k != ~0ULL) {
                const unsigned long long ck = g.ckey(k, a.slot_id[sl]);
                if ((ck >> hi) == prefix) bin = (int)((ck >> lo) & bmask);
            }
        }
        const unsigned peers = __match_any_sync(0xffffffffu, bin);
        if (bin >= 0 && lane == __ffs(peers) - 1) atomicAdd(&s_h[bin], (unsigned)__popc(peers));
    }
    __syncthreads();
    for (int b = threadIdx.x; b <= (int)bmask; b += blockDim.x)
        if (s_h[b]) atomicAdd(&a.lru_hist[p * kLruBins + b], s_h[b]);
}

__global__ void __launch_bounds__(256) k_lru_collect(InsArgs a) {
    LruGeom g;
    if (!g.load(a.lru)) return;
    unsigned long long T; int all;
    lru_select(a, g, g.digits, T, all);
    if (blockIdx.x == 0 && threadIdx.x == 0) a.lru->all = all;
    const int lane = threadIdx.x & 31;
    for (int s0 = (blockIdx.x * blockDim.x + threadIdx.x) & ~31; s0 < a.nslots; s0 += gridDim.x * blockDim.x) {
        const int sl = s0 + lane;
        bool take = false;
        unsigned long long ck = 0;
        if (sl < a.nslots) {
            const unsigned long long k = a.lru_key[sl];
            if (k != ~0ULL) { ck = g.ckey(k, a.slot_id[sl]); take = all || ck <= T; }
        }
        const unsigned bal = __ballot_sync(0xffffffffu, take);
        int p0 = 0;
        if (lane == 0 && bal) p0 = atomicAdd(&a.lru->count, __popc(bal));
        p0 = __shfl_sync(0xffffffffu, p0, 0);
        if (take) {
            const int pos = p0 + __popc(bal & ((1u << lane) - 1));
            if (pos < kLruK) a.lru_list[pos] = (ck << 32) | (unsigned)sl;
        }
    }
}

// rank by count: element e's position = the number of listed keys below it (keys are unique); a CTA
// compares 256 elements against one quarter of the list
__global__ void __launch_bounds__(256) k_lru_rank(InsArgs a) {
    __shared__ unsigned long long s_k[kLruK / 4];
    if (!a.lru->valid) return;
    const int n = min(a.lru->count, kLruK);
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    const int c0 = blockIdx.y * (kLruK / 4), c1 = min(n, c0 + kLruK / 4);
    if (blockIdx.x * blockDim.x >= n || c0 >= n) return;
    for (int i = c0 + threadIdx.x; i < c1; i += blockDim.x) s_k[i - c0] = a.lru_list[i];
    __syncthreads();
    if (e >= n) return;
    const unsigned long long k = a.lru_list[e];
    unsigned cnt = 0;
    for (int i = 0; i < c1 - c0; ++i) cnt += s_k[i] < k;
    atomicAdd(&a.lru_rank[e], cnt);
}

__global__ void __launch_bounds__(256) k_lru_scatter(InsArgs a) {
    if (!a.lru->valid) return;
    const int n = min(a.lru->count, kLruK);
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e < n) a.lru_sorted[a.lru_rank[e]] = a.lru_list[e];
}

__global__ void __launch_bounds__(kCommitThreads) k_ins_commit(InsArgs a) {
    const unsigned long long tnow = a.clock ? *a.clock : a.t;   // device clock (CUDA-graph replays advance it)
    extern __shared__ __align__(16) unsigned char smc[];
    const int tid = threadIdx.x;
    const CommitSmem lay(a.nslots, a.S, a.candK, a.rec_cap);
    uint8_t* sflag = smc;
    unsigned long long* ckey = (unsigned long long*)(smc + lay.ckey);
    int32_t* cslot = (int32_t*)(smc + lay.cslot);
    int32_t* snew = (int32_t*)(smc + lay.snew);
    int32_t* srep = (int32_t*)(smc + lay.srep);
    int32_t* soff = (int32_t*)(smc + lay.soff);
    int32_t* seq = (int32_t*)(smc + lay.seq);
    int32_t* slen = (int32_t*)(smc + lay.slen);
    int32_t* sfpos = (int32_t*)(smc + lay.sfpos);
    int32_t* clen = (int32_t*)(smc + lay.clen);
    int2* srec = (int2*)(smc + lay.srec);
    __shared__ int s_abort, s_nrec;
    __shared__ long long s_live_tokens, s_chunks, s_pinned_tok;
    __shared__ int s_fifo_head, s_fifo_count, s_next_id, s_free_top, s_num_live, s_nremoved;
    __shared__ int s_rm[kMaxSupersede];
    __shared__ unsigned long long s_red_key[kCommitThreads / 32];
    __shared__ int s_red_slot[kCommitThreads / 32];
    __shared__ int32_t s_wsum[kCommitThreads / 32 + 1];
#ifdef CP_COMMIT_PROF
    long long t_phase = clock64();
#endif

    if (tid == 0) {
        s_abort = 0; s_chunks = 0; s_pinned_tok = 0;
        if (cp_err_set(a.hdr)) s_abort = 1;
        else if (a.hdr->first_err != CP_NO_ERR_KEY) {
            const unsigned code = (unsigned)(a.hdr->first_err & 0xffffffffu);
            cp_raise(a.hdr, code_of((int)code));
            s_abort = 1;
        } else if (a.hdr->n_cand > a.MAXC) {
            cp_raise(a.hdr, CP_ERR_CAPACITY);
            s_abort = 1;
        }
        a.hdr->first_err = CP_NO_ERR_KEY;
    }
    __syncthreads();
    if (s_abort) {
        for (int j = tid; j < a.S; j += blockDim.x) { a.out_id[j] = -1; a.out_oc[j] = -1; a.out_tmp[j] = -1; }
        return;
    }
    // ---- load state
    for (int i = tid; i < a.nslots; i += blockDim.x) sflag[i] = a.slot_state[i] == CP_SLOT_LIVE ? 1 : 0;
    {   // R#32: tokens of the live pinned entries (constant through the call: they can't be removed)
        long long pt = 0;
        for (int i = tid; i < a.nslots; i += blockDim.x)
            if (a.slot_state[i] == CP_SLOT_LIVE && a.slot_pin[i] > 0) pt += a.slot_len[i];
        for (int o = 16; o; o >>= 1) pt += __shfl_xor_sync(0xffffffffu, pt, o);
        if ((tid & 31) == 0 && pt) atomicAdd((unsigned long long*)&s_pinned_tok, (unsigned long long)pt);
    }
    for (int j = tid; j < a.S; j += blockDim.x) {
        snew[j] = -1; soff[j] = 0; srep[j] = a.span_rep[j]; seq[j] = -1; slen[j] = a.span_len[j]; sfpos[j] = -1;
    }
    if (tid == 0) {
        soff[a.S] = 0;
        s_live_tokens = a.hdr->live_tokens; s_fifo_head = a.hdr->fifo_head; s_fifo_count = a.hdr->fifo_count;
        s_next_id = a.hdr->next_id; s_free_top = a.hdr->slot_free_top; s_num_live = a.hdr->num_live;
        s_nremoved = 0;
    }
    __syncthreads();
    // ---- relation CSR over new spans: (other, kind) records per span, built by the prepare (counts in
    //      k_ins_verify, offsets and records in k_ins_rel_fill)
    for (int j = tid; j <= a.S; j += blockDim.x) soff[j] = a.rel_off[j];
    if (tid == 0) s_nrec = a.rel_off[a.S];
    __syncthreads();
    // ---- capacity checks before any mutation (an insert that fails changes nothing): the supersede
    //      list of one span (its CONTAINED records bound it) and the copy-in chunk list (stored spans
    //      may overlap, so their total length can exceed max_batch_tokens)
    {
        int bad = 0;
        long long chunks = 0;
        for (int j = tid; j < a.S; j += blockDim.x) {
            chunks += (slen[j] + CP_GATHER_CHUNK - 1) / CP_GATHER_CHUNK;
            if (srep[j] != j) continue;
            int ncont = 0;
            for (int q = soff[j]; q < soff[j + 1]; ++q) ncont += a.rel_rec[q].y == REL_CONTAINED;
            bad |= ncont > kMaxSupersede;
        }
        for (int o = 16; o; o >>= 1) chunks += __shfl_xor_sync(0xffffffffu, chunks, o);
        if ((tid & 31) == 0 && chunks) atomicAdd((unsigned long long*)&s_chunks, (unsigned long long)chunks);
        if (bad) s_abort = 1;
        __syncthreads();
        if (tid == 0 && (s_abort || s_chunks > a.CH)) { cp_raise(a.hdr, CP_ERR_CAPACITY); s_abort = 1; }
        __syncthreads();
        if (s_abort) {
            for (int j = tid; j < a.S; j += blockDim.x) { a.out_id[j] = -1; a.out_oc[j] = -1; a.out_tmp[j] = -1; }
            return;
        }
    }
    const bool rec_in_smem = s_nrec <= a.rec_cap;
    if (rec_in_smem) for (int i = tid; i < s_nrec; i += blockDim.x) srec[i] = a.rel_rec[i];
    __syncthreads();
    const int2* rec = rec_in_smem ? srec : a.rel_rec;
    PROF_T(0);

    // a relation names an old slot (code >= 0) or a new span's CONTENT (code < 0: a representative);
    // that content may have been stored by any span of the same representative, and the pool holds
    // at most one live entry per content: seq[rep] is the latest slot stored or refreshed for it
    // (snew[rep] alone misses a duplicate of a Dropped representative that got stored later)
    auto resolve = [&](int code) -> int { return code >= 0 ? code : seq[srep[-1 - code]]; };
    auto is_live = [&](int code) -> bool { const int s = resolve(code); return s >= 0 && (sflag[s] & 1); };


    // ---- parallel prefix: until the first span that must be stored, nothing is stored or removed,
    //      so every span before it is decided against the initial state (duplicates only refresh
    //      last_used, which no decision reads).  In steady-state serving this is the whole batch.
    __shared__ int s_jstar;
    if (tid == 0) s_jstar = a.S;
    __syncthreads();
    for (int j = tid; j < a.S; j += blockDim.x) {
        bool decided = false;
        const int rj = srep[j];                      // duplicates share their representative's relations
        for (int q = soff[rj]; q < soff[rj + 1] && !decided; ++q) {
            const int2 rr = rec[q];
            if (rr.x >= 0 && (sflag[rr.x] & 1) && (rr.y == REL_EQ || rr.y == REL_CONTAINER)) decided = true;
        }
        if (!decided) atomicMin(&s_jstar, j);
    }
    __syncthreads();
    const int jstar = s_jstar;
    for (int j = tid; j < jstar; j += blockDim.x) {
        int dup = -1, cont = -1, cont_id = 0x7fffffff;
        const int rj = srep[j];
        for (int q = soff[rj]; q < soff[rj + 1]; ++q) {
            const int2 rr = rec[q];
            if (rr.x < 0 || !(sflag[rr.x] & 1)) continue;
            if (rr.y == REL_EQ) dup = rr.x;
            else if (rr.y == REL_CONTAINER) { const int sid = a.slot_id[rr.x]; if (sid < cont_id) { cont_id = sid; cont = rr.x; } }
        }
        if (dup >= 0) {
            a.slot_last[dup] = tnow; sflag[dup] |= 4; a.out_tmp[j] = dup; a.out_oc[j] = CP_DUPLICATE;
            seq[rj] = dup;                        // the one live entry with this content (benign equal-value race)
        } else { a.out_tmp[j] = cont; a.out_oc[j] = CP_DROPPED_CONTAINED; }
    }
    __syncthreads();
    PROF_T(1);
    // ---- LRU candidates (R#21): the K smallest live (last_used, id) keys, sorted, in shared
    //      memory.  Within this call keys only grow (a Duplicate refresh sets last_used = t >= all old
    //      values when time is monotone) and new entries sort after every old one, so evictions pop
    //      this list, skipping entries removed or refreshed since; the block-wide arg-min remains the
    //      fallback (list exhausted, non-monotone time, K = 0).
    __shared__ unsigned long long s_minl, s_maxl;
    __shared__ unsigned s_idmin, s_idmax;
    __shared__ int s_cn, s_cp, s_heap, s_hist[256], s_digit, s_rem2;
    __shared__ long long s_pending;
    if (tid == 0) { s_minl = ~0ULL; s_maxl = 0; s_idmin = 0xffffffffu; s_idmax = 0; s_cn = 0; s_cp = 0; s_heap = 0; s_pending = 0; }
    __syncthreads();
    {   // upper bound of the tokens this call can still store: if it fits the budget, no eviction happens
        long long pend = 0;
        for (int j = jstar + tid; j < a.S; j += blockDim.x) pend += slen[j];
        for (int o = 16; o; o >>= 1) pend += __shfl_xor_sync(0xffffffffu, pend, o);
        if ((tid & 31) == 0 && pend) atomicAdd((unsigned long long*)&s_pending, (unsigned long long)pend);
    }
    __syncthreads();
    // the list the prepare built (k_lru_*), if it is usable: no pin since its snapshot, a monotone clock
    // (count <= candK: the list holds EVERY snapshot key up to its threshold -- a complete prefix of the
    // LRU order, which is what makes its pops exact; a longer list would have been truncated)
    const bool prepared = a.candK > 0 && a.lru->valid && a.lru->pin_epoch == a.hdr->pin_epoch && tnow >= a.lru->maxl &&
                          a.lru->count <= a.candK;
    if (prepared && s_live_tokens + s_pending > a.capacity) {
        const unsigned long long minl = a.lru->minl;
        const unsigned idmin = a.lru->idmin;
        const int idb = 32 - __clz((int)(a.lru->idmax - idmin) | 1);
        const unsigned long long idmask = (1ULL << idb) - 1;
        const int cn = min(a.lru->count, a.candK);
        for (int p = tid; p < a.candK; p += blockDim.x) {
            if (p < cn) {
                const unsigned long long sk = a.lru_sorted[p], ck = sk >> 32;
                const int sl = (int)(sk & 0xffffffffu);
                ckey[p] = ((ck >> idb) << 32) | ((ck & idmask) + idmin);   // (last - minl) << 32 | id
                cslot[p] = sl; clen[p] = a.slot_len[sl];
            } else { ckey[p] = ~0ULL; cslot[p] = -1; clen[p] = 0; }
        }
        if (tid == 0) { s_minl = minl; s_maxl = a.lru->maxl; s_cn = cn; s_heap = 1; }
        __syncthreads();
    } else if (a.candK > 0 && s_live_tokens + s_pending > a.capacity) {
        // one pass: ranges of last_used and id over the evictable (live, unpinned) entries
        unsigned long long mn = ~0ULL, mx = 0;
        unsigned idmn = 0xffffffffu, idmx = 0;
        for (int sl = tid; sl < a.nslots; sl += blockDim.x)
            if ((sflag[sl] & 1) && a.slot_pin[sl] == 0) {
                const unsigned long long lu = a.slot_last[sl];
                const unsigned id = (unsigned)a.slot_id[sl];
                mn = lu < mn ? lu : mn; mx = lu > mx ? lu : mx;
                idmn = id < idmn ? id : idmn; idmx = id > idmx ? id : idmx;
            }
        for (int o = 16; o; o >>= 1) {
            const unsigned long long a2 = __shfl_xor_sync(0xffffffffu, mn, o), b2 = __shfl_xor_sync(0xffffffffu, mx, o);
            mn = a2 < mn ? a2 : mn; mx = b2 > mx ? b2 : mx;
            const unsigned c2 = __shfl_xor_sync(0xffffffffu, idmn, o), d2 = __shfl_xor_sync(0xffffffffu, idmx, o);
            idmn = c2 < idmn ? c2 : idmn; idmx = d2 > idmx ? d2 : idmx;
        }
        if ((tid & 31) == 0) { atomicMin(&s_minl, mn); atomicMax(&s_maxl, mx); atomicMin(&s_idmin, idmn); atomicMax(&s_idmax, idmx); }
        __syncthreads();
        PROF_T(10);
        const bool ok = s_maxl >= s_minl && (s_maxl - s_minl) < (1ULL << 32) && tnow >= s_maxl;
        if (ok) {
            const unsigned long long minl = s_minl;
            const unsigned idmin = s_idmin;
            // the radix select runs on a compact key with the same order: (last - minl) << idb | (id - idmin),
            // idb = bits of the id range, so only the digits the keys can differ in are scanned (config-5
            // churn: ~3 passes instead of 8 over the slot table)
            const int idb = 32 - __clz((int)(s_idmax - idmin) | 1);
            const int kb = idb + (64 - __clzll((long long)((s_maxl - minl) | 1)));
            const int top = ((kb + 7) / 8 - 1) * 8;
            auto ckeyof = [&](unsigned long long lu, unsigned id) -> unsigned long long {
                return ((lu - minl) << idb) | (unsigned long long)(id - idmin);
            };
            unsigned long long prefix = 0, pmask = 0;
            if (tid == 0) s_rem2 = a.candK;
            __syncthreads();
            for (int shift = top; shift >= 0; shift -= 8) {
                for (int b = tid; b < 256; b += blockDim.x) s_hist[b] = 0;
                __syncthreads();
                // 4 slots per thread in flight (their loads are issued before any histogram update); the
                // lanes of a warp that fall in one bin add once (most keys share the leading digits: plain
                // shared atomics on one bin serialise 32-way)
                for (int s0 = tid & ~31; s0 < a.nslots; s0 += 4 * blockDim.x) {     // warp-uniform trip count
                    unsigned long long lu[4]; unsigned id[4]; bool on[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const int sl = s0 + u * blockDim.x + (tid & 31);
                        on[u] = sl < a.nslots && (sflag[sl] & 1);
                        if (on[u]) { on[u] = a.slot_pin[sl] == 0; lu[u] = a.slot_last[sl]; id[u] = (unsigned)a.slot_id[sl]; }
                    }
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        int bin = -1;                                           // pinned: never evicted (R#32)
                        if (on[u]) {
                            const unsigned long long k = ckeyof(lu[u], id[u]);
                            if ((k & pmask) == prefix) bin = (int)((k >> shift) & 255);
                        }
                        const unsigned peers = __match_any_sync(0xffffffffu, bin);
                        if (bin >= 0 && (tid & 31) == __ffs(peers) - 1) atomicAdd(&s_hist[bin], __popc(peers));
                    }
                }
                __syncthreads();
                if (tid == 0) {
                    int cum = 0, rem = s_rem2, dg = 255;
                    for (int b = 0; b < 256; ++b) {
                        if (cum + s_hist[b] >= rem) { dg = b; rem -= cum; break; }
                        cum += s_hist[b];
                    }
                    s_digit = dg; s_rem2 = rem;
                }
                __syncthreads();
                prefix |= (unsigned long long)s_digit << shift;
                pmask |= 0xFFULL << shift;
                __syncthreads();
            }
            const unsigned long long T = prefix;                   // K-th smallest (or the max if fewer live)
            PROF_T(11);
            for (int s0 = tid & ~31; s0 < a.nslots; s0 += blockDim.x) {       // warp-uniform trip count
                const int sl = s0 + (tid & 31);
                bool take = false;
                unsigned long long lu = 0;
                unsigned id = 0;
                if (sl < a.nslots && (sflag[sl] & 1) && a.slot_pin[sl] == 0) {
                    lu = a.slot_last[sl]; id = (unsigned)a.slot_id[sl];
                    take = ckeyof(lu, id) <= T;
                }
                const unsigned bal = __ballot_sync(0xffffffffu, take);            // one shared atomic per warp
                int p0 = 0;
                if ((tid & 31) == 0 && bal) p0 = atomicAdd(&s_cn, __popc(bal));
                p0 = __shfl_sync(0xffffffffu, p0, 0);
                if (take) {
                    const int p = p0 + __popc(bal & ((1u << (tid & 31)) - 1));
                    if (p < a.candK) {
                        if (kb <= 32) ckey[p] = (ckeyof(lu, id) << 32) | (unsigned)sl;   // packed: one 64-bit sort key
                        else { ckey[p] = ((lu - minl) << 32) | id; cslot[p] = sl; clen[p] = a.slot_len[sl]; }
                    }
                }
            }
            __syncthreads();
            const int cn = min(s_cn, a.candK);
            if (kb <= 32) {
                // (compact key, slot) packed in 64 bits; sort only the next power of two above cn; one
                // thread per compare-exchange pair (the 3-array, thread-per-element form was ~140 us per
                // evicting batch on config-5 churn)
                int Kp = 2;
                while (Kp < cn) Kp <<= 1;
                for (int p = cn + tid; p < Kp; p += blockDim.x) ckey[p] = ~0ULL;
                __syncthreads();
                PROF_T(12);
                for (int kk = 2; kk <= Kp; kk <<= 1)
                    for (int jj = kk >> 1; jj > 0; jj >>= 1) {
                        for (int pr = tid; pr < Kp / 2; pr += blockDim.x) {
                            const int i2 = 2 * jj * (pr / jj) + (pr % jj), ix = i2 + jj;
                            const bool up = (i2 & kk) == 0;
                            const unsigned long long x = ckey[i2], y = ckey[ix];
                            if ((x > y) == up) { ckey[i2] = y; ckey[ix] = x; }
                        }
                        __syncthreads();
                    }
                // unpack to the list format the pops read: ((last - minl) << 32 | id, slot, length)
                const unsigned long long idmask = (1ULL << idb) - 1;
                for (int p = tid; p < a.candK; p += blockDim.x) {
                    if (p < cn) {
                        const unsigned long long sk = ckey[p], ck = sk >> 32;
                        const int sl = (int)(sk & 0xffffffffu);
                        ckey[p] = ((ck >> idb) << 32) | ((ck & idmask) + idmin);
                        cslot[p] = sl; clen[p] = a.slot_len[sl];
                    } else { ckey[p] = ~0ULL; cslot[p] = -1; clen[p] = 0; }
                }
                __syncthreads();
            } else {
            for (int p = cn + tid; p < a.candK; p += blockDim.x) { ckey[p] = ~0ULL; cslot[p] = -1; clen[p] = 0; }
            __syncthreads();
            PROF_T(12);
            // bitonic sort of the K candidates by key (keys are unique)
            for (int kk = 2; kk <= a.candK; kk <<= 1)
                for (int jj = kk >> 1; jj > 0; jj >>= 1) {
                    for (int i2 = tid; i2 < a.candK; i2 += blockDim.x) {
                        const int ix = i2 ^ jj;
                        if (ix > i2) {
                            const bool up = (i2 & kk) == 0;
                            const unsigned long long x = ckey[i2], y = ckey[ix];
                            if ((x > y) == up) {
                                ckey[i2] = y; ckey[ix] = x;
                                const int t2 = cslot[i2]; cslot[i2] = cslot[ix]; cslot[ix] = t2;
                                const int l2 = clen[i2]; clen[i2] = clen[ix]; clen[ix] = l2;
                            }
                        }
                    }
                    __syncthreads();
                }
            }
            if (tid == 0) { s_cn = cn; s_heap = 1; }
        }
        __syncthreads();
    }
    // ---- sequential part (warp 0).  Spans are applied in input order, 32 at a time: a Duplicate or a
    //      Dropped span changes no liveness, so every span up to the first one that must be stored is
    //      decided by its own lane against the same state; lane 0 then stores that span (supersedes,
    //      LRU evictions from the candidate list) and the next window starts after it.  Free-slot
    //      stack and free-page FIFO heads are cached in shared memory.  Page traffic is deferred:
    //      stores only record their FIFO position and removals their tail position; the block fills
    //      page lists and appends removed pages in parallel at the end.  That is exact while pops
    //      read only the FIFO's initial region and appends do not wrap onto it, and while no entry
    //      stored in this call is removed again; otherwise lane 0 materialises everything so far and
    //      continues immediately (flush).  Only an arg-min eviction (candidate list exhausted) brings
    //      the whole block in.
    __shared__ int s_stack_cache[kStackCache];
    __shared__ int s_fifo_cache[kFifoCache];
    __shared__ int s_sc_n, s_fc_n, s_fifo_head0, s_resume, s_argmin;
    __shared__ int s_defer, s_count0, s_ndef_rm;
    __shared__ long long s_appended;
    if (tid == 0) {
        s_sc_n = min(s_free_top, kStackCache);
        s_fc_n = min(s_fifo_count, kFifoCache);
        s_fifo_head0 = s_fifo_head;
        s_defer = 1; s_count0 = s_fifo_count; s_ndef_rm = 0; s_appended = 0;
    }
    __syncthreads();
    PROF_T(2);
    for (int k = tid; k < s_sc_n; k += blockDim.x) s_stack_cache[k] = a.slot_stack[s_free_top - 1 - k];
    for (int k = tid; k < s_fc_n; k += blockDim.x) s_fifo_cache[k] = a.fifo[(s_fifo_head0 + k) % a.P];
    __syncthreads();
    const int free_top0 = s_free_top;
    auto pop_slot = [&]() -> int {
        const int k = free_top0 - s_free_top;                  // pops so far
        const int slot = k < s_sc_n ? s_stack_cache[k] : a.slot_stack[s_free_top - 1];
        --s_free_top;
        return slot;
    };
    const int P32 = (int)a.P;                                  // page count (< 2^31)
    auto wrap = [&](int v) -> int { return v >= P32 ? v - P32 : v; };   // positions wrap at most once
    long long popped = 0;                                      // pages popped by this call (thread 0)
    auto fifo_at = [&](int pos) -> int {                      // pos: absolute FIFO position in [0, P)
        const int off = pos >= s_fifo_head0 ? pos - s_fifo_head0 : pos + P32 - s_fifo_head0;
        // the cached head window is valid until the FIFO could have wrapped around onto it
        return (off < s_fc_n && popped < (long long)P32 - s_fc_n) ? s_fifo_cache[off] : a.fifo[pos];
    };
    auto flush_deferred = [&]() {                              // thread 0: deferred page traffic, in order
        for (int r = 0; r < s_ndef_rm; ++r) {                  // appends land beyond the initial region
            const int sl = a.removed[r] & 0x7fffffff;
            const int npg = (a.slot_len[sl] + CP_BLOCK - 1) / CP_BLOCK;
            const int32_t* pl = a.slot_pages + (int64_t)sl * a.MP;
            for (int i = 0, pos = a.rm_pos[r]; i < npg; ++i, pos = wrap(pos + 1)) a.fifo[pos] = pl[i];
        }
        for (int j = 0; j < a.S; ++j) {                        // pops read the initial region
            if (sfpos[j] < 0) continue;
            const int npg = (slen[j] + CP_BLOCK - 1) / CP_BLOCK;
            int32_t* pl = a.slot_pages + (int64_t)snew[j] * a.MP;
            for (int i = 0, pos = sfpos[j]; i < npg; ++i, pos = wrap(pos + 1)) { pl[i] = fifo_at(pos); a.page_owner[pl[i]] = snew[j]; }
            sfpos[j] = -1;
        }
        s_defer = 0;
    };
    auto remove_serial = [&](int slot, int len) {             // pages to the FIFO tail (R#22)
        const int npg = (len + CP_BLOCK - 1) / CP_BLOCK;
        if (s_defer && ((sflag[slot] & 2) || (long long)s_count0 + s_appended + npg > (long long)P32)) flush_deferred();
        const int tail = wrap(s_fifo_head + s_fifo_count);
        if (s_defer) {
            a.rm_pos[s_nremoved] = tail;
            s_appended += npg;
            s_ndef_rm = s_nremoved + 1;
        } else {
            const int32_t* pl = a.slot_pages + (int64_t)slot * a.MP;
            for (int i0 = 0; i0 < npg; i0 += 16) {            // 16 independent loads, then the stores
                int v[16];
#pragma unroll
                for (int u = 0; u < 16; ++u) v[u] = (i0 + u < npg) ? __ldcg(pl + i0 + u) : 0;
                int pos = wrap(tail + i0);
#pragma unroll
                for (int u = 0; u < 16; ++u)
                    if (i0 + u < npg) { a.fifo[pos] = v[u]; pos = wrap(pos + 1); }
            }
        }
        s_fifo_count += npg;
        a.removed[s_nremoved++] = slot | ((sflag[slot] & 2) ? (int)0x80000000 : 0);
        sflag[slot] = 0;
        s_live_tokens -= len;
        s_num_live -= 1;
    };
    auto pop_candidate = [&](int& len) -> int {
        if (!s_heap) return -1;
        while (s_cp < s_cn) {
            const int sl = cslot[s_cp];
            const unsigned long long k = ckey[s_cp];
            if ((k >> 32) + s_minl >= tnow) return -1;             // t-group: ordered by id with refreshed/new ones
            len = clen[s_cp];
            ++s_cp;
            // live, not stored or refreshed in this call, last_used still the listed one (a prepared list
            // predates this step's match touches)
            if ((sflag[sl] & 1) && !(sflag[sl] & 6) && a.slot_last[sl] == (k >> 32) + s_minl) return sl;
        }
        return -1;
    };
    // ---- parallel apply.  The sequential loop below pays ~2K cycles per stored span (config-5 churn:
    //      ~430 stores, ~0.5 ms per batch).  When the batch's segments do not interact -- no containment
    //      between two batch contents, no live segment superseded by one span and referenced by another,
    //      no LRU victim referenced by a later span, no candidate the eviction pointer passes before the
    //      span that refreshes or supersedes it, pops inside the FIFO's initial region, at most kFastSup
    //      supersedes per span -- every decision is the one the initial state gives, and ids, slots, pages,
    //      removal order and FIFO positions are prefix sums.  The result is then exactly the sequential
    //      one (R#20-22); otherwise the sequential loop runs, from the untouched state.
    __shared__ int s_fast, s_ns;
    __shared__ long long s_s64[kCommitThreads / 32 + 1];
    __shared__ int s_why;                 // why the parallel apply was not taken (bit mask, diagnostics)
    const int Sn = a.S;
    if (tid == 0) {
        s_fast = a.force_serial ? 0 : 1; s_why = a.force_serial ? 1 : 0;
        if (s_pinned_tok > 0) { s_fast = 0; s_why |= 1024; }      // pinned entries: the sequential rules (R#32)
    }
    // f_refs / f_evpos / f_maxpos / f_supby / f_sidx come initialised (k_ins_validate) and f_last (each
    // content's last span) filled (k_ins_rep) by the prepare
    __syncthreads();
    PROF_T(5);
    for (int r = tid; r < Sn; r += blockDim.x) {                 // decision of each content vs the initial pool
        if (srep[r] != r) continue;
        int dup = -1, cont = -1, cont_id = INT_MAX, nsup = 0, suptok = 0, suppg = 0;
        bool bad = false;
        for (int q = soff[r]; q < soff[r + 1]; ++q) {
            const int2 rr = rec[q];
            if (rr.x < 0) { bad = true; break; }                   // relation between two batch contents
            if (!(sflag[rr.x] & 1)) continue;
            if (rr.y == REL_EQ) dup = rr.x;
            else if (rr.y == REL_CONTAINER) { const int sid = a.slot_id[rr.x]; if (sid < cont_id) { cont_id = sid; cont = rr.x; } }
            else { ++nsup; suptok += a.slot_len[rr.x]; suppg += (a.slot_len[rr.x] + CP_BLOCK - 1) / CP_BLOCK; }
        }
        if (bad) { s_fast = 0; atomicOr(&s_why, 2); continue; }
        const int kind = dup >= 0 ? 0 : cont >= 0 ? 1 : 2;        // 0 Duplicate, 1 Dropped, 2 store
        if (kind == 2 && nsup > kFastSup) { s_fast = 0; atomicOr(&s_why, 4); }
        a.f_kind[r] = kind; a.f_target[r] = dup >= 0 ? dup : cont;
        a.f_supcnt[r] = kind == 2 ? nsup : 0; a.f_suptok[r] = kind == 2 ? suptok : 0; a.f_suppg[r] = kind == 2 ? suppg : 0;
        a.f_sidx[r] = kind == 2 ? 1 : 0;
        const int last = a.f_last[r];
        for (int q = soff[r]; q < soff[r + 1]; ++q) {
            const int2 rr = rec[q];
            if (!(sflag[rr.x] & 1)) continue;
            atomicAdd(&a.f_refs[rr.x], 1);
            atomicMax(&a.f_maxpos[rr.x], last);                     // referenced up to the content's last span
            if (rr.y == REL_EQ) atomicMin(&a.f_evpos[rr.x], r);     // refreshed at r
            if (rr.y == REL_CONTAINED && kind == 2) {
                atomicMin(&a.f_evpos[rr.x], r);                     // superseded at r
                if (atomicCAS(&a.f_supby[rr.x], -1, r) != -1) { s_fast = 0; atomicOr(&s_why, 8); }
            }
        }
    }
    __syncthreads();
    // a live segment superseded by one span and referenced by another (f_supby >= 0 marks exactly the live
    // CONTAINED records of storing contents: walk those records, not the whole slot table)
    for (int r = tid; r < Sn; r += blockDim.x) {
        if (srep[r] != r || a.f_kind[r] != 2) continue;
        for (int q = soff[r]; q < soff[r + 1]; ++q) {
            const int2 rr = rec[q];
            if (rr.y == REL_CONTAINED && rr.x >= 0 && (sflag[rr.x] & 1) && a.f_refs[rr.x] > 1) { s_fast = 0; atomicOr(&s_why, 8); }
        }
    }
    __syncthreads();
    PROF_T(6);
    if (s_fast) {
        // store order: exclusive scan of the storing contents (a content is stored by its first span)
        const int ns = block_excl_scan<kCommitThreads>(a.f_sidx, Sn, s_wsum);
        if (tid == 0) s_ns = ns;
        for (int r = tid; r < Sn; r += blockDim.x) {
            if (srep[r] != r || a.f_kind[r] != 2) continue;
            const int k = a.f_sidx[r], m = slen[r];
            a.f_sj[k] = r;
            a.f_pgpref[k] = (m + CP_BLOCK - 1) / CP_BLOCK;
            a.f_netpref[k] = (long long)m - a.f_suptok[r];
            a.f_rmpref[k] = a.f_supcnt[r];
            a.f_suppgpref[k] = a.f_suppg[r];
        }
        __syncthreads();
        const int totpg = block_excl_scan<kCommitThreads>(a.f_pgpref, ns, s_wsum);
        const int totsup = block_excl_scan<kCommitThreads>(a.f_rmpref, ns, s_wsum);
        const int totsuppg = block_excl_scan<kCommitThreads>(a.f_suppgpref, ns, s_wsum);
        const long long totnet = block_excl_scan64<kCommitThreads>(a.f_netpref, ns, s_s64);
        (void)totpg; (void)totsup; (void)totsuppg; (void)totnet;
        __syncthreads();
        PROF_T(7);
        // ---- LRU: the victims, in candidate-list order, that the sequential evictions would pop
        const long long L0 = s_live_tokens;
        bool evict = false;
        for (int k = tid; k < ns; k += blockDim.x) evict |= L0 + a.f_netpref[k] + (long long)slen[a.f_sj[k]] - a.f_suptok[a.f_sj[k]] > a.capacity;
        evict = __syncthreads_or(evict);
        if (evict && !s_heap) { if (tid == 0) { s_fast = 0; atomicOr(&s_why, 16); } }
        __syncthreads();
        if (s_fast && evict) {
            const int cn = s_cn;
            // kept = live old entries not refreshed / superseded in this call (the pop test of the loop)
            for (int q = tid; q < cn; q += blockDim.x) {
                const int sl = cslot[q];
                a.f_vfc[q] = (sl >= 0 && (sflag[sl] & 1) && !(sflag[sl] & 4) && a.f_evpos[sl] == INT_MAX &&
                              a.slot_last[sl] == (ckey[q] >> 32) + s_minl) ? 1 : 0;
            }
            __syncthreads();
            for (int q = tid; q < cn; q += blockDim.x) a.f_vlen[q] = a.f_vfc[q];      // keep flags
            __syncthreads();
            const int nv = block_excl_scan<kCommitThreads>(a.f_vfc, cn, s_wsum);        // f_vfc[q] = kept before q
            for (int q = tid; q < cn; q += blockDim.x)
                if (a.f_vlen[q]) { const int v = a.f_vfc[q]; a.f_vslot[v] = cslot[q]; }
            __syncthreads();
            for (int v = tid; v < nv; v += blockDim.x) {
                const int L = a.slot_len[a.f_vslot[v]];
                a.f_vcum[v] = L; a.f_vcpg[v] = (L + CP_BLOCK - 1) / CP_BLOCK;
            }
            __syncthreads();
            const long long vtot = block_excl_scan64<kCommitThreads>(a.f_vcum, nv, s_s64);
            const int vtotpg = block_excl_scan<kCommitThreads>(a.f_vcpg, nv, s_wsum);
            if (tid == 0) { a.f_vcum[nv] = vtot; a.f_vcpg[nv] = vtotpg; }
            __syncthreads();
            // victims needed after store k: smallest v with L0 + net_incl(k) - vcum[v] <= capacity
            const bool complete = cn >= s_num_live;                 // the list holds every live entry
            for (int k = tid; k < ns; k += blockDim.x) {
                const int j = a.f_sj[k];
                const long long P = L0 + a.f_netpref[k] + (long long)slen[j] - a.f_suptok[j];
                int lo = 0, hi = nv;
                if (P - a.f_vcum[nv] > a.capacity) { s_fast = 0; atomicOr(&s_why, 32); lo = nv; }
                else while (lo < hi) { const int mid = (lo + hi) >> 1; if (P - a.f_vcum[mid] <= a.capacity) hi = mid; else lo = mid + 1; }
                a.f_vk[k] = lo;
            }
            (void)complete;
            __syncthreads();
            block_incl_maxscan<kCommitThreads>(a.f_vk, ns, s_wsum);
            const int Vtot = ns > 0 ? a.f_vk[ns - 1] : 0;
            // every list entry the pointer reaches (q with f_vfc[q] < Vtot): not in the t-group (the loop
            // would fall back to the arg-min), a victim not referenced after its pop, a skipped entry
            // refreshed / superseded before it
            for (int q = tid; q < cn; q += blockDim.x) {
                const int fc = a.f_vfc[q];
                if (fc >= Vtot) continue;
                if ((ckey[q] >> 32) + s_minl >= tnow) { s_fast = 0; atomicOr(&s_why, 64); continue; }
                int lo = 0, hi = ns - 1;                              // store whose eviction reaches q
                while (lo < hi) { const int mid = (lo + hi) >> 1; if (a.f_vk[mid] > fc) hi = mid; else lo = mid + 1; }
                const int jk = a.f_sj[lo], sl = cslot[q];
                if (a.f_vlen[q]) { if (a.f_maxpos[sl] > jk) { s_fast = 0; atomicOr(&s_why, 128); } }
                else if ((sflag[sl] & 1) && !(sflag[sl] & 4) && a.slot_last[sl] == (ckey[q] >> 32) + s_minl &&
                         !(a.f_evpos[sl] < jk)) { s_fast = 0; atomicOr(&s_why, 256); }
            }
        } else if (s_fast) {
            for (int k = tid; k < ns; k += blockDim.x) a.f_vk[k] = 0;
            if (tid == 0) { a.f_vcum[0] = 0; a.f_vcpg[0] = 0; }
        }
        __syncthreads();
    }
    if (s_fast) {
        // every pop reads a page that is free at that point of the sequential order: the initial free
        // pages, then the pages appended by removals before it (supersedes up to this store, evictions
        // after the earlier stores)
        for (int k = tid; k < s_ns; k += blockDim.x) {
            const int j = a.f_sj[k];
            const int end = a.f_pgpref[k] + (slen[j] + CP_BLOCK - 1) / CP_BLOCK;
            const int app = a.f_suppgpref[k] + a.f_suppg[j] + a.f_vcpg[k > 0 ? a.f_vk[k - 1] : 0];
            if (end > s_count0 + app) { s_fast = 0; atomicOr(&s_why, 512); }
        }
        __syncthreads();
        PROF_T(8);
    }
    if (s_fast) {
        // ---- apply (nothing above changed the index)
        const int ns = s_ns;
        const int tail0 = wrap(s_fifo_head0 + s_count0);
        for (int j = tid; j < Sn; j += blockDim.x) {
            const int r = srep[j], kind = a.f_kind[r];
            if (kind == 0) {
                const int X = a.f_target[r];
                a.slot_last[X] = tnow; a.out_tmp[j] = X; a.out_oc[j] = CP_DUPLICATE;
            } else if (kind == 1) {
                a.out_tmp[j] = a.f_target[r]; a.out_oc[j] = CP_DROPPED_CONTAINED;
            }
        }
        for (int k = tid; k < ns; k += blockDim.x) {
            const int j = a.f_sj[k], m = slen[j];
            const int slot = k < s_sc_n ? s_stack_cache[k] : a.slot_stack[free_top0 - 1 - k];
            a.slot_id[slot] = s_next_id + k; a.slot_len[slot] = m; a.slot_last[slot] = tnow;
            snew[j] = slot; sfpos[j] = wrap(s_fifo_head0 + a.f_pgpref[k]);
            a.out_tmp[j] = slot; a.out_oc[j] = a.f_supcnt[j] > 0 ? CP_SUPERSEDED : CP_STORED;
            // removals of this store: its supersedes (ascending id), then its LRU victims
            const int v0 = k > 0 ? a.f_vk[k - 1] : 0, v1 = a.f_vk[k];
            int base = a.f_rmpref[k] + v0;
            int pg = a.f_suppgpref[k] + a.f_vcpg[v0];
            int sup[kFastSup], ns2 = 0;
            for (int q = soff[j]; q < soff[j + 1]; ++q) {
                const int2 rr = rec[q];
                if (rr.y == REL_CONTAINED && (sflag[rr.x] & 1)) sup[ns2++] = rr.x;
            }
            for (int x = 1; x < ns2; ++x)
                for (int y = x; y > 0 && a.slot_id[sup[y]] < a.slot_id[sup[y - 1]]; --y) { const int tt = sup[y]; sup[y] = sup[y - 1]; sup[y - 1] = tt; }
            for (int x = 0; x < ns2; ++x) {
                a.removed[base] = sup[x]; a.rm_pos[base] = wrap(tail0 + pg);
                pg += (a.slot_len[sup[x]] + CP_BLOCK - 1) / CP_BLOCK; ++base;
            }
            for (int v = v0; v < v1; ++v) {
                const int sl = a.f_vslot[v];
                a.removed[base] = sl; a.rm_pos[base] = wrap(tail0 + pg);
                pg += (a.slot_len[sl] + CP_BLOCK - 1) / CP_BLOCK; ++base;
            }
        }
        __syncthreads();
        for (int j = tid; j < Sn; j += blockDim.x) {             // later spans of a stored content: Duplicates
            const int r = srep[j];
            if (r != j && a.f_kind[r] == 2) { a.out_tmp[j] = snew[r]; a.out_oc[j] = CP_DUPLICATE; }
        }
        const int Vtot = ns > 0 ? a.f_vk[ns - 1] : 0;
        const int nrm = (ns > 0 ? a.f_rmpref[ns - 1] + a.f_supcnt[a.f_sj[ns - 1]] : 0) + Vtot;
        for (int x = tid; x < nrm; x += blockDim.x) sflag[a.removed[x]] = 0;
        __syncthreads();
        for (int j = tid; j < Sn; j += blockDim.x) {
            if (srep[j] == j && a.f_kind[j] == 0) sflag[a.f_target[j]] |= 4;
            if (snew[j] >= 0) sflag[snew[j]] = 3;
        }
        if (tid == 0) {
            const int totpg = ns > 0 ? a.f_pgpref[ns - 1] + (slen[a.f_sj[ns - 1]] + CP_BLOCK - 1) / CP_BLOCK : 0;
            const int rmpg = (ns > 0 ? a.f_suppgpref[ns - 1] + a.f_suppg[a.f_sj[ns - 1]] : 0) + a.f_vcpg[Vtot];
            const long long lastnet = ns > 0 ? (long long)slen[a.f_sj[ns - 1]] - a.f_suptok[a.f_sj[ns - 1]] : 0;
            s_live_tokens = s_live_tokens + (ns > 0 ? a.f_netpref[ns - 1] + lastnet : 0) - a.f_vcum[Vtot];
            s_fifo_head = wrap(s_fifo_head0 + totpg);
            s_fifo_count = s_count0 - totpg + rmpg;
            s_next_id += ns; s_free_top = free_top0 - ns; s_num_live += ns - nrm;
            s_nremoved = nrm; s_ndef_rm = nrm; s_appended = rmpg;
            atomicAdd(&a.hdr->commits_parallel, 1);
        }
        __syncthreads();
        PROF_T(9);
    } else if (tid == 0) {
        atomicAdd(&a.hdr->commits_serial, 1);
        atomicOr(&a.hdr->commit_why, s_why);
    }
    int j0 = jstar;
    while (!s_fast) {
        if (tid < 32) {
            if (tid == 0) { s_resume = a.S; s_argmin = 0; }
            __syncwarp();
            int j = j0;
            while (j < a.S) {
                // ---- each lane decides span j + lane against the state at the window start
                const int jj = j + tid;
                int kind = 3, target = -1, rjj = 0;                // 0 Duplicate, 1 Dropped, 2 store, 3 none
                if (jj < a.S) {
                    rjj = srep[jj];
                    const int b = soff[rjj], e = soff[rjj + 1];
                    const int known = seq[rjj];                    // the pool holds at most one live entry per content
                    if (known >= 0 && (sflag[known] & 1)) target = known;
                    else {
                        if (rjj != jj && is_live(-1 - rjj)) target = resolve(-1 - rjj);   // its stored representative
                        for (int q = b; q < e && target < 0; ++q)
                            if (rec[q].y == REL_EQ && is_live(rec[q].x)) target = resolve(rec[q].x);
                    }
                    if (target >= 0) kind = 0;
                    else {
                        int cont_id = 0x7fffffff;
                        for (int q = b; q < e; ++q)
                            if (rec[q].y == REL_CONTAINER && is_live(rec[q].x)) {
                                const int sx = resolve(rec[q].x);
                                const int sid = a.slot_id[sx];
                                if (sid < cont_id) { cont_id = sid; target = sx; }
                            }
                        kind = target >= 0 ? 1 : 2;
                        if (kind == 2 && s_pinned_tok > 0) {      // R#32: it may not remove a pinned entry and
                            int bid = 0x7fffffff;                 // must fit the budget beside the pinned tokens
                            for (int q = b; q < e; ++q)
                                if (rec[q].y == REL_CONTAINED && is_live(rec[q].x)) {
                                    const int sx = resolve(rec[q].x);
                                    if (a.slot_pin[sx] > 0 && a.slot_id[sx] < bid) { bid = a.slot_id[sx]; target = sx; }
                                }
                            if (target >= 0 || s_pinned_tok + slen[jj] > a.capacity) kind = 4;
                        }
                    }
                }
                const unsigned need = __ballot_sync(0xffffffffu, kind == 2);
                const int f = need ? __ffs(need) - 1 : 32;
                if (tid < f && kind == 0) {                        // Duplicate refreshes last_used (R#20)
                    seq[rjj] = target;
                    a.slot_last[target] = tnow;
                    sflag[target] |= 4;                            // same value from every lane that writes it
                    a.out_tmp[jj] = target; a.out_oc[jj] = CP_DUPLICATE;
                } else if (tid < f && kind == 1) {
                    a.out_tmp[jj] = target; a.out_oc[jj] = CP_DROPPED_CONTAINED;
                } else if (tid < f && kind == 4) {
                    a.out_tmp[jj] = target; a.out_oc[jj] = CP_DEFERRED_PINNED;
                }
                __syncwarp();
                if (f == 32) { j += 32; continue; }
                const int js = j + f;                              // the first span that must be stored
                if (tid == 0) {
                    const int rj = srep[js];
                    const int b = soff[rj], e = soff[rj + 1];
                    // supersede: the live entries it strictly contains, ascending id
                    int n = 0;
                    for (int q = b; q < e; ++q)
                        if (rec[q].y == REL_CONTAINED && is_live(rec[q].x)) {
                            const int sx = resolve(rec[q].x);
                            bool seen = false;
                            for (int z = 0; z < n; ++z) seen |= (s_rm[z] == sx);
                            if (!seen && n < kMaxSupersede) s_rm[n++] = sx;     // n <= CONTAINED records (checked)
                        }
                    for (int x = 1; x < n; ++x)      // insertion sort by id
                        for (int y = x; y > 0 && a.slot_id[s_rm[y]] < a.slot_id[s_rm[y - 1]]; --y) {
                            const int tmp = s_rm[y]; s_rm[y] = s_rm[y - 1]; s_rm[y - 1] = tmp;
                        }
                    for (int x = 0; x < n; ++x) remove_serial(s_rm[x], a.slot_len[s_rm[x]]);
                    // store span js: id = next id, pages from the FIFO head (R#22)
                    const int m = slen[js];
                    const int slot = pop_slot();
                    const int id = s_next_id++;
                    const int npg = (m + CP_BLOCK - 1) / CP_BLOCK;
                    if (s_fifo_count < npg) cp_raise(a.hdr, CP_ERR_CAPACITY);
                    if (s_defer && popped + npg > (long long)s_count0) flush_deferred();
                    if (s_defer) sfpos[js] = s_fifo_head;
                    else {
                        int32_t* pl = a.slot_pages + (int64_t)slot * a.MP;
                        for (int i = 0, pos = s_fifo_head; i < npg; ++i, pos = wrap(pos + 1)) { pl[i] = fifo_at(pos); a.page_owner[pl[i]] = slot; }
                    }
                    popped += npg;
                    s_fifo_head = wrap(s_fifo_head + npg); s_fifo_count -= npg;
                    s_live_tokens += m; s_num_live += 1;
                    sflag[slot] = 3; snew[js] = slot; seq[rj] = slot;
                    // id / len / last_used are read by later decisions; origin and hashes are written by
                    // the parallel write-back (no global loads on this path)
                    a.slot_id[slot] = id; a.slot_len[slot] = m; a.slot_last[slot] = tnow;
                    a.out_tmp[js] = slot; a.out_oc[js] = n > 0 ? CP_SUPERSEDED : CP_STORED;
                    PROF_CNT(13, 1);
                    // LRU eviction: victim = min (last_used, id) among live entries (R#21)
                    while (s_live_tokens > a.capacity) {
                        int vlen = 0;
                        const int v = pop_candidate(vlen);
                        if (v < 0) { s_argmin = 1; s_resume = js + 1; break; }
                        remove_serial(v, vlen);
                        PROF_CNT(14, 1);
                    }
                }
                __syncwarp();
                if (s_argmin) break;
                j = js + 1;
            }
        }
        __syncthreads();
        if (!s_argmin) break;
        PROF_CNT(15, tid == 0 ? 1 : 0);
        // block-wide arg-min evictions until the budget holds, then continue after span s_resume - 1
        while (s_live_tokens > a.capacity) {
            unsigned long long best_last = ~0ULL; int best_id = 0x7fffffff, best_slot = -1;
            for (int sx = tid; sx < a.nslots; sx += blockDim.x) {
                if (!(sflag[sx] & 1) || a.slot_pin[sx] > 0) continue;
                const unsigned long long lu = a.slot_last[sx];
                const int sid = a.slot_id[sx];
                if (lu < best_last || (lu == best_last && sid < best_id)) { best_last = lu; best_id = sid; best_slot = sx; }
            }
            for (int off = 16; off; off >>= 1) {
                const unsigned long long ol = __shfl_xor_sync(0xffffffffu, best_last, off);
                const int oi = __shfl_xor_sync(0xffffffffu, best_id, off);
                const int os = __shfl_xor_sync(0xffffffffu, best_slot, off);
                if (ol < best_last || (ol == best_last && oi < best_id)) { best_last = ol; best_id = oi; best_slot = os; }
            }
            if ((tid & 31) == 0) { s_red_key[tid >> 5] = best_last; s_red_slot[tid >> 5] = best_slot; s_wsum[tid >> 5] = best_id; }
            __syncthreads();
            if (tid == 0) {
                int bs = -1, bi = 0x7fffffff; unsigned long long bl = ~0ULL;
                for (int w = 0; w < kCommitThreads / 32; ++w) {
                    if (s_red_slot[w] < 0) continue;
                    if (s_red_key[w] < bl || (s_red_key[w] == bl && s_wsum[w] < bi)) { bl = s_red_key[w]; bi = s_wsum[w]; bs = s_red_slot[w]; }
                }
                if (bs >= 0) remove_serial(bs, a.slot_len[bs]);
                else { cp_raise(a.hdr, CP_ERR_CAPACITY); s_live_tokens = 0; }   // unreachable: R#32 defers such stores
            }
            __syncthreads();
        }
        j0 = s_resume;
        __syncthreads();                 // every thread has read s_resume before thread 0 resets it
    }
    __syncthreads();
    // ---- deferred page traffic, block-parallel (warp per removal / per stored span): appended pages
    //      go beyond the FIFO's initial region; the sequential loop's pops stay inside it, the parallel
    //      apply's may reach appended pages (written first)
    if (s_defer) {
        const int cw = tid >> 5, cl = tid & 31, nw = kCommitThreads / 32;
        for (int r = cw; r < s_ndef_rm; r += nw) {
            const int sl = a.removed[r] & 0x7fffffff;
            const int npg = (a.slot_len[sl] + CP_BLOCK - 1) / CP_BLOCK;
            const int32_t* pl = a.slot_pages + (int64_t)sl * a.MP;
            for (int i = cl; i < npg; i += 32) a.fifo[wrap(a.rm_pos[r] + i)] = pl[i];
        }
        __syncthreads();                 // pops past the initial region read pages appended above (parallel apply)
        for (int j = cw; j < a.S; j += nw) {
            if (sfpos[j] < 0) continue;
            const int npg = (slen[j] + CP_BLOCK - 1) / CP_BLOCK;
            int32_t* pl = a.slot_pages + (int64_t)snew[j] * a.MP;
            for (int i = cl; i < npg; i += 32) { pl[i] = a.fifo[wrap(sfpos[j] + i)]; a.page_owner[pl[i]] = snew[j]; }
        }
    }
    __syncthreads();
    PROF_T(3);
    // ---- write back (block-parallel): removed slots return to the free stack; the new live entries
    //      get their origin / hashes and are listed, in span order, for publishing and copy-in
    const int nrm = s_nremoved, top0 = s_free_top;
    for (int r = tid; r < nrm; r += blockDim.x) a.slot_stack[top0 + r] = a.removed[r] & 0x7fffffff;
    for (int j = tid; j < a.S; j += blockDim.x) {           // soff is free now: new-live flags
        const int slot = snew[j];
        soff[j] = (slot >= 0 && (sflag[slot] & 1)) ? 1 : 0;
    }
    __syncthreads();
    const int nl = block_excl_scan<kCommitThreads>(soff, a.S, s_wsum);
    for (int j = tid; j < a.S; j += blockDim.x) {
        const int slot = snew[j];
        if (slot < 0 || !(sflag[slot] & 1)) continue;
        const int q = soff[j];
        a.slot_origin[slot] = a.span_begin[j]; a.slot_prefix[slot] = a.span_pre[j]; a.slot_full[slot] = a.span_full[j];
        a.slot_owner[slot] = 0;                              // a shared entry (the slot may have been private)
        a.cp_req[q] = a.span_req[j]; a.cp_slot[q] = slot; a.cp_dst[q] = a.span_begin[j];
        a.cp_len[q] = slen[j]; a.cp_delta[q] = j;            // cp_delta carries the span index
    }
    if (tid == 0) {
        a.hdr->n_copy = nl; a.hdr->n_new_live = nl; a.hdr->n_removed = nrm;
        a.hdr->live_tokens = s_live_tokens; a.hdr->fifo_head = s_fifo_head; a.hdr->fifo_count = s_fifo_count;
        a.hdr->next_id = s_next_id; a.hdr->slot_free_top = top0 + nrm; a.hdr->num_live = s_num_live;
    }
    __syncthreads();
    for (int i = tid; i < a.nslots; i += blockDim.x) a.slot_state[i] = (sflag[i] & 1) ? CP_SLOT_LIVE : CP_SLOT_FREE;
    // entry ids of the outcomes (the block's slot_id writes are visible after the barrier above; this was
    // the separate k_ins_outids launch)
    for (int j = tid; j < a.S; j += blockDim.x) { const int sx = a.out_tmp[j]; a.out_id[j] = sx >= 0 ? a.slot_id[sx] : -1; }
    __syncthreads();
    PROF_T(4);
}

// map the committed slot of each span to its entry id (parallel)
__global__ void k_ins_outids(InsArgs a) {
    if (cp_err_set(a.hdr)) return;
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < a.S; j += gridDim.x * blockDim.x) {
        const int s = a.out_tmp[j];
        a.out_id[j] = s >= 0 ? a.slot_id[s] : -1;
    }
}

// tombstone prefix-table entries of removed pool entries (those that were in the table); warp per slot
__global__ void k_ins_delete(InsArgs a) {
    if (cp_err_set(a.hdr)) return;
    const int n = a.hdr->n_removed;
    const int lane = threadIdx.x & 31;
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int nwarps = (gridDim.x * blockDim.x) >> 5;
    for (int r = warp; r < n; r += nwarps) {
        const int code = a.removed[r];
        if (code < 0) continue;               // stored and removed within this call: never published
        const int slot = code;
        const unsigned long long key = a.slot_prefix[slot];
        uint32_t p0 = cp_hpos(key, a.logT);
        while (true) {
            const uint32_t p = (p0 + lane) & (uint32_t)(a.T - 1);
            const unsigned long long k = a.htab[p].key;
            const bool hit = k == key && a.htab[p].slot == slot;
            const unsigned empt = __ballot_sync(0xffffffffu, k == CP_EMPTY_KEY);
            const unsigned hits = __ballot_sync(0xffffffffu, hit);
            const int lim = empt ? __ffs(empt) - 1 : 32;
            const unsigned before = lim == 32 ? hits : (hits & ((1u << lim) - 1u));
            if (before) { if (lane == __ffs(before) - 1) a.htab[p].key = CP_TOMB_KEY; break; }
            if (empt) break;
            p0 = (p0 + 32) & (uint32_t)(a.T - 1);
        }
    }
}

// SHA-256 (FIPS 180-4) over big-endian u64 token ids (R#6); one thread per entry
__device__ const uint32_t kK256[64] = {
    0x428a2f98, 0x71374491, 0xb5c0fbcf, 0xe9b5dba5, 0x3956c25b, 0x59f111f1, 0x923f82a4, 0xab1c5ed5,
    0xd807aa98, 0x12835b01, 0x243185be, 0x550c7dc3, 0x72be5d74, 0x80deb1fe, 0x9bdc06a7, 0xc19bf174,
    0xe49b69c1, 0xefbe4786, 0x0fc19dc6, 0x240ca1cc, 0x2de92c6f, 0x4a7484aa, 0x5cb0a9dc, 0x76f988da,
    0x983e5152, 0xa831c66d, 0xb00327c8, 0xbf597fc7, 0xc6e00bf3, 0xd5a79147, 0x06ca6351, 0x14292967,
    0x27b70a85, 0x2e1b2138, 0x4d2c6dfc, 0x53380d13, 0x650a7354, 0x766a0abb, 0x81c2c92e, 0x92722c85,
    0xa2bfe8a1, 0xa81a664b, 0xc24b8b70, 0xc76c51a3, 0xd192e819, 0xd6990624, 0xf40e3585, 0x106aa070,
    0x19a4c116, 0x1e376c08, 0x2748774c, 0x34b0bcb5, 0x391c0cb3, 0x4ed8aa4a, 0x5b9cca4f, 0x682e6ff3,
    0x748f82ee, 0x78a5636f, 0x84c87814, 0x8cc70208, 0x90befffa, 0xa4506ceb, 0xbef9a3f7, 0xc67178f2};

__device__ __forceinline__ uint32_t rotr32(uint32_t x, int n) { return __funnelshift_r(x, x, n); }

__device__ void sha256_compress(uint32_t H[8], const uint32_t Win[16]) {
    uint32_t W[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) W[i] = Win[i];
    uint32_t a = H[0], b = H[1], c = H[2], d = H[3], e = H[4], f = H[5], g = H[6], h = H[7];
#pragma unroll 16
    for (int t = 0; t < 64; ++t) {
        uint32_t wt;
        if (t < 16) wt = W[t];
        else {
            const uint32_t w15 = W[(t - 15) & 15], w2 = W[(t - 2) & 15];
            const uint32_t s0 = rotr32(w15, 7) ^ rotr32(w15, 18) ^ (w15 >> 3);
            const uint32_t s1 = rotr32(w2, 17) ^ rotr32(w2, 19) ^ (w2 >> 10);
            wt = W[t & 15] = W[t & 15] + s0 + W[(t - 7) & 15] + s1;
        }
        const uint32_t S1 = rotr32(e, 6) ^ rotr32(e, 11) ^ rotr32(e, 25);
        const uint32_t ch = (e & f) ^ (~e & g);
        const uint32_t T1 = h + S1 + ch + kK256[t] + wt;
        const uint32_t S0 = rotr32(a, 2) ^ rotr32(a, 13) ^ rotr32(a, 22);
        const uint32_t mj = (a & b) ^ (a & c) ^ (b & c);
        h = g; g = f; f = e; e = d + T1; d = c; c = b; b = a; a = T1 + S0 + mj;
    }
    H[0] += a; H[1] += b; H[2] += c; H[3] += d; H[4] += e; H[5] += f; H[6] += g; H[7] += h;
}

__device__ void sha256_tokens_dev(const int32_t* tau, int m, uint8_t* out) {
    uint32_t H[8] = {0x6a09e667, 0xbb67ae85, 0x3c6ef372, 0xa54ff53a, 0x510e527f, 0x9b05688c, 0x1f83d9ab, 0x5be0cd19};
    uint32_t W[16];
    const int full = m / 8;
    for (int b = 0; b < full; ++b) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int64_t v = tau[8 * b + i];
            W[2 * i] = (uint32_t)((uint64_t)v >> 32); W[2 * i + 1] = (uint32_t)(uint64_t)v;
        }
        sha256_compress(H, W);
    }
    const int rem = m - 8 * full;
    for (int i = 0; i < 16; ++i) W[i] = 0;
    for (int i = 0; i < rem; ++i) {
        const int64_t v = tau[8 * full + i];
        W[2 * i] = (uint32_t)((uint64_t)v >> 32); W[2 * i + 1] = (uint32_t)(uint64_t)v;
    }
    W[2 * rem] = 0x80000000u;
    const uint64_t bits = (uint64_t)m * 64ULL;
    if (2 * rem + 1 > 14) {
        sha256_compress(H, W);
        for (int i = 0; i < 16; ++i) W[i] = 0;
    }
    W[14] = (uint32_t)(bits >> 32); W[15] = (uint32_t)bits;
    sha256_compress(H, W);
    for (int i = 0; i < 8; ++i) {
        out[4 * i] = (uint8_t)(H[i] >> 24); out[4 * i + 1] = (uint8_t)(H[i] >> 16);
        out[4 * i + 2] = (uint8_t)(H[i] >> 8); out[4 * i + 3] = (uint8_t)H[i];
    }
}

// publish new live entries: prefix table insert, token + recompute-bit store, digest
__global__ void k_ins_publish(InsArgs a) {
    if (cp_err_set(a.hdr)) return;
    const int n = a.hdr->n_new_live;
    const int lane = threadIdx.x & 31;
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int nwarps = (gridDim.x * blockDim.x) >> 5;
    for (int q = warp; q < n; q += nwarps) {
        const int slot = a.cp_slot[q], j = a.cp_delta[q], m = a.cp_len[q];
        const int32_t* tau = span_tokens(a, j);
        for (int t = lane; t < m; t += 32) {
            const int page = a.slot_pages[(int64_t)slot * a.MP + (t >> 4)];
            a.page_tokens[(int64_t)page * CP_BLOCK + (t & 15)] = tau[t];
        }
        const int npg = (m + CP_BLOCK - 1) / CP_BLOCK;
        for (int pg = lane; pg < npg; pg += 32) {
            uint32_t v = 0;
            if (a.bits) {
                for (int z = 0; z < CP_BLOCK && pg * CP_BLOCK + z < m; ++z) {
                    const int t = pg * CP_BLOCK + z;
                    v |= ((a.bits[a.bits_off[j] + (t >> 5)] >> (t & 31)) & 1u) << z;
                }
            }
            a.page_bits[a.slot_pages[(int64_t)slot * a.MP + pg]] = (uint16_t)v;
        }
        HEntry v; v.key = a.slot_prefix[slot]; v.full = a.slot_full[slot]; v.slot = slot; v.len = m; v.pad = 0;
        const bool fresh = cp_warp_insert(a.htab, (uint32_t)(a.T - 1), a.logT, v, true);
        if (fresh && lane == 0) atomicAdd(&a.hdr->table_used, 1);
    }
}

// rebuild the prefix table when tombstones accumulate (live + tombstones > T/2)
// ---- R#32 pins: validate every listed page (owned by a live entry), apply, undo if a count went negative
__global__ void k_pin_check(DevHeader* hdr, const int32_t* pages, int64_t n, const int32_t* page_owner,
                            const uint8_t* slot_state, const int32_t* slot_pages, int32_t MP, const int32_t* slot_len) {
    if (cp_err_set(hdr)) return;
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x) {
        const int p = pages[q];
        if (p < 0) continue;
        const int s = page_owner[p];
        bool ok = s >= 0 && slot_state[s] == CP_SLOT_LIVE;
        if (ok) {                                   // the page is in its owner's current page list
            const int npg = (slot_len[s] + CP_BLOCK - 1) / CP_BLOCK;
            bool in = false;
            for (int i = 0; i < npg && !in; ++i) in = slot_pages[(int64_t)s * MP + i] == p;
            ok = in;
        }
        if (!ok) cp_raise(hdr, CP_ERR_INVALID_ARG);
    }
}
__global__ void k_pin_apply(DevHeader* hdr, const int32_t* pages, int64_t n, const int32_t* page_owner,
                            int32_t* slot_pin, int32_t delta, int32_t undo) {
    if (cp_err_set(hdr)) return;
    if (undo && !hdr->pin_neg) return;
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x) {
        const int p = pages[q];
        if (p < 0) continue;
        const int v = atomicAdd(&slot_pin[page_owner[p]], undo ? -delta : delta) + (undo ? -delta : delta);
        if (!undo && v < 0) hdr->pin_neg = 1;
    }
}
__global__ void k_pin_done(DevHeader* hdr) {
    if (hdr->pin_neg && !cp_err_set(hdr)) cp_raise(hdr, CP_ERR_INVALID_ARG);   // after the undo
    hdr->pin_neg = 0;
    hdr->pin_epoch += 1;
}

// SHA-256 digests of the published entries (thread per entry; launched on the index's side stream,
// concurrently with the table rebuild and the copy-in, which do not read digests)
__global__ void k_ins_digest(InsArgs a) {
    if (cp_err_set(a.hdr)) return;
    const int n = a.hdr->n_new_live;
    for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < n; q += gridDim.x * blockDim.x) {
        const int slot = a.cp_slot[q], j = a.cp_delta[q], m = a.cp_len[q];
        sha256_tokens_dev(span_tokens(a, j), m, a.slot_digest + (int64_t)slot * 32);
    }
}


// ---- R#33 same-user sessions: cp_index_insert_session ----------------------------------------------
// thread per request: session in range, 1 <= n <= budget / max_span_len, block table wide enough, and a
// free slot for every request (the first failing request in input order decides; nothing changes)
__global__ void k_sess_validate(InsArgs a) {
    if (blockIdx.x == 0 && threadIdx.x == 0) { a.hdr->n_removed = 0; a.hdr->n_copy = 0; a.hdr->n_new_live = 0; }
    if (cp_err_set(a.hdr)) return;
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < a.num_reqs; r += gridDim.x * blockDim.x) {
        const int o = a.session[r];
        const int64_t n = a.offsets[r + 1] - a.offsets[r];
        int bad = -1;
        if (o < 1 || o > a.max_sessions || n < 1 || ((n - 1) >> 4) >= a.max_blocks) bad = 0;
        else if (n > a.capacity || n > a.max_span_len) bad = 2;
        if (bad >= 0) atomicMin(&a.hdr->first_err, ((unsigned long long)r << 32) | (unsigned)bad);
    }
    if (blockIdx.x == 0 && threadIdx.x == 0 && a.hdr->slot_free_top < a.num_reqs)
        atomicMin(&a.hdr->first_err, ((unsigned long long)0x7FFFFFFF << 32) | 2u);
}

// one CTA: the requests in input order (thread 0 bookkeeping, block-wide LRU arg-min), the same rules as
// the oracle's orc_index_insert_session.  Slots freed here go back to the free stack at the end (so an
// evicted shared entry's slot keeps its prefix hash until k_ins_delete tombstones it).
__global__ void __launch_bounds__(256) k_sess_commit(InsArgs a) {
    const unsigned long long tnow = a.clock ? *a.clock : a.t;
    __shared__ int s_abort, s_go, s_nfree, s_ncopy, s_nrm;
    __shared__ long long s_live, s_pinned;
    __shared__ unsigned long long s_bl[8]; __shared__ int s_bi[8], s_bs[8];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    if (tid == 0) {
        s_abort = 0;
        if (cp_err_set(a.hdr)) s_abort = 1;
        else if (a.hdr->first_err != CP_NO_ERR_KEY) { cp_raise(a.hdr, code_of((int)(a.hdr->first_err & 0xffffffffu))); s_abort = 1; }
        a.hdr->first_err = CP_NO_ERR_KEY;
        s_live = a.hdr->live_tokens; s_pinned = 0; s_nfree = 0; s_ncopy = 0; s_nrm = 0;
    }
    __syncthreads();
    if (s_abort) {
        for (int r = tid; r < a.num_reqs; r += blockDim.x) { a.out_oc[r] = -1; a.out_tmp[r] = -1; }
        return;
    }
    {
        long long pt = 0;
        for (int i = tid; i < a.nslots; i += blockDim.x)
            if (a.slot_state[i] == CP_SLOT_LIVE && a.slot_pin[i] > 0) pt += a.slot_len[i];
        for (int o = 16; o; o >>= 1) pt += __shfl_xor_sync(0xffffffffu, pt, o);
        if (lane == 0 && pt) atomicAdd((unsigned long long*)&s_pinned, (unsigned long long)pt);
    }
    __syncthreads();
    DevHeader* h = a.hdr;
    const int P32 = (int)a.P;
    auto remove = [&](int sl) {                     // thread 0: pages to the FIFO tail in page-list order
        const int npg = (a.slot_len[sl] + CP_BLOCK - 1) / CP_BLOCK;
        for (int i = 0; i < npg; ++i) {
            a.fifo[(h->fifo_head + h->fifo_count) % P32] = a.slot_pages[(int64_t)sl * a.MP + i];
            h->fifo_count++;
        }
        s_live -= a.slot_len[sl]; h->num_live--;
        a.slot_state[sl] = CP_SLOT_FREE;
        const int own = a.slot_owner[sl];
        if (own > 0) { if (a.session_slot[own] == sl) a.session_slot[own] = -1; }
        else a.removed[s_nrm++] = sl;                // shared: tombstone its prefix-table entry afterwards
        a.rm_pos[s_nfree++] = sl;                    // freed slots, pushed at the end
    };
    for (int r = 0; r < a.num_reqs; ++r) {
        const int o = a.session[r];
        const int n = (int)(a.offsets[r + 1] - a.offsets[r]);
        if (tid == 0) {
            int old = a.session_slot[o];
            if (old >= 0 && !(a.slot_state[old] == CP_SLOT_LIVE && a.slot_owner[old] == o)) old = -1;
            s_go = 1;
            if ((old >= 0 && a.slot_pin[old] > 0) || s_pinned + n > a.capacity) {        // R#32
                s_go = 0;
                a.out_tmp[r] = (old >= 0 && a.slot_pin[old] > 0) ? old : -1; a.out_oc[r] = CP_DEFERRED_PINNED;
            } else {
                if (old >= 0) remove(old);
                const int slot = a.slot_stack[--h->slot_free_top];
                const int id = h->next_id++;
                const int npg = (n + CP_BLOCK - 1) / CP_BLOCK;
                for (int i = 0; i < npg; ++i) {
                    const int pg = a.fifo[h->fifo_head];
                    h->fifo_head = (h->fifo_head + 1) % P32; h->fifo_count--;
                    a.slot_pages[(int64_t)slot * a.MP + i] = pg; a.page_owner[pg] = slot;
                }
                a.slot_id[slot] = id; a.slot_len[slot] = n; a.slot_origin[slot] = 0; a.slot_last[slot] = tnow;
                a.slot_prefix[slot] = 0; a.slot_full[slot] = 0; a.slot_owner[slot] = o;
                a.slot_state[slot] = CP_SLOT_LIVE;
                a.session_slot[o] = slot;
                s_live += n; h->num_live++;
                const int q = s_ncopy++;
                a.cp_req[q] = r; a.cp_slot[q] = slot; a.cp_dst[q] = 0; a.cp_len[q] = n; a.cp_delta[q] = r;
                a.out_tmp[r] = slot; a.out_oc[r] = CP_STORED;
            }
        }
        __syncthreads();
        // LRU (R#21, R#32): victim = min (last_used, id) among live unpinned entries of any owner
        while (s_go && s_live > a.capacity) {
            unsigned long long bl = ~0ULL; int bi = 0x7fffffff, bs = -1;
            for (int sx = tid; sx < a.nslots; sx += blockDim.x) {
                if (a.slot_state[sx] != CP_SLOT_LIVE || a.slot_pin[sx] > 0) continue;
                const unsigned long long lu = a.slot_last[sx];
                const int sid = a.slot_id[sx];
                if (lu < bl || (lu == bl && sid < bi)) { bl = lu; bi = sid; bs = sx; }
            }
            for (int off = 16; off; off >>= 1) {
                const unsigned long long ol = __shfl_xor_sync(0xffffffffu, bl, off);
                const int oi = __shfl_xor_sync(0xffffffffu, bi, off), os = __shfl_xor_sync(0xffffffffu, bs, off);
                if (ol < bl || (ol == bl && oi < bi)) { bl = ol; bi = oi; bs = os; }
            }
            if (lane == 0) { s_bl[wid] = bl; s_bi[wid] = bi; s_bs[wid] = bs; }
            __syncthreads();
            if (tid == 0) {
                int v = -1; unsigned long long vb = ~0ULL; int vi = 0x7fffffff;
                for (int w = 0; w < 8; ++w)
                    if (s_bs[w] >= 0 && (s_bl[w] < vb || (s_bl[w] == vb && s_bi[w] < vi))) { vb = s_bl[w]; vi = s_bi[w]; v = s_bs[w]; }
                if (v >= 0) remove(v); else { cp_raise(h, CP_ERR_CAPACITY); s_live = 0; }   // unreachable (R#32)
            }
            __syncthreads();
        }
        __syncthreads();
    }
    if (tid == 0) {
        for (int i = 0; i < s_nfree; ++i) a.slot_stack[h->slot_free_top++] = a.rm_pos[i];
        // entries stored and evicted again within this call are neither published nor copied (their pages
        // may already belong to a later entry); freed slots are not reused within the call, so "still
        // live" identifies the survivors
        int q2 = 0;
        for (int q = 0; q < s_ncopy; ++q) {
            if (a.slot_state[a.cp_slot[q]] != CP_SLOT_LIVE) continue;
            a.cp_req[q2] = a.cp_req[q]; a.cp_slot[q2] = a.cp_slot[q]; a.cp_dst[q2] = a.cp_dst[q];
            a.cp_len[q2] = a.cp_len[q]; a.cp_delta[q2] = a.cp_delta[q]; ++q2;
        }
        h->live_tokens = s_live; h->n_removed = s_nrm; h->n_copy = q2; h->n_new_live = q2;
    }
}

// warp per stored private entry: its tokens into the token store, no recompute marks, its SHA-256 digest
__global__ void k_sess_publish(InsArgs a) {
    if (cp_err_set(a.hdr)) return;
    const int n = a.hdr->n_new_live;
    const int lane = threadIdx.x & 31;
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nwarps = (gridDim.x * blockDim.x) >> 5;
    for (int q = warp; q < n; q += nwarps) {
        const int slot = a.cp_slot[q], r = a.cp_req[q], m = a.cp_len[q];
        const int32_t* tau = a.tokens + a.offsets[r];
        for (int t = lane; t < m; t += 32)
            a.page_tokens[(int64_t)a.slot_pages[(int64_t)slot * a.MP + (t >> 4)] * CP_BLOCK + (t & 15)] = tau[t];
        for (int pg = lane; pg < (m + CP_BLOCK - 1) / CP_BLOCK; pg += 32) a.page_bits[a.slot_pages[(int64_t)slot * a.MP + pg]] = 0;
        if (lane == 0) sha256_tokens_dev(tau, m, a.slot_digest + (int64_t)slot * 32);
    }
}

__global__ void k_rebuild_check(DevHeader* hdr, int64_t T) {
    hdr->rebuild = (hdr->error == 0 && (int64_t)hdr->table_used * 2 > T) ? 1 : 0;
}
__global__ void k_rebuild_clear(DevHeader* hdr, HEntry* htab, int64_t T) {
    if (!hdr->rebuild) return;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < T; i += (int64_t)gridDim.x * blockDim.x) {
        htab[i].key = CP_EMPTY_KEY; htab[i].slot = -1; htab[i].len = 0; htab[i].full = 0;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) hdr->table_used = 0;
}
__global__ void k_rebuild_fill(DevHeader* hdr, HEntry* htab, int logT, int64_t T, const uint8_t* state,
                               const unsigned long long* prefix, const unsigned long long* full,
                               const int32_t* len, int32_t nslots, const int32_t* owner) {
    if (!hdr->rebuild) return;
    const int lane = threadIdx.x & 31;
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int nwarps = (gridDim.x * blockDim.x) >> 5;
    for (int s = warp; s < nslots; s += nwarps) {
        if (state[s] != CP_SLOT_LIVE || owner[s] != 0) continue;          // private entries are not probed
        HEntry v; v.key = prefix[s]; v.full = full[s]; v.slot = s; v.len = len[s]; v.pad = 0;
        cp_warp_insert(htab, (uint32_t)(T - 1), logT, v, false);
        if (lane == 0) atomicAdd(&hdr->table_used, 1);
    }
}

// cp_hash_prefix: one CTA per request, chunks of 8192 tokens with a carried running hash
__device__ uint64_t powmod_dev(uint64_t b, int e) {
    uint64_t p = 1;
    while (e) { if (e & 1) p = cp_mulmod(p, b); b = cp_mulmod(b, b); e >>= 1; }
    return p;
}
__global__ void __launch_bounds__(256) k_hash_prefix(const int32_t* tokens, const int64_t* offsets, uint64_t B,
                                                     uint64_t* out) {
    extern __shared__ uint64_t sm[];
    __shared__ uint64_t wtmp[16];
    __shared__ uint64_t s_carry;
    const int r = blockIdx.x;
    const int64_t o = offsets[r];
    const int n = (int)(offsets[r + 1] - o);
    const int32_t* t = tokens + o;
    uint64_t* dst = out + o + r;                       // n + 1 values for request r
    if (threadIdx.x == 0) { dst[0] = 0; s_carry = 0; }
    __syncthreads();
    for (int base = 0; base < n; base += 8192) {
        const int len = min(8192, n - base);
        cp_block_prefix_hash<256>([&](int i) { return t[base + i]; }, len, B, sm, wtmp);
        const uint64_t carry = s_carry;
        for (int i = threadIdx.x + 1; i <= len; i += blockDim.x)
            dst[base + i] = cp_addmod(cp_mulmod(carry, powmod_dev(B, i)), sm[i]);
        __syncthreads();
        if (threadIdx.x == 0) s_carry = dst[base + len];
        __syncthreads();
    }
}

}  // namespace

// ==========================================================================================
// C-ABI
// ==========================================================================================
extern "C" {

int64_t cp_pool_num_pages(const cp_config* c) {
    if (!c || c->window_len < 1) return -1;
    const int64_t cap = c->pool_capacity_tokens;
    return (cap + c->max_span_len + CP_BLOCK - 1) / CP_BLOCK + (cap + c->window_len - 1) / c->window_len + 1;
}

int32_t cp_max_pages_per_entry(const cp_config* c) {
    if (!c) return -1;
    return (c->max_span_len + CP_BLOCK - 1) / CP_BLOCK;
}

cp_status cp_index_workspace(const cp_config* cfg, size_t* sizes) {
    if (!valid_cfg(cfg) || !sizes) return CP_ERR_INVALID_ARG;
    Layout L;
    compute_layout(cfg, &L);
    const size_t elem = cfg->dtype == CP_FP32 ? 4 : 2;
    const size_t pool = (size_t)cfg->num_layers * L.P * CP_BLOCK * cfg->num_kv_heads * cfg->head_dim * elem;
    sizes[CP_WS_POOL_K] = al(pool);
    sizes[CP_WS_POOL_V] = al(pool);
    sizes[CP_WS_META] = L.meta_size;
    sizes[CP_WS_SCRATCH] = L.scr_size;
    return CP_OK;
}

cp_status cp_index_create(const cp_config* cfg, void* const* ws, void* stream, cp_index** out) {
    if (!valid_cfg(cfg) || !ws || !out) return CP_ERR_INVALID_ARG;
    for (int i = 0; i < CP_WS_COUNT; ++i) if (!ws[i] || ((uintptr_t)ws[i] & 255)) return CP_ERR_INVALID_ARG;
    cudaStream_t st = (cudaStream_t)stream;
    Layout L;
    compute_layout(cfg, &L);
    cp_index* x = new cp_index();
    std::memset(x, 0, sizeof(*x));
    x->cfg = *cfg;
    cp_index_workspace(cfg, x->ws);
    x->P = L.P; x->MP = L.MP; x->S = L.S; x->T = L.T; x->logT = L.logT;
    x->B = 2 + host_splitmix64(cfg->hash_seed) % (CP_PMOD - 3);
    x->elem = cfg->dtype == CP_FP32 ? 4 : 2;
    x->pool_k = (char*)ws[CP_WS_POOL_K]; x->pool_v = (char*)ws[CP_WS_POOL_V];
    x->meta = (char*)ws[CP_WS_META]; x->scratch = (char*)ws[CP_WS_SCRATCH];
    x->meta_bytes = L.meta_size;
    char* m = x->meta;
    x->hdr = (DevHeader*)(m + L.meta_off[0]);
    x->slot_id = (int32_t*)(m + L.meta_off[1]); x->slot_len = (int32_t*)(m + L.meta_off[2]);
    x->slot_origin = (int32_t*)(m + L.meta_off[3]); x->slot_state = (uint8_t*)(m + L.meta_off[4]);
    x->slot_prefix = (unsigned long long*)(m + L.meta_off[5]); x->slot_full = (unsigned long long*)(m + L.meta_off[6]);
    x->slot_last = (unsigned long long*)(m + L.meta_off[7]); x->slot_digest = (uint8_t*)(m + L.meta_off[8]);
    x->slot_pages = (int32_t*)(m + L.meta_off[9]); x->fifo = (int32_t*)(m + L.meta_off[10]);
    x->slot_stack = (int32_t*)(m + L.meta_off[11]); x->page_tokens = (int32_t*)(m + L.meta_off[12]);
    x->page_bits = (uint16_t*)(m + L.meta_off[13]); x->htab = (HEntry*)(m + L.meta_off[14]);
    x->pw = (unsigned long long*)(m + L.meta_off[15]);
    x->slot_pin = (int32_t*)(m + L.meta_off[16]); x->page_owner = (int32_t*)(m + L.meta_off[17]);
    x->slot_owner = (int32_t*)(m + L.meta_off[18]); x->session_slot = (int32_t*)(m + L.meta_off[19]);
    char* s = x->scratch;
    x->HS = L.HS; x->CH = L.CH; x->CS_HITS = L.CS_HITS; x->MS = L.MS; x->MAXC = L.MAXC; x->BT = L.BT; x->logBT = L.logBT;
    x->sp_entry = (int32_t*)(s + L.scr_off[0]); x->sp_slot = (int32_t*)(s + L.scr_off[1]);
    x->sp_dst = (int32_t*)(s + L.scr_off[2]); x->sp_len = (int32_t*)(s + L.scr_off[3]);
    x->sp_delta = (int32_t*)(s + L.scr_off[4]); x->req_cnt = (int32_t*)(s + L.scr_off[5]);
    x->chunk_hit = (int32_t*)(s + L.scr_off[6]); x->chunk_t0 = (int32_t*)(s + L.scr_off[7]);
    x->hit_cs = (float2*)(s + L.scr_off[8]);
    x->span_pre = (unsigned long long*)(s + L.scr_off[9]); x->span_full = (unsigned long long*)(s + L.scr_off[10]);
    x->btab = (HEntry*)(s + L.scr_off[11]); x->cand = (Cand*)(s + L.scr_off[12]);
    x->rel_off = (int32_t*)(s + L.scr_off[13]); x->rel_rec = (int32_t*)(s + L.scr_off[14]);
    x->new_slot = (int32_t*)(s + L.scr_off[15]); x->removed = (int32_t*)(s + L.scr_off[16]);
    x->cp_req = (int32_t*)(s + L.scr_off[17]); x->cp_slot = (int32_t*)(s + L.scr_off[18]);
    x->cp_dst = (int32_t*)(s + L.scr_off[19]); x->cp_len = (int32_t*)(s + L.scr_off[20]);
    x->cp_delta = (int32_t*)(s + L.scr_off[21]); x->out_tmp = (int32_t*)(s + L.scr_off[22]);
    x->row_src = (long long*)(s + L.scr_off[23]); x->row_dst = (long long*)(s + L.scr_off[24]);
    x->eq_old = (int32_t*)(s + L.scr_off[25]); x->dtab = (HEntry*)(s + L.scr_off[26]);
    x->span_rep = (int32_t*)(s + L.scr_off[27]); x->precs = (Rec16*)(s + L.scr_off[28]);
    x->rm_pos = (int32_t*)(s + L.scr_off[29]);
    x->match_g = cfg->max_req_tokens > CP_MATCH_SMEM_TOKENS ? s + L.scr_off[30] : nullptr;
    x->fscr = s + L.scr_off[31];
    x->hit_coff = (int32_t*)(s + L.scr_off[32]);
    x->unc_list = (int64_t*)(s + L.scr_off[33]);
    x->lru_scr = s + L.scr_off[34];
    x->rel_cur = (int32_t*)(s + L.scr_off[35]);
    // power table B^k, k = 0..max_span_len (host, exact)
    std::vector<unsigned long long> pw((size_t)cfg->max_span_len + 1);
    pw[0] = 1;
    for (size_t k = 1; k < pw.size(); ++k) pw[k] = host_mulmod(pw[k - 1], x->B);
    x->Bw = pw[(size_t)cfg->window_len];
    if (cudaMemcpyAsync(x->pw, pw.data(), pw.size() * 8, cudaMemcpyHostToDevice, st) != cudaSuccess) { delete x; return CP_ERR_CUDA; }
    k_init<<<592, 256, 0, st>>>(x->hdr, x->slot_id, x->slot_state, x->fifo, x->slot_stack, x->htab, x->P, x->S, x->T,
                                x->slot_pin, x->page_owner, x->slot_owner, x->session_slot, cfg->max_sessions);
    CP_COUNT_LAUNCH();
    if (cudaGetLastError() != cudaSuccess) { delete x; return CP_ERR_CUDA; }
    if (cudaStreamSynchronize(st) != cudaSuccess) { delete x; return CP_ERR_CUDA; }
    // opt-in shared memory for the large kernels
    if (cudaFuncSetAttribute(k_ins_commit, cudaFuncAttributeMaxDynamicSharedMemorySize, 180 * 1024) != cudaSuccess) {
        delete x; return CP_ERR_CUDA;
    }
    cudaFuncSetAttribute(k_ins_scan, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(k_hash_prefix, cudaFuncAttributeMaxDynamicSharedMemorySize, 80 * 1024);
    x->wk = new WorkKey();
    if (cudaStreamCreateWithFlags(&x->side, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&x->ev_fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&x->ev_join, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&x->ev_pfork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&x->ev_pjoin, cudaEventDisableTiming) != cudaSuccess) {
        delete x->wk; delete x; return CP_ERR_CUDA;
    }
    *out = x;
    return CP_OK;
}

cp_status cp_index_create_view(const cp_index* base, int32_t num_layers, int32_t num_kv_heads, int32_t layer_offset,
                               int32_t head_offset, void* pool_k, void* pool_v, cp_index** out) {
    if (!base || base->is_view || !pool_k || !pool_v || !out) return CP_ERR_INVALID_ARG;
    if (((uintptr_t)pool_k & 255) || ((uintptr_t)pool_v & 255)) return CP_ERR_INVALID_ARG;
    cp_config vc = base->cfg;
    vc.num_layers = num_layers; vc.num_kv_heads = num_kv_heads; vc.layer_offset = layer_offset; vc.head_offset = head_offset;
    if (!valid_cfg(&vc)) return CP_ERR_INVALID_ARG;
    cp_index* x = new cp_index(*base);          // the base's META / SCRATCH pointers, layout and counters
    x->cfg = vc;
    x->is_view = 1;
    x->insert_prepared = 0;
    cp_index_workspace(&vc, x->ws);
    x->ws[CP_WS_META] = 0; x->ws[CP_WS_SCRATCH] = 0;   // not owned by the view
    x->pool_k = (char*)pool_k; x->pool_v = (char*)pool_v;
    *out = x;
    return CP_OK;
}

cp_status cp_index_destroy(cp_index* x) {
    if (!x) return CP_ERR_INVALID_ARG;
    if (!x->is_view) {
        delete x->wk;
        if (x->ev_fork) cudaEventDestroy(x->ev_fork);
        if (x->ev_join) cudaEventDestroy(x->ev_join);
        if (x->ev_pfork) cudaEventDestroy(x->ev_pfork);
        if (x->ev_pjoin) cudaEventDestroy(x->ev_pjoin);
        if (x->side) cudaStreamDestroy(x->side);
    }
    delete x;
    return CP_OK;
}

uint64_t cp_index_hash_base(const cp_index* x) { return x ? x->B : 0; }

cp_status cp_index_l2_persist(cp_index* x, void* stream, float hit_ratio) {
    if (!x || !(hit_ratio >= 0.0f && hit_ratio <= 1.0f)) return CP_ERR_INVALID_ARG;
    int dev = 0;
    CP_CUDA_CHECK(cudaGetDevice(&dev));
    cudaDeviceProp prop;
    CP_CUDA_CHECK(cudaGetDeviceProperties(&prop, dev));
    if (prop.persistingL2CacheMaxSize <= 0 || prop.accessPolicyMaxWindowSize <= 0) return CP_ERR_UNSUPPORTED;
    const size_t meta = x->meta_bytes;
    const size_t win = std::min<size_t>(meta, (size_t)prop.accessPolicyMaxWindowSize);
    const size_t carve = std::min<size_t>(win, (size_t)prop.persistingL2CacheMaxSize);
    size_t cur = 0;
    CP_CUDA_CHECK(cudaDeviceGetLimit(&cur, cudaLimitPersistingL2CacheSize));
    if (hit_ratio > 0.0f && cur < carve) CP_CUDA_CHECK(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, carve));
    cudaStreamAttrValue v;
    std::memset(&v, 0, sizeof(v));
    v.accessPolicyWindow.base_ptr = x->meta;
    v.accessPolicyWindow.num_bytes = hit_ratio > 0.0f ? win : 0;
    v.accessPolicyWindow.hitRatio = hit_ratio > 0.0f ? std::min(hit_ratio, (float)carve / (float)std::max<size_t>(win, 1)) : 0.0f;
    v.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    v.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    CP_CUDA_CHECK(cudaStreamSetAttribute((cudaStream_t)stream, cudaStreamAttributeAccessPolicyWindow, &v));
    if (x->side) CP_CUDA_CHECK(cudaStreamSetAttribute(x->side, cudaStreamAttributeAccessPolicyWindow, &v));
    return CP_OK;
}

cp_status cp_index_set_clock(cp_index* x, const uint64_t* d_clock) {
    if (!x || x->is_view) return CP_ERR_INVALID_ARG;
    x->clock = reinterpret_cast<const unsigned long long*>(d_clock);
    return CP_OK;
}

cp_status cp_pin_links(cp_index* x, const int32_t* pages, int64_t n, int32_t delta, void* stream) {
    if (!x || (n > 0 && !pages) || n < 0 || (delta != 1 && delta != -1)) return CP_ERR_INVALID_ARG;
    if (n == 0) return CP_OK;
    cudaStream_t st = (cudaStream_t)stream;
    const int grid = (int)std::min<int64_t>((n + 255) / 256, cp_sm_count() * 4);
    k_pin_check<<<grid, 256, 0, st>>>(x->hdr, pages, n, x->page_owner, x->slot_state, x->slot_pages, x->MP, x->slot_len);
    CP_COUNT_LAUNCH();
    k_pin_apply<<<grid, 256, 0, st>>>(x->hdr, pages, n, x->page_owner, x->slot_pin, delta, 0);
    CP_COUNT_LAUNCH();
    k_pin_apply<<<grid, 256, 0, st>>>(x->hdr, pages, n, x->page_owner, x->slot_pin, delta, 1);   // undo if negative
    CP_COUNT_LAUNCH();
    k_pin_done<<<1, 1, 0, st>>>(x->hdr);
    CP_COUNT_LAUNCH();
    return cudaGetLastError() == cudaSuccess ? CP_OK : CP_ERR_CUDA;
}

cp_status cp_index_match_work(cp_index* x, uint64_t* out_h, int32_t reset, void* stream) {
    if (!x || !out_h) return CP_ERR_INVALID_ARG;
    CP_CUDA_CHECK(cudaStreamSynchronize((cudaStream_t)stream));
    unsigned long long w[4];
    CP_CUDA_CHECK(cudaMemcpy(w, x->hdr->match_work, sizeof(w), cudaMemcpyDeviceToHost));
    for (int i = 0; i < 4; ++i) out_h[i] = w[i];
    if (reset) {
        const unsigned long long z[4] = {0, 0, 0, 0};
        CP_CUDA_CHECK(cudaMemcpy(x->hdr->match_work, z, sizeof(z), cudaMemcpyHostToDevice));
    }
    return CP_OK;
}

cp_status cp_index_commit_stats(cp_index* x, int32_t* out_h, void* stream) {
    if (!x || !out_h) return CP_ERR_INVALID_ARG;
    CP_CUDA_CHECK(cudaStreamSynchronize((cudaStream_t)stream));
    DevHeader h;
    CP_CUDA_CHECK(cudaMemcpy(&h, x->hdr, sizeof(h), cudaMemcpyDeviceToHost));
    out_h[0] = h.commits_parallel; out_h[1] = h.commits_serial; out_h[2] = h.commit_why;
    return CP_OK;
}

uint64_t cp_kernel_launch_count(void) { return g_cp_launches.load(); }

#ifndef CP_SRC_SHA256
#define CP_SRC_SHA256 "unknown-unknown-unknown-unknown-unknown-unknown-unknown-unknown!"
#endif
const char* cp_build_info(void) { return "cp-src-sha256=" CP_SRC_SHA256 " arch=sm_100a"; }

const char* cp_status_string(cp_status s) {
    switch (s) {
        case CP_OK: return "CP_OK";
        case CP_ERR_INVALID_ARG: return "CP_ERR_INVALID_ARG";
        case CP_ERR_SENSITIVE_SPAN: return "CP_ERR_SENSITIVE_SPAN";
        case CP_ERR_SPAN_TOO_SHORT: return "CP_ERR_SPAN_TOO_SHORT";
        case CP_ERR_CAPACITY: return "CP_ERR_CAPACITY";
        case CP_ERR_CUDA: return "CP_ERR_CUDA";
        case CP_ERR_UNSUPPORTED: return "CP_ERR_UNSUPPORTED";
    }
    return "CP_ERR_UNKNOWN";
}

cp_status cp_index_last_error(cp_index* x, void* stream) {
    if (!x) return CP_ERR_INVALID_ARG;
    cudaStream_t st = (cudaStream_t)stream;
    int32_t e = 0;
    CP_CUDA_CHECK(cudaStreamSynchronize(st));
    CP_CUDA_CHECK(cudaMemcpy(&e, &x->hdr->error, 4, cudaMemcpyDeviceToHost));
    const int32_t z = 0;
    CP_CUDA_CHECK(cudaMemcpy(&x->hdr->error, &z, 4, cudaMemcpyHostToDevice));
    return (cp_status)e;
}

cp_status cp_index_snapshot(cp_index* x, cp_snapshot* o, void* stream) {
    if (!x || !o) return CP_ERR_INVALID_ARG;
    cudaStream_t st = (cudaStream_t)stream;
    CP_CUDA_CHECK(cudaStreamSynchronize(st));
    DevHeader h;
    CP_CUDA_CHECK(cudaMemcpy(&h, x->hdr, sizeof(h), cudaMemcpyDeviceToHost));
    const int S = x->S;
    std::vector<int32_t> sid(S), slen(S), sorg(S), spages((size_t)S * x->MP);
    std::vector<uint8_t> sstate(S), sdig((size_t)S * 32);
    std::vector<unsigned long long> spre(S), sfull(S), slast(S);
    CP_CUDA_CHECK(cudaMemcpy(sid.data(), x->slot_id, 4 * S, cudaMemcpyDeviceToHost));
    CP_CUDA_CHECK(cudaMemcpy(slen.data(), x->slot_len, 4 * S, cudaMemcpyDeviceToHost));
    CP_CUDA_CHECK(cudaMemcpy(sorg.data(), x->slot_origin, 4 * S, cudaMemcpyDeviceToHost));
    CP_CUDA_CHECK(cudaMemcpy(sstate.data(), x->slot_state, S, cudaMemcpyDeviceToHost));
    CP_CUDA_CHECK(cudaMemcpy(spre.data(), x->slot_prefix, 8 * S, cudaMemcpyDeviceToHost));
    CP_CUDA_CHECK(cudaMemcpy(sfull.data(), x->slot_full, 8 * S, cudaMemcpyDeviceToHost));
    CP_CUDA_CHECK(cudaMemcpy(slast.data(), x->slot_last, 8 * S, cudaMemcpyDeviceToHost));
    CP_CUDA_CHECK(cudaMemcpy(sdig.data(), x->slot_digest, 32 * (size_t)S, cudaMemcpyDeviceToHost));
    CP_CUDA_CHECK(cudaMemcpy(spages.data(), x->slot_pages, 4 * (size_t)S * x->MP, cudaMemcpyDeviceToHost));
    std::vector<int32_t> ptok;
    std::vector<uint16_t> pbits;
    if (o->tokens || o->recompute) {
        ptok.resize((size_t)x->P * CP_BLOCK);
        pbits.resize((size_t)x->P);
        CP_CUDA_CHECK(cudaMemcpy(ptok.data(), x->page_tokens, 4 * ptok.size(), cudaMemcpyDeviceToHost));
        CP_CUDA_CHECK(cudaMemcpy(pbits.data(), x->page_bits, 2 * pbits.size(), cudaMemcpyDeviceToHost));
    }
    std::vector<int> order;
    for (int s = 0; s < S; ++s) if (sstate[s] == CP_SLOT_LIVE) order.push_back(s);
    std::sort(order.begin(), order.end(), [&](int a, int b) { return sid[a] < sid[b]; });
    o->num_live = (int32_t)order.size(); o->next_id = h.next_id; o->live_tokens = h.live_tokens;
    o->fifo_count = h.fifo_count; o->error = h.error;
    const int ML = x->cfg.max_span_len;
    for (size_t q = 0; q < order.size(); ++q) {
        const int s = order[q];
        if (o->id) o->id[q] = sid[s];
        if (o->len) o->len[q] = slen[s];
        if (o->origin_pos) o->origin_pos[q] = sorg[s];
        if (o->prefix_hash) o->prefix_hash[q] = spre[s];
        if (o->full_hash) o->full_hash[q] = sfull[s];
        if (o->last_used) o->last_used[q] = slast[s];
        if (o->digest) std::memcpy(o->digest + 32 * q, &sdig[(size_t)s * 32], 32);
        if (o->pages) std::memcpy(o->pages + (size_t)q * x->MP, &spages[(size_t)s * x->MP], 4 * (size_t)x->MP);
        for (int t = 0; t < slen[s] && (o->tokens || o->recompute); ++t) {
            const int page = spages[(size_t)s * x->MP + t / CP_BLOCK];
            if (o->tokens) o->tokens[(size_t)q * ML + t] = ptok[(size_t)page * CP_BLOCK + t % CP_BLOCK];
            if (o->recompute) o->recompute[(size_t)q * ML + t] = (pbits[page] >> (t % CP_BLOCK)) & 1;
        }
    }
    if (o->owner) {
        std::vector<int32_t> own((size_t)S);
        CP_CUDA_CHECK(cudaMemcpy(own.data(), x->slot_owner, 4 * (size_t)S, cudaMemcpyDeviceToHost));
        for (size_t q = 0; q < order.size(); ++q) o->owner[q] = own[(size_t)order[q]];
    }
    if (o->pin) {
        std::vector<int32_t> pins((size_t)S);
        CP_CUDA_CHECK(cudaMemcpy(pins.data(), x->slot_pin, 4 * (size_t)S, cudaMemcpyDeviceToHost));
        for (size_t q = 0; q < order.size(); ++q) o->pin[q] = pins[(size_t)order[q]];
    }
    if (o->fifo) {
        std::vector<int32_t> f((size_t)x->P);
        CP_CUDA_CHECK(cudaMemcpy(f.data(), x->fifo, 4 * f.size(), cudaMemcpyDeviceToHost));
        for (int i = 0; i < h.fifo_count; ++i) o->fifo[i] = f[(size_t)((h.fifo_head + i) % x->P)];
    }
    return CP_OK;
}

cp_status cp_hash_prefix(const cp_batch* b, uint64_t hash_seed, uint64_t* out, void* stream) {
    if (!b || !out || b->num_reqs < 0) return CP_ERR_INVALID_ARG;
    if (b->num_reqs == 0) return CP_OK;
    if (!b->tokens || !b->offsets) return CP_ERR_INVALID_ARG;
    static bool attr = false;
    if (!attr) { cudaFuncSetAttribute(k_hash_prefix, cudaFuncAttributeMaxDynamicSharedMemorySize, 80 * 1024); attr = true; }
    const uint64_t B = 2 + host_splitmix64(hash_seed) % (CP_PMOD - 3);
    k_hash_prefix<<<b->num_reqs, 256, 8 * 8193, (cudaStream_t)stream>>>(b->tokens, b->offsets, B, out);
    CP_COUNT_LAUNCH();
    return cudaGetLastError() == cudaSuccess ? CP_OK : CP_ERR_CUDA;
}

}  // extern "C"

namespace {

// host-side checks + the kernel argument block shared by the insert phases (no device work)
cp_status ins_args(cp_index* x, const cp_batch* wb, const cp_paged_kv* kv, int32_t num_spans,
                   const int32_t* span_req, const int32_t* span_begin, const int32_t* span_len,
                   const uint32_t* bits, const int64_t* bits_off, uint64_t t, int32_t* out_id, int32_t* out_oc,
                   InsArgs& a) {
    if (!x || !wb || !kv || x->is_view) return CP_ERR_INVALID_ARG;       // a view's metadata is its base's
    if (num_spans < 0 || num_spans > x->MS) return CP_ERR_INVALID_ARG;
    if (num_spans == 0) return CP_OK;
    if (!span_req || !span_begin || !span_len || !out_id || !out_oc) return CP_ERR_INVALID_ARG;
    if (!wb->tokens || !wb->offsets || !wb->mask) return CP_ERR_INVALID_ARG;          // writer mask required
    if (wb->num_reqs < 1 || wb->num_reqs > x->cfg.max_batch_reqs || wb->total_tokens > x->cfg.max_batch_tokens) return CP_ERR_INVALID_ARG;
    if ((bits == nullptr) != (bits_off == nullptr)) return CP_ERR_INVALID_ARG;
    if (!kv->k_layers_h || !kv->v_layers_h || !kv->block_tables) return CP_ERR_INVALID_ARG;
    std::memset(&a, 0, sizeof(a));
    a.hdr = x->hdr; a.tokens = wb->tokens; a.offsets = wb->offsets; a.mask = wb->mask; a.num_reqs = wb->num_reqs;
    a.S = num_spans; a.span_req = span_req; a.span_begin = span_begin; a.span_len = span_len;
    a.bits = bits; a.bits_off = bits_off; a.t = t; a.w = x->cfg.window_len; a.B = x->B;
    a.capacity = x->cfg.pool_capacity_tokens; a.max_span_len = x->cfg.max_span_len;
    a.out_id = out_id; a.out_oc = out_oc;
    a.nslots = x->S; a.P = x->P; a.MP = x->MP;
    a.slot_id = x->slot_id; a.slot_len = x->slot_len; a.slot_origin = x->slot_origin; a.slot_state = x->slot_state;
    a.slot_prefix = x->slot_prefix; a.slot_full = x->slot_full; a.slot_last = x->slot_last;
    a.slot_digest = x->slot_digest; a.slot_pages = x->slot_pages; a.fifo = x->fifo; a.slot_stack = x->slot_stack;
    a.page_tokens = x->page_tokens; a.page_bits = x->page_bits; a.htab = x->htab; a.logT = x->logT; a.T = x->T;
    a.pw = x->pw; a.slot_pin = x->slot_pin; a.page_owner = x->page_owner; a.slot_owner = x->slot_owner;
    a.span_pre = x->span_pre; a.span_full = x->span_full; a.btab = x->btab; a.logBT = x->logBT; a.BT = x->BT;
    a.cand = x->cand; a.MAXC = x->MAXC; a.rel_off = x->rel_off; a.rel_rec = (int2*)x->rel_rec;
    a.new_slot = x->new_slot; a.removed = x->removed; a.rm_pos = x->rm_pos;
    a.cp_req = x->cp_req; a.cp_slot = x->cp_slot; a.cp_dst = x->cp_dst; a.cp_len = x->cp_len; a.cp_delta = x->cp_delta;
    {
        const size_t M1 = (size_t)x->MS + 1;
        int32_t* q = (int32_t*)x->fscr;
        int32_t** per_span[12] = {&a.f_last, &a.f_kind, &a.f_target, &a.f_supcnt, &a.f_suptok, &a.f_suppg, &a.f_sidx,
                                  &a.f_sj, &a.f_pgpref, &a.f_rmpref, &a.f_suppgpref, &a.f_vk};
        for (int k = 0; k < 12; ++k) { *per_span[k] = q; q += M1; }
        a.f_netpref = (long long*)(((uintptr_t)q + 7) & ~(uintptr_t)7);
        q = (int32_t*)(a.f_netpref + M1);
        int32_t** per_slot[4] = {&a.f_refs, &a.f_evpos, &a.f_maxpos, &a.f_supby};
        for (int k = 0; k < 4; ++k) { *per_slot[k] = q; q += x->S; }
        int32_t** per_cand[4] = {&a.f_vslot, &a.f_vlen, &a.f_vcpg, &a.f_vfc};
        for (int k = 0; k < 4; ++k) { *per_cand[k] = q; q += 4097; }
        a.f_vcum = (long long*)(((uintptr_t)q + 7) & ~(uintptr_t)7);
    }
    {
        static int fs = -1;
        if (fs < 0) { const char* e = getenv("CP_COMMIT_SERIAL"); fs = (e && atoi(e) != 0) ? 1 : 0; }
        a.force_serial = fs;
    }
    a.CH = x->CH; a.max_blocks = kv->max_blocks_per_req; a.clock = x->clock;
    if (a.max_blocks < 1) return CP_ERR_INVALID_ARG;
    a.out_tmp = x->out_tmp; a.eq_old = x->eq_old; a.dtab = x->dtab; a.span_rep = x->span_rep; a.precs = x->precs;
    {
        char* q = x->lru_scr;
        a.lru = (LruHdr*)q; q += 64;
        a.lru_key = (unsigned long long*)q; q += 8 * (size_t)x->S;
        a.lru_hist = (unsigned*)q; q += 4 * 3 * (size_t)kLruBins;
        a.lru_list = (unsigned long long*)q; q += 8 * (size_t)kLruK;
        a.lru_rank = (unsigned*)q; q += 4 * (size_t)kLruK;
        a.lru_sorted = (unsigned long long*)q;
    }
    a.rel_cur = x->rel_cur;
    // shared memory of the commit: flags + per-span arrays, then the LRU candidate list (4096 halved to
    // fit), then as many relation records as the rest of the 180 KB holds (up to kCommitRecCap; beyond: global)
    int candK = 4096;
    while (candK >= 256 && CommitSmem(x->S, num_spans, candK, 0).fixed > 180 * 1024) candK >>= 1;
    if (candK < 256) candK = 0;
    a.candK = candK;
    const size_t fixed = CommitSmem(x->S, num_spans, candK, 0).fixed;
    a.rec_cap = fixed >= 180 * 1024 ? 0 : (int)std::min<size_t>(kCommitRecCap, (180 * 1024 - fixed) / 8);
    if (CommitSmem(x->S, num_spans, candK, a.rec_cap).total > 180 * 1024) return CP_ERR_UNSUPPORTED;   // + ~35 KB static
    return CP_OK;
}

// read-only phases: validation, hashing, batch dedup, containment scan + verification (scratch only)
cp_status ins_prepare(cp_index* x, const InsArgs& a, cudaStream_t st) {
    const int num_spans = a.S;
    cp_invalidate_worklist(x);
    const int sms = cp_sm_count();
    // The prepare runs beside the step's match; it must end before the gather starts, whose persistent
    // grid holds every SM's registers until it ends (kernels queued behind it land on the critical path).
    // First the work that needs only the index as the previous commit left it: the commit's LRU
    // candidate list (it exits at once when this call cannot evict).  The LRU chain runs on the index's side stream, a branch beside the containment scans (it reads
    // only index state no prepare kernel writes), joined before the prepare returns
    if (cudaEventRecord(x->ev_pfork, st) != cudaSuccess || cudaStreamWaitEvent(x->side, x->ev_pfork, 0) != cudaSuccess)
        return CP_ERR_CUDA;
    k_lru_init<<<1, 1024, 0, x->side>>>(a); CP_COUNT_LAUNCH();
    k_lru_snap<<<sms, 256, 0, x->side>>>(a); CP_COUNT_LAUNCH();
    for (int p = 0; p < 3; ++p) { k_lru_hist<<<sms, 256, 0, x->side>>>(a, p); CP_COUNT_LAUNCH(); }
    k_lru_collect<<<sms, 256, 0, x->side>>>(a); CP_COUNT_LAUNCH();
    k_lru_rank<<<dim3(kLruK / 256, 4), 256, 0, x->side>>>(a); CP_COUNT_LAUNCH();
    k_lru_scatter<<<kLruK / 256, 256, 0, x->side>>>(a); CP_COUNT_LAUNCH();
    if (cudaEventRecord(x->ev_pjoin, x->side) != cudaSuccess) return CP_ERR_CUDA;
    const int wblocks = std::max(1, std::min(1184, (num_spans + 7) / 8));
    k_ins_validate<<<std::max<int64_t>(wblocks, std::min<int64_t>(1184, (x->BT + 255) / 256)), kValThreads, 0, st>>>(a); CP_COUNT_LAUNCH();
    k_ins_hash<<<wblocks, 256, 0, st>>>(a); CP_COUNT_LAUNCH();
    k_ins_rep<<<wblocks, 256, 0, st>>>(a); CP_COUNT_LAUNCH();
    k_ins_bucket_offsets<<<1, 1024, 0, st>>>(a); CP_COUNT_LAUNCH();
    k_ins_bucket_fill<<<(num_spans + 255) / 256, 256, 0, st>>>(a); CP_COUNT_LAUNCH();
    const size_t scan_smem = 8 * ((size_t)x->cfg.max_span_len + 1);
    k_ins_scan<<<(int)std::min<int64_t>(num_spans, sms * 6), kScanThreads, scan_smem, st>>>(a, 0); CP_COUNT_LAUNCH();
    k_ins_verify<<<sms * 4, 256, 0, st>>>(a, 0); CP_COUNT_LAUNCH();
    k_ins_flag_eq<<<sms, 256, 0, st>>>(a); CP_COUNT_LAUNCH();
    k_ins_count_need<<<64, 256, 0, st>>>(a); CP_COUNT_LAUNCH();
    k_ins_scan<<<(int)std::min<int64_t>(x->S, sms * 6), kScanThreads, scan_smem, st>>>(a, 1); CP_COUNT_LAUNCH();
    k_ins_verify<<<sms * 4, 256, 0, st>>>(a, 1); CP_COUNT_LAUNCH();
    // the commit's relation CSR over the verified candidates
    k_ins_rel_fill<<<1, 1024, 0, st>>>(a); CP_COUNT_LAUNCH();
    if (cudaStreamWaitEvent(st, x->ev_pjoin, 0) != cudaSuccess) return CP_ERR_CUDA;   // the LRU branch
    return cudaGetLastError() == cudaSuccess ? CP_OK : CP_ERR_CUDA;
}

// mutating phases: sequential apply, table updates, copy-in of the writer KV
cp_status ins_commit(cp_index* x, const InsArgs& a, const cp_batch* wb, const cp_paged_kv* kv, cudaStream_t st,
                     int32_t nviews = 0, cp_index* const* views = nullptr, const cp_paged_kv* view_kvs = nullptr) {
    const int num_spans = a.S;
    cp_invalidate_worklist(x);
    const size_t csm = CommitSmem(x->S, num_spans, a.candK, a.rec_cap).total;
    k_ins_commit<<<1, kCommitThreads, csm, st>>>(a); CP_COUNT_LAUNCH();   // writes out_id too
    k_ins_delete<<<128, 256, 0, st>>>(a); CP_COUNT_LAUNCH();
    k_ins_publish<<<std::max(1, std::min(1184, (num_spans + 7) / 8)), 256, 0, st>>>(a); CP_COUNT_LAUNCH();
    // digests beside the rest of the commit (rebuild, copy-in): fork onto the side stream, join at the end
    if (cudaEventRecord(x->ev_fork, st) != cudaSuccess || cudaStreamWaitEvent(x->side, x->ev_fork, 0) != cudaSuccess)
        return CP_ERR_CUDA;
    k_ins_digest<<<std::max(1, std::min(148, (num_spans + 127) / 128)), 128, 0, x->side>>>(a); CP_COUNT_LAUNCH();
    if (cudaEventRecord(x->ev_join, x->side) != cudaSuccess) return CP_ERR_CUDA;
    k_rebuild_check<<<1, 1, 0, st>>>(x->hdr, x->T); CP_COUNT_LAUNCH();
    k_rebuild_clear<<<256, 256, 0, st>>>(x->hdr, x->htab, x->T); CP_COUNT_LAUNCH();
    k_rebuild_fill<<<256, 256, 0, st>>>(x->hdr, x->htab, x->logT, x->T, x->slot_state, x->slot_prefix, x->slot_full, x->slot_len, x->S,
                                        x->slot_owner); CP_COUNT_LAUNCH();
    if (cudaGetLastError() != cudaSuccess) return CP_ERR_CUDA;
    // copy the writer KV rows of the published entries into their pool pages
    const cp_status cs = cp_launch_rows(x, 1, &x->hdr->n_copy, x->cp_req, x->cp_slot, x->cp_dst, x->cp_len, nullptr,
                                        x->MS, wb->offsets, nullptr, kv, 0, st, nviews, views, view_kvs);
    if (cudaStreamWaitEvent(st, x->ev_join, 0) != cudaSuccess) return CP_ERR_CUDA;   // digests done
    return cs;
}

}  // namespace

extern "C" {

cp_status cp_index_insert(cp_index* x, const cp_batch* wb, const cp_paged_kv* kv, int32_t num_spans,
                          const int32_t* span_req, const int32_t* span_begin, const int32_t* span_len,
                          const uint32_t* bits, const int64_t* bits_off, uint64_t t,
                          int32_t* out_id, int32_t* out_oc, void* stream) {
    InsArgs a;
    const cp_status s = ins_args(x, wb, kv, num_spans, span_req, span_begin, span_len, bits, bits_off, t, out_id, out_oc, a);
    if (s != CP_OK || num_spans == 0) return s;
    if (x->insert_prepared) return CP_ERR_INVALID_ARG;          // a split insert is in flight
    const cudaStream_t st = (cudaStream_t)stream;
    const cp_status p = ins_prepare(x, a, st);
    return p != CP_OK ? p : ins_commit(x, a, wb, kv, st);
}

cp_status cp_index_insert_prepare(cp_index* x, const cp_batch* wb, const cp_paged_kv* kv, int32_t num_spans,
                                  const int32_t* span_req, const int32_t* span_begin, const int32_t* span_len,
                                  const uint32_t* bits, const int64_t* bits_off, uint64_t t,
                                  int32_t* out_id, int32_t* out_oc, void* stream) {
    InsArgs a;
    const cp_status s = ins_args(x, wb, kv, num_spans, span_req, span_begin, span_len, bits, bits_off, t, out_id, out_oc, a);
    if (s != CP_OK || num_spans == 0) return s;
    if (x->insert_prepared) return CP_ERR_INVALID_ARG;
    const cp_status p = ins_prepare(x, a, (cudaStream_t)stream);
    if (p == CP_OK) x->insert_prepared = 1;
    return p;
}

cp_status cp_index_insert_commit(cp_index* x, const cp_batch* wb, const cp_paged_kv* kv, int32_t num_spans,
                                 const int32_t* span_req, const int32_t* span_begin, const int32_t* span_len,
                                 const uint32_t* bits, const int64_t* bits_off, uint64_t t,
                                 int32_t* out_id, int32_t* out_oc, void* stream) {
    InsArgs a;
    const cp_status s = ins_args(x, wb, kv, num_spans, span_req, span_begin, span_len, bits, bits_off, t, out_id, out_oc, a);
    if (s != CP_OK || num_spans == 0) return s;
    if (!x->insert_prepared) return CP_ERR_INVALID_ARG;          // commit without prepare
    x->insert_prepared = 0;
    return ins_commit(x, a, wb, kv, (cudaStream_t)stream);
}


cp_status cp_index_insert_commit_rects(cp_index* x, int32_t num_views, cp_index* const* views, const cp_batch* wb,
                                       const cp_paged_kv* kvs, int32_t num_spans, const int32_t* span_req,
                                       const int32_t* span_begin, const int32_t* span_len, const uint32_t* bits,
                                       const int64_t* bits_off, uint64_t t, int32_t* out_id, int32_t* out_oc,
                                       void* stream) {
    if (!kvs || num_views < 0 || num_views > 3 || (num_views > 0 && !views)) return CP_ERR_INVALID_ARG;
    int layers = x ? x->cfg.num_layers : 0;
    for (int i = 0; i < num_views; ++i) {      // checked before any state changes (cp_launch_rows re-checks)
        const cp_index* v = views[i];
        if (v) layers += v->cfg.num_layers;
        if (layers > CP_MAX_LAYERS) return CP_ERR_INVALID_ARG;
        const cp_paged_kv* vk = &kvs[1 + i];
        if (!v || !v->is_view || !x || v->hdr != x->hdr || vk->block_tables != kvs[0].block_tables ||
            vk->max_blocks_per_req != kvs[0].max_blocks_per_req || !vk->k_layers_h || !vk->v_layers_h)
            return CP_ERR_INVALID_ARG;
    }
    InsArgs a;
    const cp_status s = ins_args(x, wb, &kvs[0], num_spans, span_req, span_begin, span_len, bits, bits_off, t, out_id,
                                 out_oc, a);
    if (s != CP_OK || num_spans == 0) return s;
    if (!x->insert_prepared) return CP_ERR_INVALID_ARG;          // commit without prepare
    x->insert_prepared = 0;
    return ins_commit(x, a, wb, &kvs[0], (cudaStream_t)stream, num_views, views, kvs + 1);
}

cp_status cp_index_insert_session(cp_index* x, const cp_batch* wb, const cp_paged_kv* kv, uint64_t t,
                                  int32_t* out_id, int32_t* out_oc, void* stream) {
    if (!x || x->is_view || !wb || !kv || !out_id || !out_oc || x->cfg.max_sessions < 1) return CP_ERR_INVALID_ARG;
    if (wb->num_reqs == 0) return CP_OK;
    if (wb->num_reqs < 0 || wb->num_reqs > x->cfg.max_batch_reqs || wb->num_reqs > x->MS ||
        wb->total_tokens > x->cfg.max_batch_tokens || !wb->tokens || !wb->offsets || !wb->session)
        return CP_ERR_INVALID_ARG;
    if (!kv->k_layers_h || !kv->v_layers_h || !kv->block_tables || kv->max_blocks_per_req < 1) return CP_ERR_INVALID_ARG;
    if (x->insert_prepared) return CP_ERR_INVALID_ARG;
    InsArgs a;
    std::memset(&a, 0, sizeof(a));
    a.hdr = x->hdr; a.tokens = wb->tokens; a.offsets = wb->offsets; a.num_reqs = wb->num_reqs; a.S = wb->num_reqs;
    a.t = t; a.w = x->cfg.window_len; a.B = x->B; a.capacity = x->cfg.pool_capacity_tokens;
    a.max_span_len = x->cfg.max_span_len; a.out_id = out_id; a.out_oc = out_oc;
    a.nslots = x->S; a.P = x->P; a.MP = x->MP;
    a.slot_id = x->slot_id; a.slot_len = x->slot_len; a.slot_origin = x->slot_origin; a.slot_state = x->slot_state;
    a.slot_prefix = x->slot_prefix; a.slot_full = x->slot_full; a.slot_last = x->slot_last;
    a.slot_digest = x->slot_digest; a.slot_pages = x->slot_pages; a.fifo = x->fifo; a.slot_stack = x->slot_stack;
    a.page_tokens = x->page_tokens; a.page_bits = x->page_bits; a.htab = x->htab; a.logT = x->logT; a.T = x->T;
    a.pw = x->pw; a.slot_pin = x->slot_pin; a.page_owner = x->page_owner; a.slot_owner = x->slot_owner;
    a.session = wb->session; a.session_slot = x->session_slot; a.max_sessions = x->cfg.max_sessions;
    a.removed = x->removed; a.rm_pos = x->rm_pos; a.out_tmp = x->out_tmp;
    a.cp_req = x->cp_req; a.cp_slot = x->cp_slot; a.cp_dst = x->cp_dst; a.cp_len = x->cp_len; a.cp_delta = x->cp_delta;
    a.max_blocks = kv->max_blocks_per_req; a.clock = x->clock;
    cudaStream_t st = (cudaStream_t)stream;
    cp_invalidate_worklist(x);
    k_sess_validate<<<std::max(1, std::min(148, (wb->num_reqs + 255) / 256)), 256, 0, st>>>(a); CP_COUNT_LAUNCH();
    k_sess_commit<<<1, 256, 0, st>>>(a); CP_COUNT_LAUNCH();
    k_ins_outids<<<(wb->num_reqs + 255) / 256, 256, 0, st>>>(a); CP_COUNT_LAUNCH();
    k_ins_delete<<<128, 256, 0, st>>>(a); CP_COUNT_LAUNCH();
    k_sess_publish<<<std::max(1, std::min(1184, (wb->num_reqs + 7) / 8)), 256, 0, st>>>(a); CP_COUNT_LAUNCH();
    k_rebuild_check<<<1, 1, 0, st>>>(x->hdr, x->T); CP_COUNT_LAUNCH();
    k_rebuild_clear<<<256, 256, 0, st>>>(x->hdr, x->htab, x->T); CP_COUNT_LAUNCH();
    k_rebuild_fill<<<256, 256, 0, st>>>(x->hdr, x->htab, x->logT, x->T, x->slot_state, x->slot_prefix, x->slot_full, x->slot_len, x->S,
                                        x->slot_owner); CP_COUNT_LAUNCH();
    if (cudaGetLastError() != cudaSuccess) return CP_ERR_CUDA;
    return cp_launch_rows(x, 1, &x->hdr->n_copy, x->cp_req, x->cp_slot, x->cp_dst, x->cp_len, nullptr,
                          x->MS, wb->offsets, nullptr, kv, 0, st);
}

cp_status cp_index_copy_in(cp_index* v, const cp_batch* wb, const cp_paged_kv* kv, int32_t flags, void* stream) {
    if (!v || !v->is_view || !wb || !kv || !wb->offsets) return CP_ERR_INVALID_ARG;
    if (!kv->k_layers_h || !kv->v_layers_h || !kv->block_tables || kv->max_blocks_per_req < 1) return CP_ERR_INVALID_ARG;
    if (wb->num_reqs < 1 || wb->num_reqs > v->cfg.max_batch_reqs) return CP_ERR_INVALID_ARG;
    // the base's last commit left its copy-in list (entries published by that call) in the shared
    // scratch; the copy kernels re-resolve it against this view's geometry and pool
    return cp_launch_rows(v, 1, &v->hdr->n_copy, v->cp_req, v->cp_slot, v->cp_dst, v->cp_len, nullptr,
                          v->MS, wb->offsets, nullptr, kv, flags & CP_REUSE_WORKLIST, (cudaStream_t)stream);
}

}  // extern "C"

#ifdef CP_COMMIT_PROF
extern "C" cp_status cp_commit_prof_read(unsigned long long* out_h) {
    if (cudaMemcpyFromSymbol(out_h, g_commit_prof, sizeof(unsigned long long) * 16) != cudaSuccess) return CP_ERR_CUDA;
    return CP_OK;
}
#endif
