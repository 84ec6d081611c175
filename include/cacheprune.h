/*
 * cacheprune.h -- C-ABI of the B200-native CachePrune hot path (arxiv 2605.23640).
 *
 * The library implements token-granular, privacy-masked KV reuse:
 *   cp_index_insert     -- store reusable segments in the shared KV pool
 *                          (§4.3.5 KV Pool: storage format, dedup, LRU;
 *                           L403-405 §3.3 selective sharing: a masked token is never stored)
 *   cp_match_spans      -- find stored segments inside incoming prompts
 *                          (§4.2.2 C2: rolling-hash prefix filter + verification;
 *                           L724-727 §4.3.1: plan with zero placeholders)
 *   cp_gather_rerotate  -- copy the matched K/V rows into the request's paged KV cache and re-rotate
 *                          moved keys by the RoPE position delta (placement: PAPER.md L518, L726,
 *                          L781; RoPE: the paper is silent -- DESIGN.md readings R#11-14)
 *   cp_score_deviation  -- per-token inter-minus-intra attention score and top-rho selection of the
 *                          tokens to recompute (§4.2.1 C1 Step 3; rho = 25%, L1032)
 *
 * Conventions (all calls):
 *   - Pointers are DEVICE pointers unless the name ends in _h (host).  The caller owns every buffer,
 *     including the workspaces handed to cp_index_create; the library never allocates device memory.
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).  Calls are
 *     asynchronous on that stream; outputs are valid once the stream reaches them.  All calls on one
 *     index must be ordered by the caller (single writer, multiple readers: SPEC.md L351, L423).
 *   - Errors: argument errors detectable on the host return a negative cp_status synchronously with
 *     no side effects.  Errors detectable only on the device (a sensitive token inside an insert
 *     span, a request longer than the configured maximum, a full candidate buffer) are written to a
 *     sticky device error word; while it is set every later kernel of every call on that index is a
 *     no-op, and the insert that raised it changed nothing.  cp_index_last_error() synchronizes,
 *     returns and clears it.
 *   - Positions are 0-based.  Token ids are int32 >= 0.  Masks are uint8 (1 = sensitive).
 *   - Hashing: p = 2^61-1, base B = 2 + splitmix64(hash_seed) mod (p-3) ("random base";
 *     DESIGN.md R#1), tokenval = id + 1 (R#2).  Use the same hash_seed on every rank.
 */
#ifndef CACHEPRUNE_H
#define CACHEPRUNE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    CP_OK = 0,
    CP_ERR_INVALID_ARG = -1,     /* bad argument (host) or bad span range (device)             */
    CP_ERR_SENSITIVE_SPAN = -2,  /* an insert span covers a mask-1 token         */
    CP_ERR_SPAN_TOO_SHORT = -3,  /* an insert span is shorter than window_len    */
    CP_ERR_CAPACITY = -4,        /* span longer than the budget / max_span_len, buffers full  */
    CP_ERR_CUDA = -5,            /* a CUDA runtime call failed                                  */
    CP_ERR_UNSUPPORTED = -6      /* configuration or mode not built                           */
} cp_status;

enum { CP_FP32 = 0, CP_BF16 = 1 };                 /* KV storage dtype                          */
enum { CP_ROPE_NEOX = 0, CP_ROPE_GPTJ = 1 };       /* pairs (i, i+d/2) | (2i, 2i+1)  (R#12)      */
enum { CP_MATCH_NO_TOUCH = 1,                     /* cp_match_spans flags                       */
       CP_MATCH_FIXED_CHUNK = 2,                  /* NEXT-3 baseline policies (R#28-29)          */
       CP_MATCH_PREFIX_ONLY = 4 };
enum { CP_POLICY_FIXED_CHUNK = 1, CP_POLICY_PREFIX_ONLY = 2 };   /* cp_policy_spans              */
enum { CP_ZERO_RECOMPUTE = 1, CP_ZERO_UNCOVERED = 2,  /* cp_gather_rerotate flags (R#14)            */
       CP_SKIP_LINKED = 4,                         /* NEXT-2: leave linkable blocks unwritten (R#31) */
       CP_REUSE_WORKLIST = 8,                      /* pool views: reuse the sibling's work list      */
       CP_SKIP_RECOMPUTE = 16 };                   /* leave plan-2 rows unwritten (R#14 alternative) */
enum { CP_SCORE_INTER_INTRA = 0, CP_SCORE_KVDEV = 1 };
enum { CP_STORED = 0, CP_SUPERSEDED = 1, CP_DUPLICATE = 2, CP_DROPPED_CONTAINED = 3, /* insert outcomes */
       CP_DEFERRED_PINNED = 4 };   /* not stored: it would supersede a pinned entry, or the pinned tokens plus it
                                      exceed the budget (R#32); out id = the smallest pinned entry it contains, or -1 */
enum { CP_PLAN_UNCOVERED = 0, CP_PLAN_REUSED = 1, CP_PLAN_RECOMPUTE = 2 };              /* plan codes     */

typedef struct cp_index cp_index;                  /* opaque host handle */

/* Index configuration.  num_layers / num_kv_heads are THIS shard's geometry. */
typedef struct {
    int32_t  window_len;            /* prefix-filter window = minimum segment length, 128 */
    int32_t  block_size;            /* tokens per page, pool and caller caches; must be 16 (R#23)       */
    uint64_t hash_seed;             /* seeds the random hash base B                             */
    int32_t  num_layers, num_kv_heads, head_dim;
    int32_t  layer_offset, head_offset;   /* position of this shard (diagnostics only)                */
    int32_t  dtype;                 /* CP_FP32 | CP_BF16                                                 */
    int32_t  rope_style;            /* CP_ROPE_NEOX | CP_ROPE_GPTJ                                       */
    double   rope_theta;            /* 500000 (Llama-3), 10000 (toy)                                     */
    int64_t  pool_capacity_tokens;  /* LRU budget in tokens (R#21)                              */
    int32_t  max_entries;           /* live-entry slots (>= capacity/window_len + max_spans_per_insert + 1) */
    int32_t  max_span_len;          /* longest storable segment                                          */
    int32_t  max_req_tokens;        /* longest request accepted by cp_match_spans (<= 2^20); above 10240
                                       the matcher keeps its per-request arrays in SCRATCH (24 B/token) */
    int32_t  max_batch_reqs;        /* most requests per match / insert call                             */
    int64_t  max_batch_tokens;      /* most tokens per match / insert call                               */
    int32_t  max_spans_per_insert;  /* most spans per insert call                                        */
    int32_t  max_sessions;          /* same-user sessions 1..max_sessions (R#33); 0 = no session store      */
} cp_config;

enum { CP_WS_POOL_K = 0, CP_WS_POOL_V = 1, CP_WS_META = 2, CP_WS_SCRATCH = 3, CP_WS_COUNT = 4 };

/* Fill sizes_h[CP_WS_COUNT] with the byte size of each workspace the caller must allocate
 * (device memory, 256-byte aligned).  Pool K/V layout: [num_layers][num_pages][16][H][d] dtype. */
cp_status cp_index_workspace(const cp_config* cfg_h, size_t* sizes_h);

/* Physical pool pages for cfg: ceil((capacity + max_span_len)/16) + ceil(capacity/window_len) + 1,
 * enough that the token budget, not the page count, always decides eviction. */
int64_t cp_pool_num_pages(const cp_config* cfg_h);
int32_t cp_max_pages_per_entry(const cp_config* cfg_h);

/* Create an empty index inside caller-allocated workspaces ws_h[CP_WS_COUNT] (device pointers).
 * Initializes the free-page FIFO to ascending page ids and an empty hash table on `stream`. */
cp_status cp_index_create(const cp_config* cfg_h, void* const* ws_h, void* stream, cp_index** out_h);
cp_status cp_index_destroy(cp_index* idx);

/* A CSR batch of requests. */
typedef struct {
    int32_t        num_reqs;
    int64_t        total_tokens;
    const int32_t* tokens;          /* [total_tokens]                                                 */
    const int64_t* offsets;         /* [num_reqs + 1], offsets[0] = 0                                 */
    const uint8_t* mask;            /* [total_tokens] 1 = sensitive; NULL allowed for match (R#9)    */
    int32_t        max_req_len;     /* host hint: longest request in the batch (0 = cfg max)         */
    const int32_t* session;         /* [num_reqs] same-user session of each request (R#33), or NULL:
                                       1..max_sessions = that user's session, 0 = anonymous          */
} cp_batch;

/* A paged KV cache in vLLM NHD layout: per layer a K and a V tensor [num_blocks][16][H][d]. */
typedef struct {
    void* const*   k_layers_h;      /* host array [num_layers] of device pointers                    */
    void* const*   v_layers_h;
    const int32_t* block_tables;    /* [num_reqs][max_blocks_per_req] block ids                      */
    int32_t        max_blocks_per_req;
} cp_paged_kv;

/*
 * Pool views (multi-GPU load balancing).  A rank whose shard of the (layer, KV head)
 * grid is not one rectangle holds one index for a rectangle (the base) and a view per further
 * rectangle: the view has its own geometry (num_layers x num_kv_heads at layer_offset / head_offset;
 * head_dim, dtype, RoPE and every capacity are the base's) and its own pool K/V workspaces (sizes:
 * cp_index_workspace of the base's config with the view's geometry), and shares the base's META and
 * SCRATCH -- the entry table, page lists, hash table, hit and copy lists -- so one match and one
 * insert serve every rectangle of the rank.  Allowed on a view: cp_gather_rerotate (with the base's
 * cp_match_spans output; every page id is the base's), cp_link_blocks, cp_index_copy_in,
 * cp_index_snapshot / cp_index_last_error (the base's state).  cp_match_spans and the insert calls on a
 * view return CP_ERR_INVALID_ARG.  A view must be destroyed before its base; all calls on a base and
 * its views must be stream-ordered by the caller (they share scratch).
 */
cp_status cp_index_create_view(const cp_index* base, int32_t num_layers, int32_t num_kv_heads, int32_t layer_offset,
                               int32_t head_offset, void* pool_k, void* pool_v, cp_index** out_h);

/* Copy the writer K/V rows of the entries published by the base's most recent cp_index_insert /
 * cp_index_insert_commit into this view's pool pages (the view's share of that insert's copy-in;
 * no rotation; flags: 0 or CP_REUSE_WORKLIST).  writers_h / writer_kv_h: the insert's writer batch and the writer paged KV in the
 * view's geometry.  Must be stream-ordered after that commit and before the base's next insert. */
cp_status cp_index_copy_in(cp_index* view, const cp_batch* writers_h, const cp_paged_kv* writer_kv_h, int32_t flags,
                           void* stream);

/* CP_REUSE_WORKLIST (cp_gather_rerotate / cp_index_copy_in flag): the gather's work list -- chunks of
 * hits, per-token source/destination row INDICES with plan codes, per-hit cos/sin -- does not depend on
 * the layer / head geometry, so the rectangles of one rank build it once.  With the flag, the call
 * reuses the list the immediately preceding gather (or insert copy-in) of this index family built,
 * and launches only the copy kernel.  The library checks on the host that the previous list was built
 * from the same buffers (hits, batch offsets, plan, block table pointer and width, CP_SKIP_LINKED) and
 * that no match / insert ran since, else returns CP_ERR_INVALID_ARG; the caller guarantees that those
 * buffers' CONTENTS did not change in between (so all rectangles must share one block table). */

/*
 * Insert `num_spans` segments (request span_req[s], positions [span_begin[s], +span_len[s])) of
 * the writer batch, in input order, at logical time `logical_time`.  Per span: DUPLICATE (an equal
 * live segment exists: refresh its last_used), else DROPPED_CONTAINED (a live segment strictly
 * contains it), else stored -- removing every live segment it strictly contains (SUPERSEDED) --
 * on pages taken from the FIFO head, with its K/V rows copied from writer_kv unrotated; then LRU
 * eviction by (last_used, id) while live tokens exceed the budget (R#20-22).
 * recompute_bits: packed LSB-first per span starting at word bits_word_offsets[s] (device arrays;
 * NULL = no recompute marks).  out_entry_id[s]: the stored / duplicate / containing entry id.
 * Device errors (no side effects): CP_ERR_INVALID_ARG (range, or a span reaching past the writer's
 * block table), CP_ERR_SPAN_TOO_SHORT, CP_ERR_CAPACITY (len > budget or > max_span_len), CP_ERR_SENSITIVE_SPAN
 * -- the first failing span in input order decides the code; then, still before any change,
 * CP_ERR_CAPACITY if one span strictly contains more than 1024 stored or batch segments, or if the
 * spans' copy-in work list (sum of ceil(len/32)) exceeds max_batch_tokens/32 + max_spans_per_insert + 1
 * (possible only with overlapping spans).  Config limits (cp_index_workspace / create reject others):
 * max_span_len <= 25599; window_len >= 3 when max_req_tokens > 10240.
 */
cp_status cp_index_insert(cp_index* idx, const cp_batch* writers_h, const cp_paged_kv* writer_kv_h,
                          int32_t num_spans, const int32_t* span_req, const int32_t* span_begin,
                          const int32_t* span_len, const uint32_t* recompute_bits,
                          const int64_t* bits_word_offsets, uint64_t logical_time,
                          int32_t* out_entry_id, int32_t* out_outcome, void* stream);

/*
 * The same insert in two stream-ordered halves, so that its read-only work overlaps other work on the
 * index.  cp_index_insert_prepare runs validation, hashing, batch dedup and the containment scan /
 * verification: it reads the index and writes only insert scratch, so it may run on another stream
 * concurrently with cp_match_spans / cp_gather_rerotate / cp_link_blocks on this index (never with
 * another insert).  cp_index_insert_commit, called with the SAME arguments, applies the spans (dedup
 * outcomes, supersede, LRU eviction, table updates, copy-in): it must be stream-ordered after the
 * prepare and after every gather that reads hits from before it.  recompute_bits are read only by the
 * commit, so they may be produced concurrently with the prepare.  prepare + commit on one stream is
 * exactly cp_index_insert.  A commit without a pending prepare, or a second prepare (or a plain insert)
 * while one is pending, returns CP_ERR_INVALID_ARG with no side effects.
 */
cp_status cp_index_insert_prepare(cp_index* idx, const cp_batch* writers_h, const cp_paged_kv* writer_kv_h,
                                  int32_t num_spans, const int32_t* span_req, const int32_t* span_begin,
                                  const int32_t* span_len, const uint32_t* recompute_bits,
                                  const int64_t* bits_word_offsets, uint64_t logical_time,
                                  int32_t* out_entry_id, int32_t* out_outcome, void* stream);
cp_status cp_index_insert_commit(cp_index* idx, const cp_batch* writers_h, const cp_paged_kv* writer_kv_h,
                                 int32_t num_spans, const int32_t* span_req, const int32_t* span_begin,
                                 const int32_t* span_len, const uint32_t* recompute_bits,
                                 const int64_t* bits_word_offsets, uint64_t logical_time,
                                 int32_t* out_entry_id, int32_t* out_outcome, void* stream);

/*
 * cp_index_insert_commit whose copy-in also fills `num_views` (<= 3) pool views of idx, all in ONE launch
 * of the copy kernel: writer_kv_h[0] is the writer KV in idx's geometry, writer_kv_h[1 + i] in
 * views_h[i]'s (all on the SAME block_tables pointer and width).  Equivalent to the commit followed by
 * cp_index_copy_in on every view (same rows, bit for bit).  Requirements as cp_gather_rerotate_rects
 * (CP_ERR_INVALID_ARG with no side effects otherwise); the rest as cp_index_insert_commit.
 */
cp_status cp_index_insert_commit_rects(cp_index* idx, int32_t num_views, cp_index* const* views_h,
                                       const cp_batch* writers_h, const cp_paged_kv* writer_kv_h,
                                       int32_t num_spans, const int32_t* span_req, const int32_t* span_begin,
                                       const int32_t* span_len, const uint32_t* recompute_bits,
                                       const int64_t* bits_word_offsets, uint64_t logical_time,
                                       int32_t* out_entry_id, int32_t* out_outcome, void* stream);

/*
 * Same-user session reuse (NEXT-2; "If the request belongs to the same user session,
 * all KV cache can be reused without restriction.  If the request originates from a different user, it
 * applies the selective cross-user sharing policy"; R#33: exact-prefix reuse of
 * the user's own last request).  Needs cfg.max_sessions >= 1 and writers_h->session.  For each request r
 * in input order, session s = writers_h->session[r] in 1..max_sessions: the session's private entry is
 * replaced by the WHOLE request [0, n_r) -- sensitive tokens included, no recompute marks -- stored at
 * origin 0 on pages from the FIFO head (the old entry's pages go to the FIFO tail first), with its K/V
 * rows copied from writer_kv_h; then LRU eviction as for shared entries (one budget; victims = min
 * (last_used, id) among unpinned live entries of any owner).  A pinned old entry, or pinned tokens + n_r
 * over the budget, gives CP_DEFERRED_PINNED (R#32).  Private entries are never in the prefix filter:
 * they take part in no dedup / containment with shared entries and are invisible to cp_match_spans
 * except for requests of their own session.  out_entry_id / out_outcome: device int32 [num_reqs]
 * (CP_STORED or CP_DEFERRED_PINNED).  Device errors (nothing changes; the first failing request decides):
 * a session out of range, an empty request, a block table too narrow -> CP_ERR_INVALID_ARG; a request
 * longer than the budget or max_span_len, more requests than free entry slots -> CP_ERR_CAPACITY.
 * Matching: cp_match_spans with readers_h->session set gives each request of session s >= 1 the longest
 * common prefix with s's private entry as its first hit (dst 0, delta 0, hit_len = that prefix) when it
 * is >= window_len tokens, no reader-mask test (the user's own tokens), and cross-user hits only after
 * it; session 0 = anonymous.  Only without CP_MATCH_FIXED_CHUNK / CP_MATCH_PREFIX_ONLY.
 */
cp_status cp_index_insert_session(cp_index* idx, const cp_batch* writers_h, const cp_paged_kv* writer_kv_h,
                                  uint64_t logical_time, int32_t* out_entry_id, int32_t* out_outcome, void* stream);

/* Outputs of cp_match_spans (all device buffers owned by the caller). */
typedef struct {
    int32_t  max_hits;              /* capacity; must be >= sum_r floor(n_r / window_len)            */
    int32_t* num_hits;              /* [1]                                                            */
    int32_t* req_hit_offsets;       /* [num_reqs + 1]                                                 */
    int32_t* hit_req;               /* [max_hits] request index                                       */
    int32_t* hit_entry;             /* [max_hits] entry id                                            */
    int32_t* hit_slot;              /* [max_hits] pool slot of the entry (consumed by the gather)     */
    int32_t* hit_dst;               /* [max_hits] first request position covered                     */
    int32_t* hit_len;               /* [max_hits] entry length                                        */
    int32_t* hit_delta;             /* [max_hits] RoPE delta = hit_dst - entry origin (R#11)          */
    uint8_t* plan;                  /* [total_tokens] CP_PLAN_* per position                         */
    int32_t* req_covered;           /* [num_reqs] positions covered by hits                           */
    int32_t* req_recompute;         /* [num_reqs] covered positions marked for recompute              */
    int32_t* req_candidates;        /* [num_reqs] prefix-filter candidates c                 */
} cp_hits;

/*
 * Match every request against the index (a snapshot for the call): each (k, entry e) with
 * request[k..k+m_e) equal to e's tokens (and, if a reader mask is given, no mask-1 position in the
 * range) is a verified candidate; hits are assembled greedily left to right, longest first, then
 * smaller id (R#7).  Accepted hits touch last_used[e] = max(last_used[e], logical_time) unless
 * CP_MATCH_NO_TOUCH.  Device error: a request longer than cfg.max_req_tokens, or max_hits exceeded.
 *
 * Baseline policies (NEXT-3, Fig. 4, §5.7), at most one
 * of the two flags:
 *   CP_MATCH_FIXED_CHUNK -- FixedChunk(w): only the chunk-aligned windows k = c*w (k + w <= n) are
 *     probed and only entries of length w are accepted; a chunk is covered iff an equal live
 *     length-w entry exists and the chunk has no mask-1 token (Fig. 4-b).  Position-independent
 *     (delta = k - origin may be nonzero).  The chunk store is filled by cp_policy_spans (R#28).
 *   CP_MATCH_PREFIX_ONLY -- PrefixOnly: only entries stored at origin 0 whose first w tokens equal
 *     the request's first w tokens; the covered prefix is the longest common prefix with such an
 *     entry, ending where tokens diverge, at the first mask-1 token, or at the entry's end (Fig. 4-a);
 *     covered only if >= w tokens (R#29).  One hit at dst 0, delta 0, hit_len = that prefix (may be
 *     shorter than the entry), longest first then smaller id.  More origin-0 candidates than
 *     min(max_req_len, cfg.max_req_tokens) for one request: device error CP_ERR_CAPACITY.
 * Both flags set: CP_ERR_INVALID_ARG.
 */
cp_status cp_match_spans(cp_index* idx, const cp_batch* readers_h, uint64_t logical_time,
                         int32_t flags, const cp_hits* out_h, void* stream);

/*
 * For every hit h and token t < hit_len[h] at request position q = hit_dst[h] + t, and every
 * (layer, head) of the shard: V_dst[q] <- V_pool[e][t] (bit copy); K_dst[q] <- R(delta) K_pool[e][t]
 * (fp32 products with cos/sin of delta*theta_i evaluated in fp64; delta == 0 is a bit copy).  With
 * CP_ZERO_RECOMPUTE, plan-2 positions get +0.0 in K and V (zero placeholders); with
 * CP_ZERO_UNCOVERED, plan-0 positions are zeroed too (both flags = the paper-literal placeholders, R#14);
 * with CP_SKIP_RECOMPUTE, plan-2 rows are neither copied nor zeroed (the plan codes are the placeholders
 * and the engine's prefill writes those rows; CP_ZERO_RECOMPUTE is then ignored).  `hits` is the struct cp_match_spans wrote
 * (only num_hits, hit_* and plan are read).  readers_h must be the batch that was matched.
 * Device error: a block table narrower than a covered position (position >> 4 >= max_blocks_per_req)
 * -> CP_ERR_INVALID_ARG, and no row is written (the copy kernel sees the error word and exits).
 */
cp_status cp_gather_rerotate(cp_index* idx, const cp_batch* readers_h, const cp_hits* hits_h,
                             const cp_paged_kv* dst_kv_h, int32_t flags, void* stream);

/*
 * cp_gather_rerotate for every rectangle of a rank in ONE launch of the persistent copy kernel (and one
 * of the zero-placeholder kernel): the base index `idx` and `num_views` (<= 3) of its pool views
 * (cp_index_create_view), destination caches dst_kv_h[0] (the base's geometry) and dst_kv_h[1 + i]
 * (views_h[i]'s geometry); the results are exactly those of one cp_gather_rerotate per rectangle (the
 * same kernels, rows and rotations; only the work of all rectangles shares one grid, so the launch has
 * one ramp and one tail instead of one per rectangle).  Same passages, hit list and flags as
 * cp_gather_rerotate (CP_REUSE_WORKLIST is not accepted: the call builds the list itself).  Requirements
 * (CP_ERR_INVALID_ARG, no side effects otherwise): idx is not a view, every views_h[i] is a view of idx,
 * every dst_kv_h[i] has the SAME block_tables pointer and width, the rectangles' layers total at most
 * 128.  Device errors as cp_gather_rerotate.
 */
cp_status cp_gather_rerotate_rects(cp_index* idx, int32_t num_views, cp_index* const* views_h,
                                   const cp_batch* readers_h, const cp_hits* hits_h, const cp_paged_kv* dst_kv_h,
                                   int32_t flags, void* stream);

/*
 * Recompute scores and top-rho selection for `num_spans` spans.  Span s uses the
 * final-layer attention attn_h[s] (device, fp32 [heads_h[s]][n_h[s]][n_h[s]] row-major), span
 * [span_l_h[s], span_r_h[s]] (inclusive).  For i in the span, with q(x) = trunc(x * 2^40) (R#17):
 *   score(i) = sum_heads ( sum_{j < l} q(A[i][j]) - sum_{l <= j <= i} q(A[i][j]) )
 * out_scores (device int64) receives m_s scores from score_offsets_h[s]; out_bits (device uint32)
 * receives ceil(m_s/32) words from bits_word_offsets_h[s]: the first ceil(rho_num*m/rho_den) tokens in
 * (score desc, index asc) order get bit 1 (R#15-16).  max_m bounds m_s (<= 16384).
 * Fixed-point domain (the sums are exact int64): attention entries are probabilities, each head's row
 * summing to at most 1 (softmax; a bf16 export may exceed 1 by rounding -- up to 2 is fine).  A score
 * then sums at most heads * 2 * 2^40 < 2^49 in magnitude (heads <= 255): exact.  Rows summing past 2^22
 * are outside the precondition and may wrap; that is not detected.
 * mode CP_SCORE_KVDEV takes KV caches, not attention: it returns CP_ERR_UNSUPPORTED here; the
 * CacheBlend selector is cp_score_kv_deviation below.
 */
cp_status cp_score_deviation(int32_t num_spans, const float* const* attn_h, const int32_t* n_h,
                             const int32_t* heads_h, const int32_t* span_l_h, const int32_t* span_r_h,
                             int32_t rho_num, int32_t rho_den, int32_t mode, int32_t max_m,
                             int64_t* out_scores, const int64_t* score_offsets_h,
                             uint32_t* out_bits, const int64_t* bits_word_offsets_h, void* stream);

/*
 * NEXT-4: CacheBlend's recompute selector, the KV-deviation variant the paper contrasts with its own
 * score ("compares the first-layer KV of a chunk in its original context with that
 * from a full recomputation in the new context, then recomputes the top 15% of tokens with the
 * largest deviation").  The paper gives no norm; R#30 fixes it.  For span s (request
 * span_req_h[s], positions [span_l_h[s], span_r_h[s]] inclusive) and token q in it:
 *   dev(q) = sum_{h < H, c < d} |q24(Kr[q][h][c]) - q24(Kf[q][h][c])| + |q24(Vr[q][h][c]) - q24(Vf[q][h][c])|
 * with q24(x) = trunc(x * 2^24) in int64 (exact and order independent, so GPU == oracle bit for bit).
 *   reused_{k,v}: ONE layer (the first) of the request's paged cache holding the reused KV (the
 *                 cp_gather_rerotate output: re-rotated to the new positions, so the comparison is
 *                 position-consistent), vLLM NHD [blocks][16][H][d] in `dtype`;
 *   fresh_{k,v}:  the same layer from a full recomputation in the new context, same layout;
 *   *_block_tables: int32 [num_reqs][*_max_blocks] block ids (may differ between the two caches).
 * Outputs as cp_score_deviation: out_scores[score_offsets_h[s] + i] = dev(span_l + i) (int64);
 * bits from bits_word_offsets_h[s]: the first ceil(rho_num*m/rho_den) tokens in (dev desc, index asc)
 * order get bit 1 (R#15-16; CacheBlend's 15% = 3/20).  Requirements: H*d*elem_bytes a multiple of
 * 16 bytes, |x| * 2^24 * 2 * H * d < 2^63 (|x| < 2^12 for H*d = 1024), max_m <= 16384.
 */
cp_status cp_score_kv_deviation(int32_t num_spans, const int32_t* span_req_h, const int32_t* span_l_h,
                                const int32_t* span_r_h, const void* reused_k, const void* reused_v,
                                const int32_t* reused_block_tables, int32_t reused_max_blocks,
                                const void* fresh_k, const void* fresh_v, const int32_t* fresh_block_tables,
                                int32_t fresh_max_blocks, int32_t num_kv_heads, int32_t head_dim, int32_t dtype,
                                int32_t rho_num, int32_t rho_den, int32_t max_m, int64_t* out_scores,
                                const int64_t* score_offsets_h, uint32_t* out_bits,
                                const int64_t* bits_word_offsets_h, void* stream);

/*
 * NEXT-2: zero-copy page linking (the retriever "link[s] reusable segments without
 * touching the actual KV"; prefix sharing shares whole cached blocks, L245-252).  A link is possible
 * only where a request block IS a stored page (R#31): block b of request r (positions
 * [16b, 16b+16)) links to pool page page_list[e][j] iff one hit (e, dst, len, delta) of r has
 * delta == 0, dst % 16 == 0, dst <= 16b and 16b + 16 <= dst + len (j = (16b - dst)/16), and all 16
 * positions have plan code CP_PLAN_REUSED.  Writes link_table[r * max_blocks_per_req + b] = that pool
 * page, -1 for every other block b < ceil(n_r / 16) (entries beyond are not written).  The page's
 * rows are the ones cp_gather_rerotate would copy (bit copies: delta 0), so an engine may point its
 * block table at the pool page (layer l's rows at pool_k + ((l * P + page) * 16) * H * d) instead
 * of copying; cp_gather_rerotate with CP_SKIP_LINKED then leaves those destination blocks unwritten.
 * Lifetime: unpinned, a linked page stays valid until the next cp_index_insert on this index (which may
 * evict and recycle it); pinned with cp_pin_links it stays valid until released.  `hits_h`: the
 * cp_match_spans output for `readers_h` on this index state.
 * Device error: max_blocks_per_req smaller than a request's block count -> CP_ERR_INVALID_ARG.
 */
cp_status cp_link_blocks(cp_index* idx, const cp_batch* readers_h, const cp_hits* hits_h,
                         int32_t* link_table, int32_t max_blocks_per_req, void* stream);

/*
 * NEXT-2 lifetime of linked pages (R#32; vLLM-style block reference counts).  For each of the n
 * entries of `pages` (device int32; entries < 0 skipped, so a cp_link_blocks table can be passed as is)
 * the live entry owning that pool page gets `delta` pins (+1 when an engine links the block, -1 when it
 * releases it).  While an entry has pins it is never evicted (LRU victims = min (last_used, id) among
 * unpinned live entries) nor superseded: an insert span that would remove it, or whose length with the
 * pinned tokens exceeds the budget, gets CP_DEFERRED_PINNED and changes nothing -- so a pinned page is
 * never recycled and its rows stay exactly what the gather would copy.  Device error (nothing changes):
 * a page that no live entry owns, or a count that would go negative -> CP_ERR_INVALID_ARG.
 */
cp_status cp_pin_links(cp_index* idx, const int32_t* pages, int64_t n, int32_t delta, void* stream);

/*
 * NEXT-3: the spans a baseline policy stores for a writer batch (R#28-29), in
 * (request, position) order:
 *   CP_POLICY_FIXED_CHUNK -- every chunk [c*chunk_len, (c+1)*chunk_len) inside the request that has
 *     no mask-1 token ("full-chunk hashes of prior requests' chunks, invalidating
 *     sensitive-containing chunks");
 *   CP_POLICY_PREFIX_ONLY -- [0, min(first mask-1 position, n, max_len)) if at least chunk_len long.
 * writers_h: batch with mask (required).  Outputs (device, caller-owned, room for max_spans):
 * span_req / span_begin / span_len, and count_d[0] = number of spans the policy yields (may exceed
 * max_spans; only the first max_spans are written).  If count_h is non-NULL the call synchronizes
 * the stream, stores the count there and returns CP_ERR_CAPACITY when it exceeds max_spans.
 */
cp_status cp_policy_spans(const cp_batch* writers_h, int32_t policy, int32_t chunk_len, int32_t max_len,
                          int32_t max_spans, int32_t* span_req, int32_t* span_begin, int32_t* span_len,
                          int32_t* count_d, int32_t* count_h, void* stream);

/* ---- NEXT-1: on-device KV Annotator (C1 Steps 1-2) -------------------------- */

/* Workspace bytes cp_annotate_spans needs for these requests: per request 8 (n S + 3) with S = (n+5) & ~3
 * (row prefixes, rows padded so a lane's four entries are 32-B aligned)
 * + 8(n+1) (P) + 8 max_segments (segments) + 16 max_segments ceil(n/32) (partial bests), each
 * 256-B aligned. */
size_t cp_annotate_workspace(int32_t num_reqs, const int32_t* n_h, int32_t max_segments);

/*
 * For every coarse segment (maximal mask-0 run) of every request, select the substring
 * [l*, r*] with r*-l*+1 >= min_len maximising IntraAttn - InterAttn (Step 2 P:L635-639)
 * of the causal final-layer attention attn_h[r] (device fp32 [heads][n][n], heads summed, only
 * j <= i read), computed exactly in the 2^-40 fixed point of R#17 (Step 1's summed-area sums,
 * P:L600-613).  Ties: longer, then leftmost; reported only if the difference is > 0.
 * mask_h[r]: device uint8 [n] (1 = sensitive).  Outputs (device): out_nseg[r] = number of coarse
 * segments (-1 if more than max_segments); for s < out_nseg[r], at [r * max_segments + s]:
 * out_l / out_r (0-based inclusive, -1 if the segment yields no reusable span) and out_diff.
 * workspace: device, >= cp_annotate_workspace(...) bytes, caller-owned.
 * Fixed-point domain: the summed-area sums cover the whole causal triangle, so with the probabilities of
 * cp_score_deviation (each head's row summing to at most 1, 2 with bf16 rounding) they stay below
 * n * heads * 2 * 2^40: exact for n * heads < 2^22, checked (CP_ERR_INVALID_ARG).  Rows summing past 2
 * are outside the precondition and may wrap (a uniform non-normalised matrix wraps near n = 4.5K).
 */
cp_status cp_annotate_spans(int32_t num_reqs, const float* const* attn_h, const int32_t* n_h,
                            const int32_t* heads_h, const uint8_t* const* mask_h, int32_t min_len,
                            int32_t max_segments, void* workspace, size_t workspace_bytes,
                            int32_t* out_nseg, int32_t* out_l, int32_t* out_r, int64_t* out_diff, void* stream);

/* ---- test / diagnostic exports ------------------------------------------------------------- */

/* Prefix hashes of every request: out_h (device u64) gets n_r + 1 values per request starting at
 * offsets[r] + r (h[0] = 0, h[k] = h[k-1]*B + tokenval(t_k) mod p). */
cp_status cp_hash_prefix(const cp_batch* batch_h, uint64_t hash_seed, uint64_t* out_h, void* stream);

/* Host copy of the live entries, sorted by id.  Arrays are caller-allocated HOST buffers with room
 * for cfg.max_entries entries (pages: max_pages_per_entry each; tokens/recompute: max_span_len each;
 * fifo: cp_pool_num_pages).  Optional arrays may be NULL.  Synchronizes the stream. */
typedef struct {
    int32_t   num_live;
    int32_t   next_id;
    int64_t   live_tokens;
    int32_t   fifo_count;
    int32_t   error;
    int32_t*  id;
    int32_t*  len;
    int32_t*  origin_pos;
    uint64_t* prefix_hash;
    uint64_t* full_hash;
    uint64_t* last_used;
    uint8_t*  digest;               /* [32] per entry */
    int32_t*  pages;                /* [max_pages_per_entry] per entry */
    int32_t*  tokens;               /* [max_span_len] per entry, optional */
    uint8_t*  recompute;            /* [max_span_len] per entry, optional */
    int32_t*  fifo;                 /* free pages in pop order, optional */
    int32_t*  pin;                  /* per entry: linked-block pins (R#32), optional */
    int32_t*  owner;                /* per entry: 0 shared, s = private entry of session s (R#33), optional */
} cp_snapshot;
cp_status cp_index_snapshot(cp_index* idx, cp_snapshot* out_h, void* stream);

/* Device logical clock (for CUDA-graph capture of a serving step): with d_clock set (device uint64,
 * caller-owned), cp_match_spans, the insert commit and cp_index_insert_session read the logical time
 * from *d_clock when their kernels run and ignore their host `logical_time` argument -- so a captured
 * step replays with the time the caller writes there before each replay (e.g. a captured copy from a
 * pinned host scalar).  NULL restores the host argument. */
cp_status cp_index_set_clock(cp_index* idx, const uint64_t* d_clock);

/* L2 residency of the index metadata (B200: 126 MB L2 with a persisting carve-out).  Sets `stream`'s (and
 * the index's internal side stream's) access-policy window to the index's META workspace with
 * persisting hits (hit_ratio in [0, 1]; 0 clears the window) and raises the device's persisting-L2 limit
 * to the window size (capped by the device maxima) if it is lower.  The gather streams ~100 GB per step
 * through L2 with evict-first hints; without this the control-plane kernels (match, commit) find about
 * half of the entry table in DRAM.  Kernels launched in the stream afterwards (and captured into a CUDA
 * graph from it) carry the window.  Device-wide side effect: the persisting carve-out.  Returns
 * CP_ERR_UNSUPPORTED where the device has no persisting L2. */
cp_status cp_index_l2_persist(cp_index* idx, void* stream, float hit_ratio);

/* Synchronizes, returns and clears the sticky device error word (CP_OK if none). */
cp_status cp_index_last_error(cp_index* idx, void* stream);

/* Insert commits applied so far by the parallel path and by the sequential path, and the OR of the
 * reasons the sequential one was taken (diagnostic; out_h[3]; synchronizes).  Both give identical results; the parallel one needs a batch whose segments do not
 * interact (DESIGN.md §6 N4). */
cp_status cp_index_commit_stats(cp_index* idx, int32_t* out_h, void* stream);

/* Matcher work counters accumulated by cp_match_spans since creation (or the last reset), out_h[4]:
 * windows probed (n - w + 1 per request), prefix-filter candidates c, candidates that passed the
 * full-hash pre-check, and the tokens their exact verification may compare -- the O(n + c) cost of
 * P:L696-697.  reset != 0 zeroes them.  Synchronizes. */
cp_status cp_index_match_work(cp_index* idx, uint64_t* out_h, int32_t reset, void* stream);

/* Hash base B of an index (diagnostic). */
uint64_t cp_index_hash_base(const cp_index* idx);

/* Select the gather kernel variant (A/B measurement; default 0 = unroll 2, 3 CTAs/SM, dynamic item
 * schedule; 1/2/3/5 static round-robin (unroll, CTAs/SM) = (2,4)/(4,2)/(3,2)/(8,1); 4 TMA bulk copy;
 * 6/7/8/9 dynamic (3,2)/(2,4)/(4,2)/(8,1)).  Also the CP_GATHER_VARIANT environment variable. */
cp_status cp_set_gather_variant(int32_t variant);

/* Select the N3 row kernel (A/B measurement; default 0, or the CP_SCORE_VARIANT environment variable):
 * 0 one row per 8-lane group (4 rows per warp), 4 CTAs/SM; 5 16-lane groups; 6 8-lane groups with 6
 * vectors per lane at 3 CTAs/SM; 7 4-lane groups; 4 the round-1 one-warp-per-row kernel at 4 CTAs/SM and
 * 1 / 2 / 3 the same at 5 / 6 / 8 CTAs/SM.  All give identical results. */
cp_status cp_set_score_variant(int32_t variant);

/* Diagnostic: contiguous copy of `bytes` (multiple of 16) with the gather's 128-bit streaming load /
 * store instructions, ctas_per_sm x 256-thread CTAs per SM (roofline reference for the gather). */
cp_status cp_copy_diag(const void* src, void* dst, int64_t bytes, int32_t ctas_per_sm, void* stream);

/* Number of kernels this library launched since load (evidence for gpu_launches). */
uint64_t cp_kernel_launch_count(void);

const char* cp_status_string(cp_status s);

/* Build provenance: "cp-src-sha256=<64 hex digits> arch=sm_100a" -- the SHA-256 of the sources and
 * flags this library was compiled from (paper_2605_23640_b200/build.py source_hash()); static string. */
const char* cp_build_info(void);

#ifdef __cplusplus
}
#endif
#endif /* CACHEPRUNE_H */
