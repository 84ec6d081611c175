/*
 * cp_oracle.c -- plain, slow, single-threaded CPU oracle for CachePrune's
 * token-granular KV-reuse hot path (arxiv 2605.23640).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no
 * code, header, table or constant generator with the CUDA path
 * (paper_2605_23640_b200/); neither includes the other.
 *
 * Citations: "P:Lnnn" = /root/reference/PAPER.md line, "S:Lnnn" = SPEC.md line,
 * "R#k" = reading k of DESIGN.md §3 (where the paper is silent or ambiguous).
 *
 * What is computed, and how (each is the plain definition or the paper's
 * algorithm step by step; no blocking, fusion or reordering):
 *   - polynomial hash mod p = 2^61-1, random base, tokenval = id+1
 *     (R#1-3), via an exact 128-bit product and `%`;
 *   - SHA-256 (FIPS 180-4) over big-endian u64 token ids (R#6);
 *   - pool insert: validation, Duplicate -> Contained -> Supersedes, FIFO page
 *     allocation, LRU eviction by (last_used, id)   (R#20-22);
 *   - match: the plain definition -- every (k, e) with request[k..k+m_e) equal
 *     to entry e's tokens ("appears as a contiguous substring"),
 *     found by naive substring search; then greedy left-to-right assembly
 *     (R#7), plan codes, LRU touch; the NEXT-3 baseline policies
 *     FixedChunk (aligned windows, length-w entries) and PrefixOnly (longest
 *     common prefix with an origin-0 entry) restrict the same naive search
 *     (Fig. 4; R#28-29);
 *   - RoPE re-rotation of one K row by delta in fp64, one rounding (R#11-13);
 *   - recompute score inter(i) - intra(i) in 2^-40 fixed point and top
 *     ceil(rho*m) selection (R#15-19).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>

#define ORC_P ((((uint64_t)1) << 61) - 1)

enum { ORC_OK = 0, ORC_ERR_INVALID_ARG = -1, ORC_ERR_SENSITIVE_SPAN = -2,
       ORC_ERR_SPAN_TOO_SHORT = -3, ORC_ERR_CAPACITY = -4 };
enum { ORC_STORED = 0, ORC_SUPERSEDED = 1, ORC_DUPLICATE = 2, ORC_DROPPED_CONTAINED = 3, ORC_DEFERRED_PINNED = 4 };

/* ------------------------------------------------------------------------- */
/* hashing  ("polynomial rolling hash modulo 2^61-1 with a random base") */
/* ------------------------------------------------------------------------- */
uint64_t orc_splitmix64(uint64_t x) {
    uint64_t z = x + 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

/* R#1: B = 2 + splitmix64(seed) mod (p-3), so B in [2, p-2]. */
uint64_t orc_hash_base(uint64_t seed) { return 2 + orc_splitmix64(seed) % (ORC_P - 3); }

uint64_t orc_mulmod(uint64_t a, uint64_t b) {
    unsigned __int128 x = (unsigned __int128)a * (unsigned __int128)b;
    return (uint64_t)(x % ORC_P);
}

static uint64_t tokenval(int32_t t) { return (uint64_t)(int64_t)t + 1; }   /* R#2 */

/* Horner fold, most-significant first (R#3):  H(t_1..t_m) = sum_k tokenval(t_k) B^(m-k) mod p.
 * This equals sub(1, m) of the prefix array. */
uint64_t orc_poly_hash(const int32_t* t, int64_t m, uint64_t B) {
    uint64_t h = 0;
    for (int64_t k = 0; k < m; ++k) h = (orc_mulmod(h, B) + tokenval(t[k])) % ORC_P;
    return h;
}

/* Prefix-hash array h[0..n]: h[0]=0, h[k] = (h[k-1]*B + tokenval(t_k)) mod p */
void orc_prefix_hashes(const int32_t* t, int64_t n, uint64_t B, uint64_t* h) {
    h[0] = 0;
    for (int64_t k = 1; k <= n; ++k) h[k] = (orc_mulmod(h[k - 1], B) + tokenval(t[k - 1])) % ORC_P;
}

/* ------------------------------------------------------------------------- */
/* SHA-256, FIPS 180-4 ("cryptographic hash (i.e., SHA-256)")          */
/* ------------------------------------------------------------------------- */
static const uint32_t K256[64] = {
    0x428a2f98, 0x71374491, 0xb5c0fbcf, 0xe9b5dba5, 0x3956c25b, 0x59f111f1, 0x923f82a4, 0xab1c5ed5,
    0xd807aa98, 0x12835b01, 0x243185be, 0x550c7dc3, 0x72be5d74, 0x80deb1fe, 0x9bdc06a7, 0xc19bf174,
    0xe49b69c1, 0xefbe4786, 0x0fc19dc6, 0x240ca1cc, 0x2de92c6f, 0x4a7484aa, 0x5cb0a9dc, 0x76f988da,
    0x983e5152, 0xa831c66d, 0xb00327c8, 0xbf597fc7, 0xc6e00bf3, 0xd5a79147, 0x06ca6351, 0x14292967,
    0x27b70a85, 0x2e1b2138, 0x4d2c6dfc, 0x53380d13, 0x650a7354, 0x766a0abb, 0x81c2c92e, 0x92722c85,
    0xa2bfe8a1, 0xa81a664b, 0xc24b8b70, 0xc76c51a3, 0xd192e819, 0xd6990624, 0xf40e3585, 0x106aa070,
    0x19a4c116, 0x1e376c08, 0x2748774c, 0x34b0bcb5, 0x391c0cb3, 0x4ed8aa4a, 0x5b9cca4f, 0x682e6ff3,
    0x748f82ee, 0x78a5636f, 0x84c87814, 0x8cc70208, 0x90befffa, 0xa4506ceb, 0xbef9a3f7, 0xc67178f2};

static uint32_t rotr(uint32_t x, int n) { return (x >> n) | (x << (32 - n)); }

static void sha256_block(uint32_t H[8], const uint8_t blk[64]) {
    uint32_t W[64];
    for (int t = 0; t < 16; ++t)
        W[t] = ((uint32_t)blk[4 * t] << 24) | ((uint32_t)blk[4 * t + 1] << 16) |
               ((uint32_t)blk[4 * t + 2] << 8) | (uint32_t)blk[4 * t + 3];
    for (int t = 16; t < 64; ++t) {
        uint32_t s0 = rotr(W[t - 15], 7) ^ rotr(W[t - 15], 18) ^ (W[t - 15] >> 3);
        uint32_t s1 = rotr(W[t - 2], 17) ^ rotr(W[t - 2], 19) ^ (W[t - 2] >> 10);
        W[t] = W[t - 16] + s0 + W[t - 7] + s1;
    }
    uint32_t a = H[0], b = H[1], c = H[2], d = H[3], e = H[4], f = H[5], g = H[6], h = H[7];
    for (int t = 0; t < 64; ++t) {
        uint32_t S1 = rotr(e, 6) ^ rotr(e, 11) ^ rotr(e, 25);
        uint32_t ch = (e & f) ^ (~e & g);
        uint32_t T1 = h + S1 + ch + K256[t] + W[t];
        uint32_t S0 = rotr(a, 2) ^ rotr(a, 13) ^ rotr(a, 22);
        uint32_t mj = (a & b) ^ (a & c) ^ (b & c);
        uint32_t T2 = S0 + mj;
        h = g; g = f; f = e; e = d + T1; d = c; c = b; b = a; a = T1 + T2;
    }
    H[0] += a; H[1] += b; H[2] += c; H[3] += d; H[4] += e; H[5] += f; H[6] += g; H[7] += h;
}

/* SHA-256 of an arbitrary byte message (padding per FIPS 180-4 §5.1.1). */
void orc_sha256_bytes(const uint8_t* msg, uint64_t len, uint8_t out[32]) {
    uint32_t H[8] = {0x6a09e667, 0xbb67ae85, 0x3c6ef372, 0xa54ff53a,
                     0x510e527f, 0x9b05688c, 0x1f83d9ab, 0x5be0cd19};
    uint64_t full = len / 64;
    for (uint64_t b = 0; b < full; ++b) sha256_block(H, msg + 64 * b);
    uint8_t tail[128];
    memset(tail, 0, sizeof(tail));
    uint64_t rem = len - 64 * full;
    memcpy(tail, msg + 64 * full, rem);
    tail[rem] = 0x80;
    uint64_t tl = (rem + 1 + 8 <= 64) ? 64 : 128;
    uint64_t bits = len * 8;
    for (int i = 0; i < 8; ++i) tail[tl - 1 - i] = (uint8_t)(bits >> (8 * i));
    sha256_block(H, tail);
    if (tl == 128) sha256_block(H, tail + 64);
    for (int i = 0; i < 8; ++i) {
        out[4 * i] = (uint8_t)(H[i] >> 24); out[4 * i + 1] = (uint8_t)(H[i] >> 16);
        out[4 * i + 2] = (uint8_t)(H[i] >> 8); out[4 * i + 3] = (uint8_t)H[i];
    }
}

/* R#6: digest = SHA-256 over the big-endian 8-byte encoding of each token id. */
void orc_sha256_tokens(const int32_t* t, int64_t m, uint8_t out[32]) {
    uint8_t* buf = (uint8_t*)malloc((size_t)(8 * m + 1));
    for (int64_t k = 0; k < m; ++k) {
        uint64_t v = (uint64_t)(int64_t)t[k];
        for (int i = 0; i < 8; ++i) buf[8 * k + i] = (uint8_t)(v >> (56 - 8 * i));
    }
    orc_sha256_bytes(buf, (uint64_t)(8 * m), out);
    free(buf);
}

/* ------------------------------------------------------------------------- */
/* KV Pool index                                                  */
/* ------------------------------------------------------------------------- */
typedef struct {
    int32_t id, live, len, origin_pos, origin_call, origin_req;
    int32_t pin;          /* linked-block pins on its pages (R#32) */
    int32_t owner;        /* 0: shared (cross-user) entry; s >= 1: the private entry of session s (R#33) */
    uint64_t prefix_hash, full_hash, last_used;
    uint8_t digest[32];
    int32_t* tokens;      /* [len] */
    uint8_t* recompute;   /* [len] 0/1 */
    int32_t* pages;       /* [npages] */
    int32_t npages;
} orc_entry;

typedef struct {
    int32_t w, block;
    uint64_t B;
    int64_t capacity;     /* token budget (R#21) */
    int32_t num_pages;
    orc_entry* e;         /* indexed by id; ids are never reused */
    int32_t n_e, cap_e;
    int32_t* fifo;        /* circular FIFO of free page ids (R#22) */
    int32_t fifo_head, fifo_count;
    int64_t live_tokens;
    int32_t calls;
} orc_index;

orc_index* orc_index_new(int32_t window_len, uint64_t hash_seed, int64_t capacity_tokens,
                         int32_t block_size, int32_t num_pages) {
    orc_index* x = (orc_index*)calloc(1, sizeof(orc_index));
    x->w = window_len; x->block = block_size; x->B = orc_hash_base(hash_seed);
    x->capacity = capacity_tokens; x->num_pages = num_pages;
    x->cap_e = 64; x->e = (orc_entry*)calloc((size_t)x->cap_e, sizeof(orc_entry));
    x->fifo = (int32_t*)malloc(sizeof(int32_t) * (size_t)num_pages);
    for (int32_t p = 0; p < num_pages; ++p) x->fifo[p] = p;     /* initially ascending page ids */
    x->fifo_head = 0; x->fifo_count = num_pages;
    return x;
}

void orc_index_free(orc_index* x) {
    for (int32_t i = 0; i < x->n_e; ++i) { free(x->e[i].tokens); free(x->e[i].recompute); free(x->e[i].pages); }
    free(x->e); free(x->fifo); free(x);
}

uint64_t orc_index_base(const orc_index* x) { return x->B; }

static void fifo_push(orc_index* x, int32_t p) {
    x->fifo[(x->fifo_head + x->fifo_count) % x->num_pages] = p;
    x->fifo_count++;
}
static int32_t fifo_pop(orc_index* x) {
    int32_t p = x->fifo[x->fifo_head];
    x->fifo_head = (x->fifo_head + 1) % x->num_pages;
    x->fifo_count--;
    return p;
}

/* Remove a live entry: free its pages to the FIFO tail in page-list order. */
static void remove_entry(orc_index* x, orc_entry* e) {
    e->live = 0;
    x->live_tokens -= e->len;
    for (int32_t i = 0; i < e->npages; ++i) fifo_push(x, e->pages[i]);
}

/* Naive substring search: does `hay` (length n) contain `nee` (length m) contiguously? */
static int contains(const int32_t* hay, int64_t n, const int32_t* nee, int64_t m) {
    for (int64_t k = 0; k + m <= n; ++k) {
        int64_t i = 0;
        while (i < m && hay[k + i] == nee[i]) ++i;
        if (i == m) return 1;
    }
    return 0;
}

static int32_t bit_of(const uint32_t* bits, const int64_t* word_off, int32_t s, int32_t t) {
    if (!bits) return 0;
    return (int32_t)((bits[word_off[s] + t / 32] >> (t % 32)) & 1u);
}

/*
 * Insert spans in input order at logical time t (SPEC pool.insert S:L312-320).
 * Step 0 -- validate every span first (R#20/§8(b) "an insert call with any sensitive span
 *   changes nothing"): range, length >= w, length <= capacity, mask all 0
 *   (selective sharing).  The first failing span (in input order) decides the code.
 * Step 1 -- per span: DUPLICATE if a live entry has an equal SHA-256 digest (refresh last_used);
 *   else DROPPED_CONTAINED if a live entry strictly contains it (out id = smallest such id);
 *   else remove every live entry it strictly contains (ascending id), allocate pages from the
 *   FIFO head, store (id = next id), then evict LRU = min (last_used, id) until live tokens <= capacity.
 */
int32_t orc_index_insert(orc_index* x, const int32_t* tokens, const int64_t* offsets, const uint8_t* mask,
                         int32_t num_reqs, int32_t num_spans, const int32_t* span_req,
                         const int32_t* span_begin, const int32_t* span_len,
                         const uint32_t* bits, const int64_t* bits_word_offsets,
                         uint64_t t, int32_t* out_id, int32_t* out_outcome) {
    for (int32_t s = 0; s < num_spans; ++s) {
        int32_t r = span_req[s];
        if (r < 0 || r >= num_reqs) return ORC_ERR_INVALID_ARG;
        int64_t n = offsets[r + 1] - offsets[r];
        int64_t b = span_begin[s], m = span_len[s];
        if (b < 0 || m < 0 || b + m > n) return ORC_ERR_INVALID_ARG;
        if (m < x->w) return ORC_ERR_SPAN_TOO_SHORT;
        if (m > x->capacity) return ORC_ERR_CAPACITY;
        if (mask)
            for (int64_t k = 0; k < m; ++k)
                if (mask[offsets[r] + b + k]) return ORC_ERR_SENSITIVE_SPAN;
    }
    int32_t call = x->calls++;
    for (int32_t s = 0; s < num_spans; ++s) {
        int32_t r = span_req[s];
        const int32_t* tau = tokens + offsets[r] + span_begin[s];
        int32_t m = span_len[s];
        uint8_t dg[32];
        orc_sha256_tokens(tau, m, dg);
        /* Duplicate (R#20: checked first) */
        int32_t dup = -1;
        for (int32_t i = 0; i < x->n_e; ++i)
            if (x->e[i].live && !x->e[i].owner && memcmp(x->e[i].digest, dg, 32) == 0) { dup = i; break; }
        if (dup >= 0) {
            x->e[dup].last_used = t;
            out_id[s] = dup; out_outcome[s] = ORC_DUPLICATE;
            continue;
        }
        /* strictly contained in a live entry */
        int32_t cont = -1;
        for (int32_t i = 0; i < x->n_e && cont < 0; ++i)
            if (x->e[i].live && !x->e[i].owner && x->e[i].len > m && contains(x->e[i].tokens, x->e[i].len, tau, m)) cont = i;
        if (cont >= 0) { out_id[s] = cont; out_outcome[s] = ORC_DROPPED_CONTAINED; continue; }
        /* R#32 (NEXT-2 lifetime of linked pages): a span may not remove a pinned entry, and the pinned
           tokens plus the span must fit the budget (so that the LRU can always get back under it by
           evicting unpinned entries) -- otherwise it is DEFERRED_PINNED: not stored, nothing changes */
        int32_t blocked = -1;
        int64_t pinned_tok = 0;
        for (int32_t i = 0; i < x->n_e; ++i) {
            if (!x->e[i].live || x->e[i].pin == 0) continue;
            pinned_tok += x->e[i].len;
            if (blocked < 0 && !x->e[i].owner && x->e[i].len < m && contains(tau, m, x->e[i].tokens, x->e[i].len)) blocked = i;
        }
        if (blocked >= 0 || pinned_tok + m > x->capacity) {
            out_id[s] = blocked; out_outcome[s] = ORC_DEFERRED_PINNED;
            continue;
        }
        /* supersede live entries strictly contained in tau, ascending id */
        int32_t superseded = 0;
        for (int32_t i = 0; i < x->n_e; ++i)
            if (x->e[i].live && !x->e[i].owner && x->e[i].len < m && contains(tau, m, x->e[i].tokens, x->e[i].len)) {
                remove_entry(x, &x->e[i]);
                superseded = 1;
            }
        /* store */
        if (x->n_e == x->cap_e) {
            x->cap_e *= 2;
            x->e = (orc_entry*)realloc(x->e, sizeof(orc_entry) * (size_t)x->cap_e);
        }
        int32_t id = x->n_e++;
        orc_entry* e = &x->e[id];
        memset(e, 0, sizeof(*e));
        e->id = id; e->live = 1; e->len = m; e->origin_pos = span_begin[s];
        e->origin_call = call; e->origin_req = r;
        e->prefix_hash = orc_poly_hash(tau, x->w, x->B);     /* P:L680 prefix = first w tokens */
        e->full_hash = orc_poly_hash(tau, m, x->B);          /* P:L698 full-length hash */
        memcpy(e->digest, dg, 32);
        e->last_used = t;
        e->tokens = (int32_t*)malloc(sizeof(int32_t) * (size_t)m);
        memcpy(e->tokens, tau, sizeof(int32_t) * (size_t)m);
        e->recompute = (uint8_t*)malloc((size_t)m);
        for (int32_t k = 0; k < m; ++k) e->recompute[k] = (uint8_t)bit_of(bits, bits_word_offsets, s, k);
        e->npages = (m + x->block - 1) / x->block;
        e->pages = (int32_t*)malloc(sizeof(int32_t) * (size_t)e->npages);
        if (x->fifo_count < e->npages) return ORC_ERR_CAPACITY;   /* cannot happen with the sized pool */
        for (int32_t i = 0; i < e->npages; ++i) e->pages[i] = fifo_pop(x);
        x->live_tokens += m;
        out_id[s] = id; out_outcome[s] = superseded ? ORC_SUPERSEDED : ORC_STORED;
        /* LRU eviction: victim = min (last_used, id) among live, unpinned entries (R#32) */
        while (x->live_tokens > x->capacity) {
            int32_t v = -1;
            for (int32_t i = 0; i < x->n_e; ++i) {
                if (!x->e[i].live || x->e[i].pin > 0) continue;
                if (v < 0 || x->e[i].last_used < x->e[v].last_used) v = i;
            }
            remove_entry(x, &x->e[v]);
        }
    }
    return ORC_OK;
}

/*
 * Same-user sessions (R#33, "SameUserFull is modeled as exact-prefix reuse of
 * the user's own last request").  For each request in order: its session's current private entry is
 * replaced by the whole request [0, n) -- sensitive tokens included, no recompute marks -- stored at
 * origin 0 with pages from the FIFO head (the old entry's pages go to the FIFO tail first), then LRU
 * eviction as for shared entries (one budget; victims = min (last_used, id) among unpinned live entries of
 * any owner).  A pinned old entry, or pinned tokens + n over the budget, defers the request (R#32).
 * Private entries take part in no dedup / containment with shared ones; their prefix / full hashes are 0
 * (they are found through the session, never through the prefix filter).
 */
int32_t orc_index_insert_session(orc_index* x, const int32_t* tokens, const int64_t* offsets, int32_t num_reqs,
                                 const int32_t* sessions, uint64_t t, int32_t* out_id, int32_t* out_outcome) {
    for (int32_t r = 0; r < num_reqs; ++r) {
        const int64_t n = offsets[r + 1] - offsets[r];
        if (sessions[r] < 1 || n < 1) return ORC_ERR_INVALID_ARG;
        if (n > x->capacity) return ORC_ERR_CAPACITY;
    }
    int32_t call = x->calls++;
    for (int32_t r = 0; r < num_reqs; ++r) {
        const int32_t* tau = tokens + offsets[r];
        const int32_t m = (int32_t)(offsets[r + 1] - offsets[r]);
        int32_t old = -1;
        int64_t pinned_tok = 0;
        for (int32_t i = 0; i < x->n_e; ++i) {
            if (!x->e[i].live) continue;
            if (x->e[i].owner == sessions[r]) old = i;
            if (x->e[i].pin > 0) pinned_tok += x->e[i].len;
        }
        if ((old >= 0 && x->e[old].pin > 0) || pinned_tok + m > x->capacity) {
            out_id[r] = (old >= 0 && x->e[old].pin > 0) ? old : -1; out_outcome[r] = ORC_DEFERRED_PINNED;
            continue;
        }
        if (old >= 0) remove_entry(x, &x->e[old]);
        if (x->n_e == x->cap_e) {
            x->cap_e *= 2;
            x->e = (orc_entry*)realloc(x->e, sizeof(orc_entry) * (size_t)x->cap_e);
        }
        int32_t id = x->n_e++;
        orc_entry* e = &x->e[id];
        memset(e, 0, sizeof(*e));
        e->id = id; e->live = 1; e->len = m; e->origin_pos = 0; e->origin_call = call; e->origin_req = r;
        e->owner = sessions[r];
        orc_sha256_tokens(tau, m, e->digest);
        e->last_used = t;
        e->tokens = (int32_t*)malloc(sizeof(int32_t) * (size_t)m);
        memcpy(e->tokens, tau, sizeof(int32_t) * (size_t)m);
        e->recompute = (uint8_t*)calloc((size_t)m, 1);
        e->npages = (m + x->block - 1) / x->block;
        e->pages = (int32_t*)malloc(sizeof(int32_t) * (size_t)e->npages);
        if (x->fifo_count < e->npages) return ORC_ERR_CAPACITY;
        for (int32_t i = 0; i < e->npages; ++i) e->pages[i] = fifo_pop(x);
        x->live_tokens += m;
        out_id[r] = id; out_outcome[r] = ORC_STORED;
        while (x->live_tokens > x->capacity) {
            int32_t v = -1;
            for (int32_t i = 0; i < x->n_e; ++i) {
                if (!x->e[i].live || x->e[i].pin > 0) continue;
                if (v < 0 || x->e[i].last_used < x->e[v].last_used) v = i;
            }
            remove_entry(x, &x->e[v]);
        }
    }
    return ORC_OK;
}

/* ------------------------------------------------------------------------- */
/* match (P:L663-704 C2; P:L724-727 plan with zero placeholders)              */
/* ------------------------------------------------------------------------- */
typedef struct { int32_t k, m, id; } orc_cand;

static int cand_cmp(const void* a, const void* b) {       /* (k asc, m desc, id asc), R#7 */
    const orc_cand* x = (const orc_cand*)a; const orc_cand* y = (const orc_cand*)b;
    if (x->k != y->k) return x->k < y->k ? -1 : 1;
    if (x->m != y->m) return x->m > y->m ? -1 : 1;
    return x->id < y->id ? -1 : (x->id > y->id);
}

/*
 * For each request: the verified set V = {(k, e): request[k..k+m_e) == tokens(e), and (mask
 * given) mask all 0 on that range} -- the plain definition that prefix filtering + full-hash +
 * SHA-256 verification reach exactly.  candidates c = #{(k, e): request[k..k+w)
 * == first w tokens of e} (the prefix-filter hits).  Greedy assembly (R#7), plan codes
 * 0 uncovered / 1 reused / 2 recompute (entry's stored bit), then LRU touch of accepted hits
 * (max(last_used, t)) after all requests (the index is a snapshot for the call).
 * Returns the number of hits, or -1 if max_hits would overflow.
 */
/* flags: bit 0 no LRU touch; bit 1 FixedChunk; bit 2 PrefixOnly (NEXT-3). */
#define ORC_MATCH_NO_TOUCH 1
#define ORC_MATCH_FIXED_CHUNK 2
#define ORC_MATCH_PREFIX_ONLY 4

int32_t orc_match(orc_index* x, const int32_t* tokens, const int64_t* offsets, const uint8_t* mask,
                  const int32_t* sessions, int32_t num_reqs, uint64_t t, int32_t flags, int32_t max_hits,
                  int32_t* req_hit_offsets, int32_t* hit_req, int32_t* hit_entry, int32_t* hit_dst,
                  int32_t* hit_len, int32_t* hit_delta, uint8_t* plan,
                  int32_t* req_covered, int32_t* req_recompute, int32_t* req_candidates) {
    const int fixed = (flags & ORC_MATCH_FIXED_CHUNK) != 0, prefix = (flags & ORC_MATCH_PREFIX_ONLY) != 0;
    if (fixed && prefix) return -2;
    if (sessions && (fixed || prefix)) return -2;
    int32_t nh = 0;
    req_hit_offsets[0] = 0;
    for (int32_t r = 0; r < num_reqs; ++r) {
        const int32_t* q = tokens + offsets[r];
        int64_t n = offsets[r + 1] - offsets[r];
        const uint8_t* mk = mask ? mask + offsets[r] : NULL;
        uint8_t* pl = plan + offsets[r];
        memset(pl, 0, (size_t)n);
        int32_t cov = 0, rec = 0, cands = 0;
        if (prefix) {
            /* PrefixOnly (Fig. 4-a): the covered prefix ends where the tokens
             * diverge or at the first mask-1 token.  Stored prefixes are the entries at origin 0 whose
             * first w tokens equal the request's (R#29). */
            int32_t best = -1, bl = 0;
            for (int32_t i = 0; n >= x->w && i < x->n_e; ++i) {
                orc_entry* e = &x->e[i];
                if (!e->live || e->owner) continue;
                int64_t j = 0;
                while (j < x->w && q[j] == e->tokens[j]) ++j;
                if (j < x->w) continue;
                cands++;
                if (e->origin_pos != 0) continue;
                int32_t l = 0;
                while (l < e->len && l < n && q[l] == e->tokens[l] && (!mk || mk[l] == 0)) ++l;
                if (l < x->w) continue;
                if (l > bl || (l == bl && e->id < best)) { bl = l; best = e->id; }
            }
            if (best >= 0) {
                if (nh >= max_hits) return -1;
                orc_entry* e = &x->e[best];
                hit_req[nh] = r; hit_entry[nh] = e->id; hit_dst[nh] = 0; hit_len[nh] = bl; hit_delta[nh] = 0;
                nh++;
                for (int32_t z = 0; z < bl; ++z) { pl[z] = e->recompute[z] ? 2 : 1; cov++; rec += e->recompute[z]; }
            }
            req_hit_offsets[r + 1] = nh;
            req_covered[r] = cov; req_recompute[r] = rec; req_candidates[r] = cands;
            continue;
        }
        /* same-user session reuse ("all KV cache can be reused without restriction", R#33): the
           longest common prefix with the session's last request (its private entry), sensitive tokens
           included, is one hit at 0 if >= w tokens; cross-user hits then start after it */
        int64_t cursor = 0;
        if (sessions && sessions[r] >= 1) {
            for (int32_t i = 0; i < x->n_e; ++i) {
                orc_entry* e = &x->e[i];
                if (!e->live || e->owner != sessions[r]) continue;
                int32_t l = 0;
                while (l < e->len && l < n && q[l] == e->tokens[l]) ++l;
                if (l >= x->w) {
                    if (nh >= max_hits) return -1;
                    hit_req[nh] = r; hit_entry[nh] = e->id; hit_dst[nh] = 0; hit_len[nh] = l; hit_delta[nh] = 0;
                    nh++;
                    for (int32_t z = 0; z < l; ++z) { pl[z] = 1; cov++; }
                    cursor = l;
                }
                break;
            }
        }
        int64_t nc = 0, cap = 16;
        orc_cand* V = (orc_cand*)malloc(sizeof(orc_cand) * (size_t)cap);
        /* FixedChunk (Fig. 4-b): only chunk-aligned windows, only length-w entries (R#28) */
        for (int64_t k = 0; k + x->w <= n; k += fixed ? x->w : 1) {
            for (int32_t i = 0; i < x->n_e; ++i) {
                orc_entry* e = &x->e[i];
                if (!e->live || e->owner) continue;              /* private entries: their session only */
                int64_t j = 0;
                while (j < x->w && q[k + j] == e->tokens[j]) ++j;
                if (j < x->w) continue;
                cands++;
                if (fixed && e->len != x->w) continue;
                if (k + e->len > n) continue;
                while (j < e->len && q[k + j] == e->tokens[j]) ++j;
                if (j < e->len) continue;
                if (mk) {
                    int64_t z = 0;
                    while (z < e->len && mk[k + z] == 0) ++z;
                    if (z < e->len) continue;
                }
                if (nc == cap) { cap *= 2; V = (orc_cand*)realloc(V, sizeof(orc_cand) * (size_t)cap); }
                V[nc].k = (int32_t)k; V[nc].m = e->len; V[nc].id = e->id; nc++;
            }
        }
        qsort(V, (size_t)nc, sizeof(orc_cand), cand_cmp);
        for (int64_t c = 0; c < nc; ++c) {
            if (V[c].k < cursor) continue;
            if (nh >= max_hits) { free(V); return -1; }
            orc_entry* e = &x->e[V[c].id];
            hit_req[nh] = r; hit_entry[nh] = e->id; hit_dst[nh] = V[c].k; hit_len[nh] = e->len;
            hit_delta[nh] = V[c].k - e->origin_pos;        /* R#11: delta = dst - origin */
            nh++;
            for (int32_t z = 0; z < e->len; ++z) {
                pl[V[c].k + z] = e->recompute[z] ? 2 : 1;
                cov++; rec += e->recompute[z];
            }
            cursor = V[c].k + e->len;
        }
        req_hit_offsets[r + 1] = nh;
        req_covered[r] = cov; req_recompute[r] = rec; req_candidates[r] = cands;
        free(V);
    }
    if (!(flags & ORC_MATCH_NO_TOUCH))
        for (int32_t h = 0; h < nh; ++h) {
            orc_entry* e = &x->e[hit_entry[h]];
            if (e->last_used < t) e->last_used = t;
        }
    return nh;
}

/* ------------------------------------------------------------------------- */
/* snapshot accessors                                                          */
/* ------------------------------------------------------------------------- */
int32_t orc_num_ids(const orc_index* x) { return x->n_e; }
int64_t orc_live_tokens(const orc_index* x) { return x->live_tokens; }
int32_t orc_fifo_count(const orc_index* x) { return x->fifo_count; }

/* info[10] = {live, len, origin_pos, origin_call, origin_req, npages, 0,0,0,0};
 * hashes[3] = {prefix_hash, full_hash, last_used}; digest[32]; pages[npages]; tokens[len]; rec[len] */
int32_t orc_entry_get(const orc_index* x, int32_t id, int32_t* info, uint64_t* hashes, uint8_t* digest,
                      int32_t* pages, int32_t* toks, uint8_t* rec) {
    if (id < 0 || id >= x->n_e) return ORC_ERR_INVALID_ARG;
    const orc_entry* e = &x->e[id];
    info[0] = e->live; info[1] = e->len; info[2] = e->origin_pos; info[3] = e->origin_call;
    info[4] = e->origin_req; info[5] = e->npages; info[6] = e->pin; info[7] = e->owner;
    hashes[0] = e->prefix_hash; hashes[1] = e->full_hash; hashes[2] = e->last_used;
    if (digest) memcpy(digest, e->digest, 32);
    if (pages) memcpy(pages, e->pages, sizeof(int32_t) * (size_t)e->npages);
    if (toks) memcpy(toks, e->tokens, sizeof(int32_t) * (size_t)e->len);
    if (rec) memcpy(rec, e->recompute, (size_t)e->len);
    return ORC_OK;
}

/* free-page FIFO in pop order */
void orc_fifo_get(const orc_index* x, int32_t* out) {
    for (int32_t i = 0; i < x->fifo_count; ++i) out[i] = x->fifo[(x->fifo_head + i) % x->num_pages];
}

/*
 * NEXT-2: zero-copy page linking.  The paper's retriever "link[s] reusable segments without touching
 * the actual KV"; ordinary prefix reuse shares whole cached blocks.  A link is
 * possible only where a request block IS a stored page: reading R#31 links request r's block b
 * (positions [16b, 16b + 16)) to pool page pages(e)[j] iff one hit (e, dst, len, delta) of r has
 *   delta == 0, dst % 16 == 0, dst <= 16b, 16b + 16 <= dst + len   (then j = (16b - dst) / 16),
 * and all 16 positions have plan code 1 (reused, no recompute mark).  link[r * max_blocks + b] = page,
 * every other entry of the first ceil(n_r / 16) blocks = -1 (entries beyond are left as they are).
 * The hits are the ones orc_match returned for this index state.
 */
/* R#32: pin (delta > 0) or unpin (delta < 0) the entries owning the listed pool pages, once per listed
 * page (entries < 0 are skipped: a link table can be passed as is).  Every page must belong to a live
 * entry and no pin count may go negative; otherwise nothing changes and ORC_ERR_INVALID_ARG. */
int32_t orc_pin_pages(orc_index* x, const int32_t* pages, int64_t n, int32_t delta) {
    int32_t* owner = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n > 0 ? n : 1));
    int32_t rc = ORC_OK;
    for (int64_t q = 0; q < n && rc == ORC_OK; ++q) {
        owner[q] = -1;
        if (pages[q] < 0) continue;
        for (int32_t i = 0; i < x->n_e && owner[q] < 0; ++i) {
            if (!x->e[i].live) continue;
            for (int32_t j = 0; j < x->e[i].npages; ++j)
                if (x->e[i].pages[j] == pages[q]) { owner[q] = i; break; }
        }
        if (owner[q] < 0) rc = ORC_ERR_INVALID_ARG;
    }
    if (rc == ORC_OK && delta < 0) {            /* no count may go negative (counted over the whole list) */
        for (int64_t q = 0; q < n && rc == ORC_OK; ++q) {
            if (owner[q] < 0) continue;
            int64_t uses = 0;
            for (int64_t z = 0; z < n; ++z) uses += owner[z] == owner[q];
            if (x->e[owner[q]].pin + delta * uses < 0) rc = ORC_ERR_INVALID_ARG;
        }
    }
    if (rc == ORC_OK)
        for (int64_t q = 0; q < n; ++q) if (owner[q] >= 0) x->e[owner[q]].pin += delta;
    free(owner);
    return rc;
}

int32_t orc_entry_pin(const orc_index* x, int32_t id) { return (id >= 0 && id < x->n_e) ? x->e[id].pin : -1; }

int32_t orc_link_blocks(const orc_index* x, int32_t num_reqs, const int64_t* offsets, int32_t num_hits,
                        const int32_t* hit_req, const int32_t* hit_entry, const int32_t* hit_dst,
                        const int32_t* hit_len, const int32_t* hit_delta, const uint8_t* plan,
                        int32_t max_blocks, int32_t* link) {
    for (int32_t r = 0; r < num_reqs; ++r) {
        const int64_t nb = (offsets[r + 1] - offsets[r] + 15) / 16;
        if (nb > max_blocks) return ORC_ERR_INVALID_ARG;
        for (int64_t b = 0; b < nb; ++b) link[(int64_t)r * max_blocks + b] = -1;
    }
    for (int32_t h = 0; h < num_hits; ++h) {
        if (hit_entry[h] < 0 || hit_entry[h] >= x->n_e) return ORC_ERR_INVALID_ARG;
        if (hit_delta[h] != 0 || hit_dst[h] % 16 != 0) continue;
        const orc_entry* e = &x->e[hit_entry[h]];
        const int32_t r = hit_req[h];
        for (int32_t b = hit_dst[h] / 16; 16 * b + 16 <= hit_dst[h] + hit_len[h]; ++b) {
            int all_reused = 1;
            for (int32_t q = 16 * b; q < 16 * b + 16; ++q)
                if (plan[offsets[r] + q] != 1) all_reused = 0;
            if (all_reused) link[(int64_t)r * max_blocks + b] = e->pages[(16 * b - hit_dst[h]) / 16];
        }
    }
    return ORC_OK;
}

/* ------------------------------------------------------------------------- */
/* RoPE re-rotation of one stored K row (R#11-13; the paper never mentions RoPE) */
/* ------------------------------------------------------------------------- */
/* fp64 -> bf16 with one round-to-nearest-even (finite, normal-range inputs) */
static double round_bf16(double v) {
    if (v == 0.0 || !isfinite(v)) return v;
    int ex;
    double fr = frexp(v, &ex);              /* v = fr * 2^ex, 0.5 <= |fr| < 1 */
    double sc = ldexp(fr, 8);               /* 8 significant bits: |sc| in [128, 256) */
    double rn = nearbyint(sc);              /* default rounding mode: ties to even */
    return ldexp(rn, ex - 8);
}

/*
 * x: one token's K row for one layer, H heads x d dims (values of the storage dtype, widened).
 * NeoX style (R#12): pairs (i, i+d/2), theta_i = base^(-2i/d); GPT-J style: pairs (2i, 2i+1).
 * For delta == 0 the row is copied bit-for-bit; otherwise, in fp64,
 *   a = delta*theta_i, x' = x cos a - y sin a, y' = y cos a + x sin a,
 * and each output is rounded once to the storage dtype (out_bf16 = 1: bf16 RNE; 0: fp32 RNE).
 */
void orc_rerotate_row(const float* xin, int32_t H, int32_t d, int32_t gptj, double theta_base,
                      int64_t delta, int32_t out_bf16, float* out) {
    int32_t n = H * d;
    if (delta == 0) { memcpy(out, xin, sizeof(float) * (size_t)n); return; }
    for (int32_t h = 0; h < H; ++h) {
        const float* xh = xin + h * d;
        float* oh = out + h * d;
        for (int32_t i = 0; i < d / 2; ++i) {
            int32_t ia = gptj ? 2 * i : i;
            int32_t ib = gptj ? 2 * i + 1 : i + d / 2;
            double th = pow(theta_base, -2.0 * (double)i / (double)d);
            double a = (double)delta * th;
            double c = cos(a), s = sin(a);
            double xv = (double)xh[ia], yv = (double)xh[ib];
            double xo = xv * c - yv * s;
            double yo = yv * c + xv * s;
            if (out_bf16) { oh[ia] = (float)round_bf16(xo); oh[ib] = (float)round_bf16(yo); }
            else { oh[ia] = (float)xo; oh[ib] = (float)yo; }
        }
    }
}

/* ------------------------------------------------------------------------- */
/* recompute score + top-k (C1 Step 3)                             */
/* ------------------------------------------------------------------------- */
typedef struct { int64_t s; int32_t i; } orc_sc;

static int sc_cmp(const void* a, const void* b) {        /* score desc, index asc (R#16) */
    const orc_sc* x = (const orc_sc*)a; const orc_sc* y = (const orc_sc*)b;
    if (x->s != y->s) return x->s > y->s ? -1 : 1;
    return x->i < y->i ? -1 : (x->i > y->i);
}

/* R#17: q(x) = trunc(x * 2^40) as int64 */
static int64_t fixq(float x) { return (int64_t)((double)x * 1099511627776.0); }

/*
 * A: fp32 [heads][n][n] row-major attention of the final layer, heads summed (R#18).
 * Span [l, r] (0-based, inclusive; the selected substring [l*, r*] of Step 2).  For each i in [l, r]:
 *   inter(i) = sum_h sum_{j < l} q(A_h[i][j])       (attention to tokens before l*)
 *   intra(i) = sum_h sum_{l <= j <= i} q(A_h[i][j]) (attention within [l*, i],   P:L643)
 *   score(i) = inter(i) - intra(i)                   ("ranked by their inter-intra difference")
 * k = ceil(rho_num * m / rho_den) (R#15); the first k of the order (score desc, i asc) get bit 1.
 * scores[t] and bit t refer to position l + t.
 */
int32_t orc_score(const float* A, int64_t n, int32_t heads, int32_t l, int32_t r,
                  int32_t rho_num, int32_t rho_den, int64_t* scores, uint32_t* bits) {
    if (l < 0 || r < l || r >= n || rho_den <= 0 || rho_num < 0 || rho_num > rho_den) return ORC_ERR_INVALID_ARG;
    int32_t m = r - l + 1;
    orc_sc* v = (orc_sc*)malloc(sizeof(orc_sc) * (size_t)m);
    for (int32_t i = l; i <= r; ++i) {
        int64_t inter = 0, intra = 0;
        for (int32_t h = 0; h < heads; ++h) {
            const float* row = A + ((int64_t)h * n + i) * n;
            for (int32_t j = 0; j < l; ++j) inter += fixq(row[j]);
            for (int32_t j = l; j <= i; ++j) intra += fixq(row[j]);
        }
        scores[i - l] = inter - intra;
        v[i - l].s = inter - intra; v[i - l].i = i - l;
    }
    qsort(v, (size_t)m, sizeof(orc_sc), sc_cmp);
    int64_t k = ((int64_t)rho_num * m + rho_den - 1) / rho_den;
    for (int32_t w = 0; w < (m + 31) / 32; ++w) bits[w] = 0;
    for (int64_t c = 0; c < k; ++c) bits[v[c].i / 32] |= 1u << (v[c].i % 32);
    free(v);
    return ORC_OK;
}

/*
 * NEXT-4: CacheBlend's KV-deviation selector ("compares the first-layer KV of a chunk in its
 * original context with that from a full recomputation in the new context, then recomputes the top
 * 15% of tokens with the largest deviation").  The paper names no norm; reading R#30 takes the L1
 * distance over K and V in the 2^-24 fixed point q24(x) = trunc(x * 2^24):
 *   dev(t) = sum_{c < width} |q24(Kr[t][c]) - q24(Kf[t][c])| + |q24(Vr[t][c]) - q24(Vf[t][c])|
 * Rows are dense fp32 [m][width] (width = H * d; bf16 values widen to fp32 exactly).  Kr/Vr: the
 * reused (re-rotated) first-layer KV; Kf/Vf: the freshly recomputed one.  Selection as orc_score:
 * the first ceil(rho_num * m / rho_den) tokens of (dev desc, t asc) get bit 1.
 */
static int64_t fixq24(float x) { return (int64_t)((double)x * 16777216.0); }
static int64_t absdiff(int64_t a, int64_t b) { return a > b ? a - b : b - a; }

int32_t orc_kv_deviation(const float* Kr, const float* Vr, const float* Kf, const float* Vf, int64_t m,
                         int32_t width, int32_t rho_num, int32_t rho_den, int64_t* dev, uint32_t* bits) {
    if (m < 1 || width < 1 || rho_den <= 0 || rho_num < 0 || rho_num > rho_den) return ORC_ERR_INVALID_ARG;
    orc_sc* v = (orc_sc*)malloc(sizeof(orc_sc) * (size_t)m);
    for (int64_t t = 0; t < m; ++t) {
        int64_t s = 0;
        for (int32_t c = 0; c < width; ++c) {
            const int64_t o = t * width + c;
            s += absdiff(fixq24(Kr[o]), fixq24(Kf[o]));
            s += absdiff(fixq24(Vr[o]), fixq24(Vf[o]));
        }
        dev[t] = s;
        v[t].s = s; v[t].i = (int32_t)t;
    }
    qsort(v, (size_t)m, sizeof(orc_sc), sc_cmp);
    int64_t k = ((int64_t)rho_num * m + rho_den - 1) / rho_den;
    for (int64_t w = 0; w < (m + 31) / 32; ++w) bits[w] = 0;
    for (int64_t c = 0; c < k; ++c) bits[v[c].i / 32] |= 1u << (v[c].i % 32);
    free(v);
    return ORC_OK;
}

/* Re-rotate `nrows` consecutive rows (plain loop over orc_rerotate_row). */
void orc_rerotate_rows(const float* xin, int64_t nrows, int32_t H, int32_t d, int32_t gptj, double theta_base,
                       int64_t delta, int32_t out_bf16, float* out) {
    for (int64_t r = 0; r < nrows; ++r)
        orc_rerotate_row(xin + r * (int64_t)H * d, H, d, gptj, theta_base, delta, out_bf16, out + r * (int64_t)H * d);
}

/* ------------------------------------------------------------------------- */
/* C1 Steps 1-2: summed-area table + optimal substring per coarse segment     */
/* (SPEC annotator.select_reusable S:L169-177)                    */
/* ------------------------------------------------------------------------- */
/*
 * A: fp32 [heads][n][n], causal final-layer attention; values are summed over heads in the
 * 2^-40 fixed point of R#17, so every sum below is an exact integer (ties resolve identically).
 * Step 1: T[i][j] = a[i][j] + T[i-1][j] + T[i][j-1] - T[i-1][j-1], 1-based, zero border.
 * rect(x1,x2,y1,y2) = T[x2][y2] - T[x1-1][y2] - T[x2][y1-1] + T[x1-1][y1-1]
 * Coarse segments: maximal runs of mask-0 positions [a, b] (1-based).
 * Step 2: for every substring [l, r] of the segment with r - l + 1 >= min_len,
 *   diff = IntraAttn(l, r) - InterAttn(l, r) = rect(l, r, l, r) - rect(l, r, 1, l - 1)
 * choose max diff; ties -> longer, then leftmost; store only if diff > 0.
 * Outputs (0-based, inclusive) per coarse segment s: out_l[s], out_r[s] (-1 if none), out_diff[s];
 * returns the number of coarse segments (<= max_segments) or -1 if there are more.
 */
int32_t orc_annotate(const float* A, int64_t n, int32_t heads, const uint8_t* mask, int32_t min_len,
                     int32_t max_segments, int32_t* out_l, int32_t* out_r, int64_t* out_diff) {
    int64_t* T = (int64_t*)calloc((size_t)(n + 1) * (size_t)(n + 1), sizeof(int64_t));
#define TT(i, j) T[(int64_t)(i) * (n + 1) + (j)]
    for (int64_t i = 1; i <= n; ++i)
        for (int64_t j = 1; j <= n; ++j) {
            int64_t a = 0;
            for (int32_t h = 0; h < heads; ++h) a += fixq(A[((int64_t)h * n + (i - 1)) * n + (j - 1)]);
            TT(i, j) = a + TT(i - 1, j) + TT(i, j - 1) - TT(i - 1, j - 1);
        }
#define RECT(x1, x2, y1, y2) (TT(x2, y2) - TT((x1) - 1, y2) - TT(x2, (y1) - 1) + TT((x1) - 1, (y1) - 1))
    int32_t nseg = 0;
    int64_t i = 1;
    while (i <= n) {
        if (mask[i - 1]) { ++i; continue; }
        int64_t a = i;
        while (i <= n && !mask[i - 1]) ++i;
        int64_t b = i - 1;
        if (nseg >= max_segments) { free(T); return -1; }
        int32_t bl = -1, br = -1;
        int64_t bd = 0;
        for (int64_t l = a; l <= b; ++l)
            for (int64_t r = l + min_len - 1; r <= b; ++r) {
                const int64_t intra = RECT(l, r, l, r);
                const int64_t inter = l > 1 ? RECT(l, r, 1, l - 1) : 0;
                const int64_t diff = intra - inter;
                const int64_t len = r - l + 1, blen = br - bl + 1;
                if (bl < 0 || diff > bd || (diff == bd && (len > blen || (len == blen && l - 1 < bl)))) {
                    bd = diff; bl = (int32_t)(l - 1); br = (int32_t)(r - 1);
                }
            }
        if (bl >= 0 && bd <= 0) { bl = -1; br = -1; }
        out_l[nseg] = bl; out_r[nseg] = br; out_diff[nseg] = bl >= 0 ? bd : 0;
        ++nseg;
    }
#undef RECT
#undef TT
    free(T);
    return nseg;
}

/* Step 1 alone, for pins: the SAT of the fixed-point matrix (n+1)^2 with zero border. */
void orc_sat(const float* A, int64_t n, int32_t heads, int64_t* T) {
    for (int64_t j = 0; j <= n; ++j) T[j] = 0;
    for (int64_t i = 1; i <= n; ++i) {
        T[i * (n + 1)] = 0;
        for (int64_t j = 1; j <= n; ++j) {
            int64_t a = 0;
            for (int32_t h = 0; h < heads; ++h) a += fixq(A[((int64_t)h * n + (i - 1)) * n + (j - 1)]);
            T[i * (n + 1) + j] = a + T[(i - 1) * (n + 1) + j] + T[i * (n + 1) + j - 1] - T[(i - 1) * (n + 1) + j - 1];
        }
    }
}
