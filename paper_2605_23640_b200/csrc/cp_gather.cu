// cp_gather.cu -- N2 fused gather + RoPE re-rotation (placement: PAPER.md L518, L726-727, L781;
// RoPE: DESIGN.md readings R#11-14, the paper never mentions position handling).
//
// Work list: a hit list (req, slot, dst, len, delta) is cut into chunks of CP_GATHER_CHUNK tokens by
// k_rows_prep (block 0: scan + chunk list; every block: per-hit cos/sin table, angles in fp64).
// k_rows: persistent grid, static round-robin over items (chunk, layer).  Per item, 32 threads
// resolve the token rows (pool page via the entry's page list, destination block via the block
// table, plan code), then the CTA streams the rows with 128-bit loads (ld.global.nc, L1 no-allocate)
// and 128-bit streaming stores.  A "task" moves one 16-B vector of K at element i, its NeoX partner
// at i + d/2, and the same two vectors of V; K is rotated in fp32 registers:
//     K'[i] = K[i] c - K[i+d/2] s,   K'[i+d/2] = K[i+d/2] c + K[i] s,   (c, s) = (cos, sin)(delta theta_i)
// V and delta == 0 rows are bit copies; recompute rows become +0.0 (zero placeholders).
// dir 1 (insert copy-in) moves writer rows into pool pages unrotated with the same engine.
#include "cp_internal.cuh"
#include <algorithm>
#include <cstdlib>
#include <cstring>

namespace {

constexpr int kRowsThreads = 256;
constexpr int kPrepThreads = 512;
constexpr int kCodeLinked = 3;       // row-table code of a token in a linked block (CP_SKIP_LINKED): no load, no store
constexpr int kMaxRects = 4;         // rectangles per launch (a balanced-layout rank holds at most 3)

struct RowsArgs {
    DevHeader* hdr;
    int dir;
    const int32_t* count;
    const int32_t *l_req, *l_slot, *l_dst, *l_len, *l_delta;
    int64_t list_cap;
    const int64_t* req_off; const uint8_t* plan;
    const int32_t* block_tables; int32_t max_blocks;
    char* paged_k[CP_MAX_LAYERS]; char* paged_v[CP_MAX_LAYERS];
    char* pool_k; char* pool_v; int64_t P;
    const int32_t* slot_pages; int32_t MP;
    int32_t L, H, d; double theta; int32_t flags; int32_t gptj;
    int32_t LG;                      // layers per work item (small rows: several layers share one row lookup)
    int32_t* chunk_hit; int32_t* chunk_t0; int64_t CH;
    int32_t* hit_coff;                                 // [hits] first chunk of each hit (k_rows_prep)
    long long* row_src; long long* row_dst;
    float2* hit_cs; int64_t cs_hits;
    // several (layer, head) rectangles of one rank in one launch (cp_gather_rerotate_rects): rectangle r
    // covers items [rect[r].item0, rect[r + 1].item0), its layers are paged_k/v[layer0 + l]; nrect == 1:
    // the index's own rectangle (L, H, LG, pool_k/v above)
    int32_t nrect;
    struct Rect { char* pool_k; char* pool_v; int64_t item0; int32_t L, H, LG, layer0; } rect[kMaxRects + 1];
};

// k_rows_prep (one block): per-hit first chunk = exclusive scan of ceil(len/32) over the hit list, a
// thread owning a contiguous run of hits (one block scan; the chunk list itself is written by the
// whole grid in k_rows_prep2 -- one SM writing ~12K scattered entries took 17-27 us)
__global__ void __launch_bounds__(kPrepThreads) k_rows_prep(RowsArgs a) {
    __shared__ int s_scan[kPrepThreads / 32 + 1];
    if (cp_err_set(a.hdr)) return;
    const int nh = *a.count;
    if (nh > a.list_cap || nh > a.cs_hits) { if (threadIdx.x == 0) cp_raise(a.hdr, CP_ERR_CAPACITY); return; }
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int c = (nh + kPrepThreads - 1) / kPrepThreads, h0 = min(nh, tid * c), h1 = min(nh, h0 + c);
    int loc = 0;
    for (int h = h0; h < h1; ++h) loc += (a.l_len[h] + CP_GATHER_CHUNK - 1) / CP_GATHER_CHUNK;
    int inc = loc;
    for (int o = 1; o < 32; o <<= 1) { const int y = __shfl_up_sync(0xffffffffu, inc, o); if (lane >= o) inc += y; }
    if (lane == 31) s_scan[wid] = inc;
    __syncthreads();
    if (wid == 0) {
        int x = lane < kPrepThreads / 32 ? s_scan[lane] : 0, xi = x;
        for (int o = 1; o < 32; o <<= 1) { const int y = __shfl_up_sync(0xffffffffu, xi, o); if (lane >= o) xi += y; }
        if (lane < kPrepThreads / 32) s_scan[lane] = xi - x;
        if (lane == 31) s_scan[kPrepThreads / 32] = xi;
    }
    __syncthreads();
    int run = s_scan[wid] + inc - loc;
    for (int h = h0; h < h1; ++h) { a.hit_coff[h] = run; run += (a.l_len[h] + CP_GATHER_CHUNK - 1) / CP_GATHER_CHUNK; }
    if (tid == 0) {
        const int tot = s_scan[kPrepThreads / 32];
        if (tot > a.CH) { cp_raise(a.hdr, CP_ERR_CAPACITY); a.hdr->n_chunks = 0; }
        else a.hdr->n_chunks = tot;
        a.hdr->gather_next = 0;
    }
}

// k_rows_prep2 (all blocks): per-hit cos/sin (angles in fp64, R#13) and the per-token row table
// (source / destination row offsets + plan code) so the copy kernels resolve a token with one load
__global__ void __launch_bounds__(kPrepThreads) k_rows_prep2(RowsArgs a) {
    if (cp_err_set(a.hdr)) return;
    const int nh = *a.count;
    const int half = a.d / 2;
    const int64_t gt = blockIdx.x * (int64_t)blockDim.x + threadIdx.x, nt = (int64_t)gridDim.x * blockDim.x;
    if (a.dir == 0) {
        const int64_t npairs = (int64_t)nh * half;
        for (int64_t q = gt; q < npairs; q += nt) {
            const int hh = (int)(q / half), i = (int)(q % half);
            const int delta = a.l_delta[hh];
            if (delta == 0) continue;
            const double th = pow(a.theta, -2.0 * (double)i / (double)a.d);
            double sn, cs;
            sincos((double)delta * th, &sn, &cs);
            a.hit_cs[q] = make_float2((float)cs, (float)sn);
        }
    }
    const int64_t ntok = (int64_t)a.hdr->n_chunks * CP_GATHER_CHUNK;
    const int lane = threadIdx.x & 31;
    // the 32 lanes of a warp take the 32 tokens of one chunk (nt is a multiple of 32): lane 0 finds the
    // chunk's hit (largest h with hit_coff[h] <= c) and writes the chunk-list entry the copy kernel reads
    for (int64_t qb = gt - lane; qb < ntok; qb += nt) {
        const int c = (int)(qb / CP_GATHER_CHUNK), i = lane;
        int hh = 0;
        if (lane == 0) {
            int lo = 0, hi = nh - 1;
            while (lo < hi) { const int mid = (lo + hi + 1) >> 1; if (a.hit_coff[mid] <= c) lo = mid; else hi = mid - 1; }
            hh = lo;
            a.chunk_hit[c] = hh;
            a.chunk_t0[c] = (c - a.hit_coff[hh]) * CP_GATHER_CHUNK;
        }
        hh = __shfl_sync(0xffffffffu, hh, 0);
        const int64_t q = qb + lane;
        const int t = (c - a.hit_coff[hh]) * CP_GATHER_CHUNK + i;
        if (t >= a.l_len[hh]) continue;
        const int r = a.l_req[hh], k = a.l_dst[hh], slot = a.l_slot[hh];
        const int pos = k + t;                                              // position in the request
        if ((pos >> 4) >= a.max_blocks) { cp_raise(a.hdr, CP_ERR_INVALID_ARG); continue; }   // table too narrow:
                                                                           // k_rows then writes nothing
        const int page = a.slot_pages[(int64_t)slot * a.MP + (t >> 4)];
        const int blk = a.block_tables[(int64_t)r * a.max_blocks + (pos >> 4)];
        // token-row INDICES (not element offsets): the table is independent of the shard geometry, so
        // the pool views of one rank reuse it (CP_REUSE_WORKLIST); the copy kernels scale by H*d
        const long long pool_row = (long long)page * CP_BLOCK + (t & 15);
        const long long paged_row = (long long)blk * CP_BLOCK + (pos & 15);
        long long code = a.dir == 0 ? (long long)a.plan[a.req_off[r] + pos] : (long long)CP_PLAN_REUSED;
        if (a.dir == 0 && (a.flags & CP_SKIP_RECOMPUTE) && code == CP_PLAN_RECOMPUTE) code = kCodeLinked;   // untouched
        if (a.dir == 0 && (a.flags & CP_SKIP_LINKED) && code == CP_PLAN_REUSED && a.l_delta[hh] == 0 && (k & 15) == 0) {
            const int b0 = pos & ~15;                                       // >= k: k is page aligned
            if (b0 + 16 <= k + a.l_len[hh]) {                               // the block lies inside the hit
                const uint8_t* pl = a.plan + a.req_off[r] + b0;
                bool all = true;
#pragma unroll
                for (int i = 0; i < 16; ++i) all &= pl[i] == CP_PLAN_REUSED;
                if (all) code = kCodeLinked;                                // R#31: this block IS pool page t>>4
            }
        }
        a.row_src[q] = a.dir == 0 ? pool_row : paged_row;
        a.row_dst[q] = (a.dir == 0 ? paged_row : pool_row) | (code << 62);
    }
}

template <typename T> struct Vec;
template <> struct Vec<float> { static constexpr int N = 4; };
template <> struct Vec<__nv_bfloat16> { static constexpr int N = 8; };

__device__ __forceinline__ uint4 ld_stream(const void* p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
    return r;
}
__device__ __forceinline__ void st_stream(void* p, const uint4& v) {
    asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" :: "l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}

__device__ __forceinline__ void unpack(const uint4& v, float* f, float) {
    f[0] = __uint_as_float(v.x); f[1] = __uint_as_float(v.y); f[2] = __uint_as_float(v.z); f[3] = __uint_as_float(v.w);
}
__device__ __forceinline__ uint4 pack(const float* f, float) {
    return make_uint4(__float_as_uint(f[0]), __float_as_uint(f[1]), __float_as_uint(f[2]), __float_as_uint(f[3]));
}
__device__ __forceinline__ void unpack(const uint4& v, float* f, __nv_bfloat16) {
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) { f[2 * i] = __uint_as_float(w[i] << 16); f[2 * i + 1] = __uint_as_float(w[i] & 0xffff0000u); }
}
__device__ __forceinline__ uint4 pack(const float* f, __nv_bfloat16) {
    uint32_t w[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const __nv_bfloat162 b = __floats2bfloat162_rn(f[2 * i], f[2 * i + 1]);   // RNE
        w[i] = *reinterpret_cast<const uint32_t*>(&b);
    }
    return make_uint4(w[0], w[1], w[2], w[3]);
}

template <typename T, bool GPTJ, bool CREG, int UNROLL, int MINB, bool ML, bool DYN>
__global__ void __launch_bounds__(kRowsThreads, MINB) k_rows(RowsArgs a) {
    constexpr int VEC = Vec<T>::N;
    __shared__ int64_t s_src[CP_GATHER_CHUNK], s_dst[CP_GATHER_CHUNK];
    __shared__ int s_code[CP_GATHER_CHUNK];
    __shared__ float2 s_cs[256];
    __shared__ long long s_item;
    if (cp_err_set(a.hdr)) return;
    const int nchunks = a.hdr->n_chunks;
    const int tid = threadIdx.x;
    const int half = a.d / 2;
    const int hv = half / VEC;                          // vectors per half head
    const bool zero_rec = (a.flags & CP_ZERO_RECOMPUTE) != 0;
    // the rectangle's geometry: fixed for nrect == 1, switched per item otherwise (items of one
    // rectangle are contiguous, so a CTA switches rarely)
    int cur = -1, L = 0, LG = 1, layer0 = 0, ngroups = 1, rowE = 0, tpr = 1, A = kRowsThreads;
    int64_t item0 = 0, pool_layer = 0;
    const char* poolk = nullptr; const char* poolv = nullptr;
    const int64_t items = a.nrect > 1 ? a.rect[a.nrect].item0 * nchunks
                                      : (int64_t)nchunks * (ML ? (a.L + a.LG - 1) / a.LG : a.L);
    // CREG (tpr <= block): the block's first A = floor(256 / tpr) * tpr threads work with a task stride
    // of A, so a thread's column task, and so its cos/sin, is fixed; the other 256 - A threads only
    // stage the row table (A = 256 when tpr divides the block; 240 for the 3- and 6-head rectangles of
    // the balanced layout, whose per-task column arithmetic cost ~10% per unit without this)
    constexpr bool creg = CREG;
    auto task_geom = [&](int j, int& lo, int& hi, int& i0) {
        if (!GPTJ) { const int head = j / hv, sub = j - head * hv; lo = head * a.d + sub * VEC; hi = lo + half; i0 = sub * VEC; }
        else { lo = j * 2 * VEC; hi = lo + VEC; i0 = (lo % a.d) / 2; }
    };
    int lo_t = 0, hi_t = 0, i0_t = 0;
    auto set_rect = [&](int r) {
        cur = r;
        if (a.nrect > 1) {
            L = a.rect[r].L; LG = ML ? a.rect[r].LG : 1; layer0 = a.rect[r].layer0; rowE = a.rect[r].H * a.d;
            poolk = a.rect[r].pool_k; poolv = a.rect[r].pool_v; item0 = a.rect[r].item0 * nchunks;
        } else {
            L = a.L; LG = ML ? a.LG : 1; layer0 = 0; rowE = a.H * a.d; poolk = a.pool_k; poolv = a.pool_v; item0 = 0;
        }
        ngroups = (L + LG - 1) / LG;
        tpr = rowE / (2 * VEC);                                         // tasks per token row
        A = creg ? (kRowsThreads / tpr) * tpr : kRowsThreads;
        pool_layer = a.P * CP_BLOCK * (int64_t)rowE;
        task_geom(tid % tpr, lo_t, hi_t, i0_t);
    };
    // DYN: items are taken from a device counter (one atomic per item and CTA), so CTAs that drew
    // short items (hit tails, zero placeholders) take more -- no static round-robin tail imbalance
    int64_t item = blockIdx.x;
    if (DYN) {
        if (tid == 0) s_item = (long long)atomicAdd(&a.hdr->gather_next, 1ULL);
        __syncthreads();
        item = s_item;
    }
    while (item < items) {
        {
            int r = 0;
            if (a.nrect > 1) while (r + 1 < a.nrect && item >= a.rect[r + 1].item0 * nchunks) ++r;
            if (r != cur) set_rect(r);
        }
        const int li = (int)(item - item0);
        const int c = li / ngroups, lg = li - c * ngroups;
        const int l0 = lg * LG;
        const int nl = ML ? min(LG, L - l0) : 1;            // compile-time 1 on the single-layer path
        const int hh = a.chunk_hit[c], t0 = a.chunk_t0[c];
        const int len = a.l_len[hh];
        const int ntok = min(CP_GATHER_CHUNK, len - t0);
        const int delta = a.dir == 0 ? a.l_delta[hh] : 0;
        if (tid < ntok) {
            const int64_t q = (int64_t)c * CP_GATHER_CHUNK + tid;
            const long long dw = a.row_dst[q];
            s_src[tid] = a.row_src[q] * rowE;
            s_dst[tid] = (dw & ((1LL << 62) - 1)) * rowE;
            s_code[tid] = (int)((unsigned long long)dw >> 62);
        }
        float2 csr[VEC];
        if (delta != 0) {
            const float2* tab = a.hit_cs + (int64_t)hh * half;
            if (creg) {
#pragma unroll
                for (int e = 0; e < VEC; ++e) csr[e] = tab[i0_t + e];
            } else {
                for (int i = tid; i < half; i += kRowsThreads) s_cs[i] = tab[i];
            }
        }
        __syncthreads();
        // task = ((token g * nl) + layer ll) * tpr + column j  -> j = tid % tpr when tpr | block
        const int ntask = ntok * nl * tpr;
        for (int base = 0; base < ntask; base += A * UNROLL) {
            uint4 klo[UNROLL], khi[UNROLL], vlo[UNROLL], vhi[UNROLL];
            int gl[UNROLL], code[UNROLL];
#pragma unroll
            for (int u = 0; u < UNROLL; ++u) {
                const int task = base + u * A + tid;
                code[u] = -1;
                if (tid < A && task < ntask) {
                    const int row = task / tpr;                 // (g, ll) flattened
                    const int g = (ML && nl > 1) ? row / nl : row, ll = row - g * nl;
                    int lo = lo_t, hi = hi_t, i0 = i0_t;
                    if (!creg) task_geom(task - row * tpr, lo, hi, i0);
                    gl[u] = creg ? row : task;
                    code[u] = s_code[g] == kCodeLinked ? -1 : s_code[g];
                    if (code[u] >= 0 && !(code[u] == CP_PLAN_RECOMPUTE && zero_rec)) {
                        const int l = l0 + ll;
                        const T* srcK = (const T*)(a.dir == 0 ? poolk + l * pool_layer * sizeof(T) : a.paged_k[layer0 + l]);
                        const T* srcV = (const T*)(a.dir == 0 ? poolv + l * pool_layer * sizeof(T) : a.paged_v[layer0 + l]);
                        const int64_t so = s_src[g];
                        klo[u] = ld_stream(srcK + so + lo); khi[u] = ld_stream(srcK + so + hi);
                        vlo[u] = ld_stream(srcV + so + lo); vhi[u] = ld_stream(srcV + so + hi);
                    }
                }
            }
#pragma unroll
            for (int u = 0; u < UNROLL; ++u) {
                if (code[u] < 0) continue;
                int lo = lo_t, hi = hi_t, i0 = i0_t, row = gl[u];
                if (!creg) { row = gl[u] / tpr; task_geom(gl[u] - row * tpr, lo, hi, i0); }
                const int g = (ML && nl > 1) ? row / nl : row, l = l0 + (row - g * nl);
                T* dstK = (T*)(a.dir == 0 ? a.paged_k[layer0 + l] : poolk + l * pool_layer * sizeof(T));
                T* dstV = (T*)(a.dir == 0 ? a.paged_v[layer0 + l] : poolv + l * pool_layer * sizeof(T));
                const int64_t dof = s_dst[g];
                T* dk = dstK + dof;
                T* dv = dstV + dof;
                if (code[u] == CP_PLAN_RECOMPUTE && zero_rec) {
                    const uint4 z = make_uint4(0, 0, 0, 0);
                    st_stream(dk + lo, z); st_stream(dk + hi, z); st_stream(dv + lo, z); st_stream(dv + hi, z);
                    continue;
                }
                if (delta != 0) {
                    float x[VEC], y[VEC];
                    unpack(klo[u], x, T()); unpack(khi[u], y, T());
#pragma unroll
                    for (int e = 0; e < VEC; ++e) {
                        // NeoX: pair (x[e], y[e]) uses theta_{i0+e}; GPT-J: pairs inside x and inside y
                        if (!GPTJ) {
                            const float2 cs = creg ? csr[e] : s_cs[i0 + e];
                            const float xo = fmaf(x[e], cs.x, -y[e] * cs.y);
                            const float yo = fmaf(y[e], cs.x, x[e] * cs.y);
                            x[e] = xo; y[e] = yo;
                        } else if ((e & 1) == 0) {
                            const float2 c0 = creg ? csr[e / 2] : s_cs[i0 + e / 2];
                            const float2 c1 = creg ? csr[VEC / 2 + e / 2] : s_cs[i0 + VEC / 2 + e / 2];
                            const float x0 = fmaf(x[e], c0.x, -x[e + 1] * c0.y), x1 = fmaf(x[e + 1], c0.x, x[e] * c0.y);
                            const float y0 = fmaf(y[e], c1.x, -y[e + 1] * c1.y), y1 = fmaf(y[e + 1], c1.x, y[e] * c1.y);
                            x[e] = x0; x[e + 1] = x1; y[e] = y0; y[e + 1] = y1;
                        }
                    }
                    klo[u] = pack(x, T()); khi[u] = pack(y, T());
                }
                st_stream(dk + lo, klo[u]); st_stream(dk + hi, khi[u]);
                st_stream(dv + lo, vlo[u]); st_stream(dv + hi, vhi[u]);
            }
        }
        if (DYN) {
            if (tid == 0) s_item = (long long)atomicAdd(&a.hdr->gather_next, 1ULL);
            __syncthreads();
            item = s_item;
        } else {
            item += gridDim.x;
        }
        __syncthreads();
    }
}

// ============================================================================================
// TMA bulk-copy variant (cp.async.bulk + mbarrier): opt-in only (CP_GATHER_VARIANT=4), not the default.
//   warp 0      : producer -- resolves TOK token rows of the next unit (pool page / block table /
//                 plan code) and bulk-loads the K and V rows (2 KiB each for the 8B shape) into an
//                 NST-stage shared-memory ring, completing an mbarrier transaction count
//   warps 1..4  : consumers -- wait for the stage, rotate the K rows in shared memory (fp32 math,
//                 cos/sin in registers), fence.proxy.async, named barrier
//   warp 1 lane0: storer -- bulk-stores every row of the stage to its destination (zero rows come
//                 from a shared zero row), commit_group, wait_group.read -> frees the stage
// No data passes through registers except the K rows being rotated.
// ============================================================================================
constexpr int kTmaTok = 8;                 // tokens per stage
constexpr int kTmaCons = 4;                // consumer warps
constexpr int kPend = 3;                   // bulk-store groups kept in flight by the storer
constexpr int kTmaThreads = 32 * (1 + kTmaCons);

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t cnt) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(b)), "r"(cnt) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WAIT_%=;\n}\n" :: "r"(smem_u32(b)), "r"(parity) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst_smem, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 :: "r"(smem_u32(dst_smem)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src_smem, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                 :: "l"(dst), "r"(smem_u32(src_smem)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N> __device__ __forceinline__ void bulk_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read %0;" :: "n"(N) : "memory");
}
template <int N> __device__ __forceinline__ void bulk_wait_all() {
    asm volatile("cp.async.bulk.wait_group %0;" :: "n"(N) : "memory");
}
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void cons_bar() { asm volatile("bar.sync 1, %0;" :: "n"(32 * kTmaCons) : "memory"); }

struct TmaStageMeta {
    int64_t dst[kTmaTok];
    int code[kTmaTok];
    int ntok, hit, layer, delta;
};

template <typename T, bool GPTJ>
__global__ void __launch_bounds__(kTmaThreads, 1) k_rows_tma(RowsArgs a, int nst) {
    constexpr int VEC = Vec<T>::N;
    extern __shared__ __align__(128) unsigned char smx[];
    const int rowE = a.H * a.d;
    const int rowB = rowE * (int)sizeof(T);
    const int stageB = kTmaTok * 2 * rowB;
    unsigned char* ring = smx;                                            // nst * stageB
    unsigned char* zrow = smx + (size_t)nst * stageB;                     // rowB zeros
    TmaStageMeta* meta = (TmaStageMeta*)(zrow + rowB);                    // nst
    uint64_t* full = (uint64_t*)(meta + nst);                             // nst
    uint64_t* empty = full + nst;                                         // nst
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (cp_err_set(a.hdr)) return;
    const int nchunks = a.hdr->n_chunks;
    const int64_t items = (int64_t)nchunks * a.L;
    const int64_t pool_layer = a.P * CP_BLOCK * (int64_t)rowE;
    for (int i = tid; i < rowB / 16; i += blockDim.x) reinterpret_cast<uint4*>(zrow)[i] = make_uint4(0, 0, 0, 0);
    if (tid == 0) {
        for (int s = 0; s < nst; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    fence_async_smem();
    __syncthreads();
    const bool zero_rec = (a.flags & CP_ZERO_RECOMPUTE) != 0;
    const int half = a.d / 2;
    const int hv = half / VEC;
    const int tpr = rowE / (2 * VEC);

    if (warp == 0) {
        // ---------------- producer: one coalesced row-table load per item, then the stages
        int it = 0;
        for (int64_t item = blockIdx.x; item < items; item += gridDim.x) {
            const int c = (int)(item / a.L), l = (int)(item % a.L);
            const int hh = a.chunk_hit[c], t0 = a.chunk_t0[c];
            const int ntok_item = min(CP_GATHER_CHUNK, a.l_len[hh] - t0);
            const int delta = a.dir == 0 ? a.l_delta[hh] : 0;
            const char* srcK = a.dir == 0 ? a.pool_k + l * pool_layer * sizeof(T) : a.paged_k[l];
            const char* srcV = a.dir == 0 ? a.pool_v + l * pool_layer * sizeof(T) : a.paged_v[l];
            long long my_src = 0, my_dst = 0;
            if (lane < ntok_item) {
                my_src = a.row_src[(int64_t)c * CP_GATHER_CHUNK + lane] * rowE;
                const long long dw = a.row_dst[(int64_t)c * CP_GATHER_CHUNK + lane];
                my_dst = ((dw & ((1LL << 62) - 1)) * rowE) | (dw & ~((1LL << 62) - 1));
            }
            for (int u0 = 0; u0 < ntok_item; u0 += kTmaTok, ++it) {
                const int s = it % nst;
                if (it >= nst) mbar_wait(&empty[s], ((it / nst) - 1) & 1);
                const int nt = min(kTmaTok, ntok_item - u0);
                TmaStageMeta& m = meta[s];
                // lanes u0 .. u0+nt-1 own this stage's tokens
                const int g = lane - u0;
                const bool mine = g >= 0 && g < nt;
                const int code = mine ? (int)((unsigned long long)my_dst >> 62) : -1;
                if (mine) { m.dst[g] = my_dst & ((1LL << 62) - 1); m.code[g] = code; }
                if (lane == 0) { m.ntok = nt; m.hit = hh; m.layer = l; m.delta = delta; }
                const bool load = mine && code != kCodeLinked && !(code == CP_PLAN_RECOMPUTE && zero_rec);
                const unsigned nload = __popc(__ballot_sync(0xffffffffu, load));
                __syncwarp();
                if (lane == 0) mbar_expect_tx(&full[s], nload * 2u * (uint32_t)rowB);
                __syncwarp();
                if (load) {
                    unsigned char* st = ring + (size_t)s * stageB;
                    bulk_g2s(st + (size_t)g * rowB, srcK + my_src * sizeof(T), rowB, &full[s]);
                    bulk_g2s(st + (size_t)(kTmaTok + g) * rowB, srcV + my_src * sizeof(T), rowB, &full[s]);
                }
            }
        }
    } else {
        // ---------------- consumers (warps 1..kTmaCons); warp 1 lane 0 also stores
        const int ct = tid - 32;                               // 0 .. 32*kTmaCons-1
        const bool storer = ct == 0;
        int it = 0;
        for (int64_t item = blockIdx.x; item < items; item += gridDim.x) {
            const int c = (int)(item / a.L), l = (int)(item % a.L);
            const int hh = a.chunk_hit[c], t0 = a.chunk_t0[c];
            const int ntok_item = min(CP_GATHER_CHUNK, a.l_len[hh] - t0);
            char* dstK = a.dir == 0 ? a.paged_k[l] : a.pool_k + l * pool_layer * sizeof(T);
            char* dstV = a.dir == 0 ? a.paged_v[l] : a.pool_v + l * pool_layer * sizeof(T);
            const int delta = a.dir == 0 ? a.l_delta[hh] : 0;
            for (int u0 = 0; u0 < ntok_item; u0 += kTmaTok, ++it) {
                const int s = it % nst;
                mbar_wait(&full[s], (it / nst) & 1);
                const TmaStageMeta& m = meta[s];
                const int nt = m.ntok;
                unsigned char* st = ring + (size_t)s * stageB;
                if (delta != 0) {
                    const float2* tab = a.hit_cs + (int64_t)hh * half;
                    for (int task = ct; task < nt * tpr; task += 32 * kTmaCons) {
                        const int g = task / tpr, j = task - g * tpr;
                        if ((m.code[g] == CP_PLAN_RECOMPUTE && zero_rec) || m.code[g] == kCodeLinked) continue;
                        int lo, hi, i0;
                        if (!GPTJ) { const int head = j / hv, sub = j - head * hv; lo = head * a.d + sub * VEC; hi = lo + half; i0 = sub * VEC; }
                        else { lo = j * 2 * VEC; hi = lo + VEC; i0 = (lo % a.d) / 2; }
                        T* rowp = reinterpret_cast<T*>(st + (size_t)g * rowB);
                        uint4* plo = reinterpret_cast<uint4*>(rowp + lo);
                        uint4* phi = reinterpret_cast<uint4*>(rowp + hi);
                        float x[VEC], y[VEC];
                        unpack(*plo, x, T()); unpack(*phi, y, T());
#pragma unroll
                        for (int e = 0; e < VEC; ++e) {
                            if (!GPTJ) {
                                const float2 cs = __ldg(tab + i0 + e);
                                const float xo = fmaf(x[e], cs.x, -y[e] * cs.y);
                                const float yo = fmaf(y[e], cs.x, x[e] * cs.y);
                                x[e] = xo; y[e] = yo;
                            } else if ((e & 1) == 0) {
                                const float2 c0 = __ldg(tab + i0 + e / 2), c1 = __ldg(tab + i0 + VEC / 2 + e / 2);
                                const float x0 = fmaf(x[e], c0.x, -x[e + 1] * c0.y), x1 = fmaf(x[e + 1], c0.x, x[e] * c0.y);
                                const float y0 = fmaf(y[e], c1.x, -y[e + 1] * c1.y), y1 = fmaf(y[e + 1], c1.x, y[e] * c1.y);
                                x[e] = x0; x[e + 1] = x1; y[e] = y0; y[e + 1] = y1;
                            }
                        }
                        *plo = pack(x, T()); *phi = pack(y, T());
                    }
                    fence_async_smem();
                }
                cons_bar();
                if (storer) {
                    for (int g = 0; g < nt; ++g) {
                        if (m.code[g] == kCodeLinked) continue;
                        const bool z = m.code[g] == CP_PLAN_RECOMPUTE && zero_rec;
                        const int64_t d = m.dst[g];
                        bulk_s2g(dstK + d * sizeof(T), z ? zrow : st + (size_t)g * rowB, rowB);
                        bulk_s2g(dstV + d * sizeof(T), z ? zrow : st + (size_t)(kTmaTok + g) * rowB, rowB);
                    }
                    bulk_commit();
                    // keep kPend store groups in flight: stage it-kPend has been read -> free it
                    bulk_wait_read<kPend>();
                    if (it >= kPend) mbar_arrive(&empty[(it - kPend) % nst]);
                }
            }
        }
        if (storer) {
            bulk_wait_all<0>();
            for (int q = max(0, it - kPend); q < it; ++q) mbar_arrive(&empty[q % nst]);
        }
    }
}

// CP_ZERO_UNCOVERED: zero K and V rows of plan-0 positions.  k_unc_list compacts the uncovered
// positions (warp ballot + one atomic per warp; the order is irrelevant: zero stores commute); then
// k_zero_uncovered walks items (32 listed positions x layer), so the work is proportional to the
// uncovered tokens.  (The first version walked every 32-token block of the batch per layer: 1.78 ms on
// config 2 for 1.5% uncovered tokens.)
__global__ void k_unc_list(DevHeader* hdr, const uint8_t* plan, int64_t total, int64_t* list) {
    if (cp_err_set(hdr)) return;
    const int lane = threadIdx.x & 31;
    for (int64_t g0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) - lane; g0 < total;
         g0 += (int64_t)gridDim.x * blockDim.x) {
        const int64_t g = g0 + lane;
        const bool u = g < total && plan[g] == CP_PLAN_UNCOVERED;
        const unsigned b = __ballot_sync(0xffffffffu, u);
        if (!b) continue;
        int base = 0;
        if (lane == 0) base = atomicAdd(&hdr->n_unc, __popc(b));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (u) list[base + __popc(b & ((1u << lane) - 1))] = g;
    }
}

template <typename T>
__global__ void __launch_bounds__(kRowsThreads) k_zero_uncovered(RowsArgs a, int32_t R, const int64_t* list) {
    __shared__ int64_t s_dst[32];
    __shared__ int s_on[32];
    if (cp_err_set(a.hdr)) return;
    // layers are flattened over the launch's rectangles (nrect > 1: paged_k/v[rect.layer0 + l])
    const int Lt = a.nrect > 1 ? a.rect[a.nrect - 1].layer0 + a.rect[a.nrect - 1].L : a.L;
    const int nu = a.hdr->n_unc;
    const int64_t items = (int64_t)((nu + 31) / 32) * Lt;
    for (int64_t item = blockIdx.x; item < items; item += gridDim.x) {
        const int64_t b = item / Lt;
        const int l = (int)(item % Lt);
        int r = 0;
        if (a.nrect > 1) while (r + 1 < a.nrect && l >= a.rect[r + 1].layer0) ++r;
        const int rowE = (a.nrect > 1 ? a.rect[r].H : a.H) * a.d;
        if (threadIdx.x < 32) {
            const int64_t li = b * 32 + threadIdx.x;
            s_on[threadIdx.x] = 0;
            if (li < nu) {
                const int64_t g = list[li];
                int lo = 0, hi = R - 1;
                while (lo < hi) { const int mid = (lo + hi + 1) >> 1; if (a.req_off[mid] <= g) lo = mid; else hi = mid - 1; }
                const int q = (int)(g - a.req_off[lo]);
                if ((q >> 4) >= a.max_blocks) cp_raise(a.hdr, CP_ERR_INVALID_ARG);   // never write another request's blocks
                else {
                    const int blk = a.block_tables[(int64_t)lo * a.max_blocks + (q >> 4)];
                    s_dst[threadIdx.x] = ((int64_t)blk * CP_BLOCK + (q & 15)) * rowE;
                    s_on[threadIdx.x] = 1;
                }
            }
        }
        __syncthreads();
        constexpr int VEC = Vec<T>::N;
        const int vpr = rowE / VEC;
        for (int task = threadIdx.x; task < 32 * vpr; task += blockDim.x) {
            const int g = task / vpr, v = task - g * vpr;
            if (!s_on[g]) continue;
            const uint4 z = make_uint4(0, 0, 0, 0);
            st_stream((T*)a.paged_k[l] + s_dst[g] + v * VEC, z);
            st_stream((T*)a.paged_v[l] + s_dst[g] + v * VEC, z);
        }
        __syncthreads();
    }
}

int sm_count() { return cp_sm_count(); }
int rows_grid() { return sm_count() * 4; }

// variant = (UNROLL, MINB): selectable with CP_GATHER_VARIANT for A/B measurement
template <typename T, bool G, bool CR>
cp_status launch_rows_c(const RowsArgs& a, int variant, cudaStream_t st) {
    auto go = [&](auto kern) -> cp_status {
        int occ = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kRowsThreads, 0);
        const int grid = sm_count() * std::max(1, occ);
        kern<<<grid, kRowsThreads, 0, st>>>(a);
        return CP_OK;
    };
    switch (variant) {
        // static round-robin item schedules (round-1 A/B)
        case 1: return a.LG > 1 ? go(k_rows<T, G, CR, 2, 4, true, false>) : go(k_rows<T, G, CR, 2, 4, false, false>);
        case 2: return a.LG > 1 ? go(k_rows<T, G, CR, 4, 2, true, false>) : go(k_rows<T, G, CR, 4, 2, false, false>);
        case 3: return a.LG > 1 ? go(k_rows<T, G, CR, 3, 2, true, false>) : go(k_rows<T, G, CR, 3, 2, false, false>);
        case 5: return a.LG > 1 ? go(k_rows<T, G, CR, 8, 1, true, false>) : go(k_rows<T, G, CR, 8, 1, false, false>);
        // dynamic (device-counter) item schedules
        case 6: return a.LG > 1 ? go(k_rows<T, G, CR, 3, 2, true, true>) : go(k_rows<T, G, CR, 3, 2, false, true>);
        case 7: return a.LG > 1 ? go(k_rows<T, G, CR, 2, 4, true, true>) : go(k_rows<T, G, CR, 2, 4, false, true>);
        case 8: return a.LG > 1 ? go(k_rows<T, G, CR, 4, 2, true, true>) : go(k_rows<T, G, CR, 4, 2, false, true>);
        case 9: return a.LG > 1 ? go(k_rows<T, G, CR, 8, 1, true, true>) : go(k_rows<T, G, CR, 8, 1, false, true>);
        // default: unroll 2, 3 CTAs per SM, dynamic -- measured best on B200 for full rows, layer and
        // head shards and config 3 (tools/gather_ab.py, profiles/r01/gather_variants_ab_dyn.log)
        default: return a.LG > 1 ? go(k_rows<T, G, CR, 2, 3, true, true>) : go(k_rows<T, G, CR, 2, 3, false, true>);
    }
}
template <typename T, bool G>
bool launch_rows_tma(const RowsArgs& a, cudaStream_t st) {
    const int rowB = a.H * a.d * (int)sizeof(T);
    const int stageB = kTmaTok * 2 * rowB;
    if (rowB % 16) return false;
    const size_t fixed = (size_t)rowB + 0;                         // zero row
    int nst = 0;
    for (int n = 8; n >= kPend + 2; --n) {
        const size_t need = (size_t)n * stageB + fixed + n * (sizeof(TmaStageMeta) + 16) + 256;
        if (need <= 200 * 1024) { nst = n; break; }
    }
    if (!nst) return false;
    const size_t smem = (size_t)nst * stageB + fixed + nst * (sizeof(TmaStageMeta) + 16) + 256;
    static bool attr[2][2] = {{false, false}, {false, false}};
    bool& done = attr[sizeof(T) == 2][G];
    if (!done) {
        cudaFuncSetAttribute(k_rows_tma<T, G>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        done = true;
    }
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_rows_tma<T, G>, kTmaThreads, smem);
    k_rows_tma<T, G><<<sm_count() * std::max(1, occ), kTmaThreads, smem, st>>>(a, nst);
    return true;
}

template <typename T, bool G>
cp_status launch_rows_t(const RowsArgs& a, int variant, cudaStream_t st) {
    constexpr int VEC = Vec<T>::N;
    const int tpr = a.H * a.d / (2 * VEC);
    if (variant == 4 && a.nrect == 1 && launch_rows_tma<T, G>(a, st)) return CP_OK;
    if (variant == 4) variant = 0;
    return (tpr <= kRowsThreads) ? launch_rows_c<T, G, true>(a, variant, st) : launch_rows_c<T, G, false>(a, variant, st);
}

int g_variant = -1;
int gather_variant() {
    if (g_variant < 0) { const char* e = getenv("CP_GATHER_VARIANT"); g_variant = e ? atoi(e) : 0; }
    return g_variant;
}

}  // namespace

cp_status cp_launch_rows(cp_index* x, int dir, const int32_t* d_count, const int32_t* l_req, const int32_t* l_slot,
                         const int32_t* l_dst, const int32_t* l_len, const int32_t* l_delta, int64_t list_cap,
                         const int64_t* req_off, const uint8_t* plan, const cp_paged_kv* kv, int32_t flags,
                         cudaStream_t st, int32_t nviews, cp_index* const* views, const cp_paged_kv* view_kvs) {
    RowsArgs a;
    std::memset(&a, 0, sizeof(a));
    a.hdr = x->hdr; a.dir = dir; a.count = d_count;
    a.l_req = l_req; a.l_slot = l_slot; a.l_dst = l_dst; a.l_len = l_len; a.l_delta = l_delta;
    a.list_cap = list_cap; a.req_off = req_off; a.plan = plan;
    a.block_tables = kv->block_tables; a.max_blocks = kv->max_blocks_per_req;
    for (int l = 0; l < x->cfg.num_layers; ++l) {
        a.paged_k[l] = (char*)kv->k_layers_h[l]; a.paged_v[l] = (char*)kv->v_layers_h[l];
        if (!a.paged_k[l] || !a.paged_v[l]) return CP_ERR_INVALID_ARG;
    }
    a.pool_k = x->pool_k; a.pool_v = x->pool_v; a.P = x->P; a.slot_pages = x->slot_pages; a.MP = x->MP;
    a.L = x->cfg.num_layers; a.H = x->cfg.num_kv_heads; a.d = x->cfg.head_dim; a.theta = x->cfg.rope_theta;
    a.flags = flags; a.gptj = x->cfg.rope_style == CP_ROPE_GPTJ;
    const int vec = x->cfg.dtype == CP_BF16 ? 8 : 4;
    auto lg_of = [&](const cp_config& c) {
        const int tpr = c.num_kv_heads * c.head_dim / (2 * vec);
        return std::max(1, std::min(c.num_layers, 2048 / std::max(1, CP_GATHER_CHUNK * tpr)));
    };
    a.LG = lg_of(x->cfg);
    a.nrect = 1;
    if (nviews > 0) {
        // the rank's other rectangles (pool views of x) in the same launch: one persistent grid, one tail
        if (nviews + 1 > kMaxRects || !views || !view_kvs || x->is_view) return CP_ERR_INVALID_ARG;
        int64_t groups = 0;
        int layers = 0;
        for (int r = 0; r <= nviews; ++r) {
            const cp_index* v = r == 0 ? x : views[r - 1];
            const cp_paged_kv* vk = r == 0 ? kv : &view_kvs[r - 1];
            if (!v || (r > 0 && (!v->is_view || v->hdr != x->hdr))) return CP_ERR_INVALID_ARG;
            if (v->cfg.head_dim != x->cfg.head_dim || v->cfg.dtype != x->cfg.dtype || v->cfg.rope_style != x->cfg.rope_style)
                return CP_ERR_INVALID_ARG;
            if (vk->block_tables != kv->block_tables || vk->max_blocks_per_req != kv->max_blocks_per_req ||
                !vk->k_layers_h || !vk->v_layers_h) return CP_ERR_INVALID_ARG;
            if (layers + v->cfg.num_layers > CP_MAX_LAYERS) return CP_ERR_INVALID_ARG;
            auto& R = a.rect[r];
            R.pool_k = v->pool_k; R.pool_v = v->pool_v; R.L = v->cfg.num_layers; R.H = v->cfg.num_kv_heads;
            R.LG = lg_of(v->cfg); R.layer0 = layers; R.item0 = groups;
            for (int l = 0; l < R.L; ++l) {
                a.paged_k[layers + l] = (char*)vk->k_layers_h[l]; a.paged_v[layers + l] = (char*)vk->v_layers_h[l];
                if (!a.paged_k[layers + l] || !a.paged_v[layers + l]) return CP_ERR_INVALID_ARG;
            }
            layers += R.L;
            groups += (R.L + R.LG - 1) / R.LG;
            a.LG = std::max(a.LG, R.LG);                    // the launch's template choice covers every rectangle
            a.H = std::max(a.H, R.H);
        }
        a.rect[nviews + 1].item0 = groups;
        a.nrect = nviews + 1;
    }
    a.chunk_hit = x->chunk_hit; a.chunk_t0 = x->chunk_t0; a.CH = x->CH; a.hit_coff = x->hit_coff;
    a.row_src = x->row_src; a.row_dst = x->row_dst;
    a.hit_cs = x->hit_cs; a.cs_hits = x->CS_HITS;
    if (dir == 0 && !l_delta) return CP_ERR_INVALID_ARG;
    WorkKey key;
    key.valid = 1; key.dir = dir; key.cap = list_cap; key.max_blocks = kv->max_blocks_per_req;
    key.skip_linked = dir == 0 ? (flags & (CP_SKIP_LINKED | CP_SKIP_RECOMPUTE)) : 0;
    const void* kp[9] = {d_count, l_req, l_slot, l_dst, l_len, l_delta, req_off, plan, kv->block_tables};
    for (int i = 0; i < 9; ++i) key.p[i] = kp[i];
    if (flags & CP_REUSE_WORKLIST) {
        // the previous gather / copy-in of this index family built the same list (only the layer and head
        // geometry differ): rewind the dynamic item counter and run the copy kernel alone
        if (!x->wk || !x->wk->same(key)) return CP_ERR_INVALID_ARG;
        if (cudaMemsetAsync(&x->hdr->gather_next, 0, sizeof(x->hdr->gather_next), st) != cudaSuccess) return CP_ERR_CUDA;
    } else {
        k_rows_prep<<<1, kPrepThreads, 0, st>>>(a);
        CP_COUNT_LAUNCH();
        k_rows_prep2<<<sm_count() * 2, kPrepThreads, 0, st>>>(a);
        CP_COUNT_LAUNCH();
        if (x->wk) *x->wk = key;
    }
    const bool bf16 = x->cfg.dtype == CP_BF16;
    const int var = gather_variant();
    if (bf16) { if (a.gptj) launch_rows_t<__nv_bfloat16, true>(a, var, st); else launch_rows_t<__nv_bfloat16, false>(a, var, st); }
    else { if (a.gptj) launch_rows_t<float, true>(a, var, st); else launch_rows_t<float, false>(a, var, st); }
    CP_COUNT_LAUNCH();
    return cudaGetLastError() == cudaSuccess ? CP_OK : CP_ERR_CUDA;
}

extern "C" cp_status cp_set_gather_variant(int32_t v) {
    if (v < 0 || v > 9) return CP_ERR_INVALID_ARG;
    g_variant = v;
    return CP_OK;
}

namespace {
cp_status gather_rects(cp_index* x, const cp_batch* b, const cp_hits* h, const cp_paged_kv* kv, int32_t nviews,
                       cp_index* const* views, const cp_paged_kv* view_kvs, int32_t flags, void* stream) {
    if (!x || !b || !h || !kv) return CP_ERR_INVALID_ARG;
    if (!kv->k_layers_h || !kv->v_layers_h || !kv->block_tables || !b->offsets) return CP_ERR_INVALID_ARG;
    if (!h->num_hits || !h->hit_req || !h->hit_slot || !h->hit_dst || !h->hit_len || !h->hit_delta || !h->plan)
        return CP_ERR_INVALID_ARG;
    if (b->num_reqs < 0 || b->num_reqs > x->cfg.max_batch_reqs) return CP_ERR_INVALID_ARG;
    if (b->num_reqs == 0) return CP_OK;
    cudaStream_t st = (cudaStream_t)stream;
    cp_status s = cp_launch_rows(x, 0, h->num_hits, h->hit_req, h->hit_slot, h->hit_dst, h->hit_len, h->hit_delta,
                                 h->max_hits, b->offsets, h->plan, kv, flags, st, nviews, views, view_kvs);
    if (s != CP_OK) return s;
    if (flags & CP_ZERO_UNCOVERED) {
        RowsArgs a;
        std::memset(&a, 0, sizeof(a));
        a.hdr = x->hdr; a.req_off = b->offsets; a.plan = h->plan;
        a.block_tables = kv->block_tables; a.max_blocks = kv->max_blocks_per_req;
        for (int l = 0; l < x->cfg.num_layers; ++l) { a.paged_k[l] = (char*)kv->k_layers_h[l]; a.paged_v[l] = (char*)kv->v_layers_h[l]; }
        a.L = x->cfg.num_layers; a.H = x->cfg.num_kv_heads; a.d = x->cfg.head_dim;
        a.nrect = 1;
        if (nviews > 0) {                            // validated by cp_launch_rows above
            int layers = 0;
            for (int r = 0; r <= nviews; ++r) {
                const cp_index* v = r == 0 ? x : views[r - 1];
                const cp_paged_kv* vk = r == 0 ? kv : &view_kvs[r - 1];
                a.rect[r].L = v->cfg.num_layers; a.rect[r].H = v->cfg.num_kv_heads; a.rect[r].layer0 = layers;
                for (int l = 0; l < v->cfg.num_layers; ++l) {
                    a.paged_k[layers + l] = (char*)vk->k_layers_h[l]; a.paged_v[layers + l] = (char*)vk->v_layers_h[l];
                }
                layers += v->cfg.num_layers;
            }
            a.nrect = nviews + 1;
        }
        if (b->total_tokens > x->cfg.max_batch_tokens) return CP_ERR_INVALID_ARG;
        if (cudaMemsetAsync(&x->hdr->n_unc, 0, sizeof(x->hdr->n_unc), st) != cudaSuccess) return CP_ERR_CUDA;
        k_unc_list<<<sm_count() * 4, 256, 0, st>>>(x->hdr, h->plan, b->total_tokens, x->unc_list);
        CP_COUNT_LAUNCH();
        if (x->cfg.dtype == CP_BF16) k_zero_uncovered<__nv_bfloat16><<<rows_grid(), kRowsThreads, 0, st>>>(a, b->num_reqs, x->unc_list);
        else k_zero_uncovered<float><<<rows_grid(), kRowsThreads, 0, st>>>(a, b->num_reqs, x->unc_list);
        CP_COUNT_LAUNCH();
        if (cudaGetLastError() != cudaSuccess) return CP_ERR_CUDA;
    }
    return CP_OK;
}
}  // namespace

extern "C" cp_status cp_gather_rerotate(cp_index* x, const cp_batch* b, const cp_hits* h, const cp_paged_kv* kv,
                                        int32_t flags, void* stream) {
    return gather_rects(x, b, h, kv, 0, nullptr, nullptr, flags, stream);
}

extern "C" cp_status cp_gather_rerotate_rects(cp_index* x, int32_t num_views, cp_index* const* views, const cp_batch* b,
                                              const cp_hits* h, const cp_paged_kv* dst_kv, int32_t flags, void* stream) {
    if (num_views < 0 || num_views + 1 > kMaxRects || (num_views > 0 && !views) || !dst_kv) return CP_ERR_INVALID_ARG;
    if (!x || x->is_view || (flags & CP_REUSE_WORKLIST)) return CP_ERR_INVALID_ARG;
    return gather_rects(x, b, h, &dst_kv[0], num_views, views, dst_kv + 1, flags, stream);
}

// ---- NEXT-2: zero-copy page linking (R#31) ---------------------------------------------------------
namespace {
// every block b < ceil(n_r / 16) of every request -> -1; a request with more blocks than the table: error
__global__ void k_link_clear(DevHeader* hdr, const int64_t* req_off, int32_t R, int32_t* link, int32_t maxb) {
    if (cp_err_set(hdr)) return;
    const int64_t n = (int64_t)R * maxb;
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x) {
        const int r = (int)(q / maxb), b = (int)(q % maxb);
        const int64_t nb = (req_off[r + 1] - req_off[r] + 15) >> 4;
        if (b == 0 && nb > maxb) cp_raise(hdr, CP_ERR_INVALID_ARG);
        if (b < nb) link[q] = -1;
    }
}
// one warp per hit: lanes take the hit's full pages; a page links iff delta == 0, dst % 16 == 0 and
// its 16 plan codes are all CP_PLAN_REUSED
__global__ void k_link_hits(DevHeader* hdr, const int32_t* count, int32_t cap, const int32_t* h_req,
                            const int32_t* h_slot, const int32_t* h_dst, const int32_t* h_len, const int32_t* h_delta,
                            const int64_t* req_off, const uint8_t* plan, const int32_t* slot_pages, int32_t MP,
                            int32_t* link, int32_t maxb) {
    if (cp_err_set(hdr)) return;
    const int lane = threadIdx.x & 31;
    const int nh = min(*count, cap);
    for (int h = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5); h < nh;
         h += (int)(((int64_t)gridDim.x * blockDim.x) >> 5)) {
        const int dst = h_dst[h], len = h_len[h];
        if (h_delta[h] != 0 || (dst & 15) != 0) continue;
        const int r = h_req[h], slot = h_slot[h];
        const uint8_t* pl = plan + req_off[r];
        for (int j = lane; 16 * j + 16 <= len; j += 32) {
            const int b = (dst >> 4) + j;
            bool all = true;
#pragma unroll
            for (int i = 0; i < 16; ++i) all &= pl[16 * b + i] == CP_PLAN_REUSED;
            if (all && b < maxb) link[(int64_t)r * maxb + b] = slot_pages[(int64_t)slot * MP + j];
        }
    }
}
}  // namespace

extern "C" cp_status cp_link_blocks(cp_index* x, const cp_batch* b, const cp_hits* h, int32_t* link,
                                    int32_t max_blocks, void* stream) {
    if (!x || !b || !h || !link || max_blocks < 1 || !b->offsets) return CP_ERR_INVALID_ARG;
    if (!h->num_hits || !h->hit_req || !h->hit_slot || !h->hit_dst || !h->hit_len || !h->hit_delta || !h->plan)
        return CP_ERR_INVALID_ARG;
    if (b->num_reqs < 0 || b->num_reqs > x->cfg.max_batch_reqs) return CP_ERR_INVALID_ARG;
    if (b->num_reqs == 0) return CP_OK;
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t n = (int64_t)b->num_reqs * max_blocks;
    k_link_clear<<<(int)std::min<int64_t>((n + 255) / 256, sm_count() * 4), 256, 0, st>>>(x->hdr, b->offsets, b->num_reqs,
                                                                                          link, max_blocks);
    CP_COUNT_LAUNCH();
    k_link_hits<<<sm_count() * 2, 256, 0, st>>>(x->hdr, h->num_hits, h->max_hits, h->hit_req, h->hit_slot, h->hit_dst,
                                              h->hit_len, h->hit_delta, b->offsets, h->plan, x->slot_pages, x->MP,
                                              link, max_blocks);
    CP_COUNT_LAUNCH();
    return cudaGetLastError() == cudaSuccess ? CP_OK : CP_ERR_CUDA;
}

// ---- diagnostic: contiguous streaming copy with the gather's load/store instructions -----------------
// (the roofline check for the copy-shaped gather: what LDG.128.nc / STG.128.cs reach on this part)
namespace {
template <int UNROLL>
__global__ void __launch_bounds__(256) k_copy_diag(const uint4* __restrict__ src, uint4* __restrict__ dst, int64_t n16) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x * UNROLL;
    for (int64_t base = (int64_t)blockIdx.x * blockDim.x * UNROLL + threadIdx.x; base < n16; base += stride) {
        uint4 v[UNROLL];
#pragma unroll
        for (int u = 0; u < UNROLL; ++u) { const int64_t i = base + (int64_t)u * blockDim.x; if (i < n16) v[u] = ld_stream(src + i); }
#pragma unroll
        for (int u = 0; u < UNROLL; ++u) { const int64_t i = base + (int64_t)u * blockDim.x; if (i < n16) st_stream(dst + i, v[u]); }
    }
}
}  // namespace

extern "C" cp_status cp_copy_diag(const void* src, void* dst, int64_t bytes, int32_t ctas_per_sm, void* stream) {
    if (!src || !dst || bytes <= 0 || (bytes & 15) || ctas_per_sm < 1) return CP_ERR_INVALID_ARG;
    k_copy_diag<8><<<sm_count() * ctas_per_sm, 256, 0, (cudaStream_t)stream>>>((const uint4*)src, (uint4*)dst, bytes / 16);
    CP_COUNT_LAUNCH();
    return cudaGetLastError() == cudaSuccess ? CP_OK : CP_ERR_CUDA;
}
