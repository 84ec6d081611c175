// cp_score.cu -- N3 recompute score + top-rho selection (§4.2.1 C1 Step 3;
// rho = 25% default).  The paper computes the per-token inter/intra sums from a summed-area
// table on the CPU after copying the attention matrix off the GPU (L770, 383 ms at 10K tokens,
// L1201); here the attention never leaves HBM: the row sums are streamed directly.
//
//   k_score_rows_grp (default; k_score_rows = one warp per row, variant 4): one 8-lane group per span
//                  row i, 4 rows per warp; reads A_h[i][0..i] (fp32, 128-bit loads where aligned),
//                  accumulates q(x) = trunc(x * 2^40) in int64 (R#17: exact and order independent,
//                  so the GPU and the oracle agree bit for bit) with sign + for j < l*, - for j >= l*.
//   k_score_topk : one CTA per span; 8-pass MSB radix select of the k-th largest score
//                  (k = ceil(rho_num*m/rho_den), R#15), then ties at the threshold go to the smaller
//                  index (R#16) via a block scan; bits packed LSB-first.
#include "cp_internal.cuh"
#include <algorithm>
#include <cstring>
#include <climits>
#include <cstdlib>
#include <type_traits>
#include <vector>

namespace {

constexpr int kSpansPerLaunch = 900;        // 32-B descriptors: 28.8 KB of kernel parameters
constexpr int kRowThreads = 256;
constexpr int kTopkThreads = 256;

struct SpanDesc {                               // 32 B
    const float* A;
    int32_t row_begin;                          // first global row of this span within the launch
    int32_t score_off, bits_off;                // relative to the launch's output bases
    int32_t n, l;
    int32_t r_heads;                            // r | (heads << 24)
    __host__ __device__ int r() const { return r_heads & 0xffffff; }
    __host__ __device__ int heads() const { return (int)((uint32_t)r_heads >> 24); }
};
static_assert(sizeof(SpanDesc) == 32, "SpanDesc must be 32 B");

struct ScoreArgs {
    SpanDesc sp[kSpansPerLaunch];
    int32_t nsp;
    int32_t total_rows;
    int32_t rho_num, rho_den;
    long long* scores;                          // launch base (score_off is relative to it)
    uint32_t* bits;
};

// q(x) = trunc(x * 2^40): the fp32 product by a power of two is exact (no FTZ), and cvt.rzi.s64
// truncates toward zero exactly like the oracle's (int64_t)((double)x * 2^40).
__device__ __forceinline__ long long q40(float x) { return __float2ll_rz(x * 1099511627776.0f); }

__device__ __forceinline__ float4 ld_nc4(const float4* p) {
    float4 f;
    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(f.x), "=f"(f.y), "=f"(f.z), "=f"(f.w) : "l"(p));
    return f;
}

constexpr int kRowBatch = 4;                   // 16-B loads in flight per lane (2 KiB per warp); 8 measured
                                               // slower (tools/score_rows_ab.cu: issue-bound on predicated tails)

// One streaming pass over the row prefix A[i][0..i]: returns this lane's share of
//   inter - intra = sum_{j<l*} q(A[i][j]) - sum_{l*<=j<=i} q(A[i][j])
// accumulated as 2 * sum_{j<l*} q - sum_{j<=i} q (the same integers, regrouped exactly; the row sum
// is read, never assumed to be 1 -- R#27).  Scalar head up to 16-B alignment, then batches of
// kRowBatch predicated 128-bit loads per lane issued before any arithmetic, scalar tail.
__device__ __forceinline__ long long warp_row_score(const float* p, int cnt, int l, int lane) {
    long long all = 0, inter = 0;
    const int mis = (int)((reinterpret_cast<uintptr_t>(p) >> 2) & 3);
    const int head = min(cnt, mis ? 4 - mis : 0);
    if (lane < head) { const long long x = q40(__ldg(p + lane)); all += x; if (lane < l) inter += x; }
    const int nvec = (cnt - head) >> 2;
    const float4* v4 = reinterpret_cast<const float4*>(p + head);
    for (int q0 = 0; q0 < nvec; q0 += 32 * kRowBatch) {
        float4 f[kRowBatch];
#pragma unroll
        for (int u = 0; u < kRowBatch; ++u) {
            const int q = q0 + u * 32 + lane;
            f[u] = q < nvec ? ld_nc4(v4 + q) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int u = 0; u < kRowBatch; ++u) {
            const int j0 = head + 4 * (q0 + u * 32 + lane);     // column of f[u].x
            const long long x0 = q40(f[u].x), x1 = q40(f[u].y), x2 = q40(f[u].z), x3 = q40(f[u].w);
            const long long s = (x0 + x1) + (x2 + x3);
            all += s;
            if (j0 + 3 < l) inter += s;
            else if (j0 < l) inter += x0 + (j0 + 1 < l ? x1 : 0) + (j0 + 2 < l ? x2 : 0);
        }
    }
    const int t = head + 4 * nvec + lane;
    if (t < cnt) { const long long x = q40(__ldg(p + t)); all += x; if (t < l) inter += x; }
    return 2 * inter - all;
}

// One warp per span row i (all heads), a single pass over A_h[i][0..i].  MINB = CTAs per SM the
// register budget must allow (variants for A/B measurement: cp_set_score_variant).
template <int MINB>
__global__ void __launch_bounds__(kRowThreads, MINB) k_score_rows(const ScoreArgs a) {
    // the spans' first rows, staged in shared memory: the per-row binary search then costs shared
    // loads instead of a chain of dependent kernel-parameter (constant-cache) loads
    __shared__ int32_t s_rb[kSpansPerLaunch];
    for (int q = threadIdx.x; q < a.nsp; q += blockDim.x) s_rb[q] = a.sp[q].row_begin;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int warp = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
    const int nwarps = (int)(((int64_t)gridDim.x * blockDim.x) >> 5);
    for (int gr = warp; gr < a.total_rows; gr += nwarps) {
        int lo = 0, hi = a.nsp - 1;
        while (lo < hi) { const int mid = (lo + hi + 1) >> 1; if (s_rb[mid] <= gr) lo = mid; else hi = mid - 1; }
        const float* A = a.sp[lo].A;
        const int n = a.sp[lo].n, l = a.sp[lo].l, heads = a.sp[lo].heads();
        const int i = l + (gr - a.sp[lo].row_begin);
        const int score_off = a.sp[lo].score_off;
        long long acc = 0;
        for (int h = 0; h < heads; ++h)
            acc += warp_row_score(A + ((int64_t)h * n + i) * (int64_t)n, i + 1, l, lane);
#pragma unroll
        for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0) a.scores[score_off + (i - l)] = acc;
    }
}

// ---- k_score_rows_grp (default): the row kernel above with a row per SUB-lane group instead of per
// warp.  ncu of k_score_rows (profiles/r02/n3): ~457 warp instructions per row at 57% issue-active, the
// per-row setup (span search, pointers, head / tail, reduction) a third of them; with 32/SUB consecutive
// rows per warp the setup instructions serve 32/SUB rows at once, each row still read with 16-B loads
// (SUB x 16 B contiguous per instruction and row), and the reduction is log2(SUB) shuffle levels.
// Consecutive rows have nearly equal lengths, so the groups of a warp stay converged.
template <int SUB, int U>
__device__ __forceinline__ long long grp_row_score(const float* p, int cnt, int l, int sl) {
    long long all = 0, inter = 0;
    const int mis = (int)((reinterpret_cast<uintptr_t>(p) >> 2) & 3);
    const int head = min(cnt, mis ? 4 - mis : 0);
    if (sl < head) { const long long x = q40(__ldg(p + sl)); all += x; if (sl < l) inter += x; }
    const int nvec = (cnt - head) >> 2;
    const float4* v4 = reinterpret_cast<const float4*>(p + head);
    for (int q0 = 0; q0 < nvec; q0 += SUB * U) {
        float4 f[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int q = q0 + u * SUB + sl;
            f[u] = q < nvec ? ld_nc4(v4 + q) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int j0 = head + 4 * (q0 + u * SUB + sl);
            const long long x0 = q40(f[u].x), x1 = q40(f[u].y), x2 = q40(f[u].z), x3 = q40(f[u].w);
            const long long sm = (x0 + x1) + (x2 + x3);
            all += sm;
            if (j0 + 3 < l) inter += sm;
            else if (j0 < l) inter += x0 + (j0 + 1 < l ? x1 : 0) + (j0 + 2 < l ? x2 : 0);
        }
    }
    const int t = head + 4 * nvec + sl;
    if (sl < 3 && t < cnt) { const long long x = q40(__ldg(p + t)); all += x; if (t < l) inter += x; }
    return 2 * inter - all;
}

template <int SUB, int U, int MINB>
__global__ void __launch_bounds__(kRowThreads, MINB) k_score_rows_grp(const ScoreArgs a) {
    __shared__ int32_t s_rb[kSpansPerLaunch];
    for (int q = threadIdx.x; q < a.nsp; q += blockDim.x) s_rb[q] = a.sp[q].row_begin;
    __syncthreads();
    constexpr int R = 32 / SUB;                                  // rows per warp
    const int lane = threadIdx.x & 31, sg = lane / SUB, sl = lane % SUB;
    const int warp = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
    const int nwarps = (int)(((int64_t)gridDim.x * blockDim.x) >> 5);
    const int ngroups = (a.total_rows + R - 1) / R;
    for (int g = warp; g < ngroups; g += nwarps) {
        const int gr = g * R + sg;
        long long acc = 0;
        int lo = 0;
        if (gr < a.total_rows) {
            int hi = a.nsp - 1;
            while (lo < hi) { const int mid = (lo + hi + 1) >> 1; if (s_rb[mid] <= gr) lo = mid; else hi = mid - 1; }
            const float* A = a.sp[lo].A;
            const int n = a.sp[lo].n, l = a.sp[lo].l, heads = a.sp[lo].heads();
            const int i = l + (gr - s_rb[lo]);
            for (int h = 0; h < heads; ++h) acc += grp_row_score<SUB, U>(A + ((int64_t)h * n + i) * (int64_t)n, i + 1, l, sl);
        }
#pragma unroll
        for (int o = SUB / 2; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (sl == 0 && gr < a.total_rows) a.scores[a.sp[lo].score_off + (gr - s_rb[lo])] = acc;
    }
}

__global__ void __launch_bounds__(kTopkThreads) k_score_topk(const ScoreArgs a) {
    extern __shared__ __align__(16) unsigned char smt[];
    __shared__ int hist[256];
    __shared__ int s_digit, s_rem;
    __shared__ int s_wsum[kTopkThreads / 32 + 1];
    const SpanDesc& s = a.sp[blockIdx.x];
    const int m = s.r() - s.l + 1;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    unsigned long long* key = (unsigned long long*)smt;
    uint8_t* sel = (uint8_t*)(smt + 8 * (size_t)m);
    const long long kk = ((long long)a.rho_num * m + a.rho_den - 1) / a.rho_den;
    const int nwords = (m + 31) / 32;
    uint32_t* bits = a.bits + s.bits_off;
    if (kk <= 0 || kk >= m) {
        const uint32_t fill = kk <= 0 ? 0u : 0xffffffffu;
        for (int w = tid; w < nwords; w += blockDim.x) {
            const int nb = min(32, m - 32 * w);
            bits[w] = nb == 32 ? fill : (fill & ((1u << nb) - 1u));
        }
        return;
    }
    __shared__ unsigned long long s_or[kTopkThreads / 32], s_and[kTopkThreads / 32];
    unsigned long long vor = 0, vand = ~0ULL;
    for (int i = tid; i < m; i += blockDim.x) {
        const unsigned long long kx = (unsigned long long)a.scores[s.score_off + i] ^ (1ULL << 63);
        key[i] = kx; vor |= kx; vand &= kx;
    }
    for (int o = 16; o; o >>= 1) { vor |= __shfl_xor_sync(0xffffffffu, vor, o); vand &= __shfl_xor_sync(0xffffffffu, vand, o); }
    if (lane == 0) { s_or[wid] = vor; s_and[wid] = vand; }
    unsigned long long prefix = 0, pmask = 0;
    if (tid == 0) s_rem = (int)kk;
    __syncthreads();
    vor = 0; vand = ~0ULL;
    for (int w = 0; w < kTopkThreads / 32; ++w) { vor |= s_or[w]; vand &= s_and[w]; }
    // bytes on which every key agrees need no radix pass: fold them into the prefix directly
    const unsigned long long diff = vor ^ vand;                          // bits that differ somewhere
    const int top = diff ? 63 - __clzll(diff) : -1;
    const int start = top < 0 ? -8 : (top / 8) * 8;
    if (start < 56) { pmask = ~0ULL << (start + 8); prefix = vand & pmask; }
    for (int shift = start; shift >= 0; shift -= 8) {
        for (int b = tid; b < 256; b += blockDim.x) hist[b] = 0;
        __syncthreads();
        for (int i = tid; i < m; i += blockDim.x)
            if ((key[i] & pmask) == prefix) atomicAdd(&hist[(key[i] >> shift) & 255], 1);
        __syncthreads();
        if (wid == 0) {                 // warp-parallel: lane owns bins [8 lane, 8 lane + 8)
            int c[8], tot = 0;
#pragma unroll
            for (int k = 0; k < 8; ++k) { c[k] = hist[8 * lane + k]; tot += c[k]; }
            int incl = tot;             // keys in bins >= 8 lane
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) { const int y = __shfl_down_sync(0xffffffffu, incl, o); if (lane + o < 32) incl += y; }
            const int rem = s_rem, excl = incl - tot;
            __syncwarp();
            if (excl < rem && rem <= incl) {          // exactly one lane holds the k-th largest digit
                int cum = excl;
#pragma unroll
                for (int k = 7; k >= 0; --k) {
                    if (cum + c[k] >= rem) { s_digit = 8 * lane + k; s_rem = rem - cum; break; }
                    cum += c[k];
                }
            }
        }
        __syncthreads();
        prefix |= (unsigned long long)s_digit << shift;
        pmask |= 0xFFULL << shift;
        __syncthreads();
    }
    const unsigned long long T = prefix;
    const int take_eq = s_rem;                      // keys equal to T to select, smallest index first
    // rank among equals: chunked block scan
    const int c = (m + kTopkThreads - 1) / kTopkThreads, c0 = min(m, tid * c), c1 = min(m, c0 + c);
    int loc = 0;
    for (int i = c0; i < c1; ++i) loc += key[i] == T;
    int inc = loc;
    for (int o = 1; o < 32; o <<= 1) { const int y = __shfl_up_sync(0xffffffffu, inc, o); if (lane >= o) inc += y; }
    if (lane == 31) s_wsum[wid] = inc;
    __syncthreads();
    if (wid == 0) {
        int x = lane < kTopkThreads / 32 ? s_wsum[lane] : 0, xi = x;
        for (int o = 1; o < 32; o <<= 1) { const int y = __shfl_up_sync(0xffffffffu, xi, o); if (lane >= o) xi += y; }
        if (lane < kTopkThreads / 32) s_wsum[lane] = xi - x;
    }
    __syncthreads();
    int rank = s_wsum[wid] + inc - loc;
    for (int i = c0; i < c1; ++i) {
        const bool eq = key[i] == T;
        sel[i] = key[i] > T || (eq && rank < take_eq);
        rank += eq;
    }
    __syncthreads();
    for (int w = tid; w < nwords; w += blockDim.x) {
        uint32_t v = 0;
        for (int b = 0; b < 32 && 32 * w + b < m; ++b) v |= (uint32_t)sel[32 * w + b] << b;
        bits[w] = v;
    }
}

// ---------------------------------------------------------------------------------------------------
// NEXT-4: CacheBlend KV deviation (R#30).  One warp per span token: the token's K and V
// rows (H*d elements each) of the reused and the fresh first-layer caches, 16-B loads (4 tensors x
// kDevBatch vectors per lane in flight), dev = sum |q24(reused) - q24(fresh)| in exact int64.
// The scores then go through the same k_score_topk as N3.
struct KvDevArgs {
    const uint4* rk; const uint4* rv; const int32_t* rbt;
    const uint4* fk; const uint4* fv; const int32_t* fbt;
    int32_t rmaxb, fmaxb;
    int32_t vec_per_row;                        // 16-B vectors per token row (H * d * elem / 16)
};

__device__ __forceinline__ long long q24(float x) { return __float2ll_rz(x * 16777216.0f); }
__device__ __forceinline__ long long absll(long long x) { return x < 0 ? -x : x; }
__device__ __forceinline__ long long vdev(const uint4 a, const uint4 b, std::true_type) {      // 8 x bf16
    const uint32_t wa[4] = {a.x, a.y, a.z, a.w}, wb[4] = {b.x, b.y, b.z, b.w};
    long long s = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        s += absll(q24(__uint_as_float(wa[k] << 16)) - q24(__uint_as_float(wb[k] << 16)));
        s += absll(q24(__uint_as_float(wa[k] & 0xffff0000u)) - q24(__uint_as_float(wb[k] & 0xffff0000u)));
    }
    return s;
}
__device__ __forceinline__ long long vdev(const uint4 a, const uint4 b, std::false_type) {     // 4 x fp32
    return absll(q24(__uint_as_float(a.x)) - q24(__uint_as_float(b.x))) + absll(q24(__uint_as_float(a.y)) - q24(__uint_as_float(b.y))) +
           absll(q24(__uint_as_float(a.z)) - q24(__uint_as_float(b.z))) + absll(q24(__uint_as_float(a.w)) - q24(__uint_as_float(b.w)));
}
__device__ __forceinline__ uint4 ld_nc_u4(const uint4* p) {
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    return v;
}

template <bool BF16, int kDevBatch, int MINB>
__global__ void __launch_bounds__(kRowThreads, MINB) k_kvdev_rows(const ScoreArgs a, const KvDevArgs k) {
    __shared__ int32_t s_rb[kSpansPerLaunch];          // spans' first rows (see k_score_rows)
    for (int q = threadIdx.x; q < a.nsp; q += blockDim.x) s_rb[q] = a.sp[q].row_begin;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int warp = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
    const int nwarps = (int)(((int64_t)gridDim.x * blockDim.x) >> 5);
    const int V = k.vec_per_row;
    for (int gr = warp; gr < a.total_rows; gr += nwarps) {
        int lo = 0, hi = a.nsp - 1;
        while (lo < hi) { const int mid = (lo + hi + 1) >> 1; if (s_rb[mid] <= gr) lo = mid; else hi = mid - 1; }
        const int req = a.sp[lo].n, l = a.sp[lo].l;
        const int i = l + (gr - a.sp[lo].row_begin);
        const int64_t ro = ((int64_t)k.rbt[(int64_t)req * k.rmaxb + (i >> 4)] * 16 + (i & 15)) * V;
        const int64_t fo = ((int64_t)k.fbt[(int64_t)req * k.fmaxb + (i >> 4)] * 16 + (i & 15)) * V;
        long long acc = 0;
        for (int v0 = 0; v0 < V; v0 += 32 * kDevBatch) {
            uint4 x[kDevBatch][4];
#pragma unroll
            for (int u = 0; u < kDevBatch; ++u) {
                const int v = v0 + 32 * u + lane;
                const bool ok = v < V;
                const uint4 z = make_uint4(0, 0, 0, 0);
                x[u][0] = ok ? ld_nc_u4(k.rk + ro + v) : z;
                x[u][1] = ok ? ld_nc_u4(k.fk + fo + v) : z;
                x[u][2] = ok ? ld_nc_u4(k.rv + ro + v) : z;
                x[u][3] = ok ? ld_nc_u4(k.fv + fo + v) : z;
            }
#pragma unroll
            for (int u = 0; u < kDevBatch; ++u)
                acc += vdev(x[u][0], x[u][1], std::integral_constant<bool, BF16>()) +
                       vdev(x[u][2], x[u][3], std::integral_constant<bool, BF16>());
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0) a.scores[a.sp[lo].score_off + (i - l)] = acc;
    }
}

}  // namespace

namespace {

int sm_count_score() { return cp_sm_count(); }

int g_score_variant = -1;
void launch_score_rows(const ScoreArgs& a, cudaStream_t st) {
    if (g_score_variant < 0) { const char* e = getenv("CP_SCORE_VARIANT"); g_score_variant = e ? atoi(e) : 0; }
    const int sms = sm_count_score();
    auto go = [&](auto kern, int per_sm) {
        const int grid = (int)std::min<int64_t>((a.total_rows + 7) / 8, (int64_t)sms * per_sm);
        kern<<<grid, kRowThreads, 0, st>>>(a);
    };
    switch (g_score_variant) {
        // (lanes per row, 16-B vectors per lane in flight, CTAs/SM); tools/score_ab.py, config 2 (ms incl. top-k):
        // (8,4,4) 0.233-0.236; (16,4,4) 0.251; (8,6,3) 0.245; (4,4,4) 0.279; (8,2,4) 0.305; (8,8,3) 0.282;
        // round-1 warp per row (variant 4) 0.293
        case 0: go(k_score_rows_grp<8, 4, 4>, 4); return;         // default: 4 rows per warp
        case 5: go(k_score_rows_grp<16, 4, 4>, 4); return;
        case 6: go(k_score_rows_grp<8, 6, 3>, 3); return;
        case 7: go(k_score_rows_grp<4, 4, 4>, 4); return;
        default: break;
    }
    switch (g_score_variant) {
        case 1: go(k_score_rows<5>, 5); break;
        case 2: go(k_score_rows<6>, 6); break;
        case 3: go(k_score_rows<8>, 8); break;
        default: go(k_score_rows<4>, 4); break;           // variant 4: the round-1 warp-per-row kernel
    }
}

cp_status topk_smem(int32_t max_m, size_t* smem) {
    *smem = 9 * (size_t)max_m + 16;
    static size_t attr = 0;
    if (*smem > attr) {
        if (cudaFuncSetAttribute(k_score_topk, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)std::max<size_t>(*smem, 48 * 1024)) != cudaSuccess)
            return CP_ERR_CUDA;
        attr = *smem;
    }
    return CP_OK;
}

// Offsets of one launch (<= kSpansPerLaunch spans) must fit the 32-bit descriptor fields.
bool launch_fits(int s0, int nsp, const int32_t* l_h, const int32_t* r_h, const int64_t* score_off_h,
                 const int64_t* bits_off_h) {
    int64_t rows = 0;
    for (int s = s0; s < s0 + nsp; ++s) {
        if (score_off_h[s] - score_off_h[s0] > INT32_MAX || bits_off_h[s] - bits_off_h[s0] > INT32_MAX) return false;
        rows += r_h[s] - l_h[s] + 1;
    }
    return rows <= INT32_MAX - 65536;
}

// Build the descriptors of spans [s0, s0 + nsp) (A / n / heads per span as given) into `a`.
void fill_args(ScoreArgs& a, int s0, int nsp, const float* const* A_h, const int32_t* n_h, const int32_t* heads_h,
               const int32_t* l_h, const int32_t* r_h, int32_t rho_num, int32_t rho_den, int64_t* out_scores,
               const int64_t* score_off_h, uint32_t* out_bits, const int64_t* bits_off_h) {
    std::memset(&a, 0, sizeof(a));
    a.nsp = nsp;
    const int64_t sbase = score_off_h[s0], bbase = bits_off_h[s0];
    int64_t rows = 0;
    for (int q = 0; q < nsp; ++q) {
        const int s = s0 + q;
        SpanDesc d;
        d.A = A_h ? A_h[s] : nullptr; d.row_begin = (int32_t)rows;
        d.score_off = (int32_t)(score_off_h[s] - sbase); d.bits_off = (int32_t)(bits_off_h[s] - bbase);
        d.n = n_h[s]; d.l = l_h[s]; d.r_heads = r_h[s] | ((heads_h ? heads_h[s] : 1) << 24);
        a.sp[q] = d;
        rows += r_h[s] - l_h[s] + 1;
    }
    a.total_rows = (int32_t)rows; a.rho_num = rho_num; a.rho_den = rho_den;
    a.scores = (long long*)out_scores + sbase; a.bits = out_bits + bbase;
}

}  // namespace

extern "C" cp_status cp_score_deviation(int32_t num_spans, const float* const* attn_h, const int32_t* n_h,
                                        const int32_t* heads_h, const int32_t* l_h, const int32_t* r_h,
                                        int32_t rho_num, int32_t rho_den, int32_t mode, int32_t max_m,
                                        int64_t* out_scores, const int64_t* score_off_h, uint32_t* out_bits,
                                        const int64_t* bits_off_h, void* stream) {
    if (mode == CP_SCORE_KVDEV) return CP_ERR_UNSUPPORTED;            // KV caches, not attention: cp_score_kv_deviation
    if (mode != CP_SCORE_INTER_INTRA) return CP_ERR_INVALID_ARG;
    if (num_spans < 0 || rho_den <= 0 || rho_num < 0 || rho_num > rho_den || max_m < 1 || max_m > 16384) return CP_ERR_INVALID_ARG;
    if (num_spans == 0) return CP_OK;
    if (!attn_h || !n_h || !heads_h || !l_h || !r_h || !out_scores || !score_off_h || !out_bits || !bits_off_h)
        return CP_ERR_INVALID_ARG;
    for (int s = 0; s < num_spans; ++s) {          // every check before any launch: no side effects on error
        if (!attn_h[s] || n_h[s] < 1 || n_h[s] >= (1 << 24) || heads_h[s] < 1 || heads_h[s] > 255 || l_h[s] < 0 ||
            r_h[s] < l_h[s] || r_h[s] >= n_h[s] || r_h[s] - l_h[s] + 1 > max_m) return CP_ERR_INVALID_ARG;
    }
    for (int s0 = 0; s0 < num_spans; s0 += kSpansPerLaunch)
        if (!launch_fits(s0, std::min(kSpansPerLaunch, num_spans - s0), l_h, r_h, score_off_h, bits_off_h))
            return CP_ERR_INVALID_ARG;
    cudaStream_t st = (cudaStream_t)stream;
    size_t smem;
    if (topk_smem(max_m, &smem) != CP_OK) return CP_ERR_CUDA;
    std::vector<ScoreArgs> args(1);
    for (int s0 = 0; s0 < num_spans; s0 += kSpansPerLaunch) {
        ScoreArgs& a = args[0];
        fill_args(a, s0, std::min(kSpansPerLaunch, num_spans - s0), attn_h, n_h, heads_h, l_h, r_h, rho_num, rho_den,
                  out_scores, score_off_h, out_bits, bits_off_h);
        launch_score_rows(a, st);
        CP_COUNT_LAUNCH();
        k_score_topk<<<a.nsp, kTopkThreads, smem, st>>>(a);
        CP_COUNT_LAUNCH();
        if (cudaGetLastError() != cudaSuccess) return CP_ERR_CUDA;
    }
    return CP_OK;
}

extern "C" cp_status cp_score_kv_deviation(int32_t num_spans, const int32_t* req_h, const int32_t* l_h,
                                           const int32_t* r_h, const void* reused_k, const void* reused_v,
                                           const int32_t* reused_bt, int32_t reused_maxb, const void* fresh_k,
                                           const void* fresh_v, const int32_t* fresh_bt, int32_t fresh_maxb,
                                           int32_t H, int32_t d, int32_t dtype, int32_t rho_num, int32_t rho_den,
                                           int32_t max_m, int64_t* out_scores, const int64_t* score_off_h,
                                           uint32_t* out_bits, const int64_t* bits_off_h, void* stream) {
    if (num_spans < 0 || rho_den <= 0 || rho_num < 0 || rho_num > rho_den || max_m < 1 || max_m > 16384) return CP_ERR_INVALID_ARG;
    if (num_spans == 0) return CP_OK;
    if (dtype != CP_BF16 && dtype != CP_FP32) return CP_ERR_INVALID_ARG;
    const int64_t row_bytes = (int64_t)H * d * (dtype == CP_BF16 ? 2 : 4);
    if (H < 1 || d < 1 || row_bytes % 16 != 0 || row_bytes / 16 > INT32_MAX) return CP_ERR_INVALID_ARG;
    if (!req_h || !l_h || !r_h || !reused_k || !reused_v || !reused_bt || !fresh_k || !fresh_v || !fresh_bt ||
        !out_scores || !score_off_h || !out_bits || !bits_off_h || reused_maxb < 1 || fresh_maxb < 1)
        return CP_ERR_INVALID_ARG;
    for (int s = 0; s < num_spans; ++s) {
        if (req_h[s] < 0 || l_h[s] < 0 || r_h[s] < l_h[s] || r_h[s] - l_h[s] + 1 > max_m) return CP_ERR_INVALID_ARG;
        if (r_h[s] / 16 >= std::min(reused_maxb, fresh_maxb)) return CP_ERR_INVALID_ARG;   // beyond the block tables
    }
    for (int s0 = 0; s0 < num_spans; s0 += kSpansPerLaunch)
        if (!launch_fits(s0, std::min(kSpansPerLaunch, num_spans - s0), l_h, r_h, score_off_h, bits_off_h))
            return CP_ERR_INVALID_ARG;
    cudaStream_t st = (cudaStream_t)stream;
    size_t smem;
    if (topk_smem(max_m, &smem) != CP_OK) return CP_ERR_CUDA;
    KvDevArgs k;
    k.rk = (const uint4*)reused_k; k.rv = (const uint4*)reused_v; k.rbt = reused_bt; k.rmaxb = reused_maxb;
    k.fk = (const uint4*)fresh_k; k.fv = (const uint4*)fresh_v; k.fbt = fresh_bt; k.fmaxb = fresh_maxb;
    k.vec_per_row = (int32_t)(row_bytes / 16);
    std::vector<ScoreArgs> args(1);
    for (int s0 = 0; s0 < num_spans; s0 += kSpansPerLaunch) {
        ScoreArgs& a = args[0];
        // SpanDesc.n carries the request index (no attention matrix in this mode)
        fill_args(a, s0, std::min(kSpansPerLaunch, num_spans - s0), nullptr, req_h, nullptr, l_h, r_h, rho_num,
                  rho_den, out_scores, score_off_h, out_bits, bits_off_h);
        const char* ev = getenv("CP_KVDEV_VARIANT");          // A/B measurement (tools/kvdev_bench.py)
        const int var = ev ? atoi(ev) : 0;
        const int64_t want = (a.total_rows + 7) / 8;
        auto go = [&](auto kern, int per_sm) {
            kern<<<(int)std::min<int64_t>(want, (int64_t)sm_count_score() * per_sm), kRowThreads, 0, st>>>(a, k);
        };
        // (16-B loads per lane and tensor, CTAs per SM); default (1, 8): 0.524 ms vs (4, 4) 0.569 ms,
        // (2, 6) 0.578, (2, 4) 0.540 on the config-2 shape (tools/kvdev_bench.py)
        if (dtype == CP_BF16) {
            if (var == 1) go(k_kvdev_rows<true, 2, 6>, 6);
            else if (var == 2) go(k_kvdev_rows<true, 4, 4>, 4);
            else if (var == 3) go(k_kvdev_rows<true, 2, 4>, 4);
            else go(k_kvdev_rows<true, 1, 8>, 8);
        } else {
            go(k_kvdev_rows<false, 1, 8>, 8);
        }
        CP_COUNT_LAUNCH();
        k_score_topk<<<a.nsp, kTopkThreads, smem, st>>>(a);
        CP_COUNT_LAUNCH();
        if (cudaGetLastError() != cudaSuccess) return CP_ERR_CUDA;
    }
    return CP_OK;
}

extern "C" cp_status cp_set_score_variant(int32_t v) {
    if (v < 0 || v > 7) return CP_ERR_INVALID_ARG;
    g_score_variant = v;
    return CP_OK;
}
