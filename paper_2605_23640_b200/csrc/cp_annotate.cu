// cp_annotate.cu -- NEXT-1: the KV Annotator's C1 Steps 1-2 on the device (§4.2.1).
//
// The paper builds a summed-area table of the final-layer attention on the CPU after a GPU->CPU copy
// (383 ms at 10K tokens) and names GPU SAT construction as future work.  Here the
// attention never leaves HBM.  Every sum is taken in the 2^-40 fixed point of R#17 (exact int64),
// so the argmax below -- and its tie-breaks -- are bit-identical to the oracle's.
//
// For a substring [l, r] (0-based, inclusive) of a coarse segment, with row prefixes
// R(i, x) = sum_{j < x} a[i][j] (heads summed) and P(x) = sum_{i < x} R(i, i+1):
//     IntraAttn - InterAttn = sum_{i=l}^{r} (R(i, i+1) - R(i, l)) - sum_{i=l}^{r} R(i, l)
//                           = P(r+1) - P(l) - 2 * sum_{i=l}^{r} R(i, l)
// which is exactly the paper's rectangle-sum form for causal attention.
//
//   k_ann_rows : warp per (request, row i): R(i, 0..i+1) into the workspace (the SAT's row pass)
//   k_ann_segs : CTA per request: P and the coarse segments by one fused block scan
//   k_ann_best : chunk best (diff desc, length desc, l asc) of sum R(i, l) walks, coalesced across
//                starts l; flat form (thread per start, 256 starts per CTA) for many-request calls,
//                split form (32 starts per CTA, the rows cut across 8 warps, two passes) for few
//   k_ann_final: warp per segment, best over its chunks; reported only if diff > 0
#include "cp_internal.cuh"
#include <algorithm>
#include <climits>
#include <cstring>
#include <cstdlib>
#include <vector>

namespace {

constexpr int kAnnReqsPerLaunch = 512;
constexpr int kBestThreads = 256;           // k_ann_best CTA: 8 warps
constexpr int kStarts = 32;                 // starts l per k_ann_best CTA (one per lane)
constexpr int kRowWarps = kBestThreads / 32;   // the segment's rows are split across the CTA's warps
constexpr int kRowUnroll = 32;            // k_ann_best: rows of R(i, l) in flight per thread
constexpr int kRowsBatch = 2;               // k_ann_rows: 128-column chunks whose loads are in flight together

struct AnnReq {
    const float* A;          // [heads][n][n]
    const uint8_t* mask;     // [n]
    long long r_off;         // workspace byte offsets
    long long p_off;
    long long s_off;         // segments, then the per-(segment, chunk) partial bests
    int32_t n, heads;
    int32_t row_begin;       // first global row of this request within the launch
    int32_t nch;             // partial-best stride per segment: ceil(n / kStarts) (the workspace's sizing)
};

struct PartialBest { long long d; int32_t len; int32_t l; };

struct AnnArgs {
    AnnReq rq[kAnnReqsPerLaunch];
    int32_t nreq, total_rows, min_len, max_seg, nchunk, cw;   // cw: starts per k_ann_best chunk
    char* ws;
    int32_t* out_nseg;       // launch bases
    int32_t* out_l;
    int32_t* out_r;
    long long* out_diff;
};

// R layout in the workspace: row i at element 3 + i * rstride(n) (rstride a multiple of 4 >= n + 2),
// so a lane's 4 entries R(i, x0+1 .. x0+4), x0 % 4 == 0, start on a 32-B boundary (two 16-B stores)
__host__ __device__ __forceinline__ int64_t rstride(int64_t n) { return (n + 5) & ~(int64_t)3; }
__host__ __device__ __forceinline__ size_t rbytes(int64_t n) { return 8 * (size_t)(n * rstride(n) + 3); }

__device__ __forceinline__ long long q40(float x) { return __float2ll_rz(x * 1099511627776.0f); }

__device__ __forceinline__ int find_req(const AnnArgs& a, int gr) {
    int lo = 0, hi = a.nreq - 1;
    while (lo < hi) { const int mid = (lo + hi + 1) >> 1; if (a.rq[mid].row_begin <= gr) lo = mid; else hi = mid - 1; }
    return lo;
}

__global__ void __launch_bounds__(256) k_ann_rows(const AnnArgs a) {
    const int lane = threadIdx.x & 31;
    const int warp = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
    const int nwarps = (int)(((int64_t)gridDim.x * blockDim.x) >> 5);
    for (int gr = warp; gr < a.total_rows; gr += nwarps) {
        const int q = find_req(a, gr);
        const AnnReq& rq = a.rq[q];
        const int n = rq.n, i = gr - rq.row_begin;
        long long* R = reinterpret_cast<long long*>(a.ws + rq.r_off) + 3 + (int64_t)i * rstride(n);
        long long carry = 0;
        if (lane == 0) R[0] = 0;
        // a lane owns 4 consecutive columns of each 128-column chunk, kRowsBatch chunks per step: all
        // loads of a step are issued before any scan, and one warp scan serves 128 columns
        for (int base = 0; base <= i; base += 128 * kRowsBatch) {
            long long v[kRowsBatch][4];
#pragma unroll
            for (int u = 0; u < kRowsBatch; ++u) {
                const int x0 = base + u * 128 + 4 * lane;
#pragma unroll
                for (int e = 0; e < 4; ++e) v[u][e] = 0;
                for (int h = 0; h < rq.heads; ++h) {
                    const float* pa = rq.A + ((int64_t)h * n + i) * n + x0;
                    if (x0 + 3 <= i && ((uintptr_t)pa & 15) == 0) {        // one 16-B load for the 4 columns
                        const float4 f = __ldg(reinterpret_cast<const float4*>(pa));
                        v[u][0] += q40(f.x); v[u][1] += q40(f.y); v[u][2] += q40(f.z); v[u][3] += q40(f.w);
                    } else {
#pragma unroll
                        for (int e = 0; e < 4; ++e)
                            if (x0 + e <= i) v[u][e] += q40(__ldg(pa + e));
                    }
                }
            }
#pragma unroll
            for (int u = 0; u < kRowsBatch; ++u) {
                const long long p1 = v[u][0] + v[u][1], p2 = p1 + v[u][2], p3 = p2 + v[u][3];
                long long inc = p3;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) { const long long y = __shfl_up_sync(0xffffffffu, inc, o); if (lane >= o) inc += y; }
                const long long ex = carry + inc - p3;                 // sum before this lane's 4 columns
                const int x0 = base + u * 128 + 4 * lane;
                if (x0 + 3 <= i) {
                    longlong2* d2 = reinterpret_cast<longlong2*>(R + x0 + 1);
                    d2[0] = make_longlong2(ex + v[u][0], ex + p1);
                    d2[1] = make_longlong2(ex + p2, ex + p3);
                } else {
                    if (x0 <= i) R[x0 + 1] = ex + v[u][0];
                    if (x0 + 1 <= i) R[x0 + 2] = ex + p1;
                    if (x0 + 2 <= i) R[x0 + 3] = ex + p2;
                }
                carry += __shfl_sync(0xffffffffu, inc, 31);
            }
        }
    }
}

// One ordered block scan per 1024-row step computes all three: P(x+1) = P(x) + R(x, x+1) (prefix of
// row sums), the coarse segments' starts (maximal mask-0 runs, in order) and their ends (the k-th
// mask-0 position followed by a mask-1 one, or the end, closes segment k).
__global__ void __launch_bounds__(1024) k_ann_segs(const AnnArgs a) {
    __shared__ long long s_w[33];
    __shared__ int s_ws[33], s_we[33];
    __shared__ long long s_carry;
    __shared__ int s_cs, s_ce;
    const AnnReq& rq = a.rq[blockIdx.x];
    const int n = rq.n;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const long long* R = reinterpret_cast<const long long*>(a.ws + rq.r_off) + 3;
    long long* P = reinterpret_cast<long long*>(a.ws + rq.p_off);
    int2* seg = reinterpret_cast<int2*>(a.ws + rq.s_off);
    if (tid == 0) { s_carry = 0; s_cs = 0; s_ce = 0; P[0] = 0; }
    for (int b0 = 0; b0 < n; b0 += 1024) {
        const int i = b0 + tid;
        const long long v = i < n ? R[(int64_t)i * rstride(n) + i + 1] : 0;
        const bool m0 = i < n && !rq.mask[i];
        const bool start = m0 && (i == 0 || rq.mask[i - 1]);
        const bool end = m0 && (i + 1 == n || rq.mask[i + 1]);
        long long inc = v;
        int incs = start, ince = end;
        for (int o = 1; o < 32; o <<= 1) {
            const long long y = __shfl_up_sync(0xffffffffu, inc, o);
            const int ys = __shfl_up_sync(0xffffffffu, incs, o), ye = __shfl_up_sync(0xffffffffu, ince, o);
            if (lane >= o) { inc += y; incs += ys; ince += ye; }
        }
        if (lane == 31) { s_w[wid] = inc; s_ws[wid] = incs; s_we[wid] = ince; }
        __syncthreads();                                     // also orders the previous step's carries
        if (wid == 0) {
            long long x = s_w[lane], xi = x;
            int xs = s_ws[lane], xsi = xs, xe = s_we[lane], xei = xe;
            for (int o = 1; o < 32; o <<= 1) {
                const long long y = __shfl_up_sync(0xffffffffu, xi, o);
                const int ys = __shfl_up_sync(0xffffffffu, xsi, o), ye = __shfl_up_sync(0xffffffffu, xei, o);
                if (lane >= o) { xi += y; xsi += ys; xei += ye; }
            }
            s_w[lane] = xi - x; s_ws[lane] = xsi - xs; s_we[lane] = xei - xe;
            if (lane == 31) { s_w[32] = xi; s_ws[32] = xsi; s_we[32] = xei; }
        }
        __syncthreads();
        if (i < n) P[i + 1] = s_carry + s_w[wid] + inc;
        if (start) { const int k = s_cs + s_ws[wid] + incs - 1; if (k < a.max_seg) seg[k].x = i; }
        if (end) { const int k = s_ce + s_we[wid] + ince - 1; if (k < a.max_seg) seg[k].y = i; }
        __syncthreads();
        if (tid == 0) { s_carry += s_w[32]; s_cs += s_ws[32]; s_ce += s_we[32]; }
    }
    __syncthreads();
    if (tid == 0) a.out_nseg[blockIdx.x] = s_cs <= a.max_seg ? s_cs : -1;
}

struct Best { long long d; int len; int l; };
__device__ __forceinline__ bool better(const Best& x, const Best& y) {      // diff desc, length desc, l asc
    if (x.len < 0) return false;
    if (y.len < 0) return true;
    if (x.d != y.d) return x.d > y.d;
    if (x.len != y.len) return x.len > y.len;
    return x.l < y.l;
}

// Many-request launches: CTA per (request, segment, chunk of 256 starts l): thread per l walks rows i = l..b (unrolled, the row
// loads of one step issued together) accumulating sum R(i, l); P(i+1) comes from shared memory.
__global__ void __launch_bounds__(kBestThreads) k_ann_best_flat(const AnnArgs a) {
    __shared__ long long s_d[kBestThreads / 32];
    __shared__ int s_len[kBestThreads / 32], s_l[kBestThreads / 32];
    extern __shared__ long long sP[];                                       // P(sa .. sb+1)
    const int per_req = a.max_seg * a.nchunk;
    const int q = blockIdx.x / per_req, rem = blockIdx.x % per_req;
    const int s = rem / a.nchunk, ch = rem % a.nchunk;
    const AnnReq& rq = a.rq[q];
    const int nseg = a.out_nseg[q];
    if (nseg < 0 || s >= nseg) return;
    const int2 sg = reinterpret_cast<const int2*>(a.ws + rq.s_off)[s];
    PartialBest* part = reinterpret_cast<PartialBest*>(a.ws + rq.s_off + 8 * (size_t)a.max_seg);
    const int n = rq.n, sa = sg.x, sb = sg.y;
    const int lmax = sb - a.min_len + 1;                                   // last admissible start
    const int l_lo = sa + ch * kBestThreads;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    if (l_lo > lmax) return;                                                // no admissible start in this chunk
    const long long* R = reinterpret_cast<const long long*>(a.ws + rq.r_off) + 3;
    const long long* P = reinterpret_cast<const long long*>(a.ws + rq.p_off);
    for (int x = l_lo + tid; x <= sb + 1; x += kBestThreads) sP[x - l_lo] = P[x];
    __syncthreads();
    const int l = l_lo + tid;
    const bool act = l <= lmax;
    Best best{0, -1, 0};
    if (act) {
        const long long Pl = sP[l - l_lo];
        long long acc = 0;
        const int rmin = l + a.min_len - 1;
        int i = l;
        for (; i + kRowUnroll - 1 <= sb; i += kRowUnroll) {
            long long v[kRowUnroll];
#pragma unroll
            for (int u = 0; u < kRowUnroll; ++u) v[u] = __ldg(R + (int64_t)(i + u) * rstride(n) + l);
#pragma unroll
            for (int u = 0; u < kRowUnroll; ++u) {
                acc += v[u];
                if (i + u >= rmin) {
                    const Best c{sP[i + u + 1 - l_lo] - Pl - 2 * acc, i + u - l + 1, l};
                    if (better(c, best)) best = c;
                }
            }
        }
        for (; i <= sb; ++i) {
            acc += __ldg(R + (int64_t)i * rstride(n) + l);
            if (i >= rmin) {
                const Best c{sP[i + 1 - l_lo] - Pl - 2 * acc, i - l + 1, l};
                if (better(c, best)) best = c;
            }
        }
    }
    for (int o = 16; o; o >>= 1) {
        const Best y{__shfl_xor_sync(0xffffffffu, best.d, o), __shfl_xor_sync(0xffffffffu, best.len, o),
                     __shfl_xor_sync(0xffffffffu, best.l, o)};
        if (better(y, best)) best = y;
    }
    if (lane == 0) { s_d[wid] = best.d; s_len[wid] = best.len; s_l[wid] = best.l; }
    __syncthreads();
    if (tid == 0) {
        Best b{0, -1, 0};
        for (int w = 0; w < kBestThreads / 32; ++w) { const Best y{s_d[w], s_len[w], s_l[w]}; if (better(y, b)) b = y; }
        PartialBest pb; pb.d = b.d; pb.len = b.len; pb.l = b.l;
        part[s * rq.nch + ch] = pb;
    }
}

// Few-request launches (the flat kernel would fill a fraction of the SMs and its critical path is a
// whole segment): CTA per (request, segment, chunk of 32 starts l): lane = start, warp w = one of 8 contiguous row
// ranges of the segment.  Pass 1: each warp sums R(i, l) over its rows i >= l; the per-warp sums are
// scanned in shared memory, so pass 2 walks each row range from its exact prefix and evaluates
// P(i+1) - P(l) - 2 * sum_{k=l}^{i} R(k, l) for every admissible end i.  The critical path is one
// eighth of the segment, at the price of reading R twice.
__global__ void __launch_bounds__(kBestThreads) k_ann_best_split(const AnnArgs a) {
    __shared__ long long s_sum[kRowWarps][kStarts];
    __shared__ long long s_d[kRowWarps];
    __shared__ int s_len[kRowWarps], s_l[kRowWarps];
    const int per_req = a.max_seg * a.nchunk;
    const int q = blockIdx.x / per_req, rem = blockIdx.x % per_req;
    const int s = rem / a.nchunk, ch = rem % a.nchunk;
    const AnnReq& rq = a.rq[q];
    const int nseg = a.out_nseg[q];
    if (nseg < 0 || s >= nseg) return;
    const int2 sg = reinterpret_cast<const int2*>(a.ws + rq.s_off)[s];
    PartialBest* part = reinterpret_cast<PartialBest*>(a.ws + rq.s_off + 8 * (size_t)a.max_seg);
    const int n = rq.n, sa = sg.x, sb = sg.y;
    const int lmax = sb - a.min_len + 1;                                   // last admissible start
    const int l_lo = sa + ch * kStarts;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    if (l_lo > lmax) return;                                                // no admissible start in this chunk
    const long long* R = reinterpret_cast<const long long*>(a.ws + rq.r_off) + 3;
    const long long* P = reinterpret_cast<const long long*>(a.ws + rq.p_off);
    const int l = l_lo + lane;
    const bool act = l <= lmax;
    const int cs = (sb - l_lo + kRowWarps) / kRowWarps;                    // rows l_lo..sb split in 8
    const int r0 = max(l_lo + wid * cs, l), r1 = min(sb, l_lo + (wid + 1) * cs - 1);
    // pass 1: this warp's partial sum of R(i, l)
    long long part_sum = 0;
    if (act) {
        int i = r0;
        for (; i + kRowUnroll - 1 <= r1; i += kRowUnroll) {
            long long v[kRowUnroll];
#pragma unroll
            for (int u = 0; u < kRowUnroll; ++u) v[u] = __ldg(R + (int64_t)(i + u) * rstride(n) + l);
#pragma unroll
            for (int u = 0; u < kRowUnroll; ++u) part_sum += v[u];
        }
        for (; i <= r1; ++i) part_sum += __ldg(R + (int64_t)i * rstride(n) + l);
    }
    s_sum[wid][lane] = part_sum;
    __syncthreads();
    long long acc = 0;
    for (int w = 0; w < wid; ++w) acc += s_sum[w][lane];                   // rows before r0 (and >= l)
    // pass 2: candidates (l, i) for i in this warp's rows
    Best best{0, -1, 0};
    if (act && r0 <= r1) {
        const long long Pl = __ldg(P + l);
        const int rmin = l + a.min_len - 1;
        int i = r0;
        for (; i + kRowUnroll - 1 <= r1; i += kRowUnroll) {
            long long v[kRowUnroll], pv[kRowUnroll];
#pragma unroll
            for (int u = 0; u < kRowUnroll; ++u) {
                v[u] = __ldg(R + (int64_t)(i + u) * rstride(n) + l);
                pv[u] = __ldg(P + i + u + 1);
            }
#pragma unroll
            for (int u = 0; u < kRowUnroll; ++u) {
                acc += v[u];
                if (i + u >= rmin) {
                    const Best c{pv[u] - Pl - 2 * acc, i + u - l + 1, l};
                    if (better(c, best)) best = c;
                }
            }
        }
        for (; i <= r1; ++i) {
            acc += __ldg(R + (int64_t)i * rstride(n) + l);
            if (i >= rmin) {
                const Best c{__ldg(P + i + 1) - Pl - 2 * acc, i - l + 1, l};
                if (better(c, best)) best = c;
            }
        }
    }
    for (int o = 16; o; o >>= 1) {
        const Best y{__shfl_xor_sync(0xffffffffu, best.d, o), __shfl_xor_sync(0xffffffffu, best.len, o),
                     __shfl_xor_sync(0xffffffffu, best.l, o)};
        if (better(y, best)) best = y;
    }
    if (lane == 0) { s_d[wid] = best.d; s_len[wid] = best.len; s_l[wid] = best.l; }
    __syncthreads();
    if (tid == 0) {
        Best b{0, -1, 0};
        for (int w = 0; w < kRowWarps; ++w) { const Best y{s_d[w], s_len[w], s_l[w]}; if (better(y, b)) b = y; }
        PartialBest pb; pb.d = b.d; pb.len = b.len; pb.l = b.l;
        part[s * rq.nch + ch] = pb;
    }
}

// warp per (request, segment): lanes stride over the chunks' partial bests, then a shuffle reduction
__global__ void k_ann_final(const AnnArgs a) {
    const int t = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5), lane = threadIdx.x & 31;
    if (t >= a.nreq * a.max_seg) return;
    const int q = t / a.max_seg, s = t % a.max_seg;
    const int nseg = a.out_nseg[q];
    if (nseg < 0 || s >= nseg) return;
    const AnnReq& rq = a.rq[q];
    const int2 sg = reinterpret_cast<const int2*>(a.ws + rq.s_off)[s];
    const PartialBest* part = reinterpret_cast<const PartialBest*>(a.ws + rq.s_off + 8 * (size_t)a.max_seg);
    const int lmax = sg.y - a.min_len + 1;
    Best b{0, -1, 0};
    for (int ch = lane; ch < a.nchunk && sg.x + ch * a.cw <= lmax; ch += 32) {
        const PartialBest pb = part[s * rq.nch + ch];
        const Best y{pb.d, pb.len, pb.l};
        if (better(y, b)) b = y;
    }
    for (int o = 16; o; o >>= 1) {
        const Best y{__shfl_xor_sync(0xffffffffu, b.d, o), __shfl_xor_sync(0xffffffffu, b.len, o),
                     __shfl_xor_sync(0xffffffffu, b.l, o)};
        if (better(y, b)) b = y;
    }
    if (lane) return;
    const bool ok = b.len > 0 && b.d > 0;
    a.out_l[t] = ok ? b.l : -1;
    a.out_r[t] = ok ? b.l + b.len - 1 : -1;
    a.out_diff[t] = ok ? b.d : 0;
}

size_t align256(size_t v) { return (v + 255) & ~(size_t)255; }

}  // namespace

extern "C" size_t cp_annotate_workspace(int32_t num_reqs, const int32_t* n_h, int32_t max_segments) {
    if (num_reqs <= 0 || !n_h || max_segments <= 0) return 0;
    size_t tot = 0;
    for (int r = 0; r < num_reqs; ++r) {
        const size_t n = (size_t)std::max(n_h[r], 0);
        const size_t nch = (n + kStarts - 1) / kStarts;
        tot += align256(rbytes((int64_t)n)) + align256(8 * (n + 1)) + align256(8 * (size_t)max_segments + 16 * (size_t)max_segments * nch);
    }
    return tot;
}

extern "C" cp_status cp_annotate_spans(int32_t num_reqs, const float* const* attn_h, const int32_t* n_h,
                                       const int32_t* heads_h, const uint8_t* const* mask_h, int32_t min_len,
                                       int32_t max_segments, void* workspace, size_t workspace_bytes,
                                       int32_t* out_nseg, int32_t* out_l, int32_t* out_r, int64_t* out_diff,
                                       void* stream) {
    if (num_reqs < 0 || min_len < 1 || max_segments < 1) return CP_ERR_INVALID_ARG;
    if (num_reqs == 0) return CP_OK;
    if (!attn_h || !n_h || !heads_h || !mask_h || !workspace || !out_nseg || !out_l || !out_r || !out_diff)
        return CP_ERR_INVALID_ARG;
    if (workspace_bytes < cp_annotate_workspace(num_reqs, n_h, max_segments)) return CP_ERR_CAPACITY;
    for (int r = 0; r < num_reqs; ++r)
        if (!attn_h[r] || !mask_h[r] || n_h[r] < 1 || heads_h[r] < 1 || n_h[r] > (1 << 20) ||
            (int64_t)n_h[r] * heads_h[r] >= (1LL << 22))       // int64 domain of the 2^-40 sums (header)
            return CP_ERR_INVALID_ARG;
    cudaStream_t st = (cudaStream_t)stream;
    std::vector<AnnArgs> hold(1);
    size_t off = 0;
    for (int r0 = 0; r0 < num_reqs; r0 += kAnnReqsPerLaunch) {
        AnnArgs& a = hold[0];
        std::memset(&a, 0, sizeof(a));
        a.nreq = std::min(kAnnReqsPerLaunch, num_reqs - r0);
        long long rows = 0;
        int64_t nmax = 1;
        for (int q = 0; q < a.nreq; ++q) {
            const int r = r0 + q;
            const size_t n = (size_t)n_h[r];
            AnnReq& d = a.rq[q];
            d.A = attn_h[r]; d.mask = mask_h[r]; d.n = n_h[r]; d.heads = heads_h[r];
            d.r_off = (long long)off; off += align256(rbytes((int64_t)n));
            d.p_off = (long long)off; off += align256(8 * (n + 1));
            d.s_off = (long long)off;
            d.nch = (int32_t)((n_h[r] + kStarts - 1) / kStarts);
            off += align256(8 * (size_t)max_segments + 16 * (size_t)max_segments * ((n + kStarts - 1) / kStarts));
            nmax = std::max<int64_t>(nmax, (int64_t)n);
            d.row_begin = (int32_t)rows;
            rows += n_h[r];
        }
        if (rows > INT32_MAX) return CP_ERR_INVALID_ARG;
        a.total_rows = (int32_t)rows; a.min_len = min_len; a.max_seg = max_segments;
        // flat (thread per start, whole segment per thread) when the launch already has a couple of
        // waves of 256-start chunks and P fits in shared memory; otherwise split the rows across warps
        const size_t psmem = 8 * ((size_t)nmax + 2);
        const char* ev = getenv("CP_ANN_VARIANT");            // A/B and parity: 1 = flat, 2 = split, else auto
        const int var = ev ? atoi(ev) : 0;
        const bool fits = psmem <= 200 * 1024;
        const bool flat = fits && (var == 1 || (var != 2 && (long long)a.nreq * ((nmax + kBestThreads - 1) / kBestThreads) >=
                                                                2LL * cp_sm_count()));
        a.cw = flat ? kBestThreads : kStarts;
        a.nchunk = (int32_t)((nmax + a.cw - 1) / a.cw);
        a.ws = (char*)workspace;
        a.out_nseg = out_nseg + r0;
        a.out_l = out_l + (int64_t)r0 * max_segments;
        a.out_r = out_r + (int64_t)r0 * max_segments;
        a.out_diff = (long long*)out_diff + (int64_t)r0 * max_segments;
        k_ann_rows<<<(int)std::min<long long>((rows + 7) / 8, (long long)cp_sm_count() * 16), 256, 0, st>>>(a);
        CP_COUNT_LAUNCH();
        k_ann_segs<<<a.nreq, 1024, 0, st>>>(a);
        CP_COUNT_LAUNCH();
        const long long nblk = (long long)a.nreq * max_segments * a.nchunk;
        if (nblk > INT32_MAX) return CP_ERR_INVALID_ARG;
        if (flat) {
            static bool attr = false;
            if (!attr) { cudaFuncSetAttribute(k_ann_best_flat, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024); attr = true; }
            k_ann_best_flat<<<(int)nblk, kBestThreads, psmem, st>>>(a);
        } else {
            k_ann_best_split<<<(int)nblk, kBestThreads, 0, st>>>(a);
        }
        CP_COUNT_LAUNCH();
        k_ann_final<<<(a.nreq * max_segments + 7) / 8, 256, 0, st>>>(a);
        CP_COUNT_LAUNCH();
        if (cudaGetLastError() != cudaSuccess) return CP_ERR_CUDA;
    }
    return CP_OK;
}
