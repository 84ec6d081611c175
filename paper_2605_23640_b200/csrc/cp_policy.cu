// cp_policy.cu -- NEXT-3: the spans the baseline policies store (PAPER.md
// Fig. 4, §5.7; R#28-29).
//
// One CTA of 1024 threads (the span lists are a few thousand entries; the cost is one pass over the
// writers' masks), output in (request, position) order by an ordered block-wide compaction:
//   FixedChunk  -- flattened chunk index g over all requests (per-request chunk counts n_r / L
//                  scanned into shared memory, g -> r by binary search); a thread checks one
//                  chunk's L mask bytes; kept chunks are compacted 1024 at a time.
//   PrefixOnly  -- one warp per request finds the first mask-1 position (ballot over 32 bytes per
//                  step, stopping at min(n, max_len)); requests with a prefix >= L are compacted.
#include "cp_internal.cuh"
#include <algorithm>

namespace {

constexpr int kPT = 1024;

// Exclusive scan of one flag per thread; returns this thread's rank among set flags and writes the
// block total to *total.
__device__ __forceinline__ int block_rank(bool flag, int* wsum, int* total) {
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const unsigned b = __ballot_sync(0xffffffffu, flag);
    const int in_warp = __popc(b & ((1u << lane) - 1u));
    if (lane == 0) wsum[wid] = __popc(b);
    __syncthreads();
    if (wid == 0) {
        const int x = wsum[lane];           // kPT / 32 == 32 warps
        int xi = x;
        for (int o = 1; o < 32; o <<= 1) { const int y = __shfl_up_sync(0xffffffffu, xi, o); if (lane >= o) xi += y; }
        wsum[lane] = xi - x;
        if (lane == 31) wsum[32] = xi;
    }
    __syncthreads();
    const int r = wsum[wid] + in_warp;
    *total = wsum[32];
    __syncthreads();
    return r;
}

struct PolicyArgs {
    const int64_t* offsets; const uint8_t* mask; int32_t R;
    int32_t policy, L, max_len, max_spans;
    int32_t *span_req, *span_begin, *span_len, *count;
};

__global__ void __launch_bounds__(kPT) k_policy_spans(PolicyArgs a) {
    extern __shared__ int32_t cc[];          // FixedChunk: [R + 1] chunk prefix counts; PrefixOnly: [R] prefix lengths
    __shared__ int wsum[33];
    __shared__ int s_carry;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    int total = 0, carry = 0;
    if (a.policy == CP_POLICY_FIXED_CHUNK) {
        // chunk counts per request, exclusive scan into cc[0..R]
        if (tid == 0) s_carry = 0;
        __syncthreads();
        for (int b0 = 0; b0 < a.R; b0 += kPT) {
            const int r = b0 + tid;
            const int v = r < a.R ? (int)((a.offsets[r + 1] - a.offsets[r]) / a.L) : 0;
            int inc = v;
            for (int o = 1; o < 32; o <<= 1) { const int y = __shfl_up_sync(0xffffffffu, inc, o); if (lane >= o) inc += y; }
            if (lane == 31) wsum[wid] = inc;
            __syncthreads();
            if (wid == 0) {
                const int x = wsum[lane];
                int xi = x;
                for (int o = 1; o < 32; o <<= 1) { const int y = __shfl_up_sync(0xffffffffu, xi, o); if (lane >= o) xi += y; }
                wsum[lane] = xi - x;
                if (lane == 31) wsum[32] = xi;
            }
            __syncthreads();
            if (r < a.R) cc[r] = s_carry + wsum[wid] + inc - v;
            __syncthreads();
            if (tid == 0) s_carry += wsum[32];
            __syncthreads();
        }
        if (tid == 0) cc[a.R] = s_carry;
        __syncthreads();
        const int G = cc[a.R];
        for (int g0 = 0; g0 < G; g0 += kPT) {
            const int g = g0 + tid;
            bool keep = false;
            int r = 0, c = 0;
            if (g < G) {
                int lo = 0, hi = a.R - 1;            // last r with cc[r] <= g
                while (lo < hi) { const int mid = (lo + hi + 1) >> 1; if (cc[mid] <= g) lo = mid; else hi = mid - 1; }
                r = lo; c = g - cc[r];
                const uint8_t* m = a.mask + a.offsets[r] + (int64_t)c * a.L;
                keep = true;
                for (int i = 0; i < a.L; ++i) if (m[i]) { keep = false; break; }
            }
            const int rank = block_rank(keep, wsum, &total);
            if (keep && carry + rank < a.max_spans) {
                a.span_req[carry + rank] = r; a.span_begin[carry + rank] = c * a.L; a.span_len[carry + rank] = a.L;
            }
            carry += total;
        }
    } else {
        // prefix length per request: first mask-1 position, capped at min(n, max_len)
        for (int r = wid; r < a.R; r += kPT / 32) {
            const int64_t o = a.offsets[r];
            const int lim = (int)min((int64_t)a.max_len, a.offsets[r + 1] - o);
            int p = lim;
            for (int i0 = 0; i0 < lim; i0 += 32) {
                const int i = i0 + lane;
                const unsigned b = __ballot_sync(0xffffffffu, i < lim && a.mask[o + i]);
                if (b) { p = i0 + __ffs(b) - 1; break; }
            }
            if (lane == 0) cc[r] = p;
        }
        __syncthreads();
        for (int b0 = 0; b0 < a.R; b0 += kPT) {
            const int r = b0 + tid;
            const bool keep = r < a.R && cc[r] >= a.L;
            const int rank = block_rank(keep, wsum, &total);
            if (keep && carry + rank < a.max_spans) {
                a.span_req[carry + rank] = r; a.span_begin[carry + rank] = 0; a.span_len[carry + rank] = cc[r];
            }
            carry += total;
        }
    }
    if (tid == 0) *a.count = carry;
}

}  // namespace

extern "C" cp_status cp_policy_spans(const cp_batch* b, int32_t policy, int32_t chunk_len, int32_t max_len,
                                     int32_t max_spans, int32_t* span_req, int32_t* span_begin, int32_t* span_len,
                                     int32_t* count_d, int32_t* count_h, void* stream) {
    if (!b || !count_d || chunk_len < 1 || max_spans < 0 || b->num_reqs < 0) return CP_ERR_INVALID_ARG;
    if (policy != CP_POLICY_FIXED_CHUNK && policy != CP_POLICY_PREFIX_ONLY) return CP_ERR_INVALID_ARG;
    if (policy == CP_POLICY_PREFIX_ONLY && max_len < chunk_len) return CP_ERR_INVALID_ARG;
    if (max_spans > 0 && (!span_req || !span_begin || !span_len)) return CP_ERR_INVALID_ARG;
    cudaStream_t st = (cudaStream_t)stream;
    if (b->num_reqs == 0) {
        CP_CUDA_CHECK(cudaMemsetAsync(count_d, 0, 4, st));
    } else {
        if (!b->offsets || !b->mask) return CP_ERR_INVALID_ARG;
        const size_t smem = 4 * ((size_t)b->num_reqs + 1);
        if (smem > 200 * 1024) return CP_ERR_UNSUPPORTED;
        static int attr_set = 0;
        if (!attr_set) { cudaFuncSetAttribute(k_policy_spans, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024); attr_set = 1; }
        PolicyArgs a{b->offsets, b->mask, b->num_reqs, policy, chunk_len, max_len, max_spans,
                     span_req, span_begin, span_len, count_d};
        k_policy_spans<<<1, kPT, smem, st>>>(a);
        CP_COUNT_LAUNCH();
        if (cudaGetLastError() != cudaSuccess) return CP_ERR_CUDA;
    }
    if (count_h) {
        CP_CUDA_CHECK(cudaMemcpyAsync(count_h, count_d, 4, cudaMemcpyDeviceToHost, st));
        CP_CUDA_CHECK(cudaStreamSynchronize(st));
        if (*count_h > max_spans) return CP_ERR_CAPACITY;
    }
    return CP_OK;
}
