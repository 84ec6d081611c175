// score_rows_ab.cu -- A/B microbenchmark of the N3 row-sum inner loop (not part of the library).
// 256 requests x causal fp32 [n x n] attention (n = 1536), span rows [l, n) with l = 160: the
// config-2 shape of k_score_rows.  Variants: q(x) via F2I.S64 or via integer decode of the fp32
// bits; loads in flight per lane.  Prints GB/s of algorithmic bytes (row prefixes read).
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/score_ab tools/score_rows_ab.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ long long q40_cvt(float x) { return __float2ll_rz(x * 1099511627776.0f); }
// trunc(x * 2^40) from the bits: |x| < 2^23 finite; denormals give 0 (as x*2^40 < 1 for them)
__device__ __forceinline__ long long q40_int(float x) {
    const uint32_t u = __float_as_uint(x);
    const int E = (u >> 23) & 255;
    const long long mant = (long long)((u & 0x7FFFFFu) | 0x800000u);
    const int sh = E - 110;
    long long q = sh >= 0 ? (mant << sh) : (sh > -24 ? (mant >> -sh) : 0);
    q = E ? q : 0;
    return (u >> 31) ? -q : q;
}

__device__ __forceinline__ float4 ld_nc4(const float4* p) {
    float4 f;
    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(f.x), "=f"(f.y), "=f"(f.z), "=f"(f.w) : "l"(p));
    return f;
}

template <int B, bool INT>
__global__ void __launch_bounds__(256) k_rows(const float* A, int n, int l, int reqs, long long* out) {
    const int lane = threadIdx.x & 31;
    const int warp = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
    const int nwarps = (int)(((int64_t)gridDim.x * blockDim.x) >> 5);
    const int rows_per = n - l, total = rows_per * reqs;
    for (int gr = warp; gr < total; gr += nwarps) {
        const int req = gr / rows_per, i = l + gr % rows_per;
        const float* p = A + ((int64_t)req * n + i) * n;
        const int cnt = i + 1, nvec = cnt >> 2;
        const float4* v4 = reinterpret_cast<const float4*>(p);
        long long all = 0, inter = 0;
        for (int q0 = 0; q0 < nvec; q0 += 32 * B) {
            float4 f[B];
#pragma unroll
            for (int u = 0; u < B; ++u) {
                const int q = q0 + u * 32 + lane;
                f[u] = q < nvec ? ld_nc4(v4 + q) : make_float4(0.f, 0.f, 0.f, 0.f);
            }
#pragma unroll
            for (int u = 0; u < B; ++u) {
                const int j0 = 4 * (q0 + u * 32 + lane);
                long long x0, x1, x2, x3;
                if (INT) { x0 = q40_int(f[u].x); x1 = q40_int(f[u].y); x2 = q40_int(f[u].z); x3 = q40_int(f[u].w); }
                else { x0 = q40_cvt(f[u].x); x1 = q40_cvt(f[u].y); x2 = q40_cvt(f[u].z); x3 = q40_cvt(f[u].w); }
                const long long s = (x0 + x1) + (x2 + x3);
                all += s;
                if (j0 + 3 < l) inter += s;
                else if (j0 < l) inter += x0 + (j0 + 1 < l ? x1 : 0) + (j0 + 2 < l ? x2 : 0);
            }
        }
        const int t = 4 * nvec + lane;
        if (t < cnt) { const long long x = INT ? q40_int(p[t]) : q40_cvt(p[t]); all += x; if (t < l) inter += x; }
        long long acc = 2 * inter - all;
        for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0) out[gr] = acc;
    }
}

// double-buffered: batch k+1 is in flight while batch k is summed
template <int B>
__global__ void __launch_bounds__(256) k_rows_db(const float* A, int n, int l, int reqs, long long* out) {
    const int lane = threadIdx.x & 31;
    const int warp = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
    const int nwarps = (int)(((int64_t)gridDim.x * blockDim.x) >> 5);
    const int rows_per = n - l, total = rows_per * reqs;
    for (int gr = warp; gr < total; gr += nwarps) {
        const int req = gr / rows_per, i = l + gr % rows_per;
        const float* p = A + ((int64_t)req * n + i) * n;
        const int cnt = i + 1, nvec = cnt >> 2;
        const float4* v4 = reinterpret_cast<const float4*>(p);
        long long all = 0, inter = 0;
        float4 cur[B], nxt[B];
#pragma unroll
        for (int u = 0; u < B; ++u) { const int q = u * 32 + lane; cur[u] = q < nvec ? ld_nc4(v4 + q) : make_float4(0.f, 0.f, 0.f, 0.f); }
        for (int q0 = 0; q0 < nvec; q0 += 32 * B) {
            const bool more = q0 + 32 * B < nvec;
            if (more) {
#pragma unroll
                for (int u = 0; u < B; ++u) { const int q = q0 + 32 * B + u * 32 + lane; nxt[u] = q < nvec ? ld_nc4(v4 + q) : make_float4(0.f, 0.f, 0.f, 0.f); }
            }
#pragma unroll
            for (int u = 0; u < B; ++u) {
                const int j0 = 4 * (q0 + u * 32 + lane);
                const long long x0 = q40_cvt(cur[u].x), x1 = q40_cvt(cur[u].y), x2 = q40_cvt(cur[u].z), x3 = q40_cvt(cur[u].w);
                const long long s = (x0 + x1) + (x2 + x3);
                all += s;
                if (j0 + 3 < l) inter += s;
                else if (j0 < l) inter += x0 + (j0 + 1 < l ? x1 : 0) + (j0 + 2 < l ? x2 : 0);
            }
            if (more) {
#pragma unroll
                for (int u = 0; u < B; ++u) cur[u] = nxt[u];
            }
        }
        const int t = 4 * nvec + lane;
        if (t < cnt) { const long long x = q40_cvt(p[t]); all += x; if (t < l) inter += x; }
        long long acc = 2 * inter - all;
        for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0) out[gr] = acc;
    }
}

// two rows per warp: both rows' batches are issued together (twice the bytes in flight per warp)
template <int B>
__global__ void __launch_bounds__(256) k_rows_pair(const float* A, int n, int l, int reqs, long long* out) {
    const int lane = threadIdx.x & 31;
    const int warp = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
    const int nwarps = (int)(((int64_t)gridDim.x * blockDim.x) >> 5);
    const int rows_per = n - l, total = rows_per * reqs;
    for (int g2 = warp; 2 * g2 < total; g2 += nwarps) {
        const float* p[2]; int cnt[2], nvec[2], grs[2];
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            const int gr = min(2 * g2 + k, total - 1);
            grs[k] = 2 * g2 + k;
            const int req = gr / rows_per, i = l + gr % rows_per;
            p[k] = A + ((int64_t)req * n + i) * n;
            cnt[k] = (2 * g2 + k < total) ? i + 1 : 0;
            nvec[k] = cnt[k] >> 2;
        }
        long long all[2] = {0, 0}, inter[2] = {0, 0};
        const int nmax = max(nvec[0], nvec[1]);
        for (int q0 = 0; q0 < nmax; q0 += 32 * B) {
            float4 f[2][B];
#pragma unroll
            for (int k = 0; k < 2; ++k)
#pragma unroll
                for (int u = 0; u < B; ++u) {
                    const int q = q0 + u * 32 + lane;
                    f[k][u] = q < nvec[k] ? ld_nc4(reinterpret_cast<const float4*>(p[k]) + q) : make_float4(0.f, 0.f, 0.f, 0.f);
                }
#pragma unroll
            for (int k = 0; k < 2; ++k)
#pragma unroll
                for (int u = 0; u < B; ++u) {
                    const int j0 = 4 * (q0 + u * 32 + lane);
                    const long long x0 = q40_cvt(f[k][u].x), x1 = q40_cvt(f[k][u].y), x2 = q40_cvt(f[k][u].z), x3 = q40_cvt(f[k][u].w);
                    const long long s4 = (x0 + x1) + (x2 + x3);
                    all[k] += s4;
                    if (j0 + 3 < l) inter[k] += s4;
                    else if (j0 < l) inter[k] += x0 + (j0 + 1 < l ? x1 : 0) + (j0 + 2 < l ? x2 : 0);
                }
        }
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            const int t = 4 * nvec[k] + lane;
            if (t < cnt[k]) { const long long x = q40_cvt(p[k][t]); all[k] += x; if (t < l) inter[k] += x; }
            long long acc = 2 * inter[k] - all[k];
            for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
            if (lane == 0 && grs[k] < total) out[grs[k]] = acc;
        }
    }
}

__global__ void fill(float* A, int64_t N) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < N; k += (int64_t)gridDim.x * blockDim.x) {
        uint32_t h = (uint32_t)(k * 2654435761u) ^ (uint32_t)(k >> 17);
        h ^= h >> 13; h *= 0x5bd1e995u; h ^= h >> 15;
        A[k] = (h >> 8) * (1.0f / 16777216.0f) * 0.01f;
    }
}

template <int B, bool INT, bool DB = false>
void run(const char* name, const float* A, int n, int l, int reqs, long long* out, long long* ref, int blocks_per_sm) {
    const int grid = 148 * blocks_per_sm;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    auto go = [&]() {
        if (INT && DB) k_rows_pair<B><<<grid, 256>>>(A, n, l, reqs, out);
        else if (DB) k_rows_db<B><<<grid, 256>>>(A, n, l, reqs, out);
        else k_rows<B, INT><<<grid, 256>>>(A, n, l, reqs, out);
    };
    for (int w = 0; w < 3; ++w) go();
    cudaEventRecord(e0);
    const int it = 10;
    for (int w = 0; w < it; ++w) go();
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= it;
    double bytes = 0;
    for (int i = l; i < n; ++i) bytes += 4.0 * ((i + 1) & ~3) ;
    bytes *= reqs;
    int bad = 0;
    if (ref) {
        static long long h1[1 << 20], h2[1 << 20];
        const int tot = (n - l) * reqs;
        cudaMemcpy(h1, out, 8 * (size_t)tot, cudaMemcpyDeviceToHost);
        cudaMemcpy(h2, ref, 8 * (size_t)tot, cudaMemcpyDeviceToHost);
        for (int k = 0; k < tot; ++k) bad += h1[k] != h2[k];
    }
    printf("%-22s blocks/SM %d  %.3f ms  %.0f GB/s  mismatches %d\n", name, blocks_per_sm, ms, bytes / ms / 1e6, bad);
}

int main() {
    const int n = 1536, l = 160, reqs = 256;
    const int64_t N = (int64_t)reqs * n * n;
    float* A; long long *out, *ref;
    cudaMalloc(&A, N * 4); cudaMalloc(&out, 8ll * reqs * n); cudaMalloc(&ref, 8ll * reqs * n);
    fill<<<148 * 8, 256>>>(A, N);
    k_rows<8, false><<<148 * 8, 256>>>(A, n, l, reqs, ref);
    cudaDeviceSynchronize();
    for (int nn : {1536}) {           // rows must be 16-B aligned here (n % 4 == 0)
      for (int bps : {2, 3, 4, 6}) {
        run<4, false>("cvt B4", A, nn, l, reqs, out, ref, bps);
        run<4, true, true>("pair B4", A, nn, l, reqs, out, ref, bps);
        run<2, true, true>("pair B2", A, nn, l, reqs, out, ref, bps);
      }
    }
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
