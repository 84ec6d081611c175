// cp_match.cu -- N1 span matcher (§4.2.2 C2; plan codes L724-727 §4.3.1).
//
// One CTA per request (512 threads):
//   1. prefix hashes h[0..n] of the request by a block-wide scan of (hash, B^len) pairs
//   2. every thread slides its windows W[k] = h[k+w] - h[k] B^w and probes the pool's prefix hash
//      table (open addressing, 16-B entries, L2 resident) -- the prefix filter;
//      each probe hit is a candidate (counted: c of P:L697) and gets the O(1) full-length hash
//      pre-check against the entry's full hash
//   3. one warp per surviving candidate compares the tokens exactly (and the reader mask, R#9);
//      exact comparison replaces the paper's SHA-256 equality (R#5): same result, no collision risk
//   4. warp 0 assembles hits greedily left to right with ballot scans (R#7).  The pool is
//      containment-free (R#20), so at most one verified entry starts at any position k.
//   5. hits -> sparse per-request scratch, LRU touch (atomicMax), plan codes + stats
//   6. the last CTA to finish (ticket) scans the per-request hit counts and compacts the hits
//      into the caller's dense arrays -- no extra launch, no host round trip.
// NEXT-3 baseline policies (R#28-29) reuse the same CTA: FixedChunk probes only the chunk-aligned
// windows and accepts only length-w entries (steps 3-4 unchanged); PrefixOnly probes window 0,
// collects the origin-0 entries and replaces steps 3-4 by a warp-per-candidate longest common
// prefix (ballot over 32 tokens per step) and a warp max over (prefix length, -id).
#include "cp_internal.cuh"
#include <algorithm>
#include <cstring>

namespace {

constexpr int kNT = 512;

#ifdef CP_MATCH_PROF
// diagnostic build only: per-phase clock64 cycles of thread 0, summed over CTAs
__device__ unsigned long long g_match_prof[8];
#define MPROF(i) do { if (tid == 0) { const long long c_ = clock64(); atomicAdd(&g_match_prof[i], (unsigned long long)(c_ - t_m)); t_m = c_; } } while (0)
#else
#define MPROF(i) do {} while (0)
#endif

struct MatchArgs {
    DevHeader* hdr;
    const int32_t* tokens; const int64_t* offsets; const uint8_t* mask; int32_t R;
    unsigned long long t; int32_t no_touch; int32_t policy;   // 0 selective, 1 FixedChunk, 2 PrefixOnly
    int32_t w; uint64_t B; uint64_t Bw; const unsigned long long* pw;
    const HEntry* htab; int logT; int64_t T;
    const int32_t* slot_id; const int32_t* slot_len; const int32_t* slot_origin;
    const unsigned long long* slot_full; unsigned long long* slot_last;
    const int32_t* slot_pages; int32_t MP; const int32_t* page_tokens; const uint16_t* page_bits;
    int32_t nmax;                      // shared memory is sized for requests of <= nmax tokens
    char* gscr;                        // long requests: per-request arrays in global scratch (else null)
    int32_t dyn_smem;                  // dynamic shared memory bytes of this launch
    int32_t *sp_entry, *sp_slot, *sp_dst, *sp_len, *sp_delta, *req_cnt;
    int32_t max_hits; int32_t* num_hits; int32_t* req_hit_offsets;
    int32_t *hit_req, *hit_entry, *hit_slot, *hit_dst, *hit_len, *hit_delta;
    uint8_t* plan; int32_t *req_covered, *req_recompute, *req_candidates;
    // R#33 same-user sessions (session == nullptr: none)
    const int32_t* session; const int32_t* session_slot; const int32_t* slot_owner; const uint8_t* slot_state;
    int32_t max_sessions;
    const unsigned long long* clock;   // cp_index_set_clock: logical time read on the device (else t)
};

struct MatchSmem {
    size_t h, vslot, tok, clist, hk, hs, hm, total;
    __host__ __device__ MatchSmem(int nmax, int w) {
        const int hmax = nmax / w + 1;
        h = 0;
        vslot = h + 8 * ((size_t)nmax + 1);
        tok = vslot + 4 * (size_t)nmax;
        clist = tok + 4 * (size_t)nmax;
        hk = clist + 4 * (size_t)nmax;
        hs = hk + 4 * (size_t)hmax;
        hm = hs + 4 * (size_t)hmax;
        total = hm + 4 * (size_t)hmax;
    }
};

// G: the per-request arrays (prefix hashes, window slots, tokens, candidates, hits) live in global
// scratch at 24 * offsets[r] + 64 * r (laid out for the request's own length) instead of shared memory
template <bool G>
__global__ void __launch_bounds__(kNT) k_match(MatchArgs a) {
    extern __shared__ __align__(16) unsigned char sm[];
    __shared__ uint64_t wtmp[2 * (kNT / 32)];
    __shared__ int s_nc, s_cands, s_nh, s_cov, s_rec, s_last, s_vtok, s_pslot, s_plen;
    __shared__ int s_scan[kNT / 32 + 1];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int r = blockIdx.x;
    const int64_t off = a.offsets[r];
    const int n = (int)(a.offsets[r + 1] - off);
    const MatchSmem L(G ? max(n, 1) : a.nmax, a.w);
    unsigned char* base = G ? reinterpret_cast<unsigned char*>(a.gscr) + 24 * off + 64 * (int64_t)r : sm;
    uint64_t* h = (uint64_t*)(base + L.h);
    int32_t* vslot = (int32_t*)(base + L.vslot);
    int32_t* tok = (int32_t*)(base + L.tok);
    int32_t* clist = (int32_t*)(base + L.clist);
    int32_t* hk = (int32_t*)(base + L.hk);
    int32_t* hs = (int32_t*)(base + L.hs);
    int32_t* hm = (int32_t*)(base + L.hm);
    const bool skip = cp_err_set(a.hdr) || n > a.nmax;
    if (tid == 0 && !cp_err_set(a.hdr) && n > a.nmax) cp_raise(a.hdr, CP_ERR_INVALID_ARG);
    if (tid == 0) { s_nc = 0; s_cands = 0; s_nh = 0; s_cov = 0; s_rec = 0; s_vtok = 0; }
    int nh = 0;
#ifdef CP_MATCH_PROF
    long long t_m = clock64();
#endif
    if (!skip) {
        // ---- 1. tokens + prefix hashes
        for (int i = tid; i < n; i += kNT) tok[i] = a.tokens[off + i];
        __syncthreads();
        cp_block_prefix_hash<kNT>([&](int i) { return tok[i]; }, n, a.B, h, wtmp);
        const int nw = n - a.w + 1;                  // number of windows (may be <= 0)
        for (int k = tid; k < nw; k += kNT) vslot[k] = -1;
        __syncthreads();
        MPROF(0);
        // ---- 2. rolling windows -> prefix filter -> O(1) full-hash pre-check (warp-level probing)
        // windows examined: every k (the method), k = c*w (FixedChunk), k = 0 (PrefixOnly)
        const int kstep = a.policy == 1 ? a.w : 1;
        const int nwin = a.policy == 0 ? nw : a.policy == 1 ? n / a.w : (nw > 0 ? 1 : 0);
        int my_cands = 0;
        const int wbase = tid & ~31;
        for (int base = 0; base < nwin; base += kNT) {
            const int c = base + tid;
            const bool act = c < nwin;
            const uint64_t W = act ? cp_subhash(h, c * kstep, a.w, a.Bw) : 0;
            cp_warp_probe<true>(a.htab, (uint32_t)(a.T - 1), a.logT, W, act, [&](int owner, const HEntry& e) {
                ++my_cands;
                const int kk = (base + wbase + owner) * kstep;
                const int m = e.len;
                if (a.policy == 2) {
                    // PrefixOnly: stored prefixes are the entries at origin 0 (R#29)
                    if (__ldg(a.slot_origin + e.slot) == 0) {
                        const int i = atomicAdd(&s_nc, 1);
                        if (i < a.nmax) clist[i] = e.slot;
                    }
                } else if ((a.policy == 0 || m == a.w) && kk + m <= n &&
                           cp_subhash(h, kk, m, __ldg(a.pw + m)) == e.full) {
                    // containment-free pool: at most one true match starts at kk (first writer wins)
                    if (atomicCAS(&vslot[kk], -1, e.slot) == -1) clist[atomicAdd(&s_nc, 1)] = kk;
                }
            });
        }
        // warp-aggregated candidate count
        for (int o = 16; o; o >>= 1) my_cands += __shfl_xor_sync(0xffffffffu, my_cands, o);
        if (lane == 0 && my_cands) atomicAdd(&s_cands, my_cands);
        __syncthreads();
        MPROF(1);
        const uint8_t* mk = a.mask ? a.mask + off : nullptr;
        if (a.policy == 2) {
            // ---- 3'. PrefixOnly: longest common prefix with each origin-0 candidate, one warp each
            if (tid == 0 && s_nc > a.nmax) cp_raise(a.hdr, CP_ERR_CAPACITY);
            const int nc = min(s_nc, a.nmax);
            for (int c = wid; c < nc; c += kNT / 32) {
                const int slot = clist[c];
                const int lim = min(__ldg(a.slot_len + slot), n);
                const int32_t* pg = a.slot_pages + (int64_t)slot * a.MP;
                int l = lim;
                for (int i0 = 0; i0 < lim; i0 += 32) {
                    const int i = i0 + lane;
                    bool stop = true;
                    if (i < lim) {
                        const int32_t et = __ldg(a.page_tokens + (int64_t)__ldg(pg + (i >> 4)) * CP_BLOCK + (i & 15));
                        stop = et != tok[i] || (mk && mk[i]);
                    }
                    const unsigned b = __ballot_sync(0xffffffffu, stop);
                    if (b) { l = i0 + __ffs(b) - 1; break; }
                }
                if (lane == 0) vslot[c] = l;
            }
            __syncthreads();
            // ---- 4'. the longest prefix, then the smaller id; covered only if >= w (R#29)
            if (wid == 0) {
                unsigned long long best = 0;
                for (int c = lane; c < nc; c += 32) {
                    const int l = vslot[c];
                    if (l < a.w) continue;
                    const unsigned long long key = ((unsigned long long)l << 32) |
                                                   (unsigned)(0x7fffffff - __ldg(a.slot_id + clist[c]));
                    best = key > best ? key : best;
                }
                for (int o = 16; o; o >>= 1) {
                    const unsigned long long y = __shfl_xor_sync(0xffffffffu, best, o);
                    best = y > best ? y : best;
                }
                if (best) {
                    for (int c = lane; c < nc; c += 32) {
                        const int l = vslot[c];
                        if (l >= a.w && (unsigned)(0x7fffffff - __ldg(a.slot_id + clist[c])) == (unsigned)(best & 0xffffffffu)) {
                            hk[0] = 0; hs[0] = clist[c]; hm[0] = l;
                        }
                    }
                }
                if (lane == 0) s_nh = best ? 1 : 0;
            }
            __syncthreads();
        } else {
        // ---- 3. exact verification.  Few candidates (the usual case: the full-hash pre-check leaves the
        //      true occurrences): work items are (candidate, 256-token chunk), dealt round-robin over the
        //      warps, so one long segment no longer runs on one warp while the others idle; a chunk that
        //      differs or covers a masked token marks its candidate (sign bit of clist).  Many candidates:
        //      one warp per candidate, stopping at the first difference.  8 tokens per lane in flight (the
        //      page-list and token-store loads of a step are issued before any compare).
        const int nc = s_nc;
        constexpr int U = 8, CHK = 32 * U, NW = kNT / 32;
        auto chunk_bad = [&](int k, const int32_t* pg, int m, int i0) -> int {
            int32_t et[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int i = i0 + 32 * u + lane;
                et[u] = i < m ? __ldg(a.page_tokens + (int64_t)__ldg(pg + (i >> 4)) * CP_BLOCK + (i & 15)) : 0;
            }
            int bad = 0;
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int i = i0 + 32 * u + lane;
                if (i < m) {
                    bad |= (et[u] != tok[k + i]);
                    if (mk) bad |= mk[k + i];
                }
            }
            return __any_sync(0xffffffffu, bad);
        };
        if (nc <= 4 * NW) {
            int gbase = 0;                                  // global index of candidate c's first chunk
            for (int c = 0; c < nc; ++c) {
                const int k = clist[c] & 0x7fffffff;
                const int slot = vslot[k];
                const int m = __ldg(a.slot_len + slot);
                const int nch = (m + CHK - 1) / CHK;
                const int first = gbase % NW;               // the warp of chunk 0
                if (wid == first && lane == 0) atomicAdd(&s_vtok, m);   // work counter: tokens a verification may compare
                const int32_t* pg = a.slot_pages + (int64_t)slot * a.MP;
                for (int ch = (wid - first + NW) % NW; ch < nch; ch += NW)
                    if (chunk_bad(k, pg, m, ch * CHK) && lane == 0) atomicOr(&clist[c], (int)0x80000000);
                gbase += nch;
            }
            __syncthreads();
            for (int c = tid; c < nc; c += kNT)
                if (clist[c] < 0) vslot[clist[c] & 0x7fffffff] = -1;
        } else {
            for (int c = wid; c < nc; c += NW) {
                const int k = clist[c];
                const int slot = vslot[k];
                const int m = __ldg(a.slot_len + slot);
                const int32_t* pg = a.slot_pages + (int64_t)slot * a.MP;
                if (lane == 0) atomicAdd(&s_vtok, m);             // work counter: tokens a verification may compare
                int bad = 0;
                for (int i0 = 0; i0 < m && !bad; i0 += CHK) bad = chunk_bad(k, pg, m, i0);
                if (bad && lane == 0) vslot[k] = -1;
            }
        }
        __syncthreads();
        MPROF(2);
        // ---- 3b. same-user session (R#33): the longest common prefix with the session's
        //      private entry (its last request, sensitive tokens included: no mask test), one hit at 0 if
        //      >= w tokens; the cross-user greedy then starts after it
        if (wid == 0) {
            int ps = -1, L = 0;
            if (a.session) {
                const int o = a.session[r];
                if (o >= 1 && o <= a.max_sessions) {
                    ps = a.session_slot[o];
                    if (ps >= 0 && !(a.slot_state[ps] == CP_SLOT_LIVE && a.slot_owner[ps] == o)) ps = -1;
                }
                if (ps >= 0) {
                    const int lim = min(__ldg(a.slot_len + ps), n);
                    const int32_t* pg = a.slot_pages + (int64_t)ps * a.MP;
                    L = lim;
                    for (int i0 = 0; i0 < lim; i0 += 32) {
                        const int i = i0 + lane;
                        const bool stop = i < lim &&
                            __ldg(a.page_tokens + (int64_t)__ldg(pg + (i >> 4)) * CP_BLOCK + (i & 15)) != tok[i];
                        const unsigned bs = __ballot_sync(0xffffffffu, stop);
                        if (bs) { L = i0 + __ffs(bs) - 1; break; }
                    }
                    if (L < a.w) { ps = -1; L = 0; }
                }
            }
            if (lane == 0) { s_pslot = ps; s_plen = L; }
        }
        __syncthreads();
        // ---- 4. greedy left-to-right assembly (warp 0)
        if (wid == 0) {
            int cursor = 0;
            if (s_pslot >= 0) {
                if (lane == 0) { hk[0] = 0; hs[0] = s_pslot; hm[0] = s_plen; }
                nh = 1;
                cursor = s_plen;
            }
            while (cursor < nw) {
                const int k = cursor + lane;
                const int v = k < nw ? vslot[k] : -1;
                const unsigned bal = __ballot_sync(0xffffffffu, v >= 0);
                if (!bal) { cursor += 32; continue; }
                const int f = __ffs(bal) - 1;
                const int kk = cursor + f;
                const int slot = __shfl_sync(0xffffffffu, v, f);
                const int m = __ldg(a.slot_len + slot);
                if (lane == 0) { hk[nh] = kk; hs[nh] = slot; hm[nh] = m; }
                ++nh;
                cursor = kk + m;
            }
            if (lane == 0) s_nh = nh;
        }
        __syncthreads();
        }   // policy != PrefixOnly
        nh = s_nh;
        // ---- 5. sparse hits + LRU touch
        const int64_t base = off / a.w + r;
        for (int i = tid; i < nh; i += kNT) {
            const int slot = hs[i];
            a.sp_entry[base + i] = __ldg(a.slot_id + slot);
            a.sp_slot[base + i] = slot;
            a.sp_dst[base + i] = hk[i];
            a.sp_len[base + i] = hm[i];
            a.sp_delta[base + i] = hk[i] - __ldg(a.slot_origin + slot);      // R#11
            if (!a.no_touch) atomicMax(a.slot_last + slot, a.clock ? *a.clock : a.t);
        }
        // ---- plan codes (0 uncovered / 1 reused / 2 recompute) and stats
        int cov = 0, rec = 0;
        for (int q = tid; q < n; q += kNT) {
            uint8_t code = CP_PLAN_UNCOVERED;
            int lo = 0, hi = nh - 1, found = -1;
            while (lo <= hi) {
                const int mid = (lo + hi) >> 1;
                if (hk[mid] <= q) { found = mid; lo = mid + 1; } else hi = mid - 1;
            }
            if (found >= 0 && q < hk[found] + hm[found]) {
                const int tt = q - hk[found];
                const int page = __ldg(a.slot_pages + (int64_t)hs[found] * a.MP + (tt >> 4));
                const int bit = (__ldg(a.page_bits + page) >> (tt & 15)) & 1;
                code = bit ? CP_PLAN_RECOMPUTE : CP_PLAN_REUSED;
                ++cov; rec += bit;
            }
            a.plan[off + q] = code;
        }
        for (int o = 16; o; o >>= 1) { cov += __shfl_xor_sync(0xffffffffu, cov, o); rec += __shfl_xor_sync(0xffffffffu, rec, o); }
        if (lane == 0) { atomicAdd(&s_cov, cov); atomicAdd(&s_rec, rec); }
        __syncthreads();
        MPROF(3);
        if (tid == 0) {
            a.req_cnt[r] = nh;
            a.req_covered[r] = s_cov; a.req_recompute[r] = s_rec; a.req_candidates[r] = s_cands;
            // work counters (O(n + c)): windows probed, prefix-filter candidates, candidates
            // through the full-hash pre-check, tokens their verification may compare
            const int nwin_w = a.policy == 0 ? max(0, n - a.w + 1) : a.policy == 1 ? n / a.w : (n >= a.w ? 1 : 0);
            atomicAdd(&a.hdr->match_work[0], (unsigned long long)nwin_w);
            atomicAdd(&a.hdr->match_work[1], (unsigned long long)s_cands);
            atomicAdd(&a.hdr->match_work[2], (unsigned long long)s_nc);
            atomicAdd(&a.hdr->match_work[3], (unsigned long long)s_vtok);
        }
    } else if (tid == 0) {
        a.req_cnt[r] = 0;
    }
    // ---- 6. last CTA: scan counts and compact into the dense output
    __threadfence();
    __syncthreads();
    if (tid == 0) s_last = (atomicAdd(&a.hdr->match_done, 1u) == (unsigned)(a.R - 1));
    __syncthreads();
    MPROF(4);
    if (!s_last) return;
    __threadfence();
    if (cp_err_set(a.hdr)) return;
    // exclusive scan over R counts in chunks of kNT; the request table (hit offset, sparse source
    // offset) is also kept in the dynamic shared memory, free by now, when it fits
    const bool tab_smem = 8 * ((size_t)a.R + 1) <= (size_t)a.dyn_smem;
    int32_t* s_off = reinterpret_cast<int32_t*>(sm);
    int32_t* s_src = s_off + (a.R + 1);
    int carry = 0;
    for (int b0 = 0; b0 < a.R; b0 += kNT) {
        const int i = b0 + tid;
        const int v = i < a.R ? *((volatile int32_t*)&a.req_cnt[i]) : 0;
        int inc = v;
        for (int o = 1; o < 32; o <<= 1) { const int y = __shfl_up_sync(0xffffffffu, inc, o); if (lane >= o) inc += y; }
        if (lane == 31) s_scan[wid] = inc;
        __syncthreads();
        if (wid == 0) {
            int x = lane < kNT / 32 ? s_scan[lane] : 0, xi = x;
            for (int o = 1; o < 32; o <<= 1) { const int y = __shfl_up_sync(0xffffffffu, xi, o); if (lane >= o) xi += y; }
            if (lane < kNT / 32) s_scan[lane] = xi - x;
            if (lane == 31) s_scan[kNT / 32] = xi;
        }
        __syncthreads();
        if (i < a.R) {
            a.req_hit_offsets[i] = carry + s_scan[wid] + inc - v;
            if (tab_smem) { s_off[i] = carry + s_scan[wid] + inc - v; s_src[i] = (int32_t)(a.offsets[i] / a.w + i); }
        }
        carry += s_scan[kNT / 32];
        __syncthreads();
    }
    if (tab_smem && tid == 0) s_off[a.R] = carry;
    if (tid == 0) {
        a.req_hit_offsets[a.R] = carry;
        if (carry > a.max_hits) cp_raise(a.hdr, CP_ERR_CAPACITY);
        else *a.num_hits = carry;
        a.hdr->match_done = 0;
    }
    __threadfence_block();
    __syncthreads();
    if (carry > a.max_hits) return;
    if (tab_smem) {
        // thread per hit: its request by binary search over the offsets, then one round trip
        for (int hh = tid; hh < carry; hh += kNT) {
            int lo = 0, hi = a.R - 1;
            while (lo < hi) { const int mid = (lo + hi + 1) >> 1; if (s_off[mid] <= hh) lo = mid; else hi = mid - 1; }
            const int64_t src = s_src[lo] + (hh - s_off[lo]);
            a.hit_req[hh] = lo;
            a.hit_entry[hh] = *((volatile int32_t*)&a.sp_entry[src]);
            a.hit_slot[hh] = *((volatile int32_t*)&a.sp_slot[src]);
            a.hit_dst[hh] = *((volatile int32_t*)&a.sp_dst[src]);
            a.hit_len[hh] = *((volatile int32_t*)&a.sp_len[src]);
            a.hit_delta[hh] = *((volatile int32_t*)&a.sp_delta[src]);
        }
        return;
    }
    for (int rr = wid; rr < a.R; rr += kNT / 32) {
        const int cnt = *((volatile int32_t*)&a.req_cnt[rr]);
        const int dst0 = a.req_hit_offsets[rr];
        const int64_t src0 = a.offsets[rr] / a.w + rr;
        for (int i = lane; i < cnt; i += 32) {
            a.hit_req[dst0 + i] = rr;
            a.hit_entry[dst0 + i] = *((volatile int32_t*)&a.sp_entry[src0 + i]);
            a.hit_slot[dst0 + i] = *((volatile int32_t*)&a.sp_slot[src0 + i]);
            a.hit_dst[dst0 + i] = *((volatile int32_t*)&a.sp_dst[src0 + i]);
            a.hit_len[dst0 + i] = *((volatile int32_t*)&a.sp_len[src0 + i]);
            a.hit_delta[dst0 + i] = *((volatile int32_t*)&a.sp_delta[src0 + i]);
        }
    }
}

}  // namespace

extern "C" cp_status cp_match_spans(cp_index* x, const cp_batch* b, uint64_t t, int32_t flags, const cp_hits* o,
                                    void* stream) {
    if (x && x->is_view) return CP_ERR_INVALID_ARG;          // views gather with their base's hits
    cp_invalidate_worklist(x);                               // it rewrites the hits a gather list was built from
    if (!x || !b || !o) return CP_ERR_INVALID_ARG;
    if ((flags & CP_MATCH_FIXED_CHUNK) && (flags & CP_MATCH_PREFIX_ONLY)) return CP_ERR_INVALID_ARG;
    if (b->num_reqs < 0 || b->num_reqs > x->cfg.max_batch_reqs || b->total_tokens > x->cfg.max_batch_tokens) return CP_ERR_INVALID_ARG;
    if (!o->num_hits || !o->req_hit_offsets || !o->hit_req || !o->hit_entry || !o->hit_slot || !o->hit_dst ||
        !o->hit_len || !o->hit_delta || !o->plan || !o->req_covered || !o->req_recompute || !o->req_candidates)
        return CP_ERR_INVALID_ARG;
    cudaStream_t st = (cudaStream_t)stream;
    if (b->num_reqs == 0) {
        CP_CUDA_CHECK(cudaMemsetAsync(o->num_hits, 0, 4, st));
        CP_CUDA_CHECK(cudaMemsetAsync(o->req_hit_offsets, 0, 4, st));
        return CP_OK;
    }
    if (!b->tokens || !b->offsets) return CP_ERR_INVALID_ARG;
    int nmax = b->max_req_len > 0 ? std::min(b->max_req_len, x->cfg.max_req_tokens) : x->cfg.max_req_tokens;
    nmax = std::max(nmax, 1);
    MatchArgs a;
    std::memset(&a, 0, sizeof(a));
    a.hdr = x->hdr; a.tokens = b->tokens; a.offsets = b->offsets; a.mask = b->mask; a.R = b->num_reqs;
    a.t = t; a.no_touch = (flags & CP_MATCH_NO_TOUCH) ? 1 : 0; a.clock = x->clock;
    a.policy = (flags & CP_MATCH_FIXED_CHUNK) ? 1 : (flags & CP_MATCH_PREFIX_ONLY) ? 2 : 0;
    a.w = x->cfg.window_len; a.B = x->B; a.Bw = x->Bw; a.pw = x->pw;
    a.htab = x->htab; a.logT = x->logT; a.T = x->T;
    a.slot_id = x->slot_id; a.slot_len = x->slot_len; a.slot_origin = x->slot_origin; a.slot_full = x->slot_full;
    a.slot_last = x->slot_last; a.slot_pages = x->slot_pages; a.MP = x->MP; a.page_tokens = x->page_tokens;
    a.page_bits = x->page_bits; a.nmax = nmax;
    a.sp_entry = x->sp_entry; a.sp_slot = x->sp_slot; a.sp_dst = x->sp_dst; a.sp_len = x->sp_len;
    a.sp_delta = x->sp_delta; a.req_cnt = x->req_cnt;
    a.max_hits = o->max_hits; a.num_hits = o->num_hits; a.req_hit_offsets = o->req_hit_offsets;
    a.hit_req = o->hit_req; a.hit_entry = o->hit_entry; a.hit_slot = o->hit_slot; a.hit_dst = o->hit_dst;
    a.hit_len = o->hit_len; a.hit_delta = o->hit_delta; a.plan = o->plan;
    a.req_covered = o->req_covered; a.req_recompute = o->req_recompute; a.req_candidates = o->req_candidates;
    if (b->session) {                              // R#33: sessions only with the method's own policy
        if (a.policy != 0 || x->cfg.max_sessions < 1) return CP_ERR_INVALID_ARG;
        a.session = b->session; a.session_slot = x->session_slot; a.slot_owner = x->slot_owner;
        a.slot_state = x->slot_state; a.max_sessions = x->cfg.max_sessions;
    }
    static int attr_set = 0;
    if (!attr_set) {
        cudaFuncSetAttribute(k_match<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 210 * 1024);
        cudaFuncSetAttribute(k_match<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 210 * 1024);
        attr_set = 1;
    }
    const bool global = nmax > CP_MATCH_SMEM_TOKENS;
    if (global && !x->match_g) return CP_ERR_UNSUPPORTED;
    // long requests: arrays in scratch; the dynamic shared memory only holds the compaction table
    const size_t smem = global ? std::min<size_t>(8 * ((size_t)b->num_reqs + 1), 48 * 1024) : MatchSmem(nmax, a.w).total;
    if (smem > 210 * 1024) return CP_ERR_UNSUPPORTED;
    a.gscr = x->match_g; a.dyn_smem = (int32_t)smem;
    CP_CUDA_CHECK(cudaMemsetAsync(&x->hdr->match_done, 0, 4, st));
    if (global) k_match<true><<<b->num_reqs, kNT, smem, st>>>(a);
    else k_match<false><<<b->num_reqs, kNT, smem, st>>>(a);
    CP_COUNT_LAUNCH();
    return cudaGetLastError() == cudaSuccess ? CP_OK : CP_ERR_CUDA;
}

#ifdef CP_MATCH_PROF
extern "C" cp_status cp_match_prof_read(unsigned long long* out_h) {
    if (cudaMemcpyFromSymbol(out_h, g_match_prof, sizeof(unsigned long long) * 8) != cudaSuccess) return CP_ERR_CUDA;
    return CP_OK;
}
#endif
