// Per-column walk budgets (replaces walker.allocate_walks / largest_remainder,
// /root/reference/pkg/src/mcfunm/walker.py:148-170) without a sort:
//   N_i = floor(p_i N_s); the residue R = N_s - sum N_i goes to the R largest
//   remainders, ties to the lowest index (the reference's stable argsort of
//   -remainder), p_i = 0 never selected ahead of p_i > 0.
// The R-th largest remainder is found by an 8-pass MSB-first radix select on
// the remainder's IEEE bits (non-negative doubles order like their bits).
#include <cstddef>
#include <cstdlib>
#include <cstring>

#include "mcf_internal.cuh"

namespace mcf {

// Largest-remainder selection without a sort:
//   1 k_alloc_floor  N_i = floor(p_i N), remainder key, Sum N_i and a 1024-bucket
//                    histogram of the remainders (floor(rem * 1024)); the last
//                    block finds the bucket b* that holds the R-th largest.
//   2 k_alloc_level2 1024 sub-buckets of b* with min/max: usually pins the
//                    threshold key T (a single distinct value) and the number
//                    I of keys == T to take.
//   3 k_alloc_cands + k_alloc_select (only when level 2 did not resolve T):
//                    one CTA, exact select among the candidates.
//   4 k_alloc_scan   one single-pass scan of the pair (a_i, b_i) =
//                    (N_i + [key_i > T], [key_i == T]): ties go to the lowest
//                    indices (the reference's stable argsort), so the final
//                    N_i = a_i + [b_i and ties before i < I] and
//                    walk_pre[i] = sum_{j<i} a_j + min(I, ties before i);
//                    the same pass fills the walk-block -> column map.
// p_i = 0 keys (0) sit below every positive remainder; they are only reached
// when R exceeds the number of positive p_i (then b* = -1 covers them).
constexpr int NBUCKET = 1024;

struct AllocState {
    unsigned long long total_floor;  // sum of floor(p N)
    unsigned long long n_pos;        // entries with p > 0
    long long left;                  // residue R
    long long need;                  // to take inside bucket b*
    int bstar;                       // bucket holding the R-th largest (-1: the p == 0 keys)
    unsigned done;
    unsigned ncand;
    unsigned long long T;            // threshold key
    long long I;                     // how many of the keys == T to take (lowest indices)
    unsigned long long ncmin, cmax;  // ~(smallest candidate key), largest candidate key
    int b2;                          // sub-bucket of b* holding the R-th largest (-1: none / not refined)
    int resolved;                    // T and the tie count are known (no candidate pass needed)
    unsigned hist[NBUCKET];
    unsigned hist2[NBUCKET];
    unsigned long long nmin2[NBUCKET], max2[NBUCKET];  // ~min / max key per sub-bucket (zero-initialised)
};

// N_i = floor(p_i N) and the remainder key (IEEE bits of the remainder + 1;
// 0 for p_i = 0), recomputed from p by every pass instead of stored
__device__ __forceinline__ void floor_key(double pi, double total, long long &got, unsigned long long &k) {
    const double want = __dmul_rn(pi, total);
    const double fl = floor(want);
    got = (long long)fl;
    k = pi != 0.0 ? (unsigned long long)__double_as_longlong(__dsub_rn(want, fl)) + 1ull : 0ull;
}

__device__ __forceinline__ int rem_bucket(unsigned long long key) {
    if (key == 0) return -1;
    const double rem = __longlong_as_double((long long)(key - 1));
    const int b = (int)(rem * NBUCKET);
    return b < NBUCKET ? b : NBUCKET - 1;
}

// second level: position inside bucket b (monotone in the remainder)
__device__ __forceinline__ int rem_sub(unsigned long long key, int b) {
    const double rem = __longlong_as_double((long long)(key - 1));
    const int s = (int)((rem * NBUCKET - b) * NBUCKET);
    return s < 0 ? 0 : (s < NBUCKET ? s : NBUCKET - 1);
}

// top-down search over 1024 counts held 4 per thread (256 threads): the bin
// with count(above) < R <= count(above) + count(bin); returns via *bin/*need
__device__ void find_bin(const unsigned *cnt, long long R, int *bin, long long *need) {
    __shared__ long long wsum[8];
    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
    long long c4[4], own = 0;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        c4[u] = (long long)atomicAdd(const_cast<unsigned *>(&cnt[NBUCKET - 1 - (4 * t + u)]), 0u);
        own += c4[u];
    }
    long long x = own;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        long long y = __shfl_up_sync(MCF_FULL, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) wsum[w] = x;
    __syncthreads();
    long long above = x - own;
    for (int j = 0; j < w; ++j) above += wsum[j];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        if (above < R && R <= above + c4[u]) {
            *bin = NBUCKET - 1 - (4 * t + u);
            *need = R - above;
        }
        above += c4[u];
    }
    __syncthreads();
}

// block-parallel search from the top bucket: thread t holds bucket NBUCKET-1-t*4..; finds b with
// count(above b) < R <= count(above b) + hist[b]
__global__ void __launch_bounds__(256, 4) k_alloc_floor(const double *__restrict__ p, long long n, double total,
                                                        long long n_walks, AllocState *st) {
    __shared__ unsigned h[NBUCKET];
    __shared__ bool last;
    for (int b = threadIdx.x; b < NBUCKET; b += blockDim.x) h[b] = 0;
    __syncthreads();
    long long got_sum = 0, pos = 0;
    const long long stride = (long long)gridDim.x * blockDim.x;
    // warp-uniform trip count (the bucket vote below is warp-wide)
    for (long long w0 = (long long)blockIdx.x * blockDim.x + (threadIdx.x & ~31); w0 < n; w0 += 4 * stride) {
        const long long i0 = w0 + (threadIdx.x & 31);
        double pv[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) pv[u] = i0 + u * stride < n ? p[i0 + u * stride] : 0.0;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const long long i = i0 + u * stride;
            long long got;
            unsigned long long k;
            floor_key(pv[u], total, got, k);
            const int bk = (i < n && k) ? rem_bucket(k) : -1;
            const int b0 = __shfl_sync(MCF_FULL, bk, 0);
            if (__all_sync(MCF_FULL, bk == b0)) {  // equal-degree runs share a bucket
                if ((threadIdx.x & 31) == 0 && b0 >= 0) atomicAdd(&h[b0], 32u);
            } else if (bk >= 0) {
                atomicAdd(&h[bk], 1u);
            }
            if (i < n) {
                got_sum += got;
                pos += k ? 1 : 0;
            }
        }
    }
    got_sum = warp_sum_ll(got_sum);  // one global atomic per CTA, not per warp
    pos = warp_sum_ll(pos);
    __shared__ unsigned long long cta_sum[2];
    if (threadIdx.x < 2) cta_sum[threadIdx.x] = 0;
    __syncthreads();
    if ((threadIdx.x & 31) == 0) {
        if (got_sum) atomicAdd(&cta_sum[0], (unsigned long long)got_sum);
        if (pos) atomicAdd(&cta_sum[1], (unsigned long long)pos);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        if (cta_sum[0]) atomicAdd(&st->total_floor, cta_sum[0]);
        if (cta_sum[1]) atomicAdd(&st->n_pos, cta_sum[1]);
    }
    for (int b = threadIdx.x; b < NBUCKET; b += blockDim.x)
        if (h[b]) atomicAdd(&st->hist[b], h[b]);
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(&st->done, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!last) return;
    __threadfence();
    const long long R = n_walks - (long long)atomicAdd(&st->total_floor, 0ull);
    const long long npos = (long long)atomicAdd(&st->n_pos, 0ull);
    if (threadIdx.x == 0) {
        st->left = R;
        st->bstar = -2;  // nothing to select
        st->need = 0;
        st->done = 0;
        st->ncand = 0;
        st->b2 = -1;
        st->resolved = 0;
        if (R > npos) {  // every positive key, plus the lowest-index p == 0 entries
            st->bstar = -1;
            st->need = R - npos;
            st->T = 0;
            st->I = R - npos;
            st->resolved = 1;
        }
    }
    __syncthreads();
    if (R > 0 && R <= npos) find_bin(st->hist, R, &st->bstar, &st->need);
}

// Level 2: histogram of bucket b* into 1024 sub-buckets with per-sub-bucket
// min/max key; the last block picks the sub-bucket, and if it holds a single
// distinct value (the usual case: equal-degree ties) T is resolved here.
__global__ void __launch_bounds__(256, 4) k_alloc_level2(const double *__restrict__ p, long long n, double total,
                                                         AllocState *st) {
    __shared__ unsigned h[NBUCKET];
    __shared__ unsigned long long mn[NBUCKET], mx[NBUCKET];
    __shared__ bool last;
    const int bstar = st->bstar;
    if (bstar < 0) return;
    for (int b = threadIdx.x; b < NBUCKET; b += blockDim.x) {
        h[b] = 0;
        mn[b] = ~0ull;
        mx[b] = 0;
    }
    __syncthreads();
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long base = (long long)blockIdx.x * blockDim.x; base < n; base += 4 * stride) {
        double pv[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const long long i = base + u * stride + threadIdx.x;
            pv[u] = i < n ? p[i] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            long long got;
            unsigned long long k;
            floor_key(pv[u], total, got, k);
            const bool in = k && rem_bucket(k) == bstar;
            const int sb = in ? rem_sub(k, bstar) : -1;
            const int s0 = __shfl_sync(MCF_FULL, sb, 0);
            const unsigned long long k0 = __shfl_sync(MCF_FULL, k, 0);
            if (__all_sync(MCF_FULL, in && k == k0)) {  // one tied key across the warp
                if ((threadIdx.x & 31) == 0) {
                    atomicAdd(&h[s0], 32u);
                    atomicMin(&mn[s0], k0);
                    atomicMax(&mx[s0], k0);
                }
            } else if (in) {
                atomicAdd(&h[sb], 1u);
                atomicMin(&mn[sb], k);
                atomicMax(&mx[sb], k);
            }
        }
    }
    __syncthreads();
    for (int b = threadIdx.x; b < NBUCKET; b += blockDim.x) {
        if (h[b]) {
            atomicAdd(&st->hist2[b], h[b]);
            atomicMax(&st->nmin2[b], ~mn[b]);
            atomicMax(&st->max2[b], mx[b]);
        }
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(&st->done, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!last) return;
    __threadfence();
    int b2 = -1;
    long long need2 = 0;
    __shared__ int s_b2;
    __shared__ long long s_need2;
    if (threadIdx.x == 0) s_b2 = -1;
    __syncthreads();
    find_bin(st->hist2, st->need, &s_b2, &s_need2);
    b2 = s_b2;
    need2 = s_need2;
    if (threadIdx.x == 0) {
        st->b2 = b2;
        st->need = need2;
        const unsigned long long lo = ~atomicAdd(&st->nmin2[b2], 0ull), hi = atomicMax(&st->max2[b2], 0ull);
        if (lo == hi) {  // single distinct value: it is the threshold
            st->T = lo;
            st->I = need2;
            st->resolved = 1;
        }
    }
}

__global__ void k_alloc_cands(const double *__restrict__ p, long long n, double total, AllocState *st,
                              unsigned long long *__restrict__ ckey) {
    const int bstar = st->bstar, b2 = st->b2;
    if (bstar < 0 || st->resolved) return;
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long base = (long long)blockIdx.x * blockDim.x; base < n; base += stride) {
        const long long i = base + threadIdx.x;
        long long got;
        unsigned long long kk = 0;
        if (i < n) floor_key(p[i], total, got, kk);
        const bool in = kk && rem_bucket(kk) == bstar && rem_sub(kk, bstar) == b2;
        const unsigned m = __ballot_sync(MCF_FULL, in);
        if (!m) continue;
        unsigned pos = 0;
        if ((threadIdx.x & 31) == 0) pos = atomicAdd(&st->ncand, (unsigned)__popc(m));
        pos = __shfl_sync(MCF_FULL, pos, 0);
        unsigned long long mn = in ? kk : ~0ull, mx = in ? kk : 0ull;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const unsigned long long a = __shfl_xor_sync(MCF_FULL, mn, o), b = __shfl_xor_sync(MCF_FULL, mx, o);
            mn = a < mn ? a : mn;
            mx = b > mx ? b : mx;
        }
        if ((threadIdx.x & 31) == 0) {
            atomicMax(&st->ncmin, ~mn);
            atomicMax(&st->cmax, mx);
        }
        if (in) ckey[pos + __popc(m & lanemask_lt())] = kk;
    }
}

// Exact k-th largest key among the C candidates (MSB-first 8-bit radix).
// Ties are the common case (equal-degree nodes share p): a bucket holding one
// distinct value is answered from the min/max, and warps whose keys share a
// digit add once.  The index tie-break is a scan afterwards.
__global__ void __launch_bounds__(1024) k_alloc_select(const unsigned long long *__restrict__ ckey, AllocState *st) {
    __shared__ unsigned h[256];
    __shared__ unsigned long long s_pre, s_mask;
    __shared__ long long s_k;
    __shared__ long long wsum[32];
    if (st->bstar == -2 || st->resolved) return;
    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
    if (~st->ncmin == st->cmax) {  // a single distinct value: it is the threshold
        if (t == 0) {
            st->T = st->cmax;
            st->I = st->need;
        }
        return;
    }
    const unsigned C = st->ncand;
    // (1) distinct values with their counts in a shared hash (ties are few, large groups)
    constexpr int HS = 2048;
    __shared__ unsigned long long hk[HS];
    __shared__ unsigned hc[HS];
    __shared__ unsigned s_nd;
    __shared__ int s_over;
    for (int j = t; j < HS; j += blockDim.x) {
        hk[j] = ~0ull;
        hc[j] = 0;
    }
    if (t == 0) {
        s_nd = 0;
        s_over = 0;
    }
    __syncthreads();
    for (unsigned base = 0; base < C && !s_over; base += blockDim.x) {
        const unsigned c = base + t;
        const bool valid = c < C;
        const unsigned long long k = valid ? ckey[c] : 0ull;
        const unsigned m = __ballot_sync(MCF_FULL, valid);
        const unsigned long long d0 = __shfl_sync(MCF_FULL, k, 0);
        const bool same = __all_sync(MCF_FULL, !valid || k == d0);
        if (same ? (lane == 0) : valid) {
            const unsigned cnt = same ? (unsigned)__popc(m) : 1u;
            const unsigned long long kk = same ? d0 : k;
            unsigned slot = (unsigned)((kk * 0x9E3779B97F4A7C15ull) >> 53);  // 11 bits
            for (int probe = 0; probe < HS; ++probe) {
                unsigned long long cur = hk[slot];
                if (cur == ~0ull) {
                    cur = atomicCAS(&hk[slot], ~0ull, kk);
                    if (cur == ~0ull) {
                        if (atomicAdd(&s_nd, 1u) >= HS / 2) s_over = 1;
                        cur = kk;
                    }
                }
                if (cur == kk) {
                    atomicAdd(&hc[slot], cnt);
                    break;
                }
                slot = (slot + 1) & (HS - 1);
            }
        }
        __syncthreads();
    }
    __syncthreads();
    if (!s_over) {
        // the k-th largest: count above each distinct value (distinct values <= HS/2)
        const long long need = st->need;
        for (int j = t; j < HS; j += blockDim.x) {
            const unsigned long long v = hk[j];
            if (v == ~0ull) continue;
            long long above = 0;
            for (int f = 0; f < HS; ++f)
                if (hk[f] != ~0ull && hk[f] > v) above += hc[f];
            if (above < need && need <= above + (long long)hc[j]) {
                st->T = v;
                st->I = need - above;
            }
        }
        return;
    }
    // (2) fallback: exact MSB-first radix over the candidates
    if (t == 0) {
        s_pre = 0;
        s_mask = 0;
        s_k = st->need;
    }
    for (int shift = 56; shift >= 0; shift -= 8) {
        if (t < 256) h[t] = 0;
        __syncthreads();
        const unsigned long long pre = s_pre, msk = s_mask;
        for (unsigned base = 0; base < C; base += blockDim.x) {  // warp-uniform trip count
            const unsigned c = base + t;
            const unsigned long long k = c < C ? ckey[c] : ~0ull;
            const bool in = c < C && (k & msk) == pre;
            const unsigned dig = in ? (unsigned)((k >> shift) & 255u) : 256u;
            const unsigned d0 = __shfl_sync(MCF_FULL, dig, 0);
            if (__all_sync(MCF_FULL, dig == d0)) {
                if (lane == 0 && d0 < 256u) atomicAdd(&h[d0], 32u);
            } else if (in) {
                atomicAdd(&h[dig], 1u);
            }
        }
        __syncthreads();
        long long own = t < 256 ? h[255 - t] : 0;  // bins from the top (largest keys first)
        long long x = own;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            long long y = __shfl_up_sync(MCF_FULL, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) wsum[w] = x;
        __syncthreads();
        long long before = x - own;
        for (int j = 0; j < w; ++j) before += wsum[j];
        const long long k = s_k;
        __syncthreads();
        if (t < 256 && before < k && k <= before + own) {
            s_pre = pre | ((unsigned long long)(255 - t) << shift);
            s_mask = msk | (255ull << shift);
            s_k = k - before;
        }
        __syncthreads();
    }
    if (t == 0) {
        st->T = s_pre;
        st->I = s_k;  // ties (key == T) to take, lowest indices first
    }
}

__global__ void __launch_bounds__(SCAN_T, 2) k_alloc_scan(const double *__restrict__ p, long long n, double total,
                                                          const AllocState *st, long long *__restrict__ ni,
                                                          long long *__restrict__ walk_pre, int *__restrict__ blk_col,
                                                          unsigned long long *sa, unsigned long long *sb,
                                                          unsigned *tile_ctr) {
    __shared__ unsigned s_tile;
    if (threadIdx.x == 0) s_tile = atomicAdd(tile_ctr, 1u);
    __syncthreads();
    const long long tile = s_tile;
    const bool select = st->bstar != -2;
    const unsigned long long T = select ? st->T : 0ull;
    const long long I = select ? st->I : 0;
    const long long base = tile * SCAN_TILE + (long long)(threadIdx.x >> 5) * 32 * SCAN_I + (threadIdx.x & 31);
    long long a[SCAN_I], b[SCAN_I], ea[SCAN_I], eb[SCAN_I];
#pragma unroll
    for (int k = 0; k < SCAN_I; ++k) {
        const long long j = base + 32 * k;
        a[k] = b[k] = 0;
        if (j < n) {
            long long got;
            unsigned long long kj;
            floor_key(p[j], total, got, kj);
            a[k] = got + ((select && kj > T) ? 1 : 0);
            b[k] = (select && kj == T) ? 1 : 0;
        }
    }
    tile_scan<true>(tile, a, b, ea, eb, sa, sb);
    constexpr long long B = 1ll << WALK_BLK_SHIFT;
#pragma unroll
    for (int k = 0; k < SCAN_I; ++k) {
        const long long j = base + 32 * k;
        if (j < n) {
            const long long nj = a[k] + ((b[k] && eb[k] < I) ? 1 : 0);
            const long long w0 = ea[k] + (eb[k] < I ? eb[k] : I);
            if (ni) ni[j] = nj;
            walk_pre[j] = w0;
            if (blk_col)
                for (long long blk = (w0 + B - 1) >> WALK_BLK_SHIFT; blk * B < w0 + nj; ++blk) blk_col[blk] = (int)j;
            if (j == n - 1) {
                const long long tb = eb[k] + b[k];
                walk_pre[n] = ea[k] + a[k] + (tb < I ? tb : I);
            }
        }
    }
}

// ---------------------------------------------------------------------------
// The whole allocation in ONE persistent kernel (n <= sm_count * 1024 * 8):
// one CTA per SM, every lane keeps its p values in registers (warp-striped,
// coalesced), and the passes above become phases separated by grid barriers:
//   phase 1  floor sums + remainder-value histogram (1024 buckets)
//   phase 2  refinement levels: every CTA reads the merged histogram, finds
//            the bin holding the R-th largest key (redundantly, identically),
//            and, unless that bin holds one distinct key, histograms the bin's
//            key range 1024-way again (<= 7 levels for 64-bit keys)
//   phase 3  the (N_i + [key > T], [key == T]) scan: warp and CTA totals,
//            CTA prefixes after one more barrier, then N_i, walk_pre and the
//            walk-block map.
// p is read once; no other kernel runs.  The grid never exceeds one CTA per
// SM, so every CTA is resident and the spin barriers cannot deadlock.
// ---------------------------------------------------------------------------
constexpr int AF_T = 1024, AF_W = AF_T / 32, AF_KMAX = 8, AF_LEVELS = 8, AF_MAXG = 1024;
constexpr int AF_REP = 8;    // replicas of the merged level-0 counts: CTA c adds into copy c % 8
constexpr int AF_REP_L = 8;  // replicas of the refinement levels

struct AllocFused {
    // ---- zeroed by the host (cudaMemsetAsync up to `lvl`)
    unsigned bar;
    unsigned pad_[31];
    unsigned flag;  // own 128-B line
    unsigned pad2_[31];
    unsigned cnt0[AF_REP][NBUCKET];  // level 0: remainder-value buckets
    unsigned long long trace[32];    // MCF_ALLOC_TRACE builds: CTA 0 phase timestamps
    // ---- refinement levels, zeroed by the CTAs during phase 1 (first used after barrier 1)
    struct Level {
        unsigned cnt[AF_REP_L][NBUCKET];
        unsigned long long nmin[AF_REP_L][NBUCKET], max[AF_REP_L][NBUCKET];  // ~min, max key per bin
    } lvl[AF_LEVELS];
    long long blk_a[AF_MAXG], blk_b[AF_MAXG];  // written before they are read
};

#ifdef MCF_ALLOC_TRACE
#define AF_TRACE(F, i)                                                              \
    do {                                                                            \
        if (blockIdx.x == 0 && threadIdx.x == 0) {                                  \
            unsigned long long t_;                                                  \
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                  \
            (F)->trace[i] = t_;                                                     \
        }                                                                           \
    } while (0)
#else
#define AF_TRACE(F, i) \
    do {               \
    } while (0)
#endif

// Grid barrier: arrivals count on one word, the last arriver publishes the
// phase on a flag in another line, and the other CTAs poll only that flag
// (with back-off) -- polling the counter itself slows the arrivals down.
__device__ __forceinline__ void grid_barrier(unsigned *bar, unsigned *flag, unsigned phase, unsigned G) {
    __syncthreads();  // the CTA's writes happen-before thread 0's release below
    if (threadIdx.x == 0) {
        unsigned old;
        asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(bar) : "memory");
        if (old == G * phase - 1) {
            asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(flag), "r"(phase) : "memory");
        } else {
            while (true) {
                unsigned v;
                asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory");
                if (v >= phase) break;
                __nanosleep(64);
            }
        }
    }
    __syncthreads();
}

// 1024 bins, one per thread, searched from the top: the bin with
// count(above) < R <= count(above) + count(bin).  Every thread gets the answer.
template <int REP>
__device__ __forceinline__ void find_bin_all(const unsigned (*cnt)[NBUCKET], long long R, int &bin, long long &need) {
    __shared__ long long wt[AF_W];
    __shared__ int s_bin;
    __shared__ long long s_need;
    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
    const int b = NBUCKET - 1 - t;
    long long c = 0;
#pragma unroll
    for (int r = 0; r < REP; ++r) c += (long long)__ldcg(cnt[r] + b);
    const long long inc = warp_incl_scan(c);
    if (lane == 31) wt[w] = inc;
    if (t == 0) s_bin = -1;
    __syncthreads();
    long long above = inc - c;
    for (int j = 0; j < w; ++j) above += wt[j];
    if (above < R && R <= above + c) {
        s_bin = b;
        s_need = R - above;
    }
    __syncthreads();
    bin = s_bin;
    need = s_need;
    __syncthreads();
}

// OnesR (optional, funm_action with v = 1): the same pass also writes
// r = A 1 (the row sums; rows holding a negative value summed with signs)
// into r and the walk headers, and zeroes the walk statistics -- so one
// kernel prepares everything the walks need.
struct OnesR {
    NodeHdr *hdr;
    const double *vals;
    double *r;
    long long *stats;
};

__global__ void __launch_bounds__(AF_T, 1) k_alloc_fused(const double *__restrict__ p, long long n, double total,
                                                        long long n_walks, int K, AllocFused *F,
                                                        long long *__restrict__ ni, long long *__restrict__ walk_pre,
                                                        int *__restrict__ blk_col, OnesR ones) {
    __shared__ unsigned h[NBUCKET];
    __shared__ unsigned long long smn[NBUCKET], smx[NBUCKET];
    __shared__ long long s_wa[AF_W], s_wb[AF_W], s_pa, s_pb;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const unsigned G = gridDim.x;
    const long long base = ((long long)blockIdx.x * AF_W + w) * 32 * K + lane;
    AF_TRACE(F, 0);
#ifdef MCF_ALLOC_TRACE
    if (threadIdx.x == 0) {
        unsigned long long t_;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));
        atomicMax(&F->trace[28], t_);  // last CTA to start
    }
#endif
    double pv[AF_KMAX];
#pragma unroll
    for (int k = 0; k < AF_KMAX; ++k) {
        const long long j = base + 32ll * k;
        pv[k] = (k < K && j < n) ? p[j] : -1.0;  // -1: padding
    }
    if (ones.stats && blockIdx.x == 0 && threadIdx.x < 4) ones.stats[threadIdx.x] = 0;
    if (ones.r) {  // r = A 1 for the same rows (warp-striped, coalesced header reads)
#pragma unroll
        for (int k = 0; k < AF_KMAX; ++k) {
            const long long j = base + 32ll * k;
            if (k >= K || j >= n) break;
            const NodeHdr hj = load_hdr(ones.hdr + j);
            double rs = hj.deg ? hj.rsum : 0.0;
            if (hj.flags & HDR_HAS_NEG) {
                rs = 0.0;
                for (int t = 0; t < hj.deg; ++t) rs = __dadd_rn(rs, ones.vals[hj.start + t]);
            }
            ones.r[j] = rs;
            ones.hdr[j].aux = rs;
        }
    }
    // ---- phase 1: floor sums, remainder buckets ------------------------------
    for (int b = threadIdx.x; b < NBUCKET; b += AF_T) h[b] = 0;
    __syncthreads();
    long long fsum = 0, pos = 0;
#pragma unroll
    for (int k = 0; k < AF_KMAX; ++k) {
        if (k >= K) break;
        long long got = 0;
        unsigned long long key = 0;
        if (pv[k] >= 0.0) floor_key(pv[k], total, got, key);
        fsum += got;
        if (key) {
            ++pos;
            atomicAdd(&h[rem_bucket(key)], 1u);
        }
    }
    fsum = warp_sum_ll(fsum);  // CTA totals to per-CTA slots (no same-address atomics)
    pos = warp_sum_ll(pos);
    if (lane == 0) {
        s_wa[w] = fsum;
        s_wb[w] = pos;
    }
    __syncthreads();
    if (w == 0) {
        const long long a = warp_sum_ll(lane < AF_W ? s_wa[lane] : 0), b = warp_sum_ll(lane < AF_W ? s_wb[lane] : 0);
        if (lane == 0) {
            F->blk_a[blockIdx.x] = a;
            F->blk_b[blockIdx.x] = b;
        }
    }
#ifdef MCF_ALLOC_TRACE
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long t_;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));
        atomicMax(&F->trace[29], t_);  // last CTA done with its shared histogram
    }
#endif
#ifndef MCF_ALLOC_NOFLUSH
    for (int b = threadIdx.x; b < NBUCKET; b += AF_T)
        if (h[b]) atomicAdd(&F->cnt0[blockIdx.x % AF_REP][b], h[b]);
    {  // zero the refinement levels (1.1 MB) while the other CTAs finish phase 1
        uint4 *z = reinterpret_cast<uint4 *>(&F->lvl[0]);
        const long long words = (long long)sizeof(F->lvl) / 16;
        for (long long i = (long long)blockIdx.x * AF_T + threadIdx.x; i < words; i += (long long)G * AF_T)
            z[i] = make_uint4(0, 0, 0, 0);
    }
#endif
#ifdef MCF_ALLOC_TRACE
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long t_;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));
        atomicMax(&F->trace[30], t_);  // last CTA done flushing
    }
#endif
    AF_TRACE(F, 1);
    unsigned phase = 1;
    grid_barrier(&F->bar, &F->flag, phase, G);
    ++phase;
    AF_TRACE(F, 2);
    // ---- phase 2: the threshold key T and the ties to take I -----------------
    {
        long long a = 0, b = 0;
        for (int j = threadIdx.x; j < (int)G; j += AF_T) {
            a += __ldcg(&F->blk_a[j]);
            b += __ldcg(&F->blk_b[j]);
        }
        a = warp_sum_ll(a);
        b = warp_sum_ll(b);
        if (lane == 0) {
            s_wa[w] = a;
            s_wb[w] = b;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            long long sa = 0, sb = 0;
            for (int j = 0; j < AF_W; ++j) {
                sa += s_wa[j];
                sb += s_wb[j];
            }
            s_pa = sa;
            s_pb = sb;
        }
        __syncthreads();
    }
    const long long R = n_walks - s_pa;  // sum of floor(p N)
    const long long npos = s_pb;        // entries with p > 0
    __syncthreads();
    unsigned long long T = ~0ull;  // R == 0: nothing selected
    long long I = 0;
    if (R > npos) {  // every positive key, then the lowest-index p == 0 entries
        T = 0;
        I = R - npos;
    } else if (R > 0) {
        int bin;
        long long need;
        find_bin_all<AF_REP>(F->cnt0, R, bin, need);
        // bucket b holds the remainders in [b/1024, (b+1)/1024) (exact: the
        // scaling by 1024 is a power of two), i.e. these keys:
        unsigned long long lo = (unsigned long long)__double_as_longlong((double)bin / NBUCKET) + 1ull;
        unsigned long long hi = (unsigned long long)__double_as_longlong((double)(bin + 1) / NBUCKET);
        for (int lvl = 1; lo != hi && lvl < AF_LEVELS; ++lvl) {
            const unsigned long long width = (hi - lo) / NBUCKET + 1;
            for (int b = threadIdx.x; b < NBUCKET; b += AF_T) {
                h[b] = 0;
                smn[b] = ~0ull;
                smx[b] = 0;
            }
            __syncthreads();
            // tied keys are the common case here: a warp counts a run of one key
            // in registers and updates shared memory once per run (every warp
            // hitting the same three shared words per item serialised the CTA)
            unsigned long long run_key = 0;
            unsigned run_cnt = 0;
#pragma unroll
            for (int k = 0; k < AF_KMAX; ++k) {
                if (k >= K) break;
                long long got;
                unsigned long long key = 0;
                if (pv[k] > 0.0) floor_key(pv[k], total, got, key);
                const bool in = key && key >= lo && key <= hi;
                const unsigned m = __ballot_sync(MCF_FULL, in);
                if (!m) continue;
                const unsigned long long k0 = __shfl_sync(MCF_FULL, key, __ffs(m) - 1);
                if (__all_sync(MCF_FULL, !in || key == k0)) {
                    if (k0 != run_key) {
                        if (run_cnt && lane == 0) {
                            const int bk = (int)((run_key - lo) / width);
                            atomicAdd(&h[bk], run_cnt);
                            atomicMin(&smn[bk], run_key);
                            atomicMax(&smx[bk], run_key);
                        }
                        run_key = k0;
                        run_cnt = 0;
                    }
                    run_cnt += __popc(m);
                } else {
                    const unsigned grp = __match_any_sync(MCF_FULL, in ? key : 0ull);
                    if (in && lane == __ffs(grp) - 1) {
                        const int bk = (int)((key - lo) / width);
                        atomicAdd(&h[bk], (unsigned)__popc(grp));
                        atomicMin(&smn[bk], key);
                        atomicMax(&smx[bk], key);
                    }
                }
            }
            if (run_cnt && lane == 0) {
                const int bk = (int)((run_key - lo) / width);
                atomicAdd(&h[bk], run_cnt);
                atomicMin(&smn[bk], run_key);
                atomicMax(&smx[bk], run_key);
            }
            __syncthreads();
            for (int b = threadIdx.x; b < NBUCKET; b += AF_T) {
                if (h[b]) {
                    const int rep = blockIdx.x % AF_REP_L;
                    atomicAdd(&F->lvl[lvl].cnt[rep][b], h[b]);
                    atomicMax(&F->lvl[lvl].nmin[rep][b], ~smn[b]);
                    atomicMax(&F->lvl[lvl].max[rep][b], smx[b]);
                }
            }
            AF_TRACE(F, 2 + 2 * lvl - 1);
#ifdef MCF_ALLOC_TRACE
            __syncthreads();
            if (threadIdx.x == 0 && lvl == 1) {
                unsigned long long t_;
                asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));
                atomicMax(&F->trace[27], t_);  // last CTA done with level 1
            }
#endif
            grid_barrier(&F->bar, &F->flag, phase, G);
    ++phase;
            AF_TRACE(F, 2 + 2 * lvl);
            find_bin_all<AF_REP_L>(F->lvl[lvl].cnt, need, bin, need);
            unsigned long long nmn = 0, mx = 0;
#pragma unroll
            for (int r = 0; r < AF_REP_L; ++r) {
                const unsigned long long a = __ldcg(&F->lvl[lvl].nmin[r][bin]), b = __ldcg(&F->lvl[lvl].max[r][bin]);
                nmn = a > nmn ? a : nmn;
                mx = b > mx ? b : mx;
            }
            lo = ~nmn;
            hi = mx;
        }
        T = lo;  // a single distinct key remains (64-bit keys need <= 7 levels)
        I = need;
    }
    AF_TRACE(F, 20);
    // ---- phase 3: N_i and walk_pre -----------------------------------------
    long long ta = 0, tb = 0;
#pragma unroll
    for (int k = 0; k < AF_KMAX; ++k) {
        if (k >= K) break;
        if (pv[k] < 0.0) continue;
        long long got;
        unsigned long long key;
        floor_key(pv[k], total, got, key);
        ta += got + (key > T ? 1 : 0);
        tb += key == T ? 1 : 0;
    }
    ta = warp_sum_ll(ta);
    tb = warp_sum_ll(tb);
    if (lane == 0) {
        s_wa[w] = ta;
        s_wb[w] = tb;
    }
    __syncthreads();
    if (w == 0) {  // exclusive warp offsets inside the CTA, CTA totals to global
        const long long va = lane < AF_W ? s_wa[lane] : 0, vb = lane < AF_W ? s_wb[lane] : 0;
        const long long ia = warp_incl_scan(va), ib = warp_incl_scan(vb);
        if (lane < AF_W) {
            s_wa[lane] = ia - va;
            s_wb[lane] = ib - vb;
        }
        if (lane == 31) {
            F->blk_a[blockIdx.x] = ia;
            F->blk_b[blockIdx.x] = ib;
        }
    }
    AF_TRACE(F, 21);
    grid_barrier(&F->bar, &F->flag, phase, G);
    ++phase;
    AF_TRACE(F, 22);
    {  // CTA prefix: sum of the totals of the CTAs before this one
        long long a = 0, b = 0;
        for (int j = threadIdx.x; j < (int)blockIdx.x; j += AF_T) {
            a += __ldcg(&F->blk_a[j]);
            b += __ldcg(&F->blk_b[j]);
        }
        a = warp_sum_ll(a);
        b = warp_sum_ll(b);
        __shared__ long long s_ra[AF_W], s_rb[AF_W];
        if (lane == 0) {
            s_ra[w] = a;
            s_rb[w] = b;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            long long sa = 0, sb = 0;
            for (int j = 0; j < AF_W; ++j) {
                sa += s_ra[j];
                sb += s_rb[j];
            }
            s_pa = sa;
            s_pb = sb;
        }
        __syncthreads();
    }
    long long ra = s_pa + s_wa[w], rb = s_pb + s_wb[w];
    constexpr long long B = 1ll << WALK_BLK_SHIFT;
#pragma unroll
    for (int k = 0; k < AF_KMAX; ++k) {
        if (k >= K) break;
        const long long j = base + 32ll * k;
        long long a = 0, t = 0;
        if (pv[k] >= 0.0) {
            long long got;
            unsigned long long key;
            floor_key(pv[k], total, got, key);
            a = got + (key > T ? 1 : 0);
            t = key == T ? 1 : 0;
        }
        const long long xa = warp_incl_scan(a), xb = warp_incl_scan(t);
        const long long ea = ra + xa - a, eb = rb + xb - t;
        if (j < n) {
            const long long nj = a + ((t && eb < I) ? 1 : 0);
            const long long w0 = ea + (eb < I ? eb : I);
            if (ni) ni[j] = nj;
            walk_pre[j] = w0;
            if (blk_col)
                for (long long blk = (w0 + B - 1) >> WALK_BLK_SHIFT; blk * B < w0 + nj; ++blk) blk_col[blk] = (int)j;
            if (j == n - 1) walk_pre[n] = ea + a + (eb + t < I ? eb + t : I);
        }
        ra += __shfl_sync(MCF_FULL, xa, 31);
        rb += __shfl_sync(MCF_FULL, xb, 31);
    }
    AF_TRACE(F, 23);
}

// fused_scratch: caller-provided AllocFused whose first fused_scratch_zero_bytes()
// are already zero (one memset for several scratch blocks), or null
static int allocate(mcf_graph *g, long long n_walks, long long *ni, long long *walk_pre, int *blk_col,
                    cudaStream_t s, void *fused_scratch = nullptr, double *r_ones = nullptr,
                    long long *stats_zero = nullptr) {
    MCF_ARG(g && walk_pre, "mcf_allocate_walks: null argument");  // ni may be null internally (not stored)
    MCF_ARG(n_walks >= 1, "n_walks must be at least 1");  // walker.py:168-169
    MCF_ARG(n_walks < (1ll << 53), "n_walks must be below 2^53");
    const long long n = g->n;
    if (n == 0) {
        MCF_CUDA(cudaMemsetAsync(walk_pre, 0, sizeof(long long), s));
        return MCF_OK;
    }
    const char *path = getenv("MCF_ALLOC_PATH");
    const int G = sm_count() < AF_MAXG ? sm_count() : AF_MAXG;
    const long long K = (n + (long long)G * AF_T - 1) / ((long long)G * AF_T);
    if (K <= AF_KMAX && !(path && !strcmp(path, "passes"))) {  // one persistent kernel
        const bool own = fused_scratch == nullptr;
        AllocFused *F = reinterpret_cast<AllocFused *>(fused_scratch);
        if (own) {
            MCF_CUDA(cudaMallocAsync(&F, sizeof(AllocFused), s));
            MCF_CUDA(cudaMemsetAsync(F, 0, offsetof(AllocFused, lvl), s));
        }
        k_alloc_fused<<<G, AF_T, 0, s>>>(g->init_prob, n, (double)n_walks, n_walks, (int)K, F, ni, walk_pre, blk_col,
                                         OnesR{g->hdr, g->vals, r_ones, stats_zero});
        mcf::note_launch();
        MCF_LAUNCHED("k_alloc_fused");
        if (own) MCF_CUDA(cudaFreeAsync(F, s));
        return MCF_OK;
    }
    // one zero-initialised block: selection state + the budget scan's look-back words
    const long long tiles = (n + SCAN_TILE - 1) / SCAN_TILE;
    const size_t state_bytes = (sizeof(AllocState) + 15) & ~size_t(15);
    char *blk = nullptr;
    unsigned long long *ckey = nullptr;
    MCF_CUDA(cudaMallocAsync(&blk, state_bytes + sizeof(unsigned long long) * (2 * tiles + 2), s));
    AllocState *st = reinterpret_cast<AllocState *>(blk);
    unsigned long long *sa = reinterpret_cast<unsigned long long *>(blk + state_bytes), *sb = sa + tiles;
    unsigned *ctr = reinterpret_cast<unsigned *>(sb + tiles);
    MCF_CUDA(cudaMemsetAsync(blk, 0, state_bytes + sizeof(unsigned long long) * (2 * tiles + 2), s));
    MCF_CUDA(cudaMallocAsync(&ckey, sizeof(unsigned long long) * n, s));  // candidates (rarely written)
    const double total = (double)n_walks;
    const int grid = sm_count() * 2;
    k_alloc_floor<<<grid, 256, 0, s>>>(g->init_prob, n, total, n_walks, st);
    mcf::note_launch();
    k_alloc_level2<<<grid, 256, 0, s>>>(g->init_prob, n, total, st);
    mcf::note_launch();
    k_alloc_cands<<<grid, 256, 0, s>>>(g->init_prob, n, total, st, ckey);
    mcf::note_launch();
    k_alloc_select<<<1, 1024, 0, s>>>(ckey, st);
    mcf::note_launch();
    k_alloc_scan<<<(unsigned)tiles, SCAN_T, 0, s>>>(g->init_prob, n, total, st, ni, walk_pre, blk_col, sa, sb, ctr);
    mcf::note_launch();
    MCF_LAUNCHED("allocate");
    MCF_CUDA(cudaFreeAsync(ckey, s));
    MCF_CUDA(cudaFreeAsync(blk, s));
    return MCF_OK;
}

int allocate_walks(mcf_graph *g, long long n_walks, long long *ni, long long *walk_pre, int *blk_col,
                   cudaStream_t s, void *fused_scratch, double *r_ones, long long *stats_zero) {
    return allocate(g, n_walks, ni, walk_pre, blk_col, s, fused_scratch, r_ones, stats_zero);
}

size_t fused_scratch_bytes() { return sizeof(AllocFused); }
size_t fused_scratch_zero_bytes() { return offsetof(AllocFused, lvl); }
bool fused_alloc_applies(const mcf_graph *g) {
    const char *path = getenv("MCF_ALLOC_PATH");
    const int G = sm_count() < AF_MAXG ? sm_count() : AF_MAXG;
    const long long K = (g->n + (long long)G * AF_T - 1) / ((long long)G * AF_T);
    return g->n > 0 && K <= AF_KMAX && !(path && !strcmp(path, "passes"));
}

}  // namespace mcf

extern "C" int mcf_allocate_walks(mcf_graph *g, int64_t n_walks, int64_t *ni, int64_t *walk_pre, void *stream) {
    if (!ni) {
        mcf::set_error("mcf_allocate_walks: null argument");
        return MCF_ERR_ARGUMENT;
    }
    return mcf::allocate(g, (long long)n_walks, (long long *)ni, (long long *)walk_pre, nullptr, (cudaStream_t)stream);
}
