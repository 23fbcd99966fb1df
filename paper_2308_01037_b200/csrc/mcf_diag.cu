// Diagonal estimator (Alg. 2 + Eq. 20, :267-305).
//
//   1. k_walk_emit   one lane per walk (same walk engine as the action path)
//                    writes its emissions (state, zeta_{k+2} W_k) into fixed
//                    slots of an emission buffer, column-contiguous.
//   2. k_diag_q      one CTA per walked column c (persistent, work counter):
//                    builds Q_c in a shared-memory hash table (global-memory
//                    table for very wide columns) and, for every stored entry
//                    (i, c), writes pcol[(i,c)] = a_ic <Q_c, C_i> -- the
//                    column's whole contribution to Eq. 20.  Q_c is summed in
//                    a fixed order (emission order within a warp, warps in
//                    index order), so results are deterministic.
//   3. k_diag_final  d_i = zeta_0 + zeta_1 a_ii + sum_c pcol[(i,c)], rows in
//                    fixed order (mcf_diag_combine).
// Partials per CSC entry make the result independent of how columns are
// split across batches, CTAs or GPUs.
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include <cooperative_groups.h>

#include "mcf_internal.cuh"

namespace cg = cooperative_groups;

namespace mcf {

// implemented in mcf_walk.cu (shares the walk engine with the action path)
int check_params(const mcf_graph *g, const mcf_walk_params *p, const long long *walk_pre, long long cb, long long ce);
int launch_walk_emit(mcf_graph *g, const mcf_walk_params *p, const long long *walk_pre, long long cb, long long ce,
                     long long nwalks, int mode, const long long *walk_off, const int *entries, long long slot_len,
                     long long off_base, long long *eaux, int *est, double *ewt, unsigned long long *colmax,
                     long long *stats, int *err, cudaStream_t s, int max_sms = 0);
enum { EMIT_FIXED = 0, EMIT_REPLAY = 1, EMIT_COUNT = 2, EMIT_EXPLICIT = 3 };

}  // namespace mcf

namespace mcf {

constexpr int Q_THREADS = 1024;  // one CTA per SM (the 224-KB table): 32 warps hide the combine's latency
constexpr int Q_WARPS = Q_THREADS / 32;
constexpr int SCAP = 16384;  // shared table slots: 16384 * (4 + 8) B = 192 KB
constexpr int FILTER_WORDS = 8192;  // 32 KB Bloom filter (262144 bits) in front of every combine lookup
constexpr int EMPTY_KEY = -1;
constexpr int DENSE_N = SCAP * 12 / 8;  // node ids a dense Q_c covers in the table's shared memory (24576)

struct QArgs {
    const long long *__restrict__ walk_pre;
    long long wb;        // first walk of the batch
    long long slot_len;  // fixed slots per walk (0 -> eoff or replay layout)
    const long long *__restrict__ eoff;      // explicit layout (relative to wb), or null
    const long long *__restrict__ walk_off;
    long long off_base;
    const int *__restrict__ est;
    const double *__restrict__ ewt;
    const long long *__restrict__ csc_ptr;
    const int *__restrict__ csc_rows;
    const double *__restrict__ csc_vals;
    long long n;
    long long col_begin, col_end;
    double *__restrict__ pcol;
    int uniform;   // every stored value equals `value`: the combine skips csc_vals
    int push_pct;  // push (bitmap tests) when deg(i) > push_pct/100 * |supp Q_c|
    double value;
    const unsigned long long *__restrict__ colmax;  // per-column max |weight| bits (from the walk kernel)
    int *gkeys;
    long long *gvals;
    long long gcap;
    unsigned long long *counter;
    // big columns (combine work > BIG_WORK probes): Q_c handed to k_diag_big
    struct BigRec *big;         // records
    unsigned *n_big;            // record counter
    unsigned max_big;
    int *pool_keys;             // persisted tables
    long long *pool_vals;
    int *pool_E;                // fixed-point exponent per record
    int *lkeys;                 // per-CTA support list of Q_c (push path), gcap_l entries per CTA
    long long *lvals;
    long long lcap;
    int *pool_nsupp;            // support-list length per big record (lists live after the table in the pool)
    // hub-row bitmaps (uniform-value graphs): hub_of[i] = bitmap index or -1
    const int *hub_of;
    const unsigned *hub_bits;
    long long hub_words;
    unsigned long long *pool_used, pool_cap;
    unsigned *pool_filt;        // FILTER_WORDS per record
    unsigned long long *prof;   // MCF_DIAG_PROF=1: combine counters (profiling only, else null)
    int *llist;                 // per-CTA lists of long (i, c) entries (~t: push), llcap each
    long long llcap;
    int *lbase;                 // k_diag_q: first piece of each listed entry, its piece sum,
    unsigned long long *lacc;   // and the piece -> entry map (ocap per CTA)
    int *lown;
    long long ocap;
    long long long_work;        // LONG_WORK: split threshold of the cluster kernels (MCF_DIAG_LONG_WORK)
    long long long_work_q;      // k_diag_q's (MCF_DIAG_LONG_WORK_Q; measured best lower: one CTA per column)
    long long big_work;         // BIG_WORK (MCF_DIAG_BIG_WORK overrides: tests)
    long long chunk_q;          // ids / support tests per shared piece of a long entry: k_diag_q (MCF_DIAG_CHUNK_Q)
    long long chunk_c;          // ... and the cluster kernels (MCF_DIAG_CHUNK)
    long long cl_base;          // first scratch region of the cluster kernels' CTAs (= k_diag_q's grid)
    int cl_maxk;                // > 0: columns whose table needs a cluster of <= cl_maxk CTAs go to k_diag_qc
    int opt;                    // MCF_DIAG_OPT: OPT_PIPE | OPT_SPEC | OPT_BLOCKED | OPT_EXACT
    unsigned *cbits;            // OPT_EXACT: per-cluster exact membership bitmap of Q_c's keys (n bits each)
    long long cwords;
};

// prof slots: 0 pull pairs, 1 pull ids, 2 pull filter passes, 3 push pairs, 4 push tests, 5 push hits,
// 6 emissions, 7 support, 8 columns, 9 big columns, 10 cycles Q build, 11 cycles combine, 12 pull hits
// per table class (0 k_diag_q shared table, 1 k_diag_q global table, 2 dense,
// 3 clusters, 4 k_diag_big): pull pairs, ids, filter passes, hits, push pairs,
// tests, push hits, spare
constexpr int PROF_BASE = 20, PROF_CLS = 8, PROF_NCLS = 5;
constexpr int PROF_PH = PROF_BASE + PROF_CLS * PROF_NCLS;  // cluster phase cycles (rank 0): 6 slots
constexpr int PROF_SLOTS = PROF_PH + 8;  // 16..18: cluster-kernel columns, cycles, emissions

__device__ __forceinline__ int ld_relaxed_i32(const int *p) {
    int v;
    asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed_i32(int *p, int v) {
    asm volatile("st.relaxed.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ int ld_volatile_i32(const int *p) { return *(const volatile int *)p; }

struct BigRec {
    long long c;      // column
    long long off;    // table offset in the pool
    unsigned cap;     // table slots (power of two)
    unsigned cn;      // entries of C_c
};

constexpr long long BIG_WORK = 1ll << 20;
constexpr int MAX_LONG = 64;            // parked long (i, c) entries per column
constexpr long long CHUNK = 1024;       // ids / support tests per shared range of a long entry
constexpr long long LONG_WORK = 2 * CHUNK;
constexpr long long LONG_WORK_Q = CHUNK / 2;  // Chung-Lu 1.6e7: 9.6 -> 9.3 s (R-MAT 2^22 prefers 2048 in the clusters)
// cluster tables are sized for load <= CL_LOAD_NUM / CL_LOAD_DEN (by emission count)
#ifndef CL_LOAD_NUM
#define CL_LOAD_NUM 1
#define CL_LOAD_DEN 1
#endif
constexpr long long SMALL_NEED = (3ll * SCAP - 4) / 4;  // largest table need one CTA's shared table holds (load <= 3/4)

// Cluster size whose distributed shared table (K x SCAP slots, load <= 3/4)
// holds a column of `need` (<= emissions) entries: 0 if one CTA's table does,
// or none of 2/4/8 (<= maxk) does (then k_diag_q's global table).
__device__ __forceinline__ int cluster_class(long long need, int maxk) {
    if (need <= SMALL_NEED) return 0;
    for (int k = 2; k <= maxk; k <<= 1)
        if ((long long)k * SCAP * CL_LOAD_DEN >= need * CL_LOAD_NUM + 4) return k;
    return 0;
}  // combine probes above which a column's Q_c is shared GPU-wide

__device__ __forceinline__ long long slot_of(const QArgs &a, long long g) {
    if (a.slot_len > 0) return (g - a.wb) * a.slot_len;
    if (a.eoff) return a.eoff[g - a.wb];
    return a.walk_off[g] - a.off_base + (g - a.wb);
}

// Fibonacci hashing: the HIGH bits of key * 2^32/phi (the low bits of the
// product depend only on the key's low bits, so keys equal mod the table size
// would share a probe chain).  mask = cap - 1, cap a power of two >= 32.
__device__ __forceinline__ uint32_t hash_slot(int key, uint32_t mask) {
    return (uint32_t)(((uint64_t)((uint32_t)key * 0x9E3779B1u) * (uint64_t)(mask + 1)) >> 32);
}

__device__ __forceinline__ int find_or_insert(int *keys, uint32_t mask, int key) {
    uint32_t s = hash_slot(key, mask);
    while (true) {
        int k = keys[s];
        if (k == key) return (int)s;
        if (k == EMPTY_KEY) {
            int old = atomicCAS(&keys[s], EMPTY_KEY, key);
            if (old == EMPTY_KEY || old == key) return (int)s;
        }
        s = (s + 1) & mask;
    }
}

__device__ __forceinline__ long long lookup(const int *keys, const long long *vals, uint32_t mask, int key,
                                            bool spec = false) {
    if (!keys) return vals[key];  // dense table (small graphs): Q_c indexed by node id
    uint32_t s = hash_slot(key, mask);
    if (spec) {  // the home slot's value loaded with its key: one round trip for a hit at home
        const int k = keys[s];
        const long long v = vals[s];
        if (k == key) return v;
        if (k == EMPTY_KEY) return 0;
        s = (s + 1) & mask;
    }
    while (true) {
        int k = keys[s];
        if (k == key) return vals[s];
        if (k == EMPTY_KEY) return 0;
        s = (s + 1) & mask;
    }
}

// int64 add into shared memory as two native 32-bit atomics (the 64-bit
// shared atomicAdd is a CAS loop, which hot keys turn into long spins): the
// low word's returned old value tells the one adder that wrapped it to carry.
// The slot holds the exact sum mod 2^64 (two's complement) once all adds land.
__device__ __forceinline__ void smem_add_i64(long long *p, long long v) {
    unsigned *w = reinterpret_cast<unsigned *>(p);
    const unsigned long long u = (unsigned long long)v;
    const unsigned lo = (unsigned)u, hi = (unsigned)(u >> 32);
    const unsigned old = atomicAdd(w, lo);
    const unsigned up = hi + (old + lo < old ? 1u : 0u);
    if (up) atomicAdd(w + 1, up);
}

// sum of v over the lanes of `mask` (the caller's match group), exact mod
// 2^64: three digit sums of <= 22 bits each never overflow 32 bits
__device__ __forceinline__ long long group_sum_i64(unsigned mask, long long v) {
    const unsigned long long u = (unsigned long long)v;
    const unsigned long long s0 = __reduce_add_sync(mask, (unsigned)(u & 0x3FFFFFull));
    const unsigned long long s1 = __reduce_add_sync(mask, (unsigned)((u >> 22) & 0x1FFFFFull));
    const unsigned long long s2 = __reduce_add_sync(mask, (unsigned)(u >> 43));
    return (long long)(s0 + (s1 << 22) + (s2 << 43));
}

// Bloom bit of a key (independent of the table hash).  Most combine lookups
// miss (C_i entries no walk from c visited): the filter answers them with one
// shared-memory word instead of a linear-probing chain.
__device__ __forceinline__ uint32_t filter_bit(int key) { return ((uint32_t)key * 0x85EBCA6Bu) >> 14; }
__device__ __forceinline__ uint32_t filter_bit2(int key) { return ((uint32_t)key * 0xC2B2AE35u) >> 14; }

// Two bits per key (k = 2): at the ~10^4 keys of a shared-memory Q_c the false
// positive rate drops from ~4% to ~0.2%, at 6.5e4 from 22% to 15%.
// Blocked variant (MCF_DIAG_OPT bit 4): three bits of ONE 32-bit word, so a
// test is a single shared-memory load instead of two.
__device__ __forceinline__ uint32_t filter_block_mask(int key) {
    const uint32_t h = (uint32_t)key * 0xC2B2AE35u;
    return (1u << (h >> 27)) | (1u << ((h >> 22) & 31u)) | (1u << ((h >> 17) & 31u));
}
__device__ __forceinline__ uint32_t filter_block_word(int key) { return ((uint32_t)key * 0x85EBCA6Bu) >> 19; }

__device__ __forceinline__ bool filter_test(const unsigned *filt, int key, bool blocked = false) {
    if (blocked) {
        const uint32_t m = filter_block_mask(key);
        return (filt[filter_block_word(key)] & m) == m;
    }
    const uint32_t b = filter_bit(key), b2 = filter_bit2(key);
    return ((filt[b >> 5] >> (b & 31)) & (filt[b2 >> 5] >> (b2 & 31)) & 1u) != 0;
}

__device__ __forceinline__ void filter_add(unsigned *filt, int key, bool blocked = false) {
    if (blocked) {
        atomicOr(&filt[filter_block_word(key)], filter_block_mask(key));
        return;
    }
    const uint32_t b = filter_bit(key), b2 = filter_bit2(key);
    atomicOr(&filt[b >> 5], 1u << (b & 31));
    atomicOr(&filt[b2 >> 5], 1u << (b2 & 31));
}

enum { OPT_SPEC = 2, OPT_BLOCKED = 4, OPT_EXACT = 8, OPT_CBATCH = 16 };  // (bit 1: a pipelined scan, measured no gain, removed)
constexpr int DIAG_OPT_DEFAULT = OPT_EXACT;  // measured: exact bitmap on (-0.5%), batched DSMEM probes off (+5%)

// Uniform-value graphs: the fixed-point sum over one range of the (i, c) work,
// warp-reduced.
//   pull (push == false): C_i entries [lo, hi) -- coalesced row ids, Bloom
//         filter, hash lookup;
//   push (push == true):  support-list positions [lo, hi) tested against hub
//         row i's bitmap (cost min(deg i, |supp Q_c|) instead of deg i).
// The ranges of one pair can be split over warps: integer adds commute, so the
// sum does not depend on the split, the path or any order (deterministic).
// Q_c in this CTA's shared memory (or its global table, or dense by node id)
struct LocalTable {
    const int *keys;  // null: dense Q_c indexed by node id
    const long long *vals;
    uint32_t mask;
    bool global;      // table in global memory: probes batched (see uniform_partial)
    static constexpr bool can_batch = true;
    __device__ __forceinline__ bool batched() const { return global; }
    __device__ __forceinline__ long long get(int key, bool spec = false) const {
        return lookup(keys, vals, mask, key, spec);
    }
    __device__ __forceinline__ int key_at(uint32_t s) const { return keys[s]; }
    __device__ __forceinline__ long long val_at(uint32_t s) const { return vals[s]; }
    __device__ __forceinline__ bool maybe(int) const { return true; }
};

template <class Table>
__device__ __forceinline__ long long uniform_partial(const QArgs &a, const Table &tab, const int *lkeys,
                                                     const long long *lvals, const unsigned *filt, int i, bool push,
                                                     long long lo, long long hi, int lane, int pcls = 0) {
    long long acc = 0;
    if (push) {
        const unsigned *bits = a.hub_bits + (long long)__ldg(a.hub_of + i) * a.hub_words;
        // PUSH_U tests in flight per lane: key load, then the dependent bitmap word
        constexpr int PUSH_U = 4;
        int hits = 0;
        for (long long t0 = lo; t0 < hi; t0 += 32 * PUSH_U) {
            int kv[PUSH_U];
            unsigned wv[PUSH_U];
#pragma unroll
            for (int u = 0; u < PUSH_U; ++u) {
                const long long t = t0 + 32 * u + lane;
                kv[u] = t < hi ? lkeys[t] : -1;
            }
#pragma unroll
            for (int u = 0; u < PUSH_U; ++u) wv[u] = kv[u] >= 0 ? __ldg(bits + (kv[u] >> 5)) : 0u;
#pragma unroll
            for (int u = 0; u < PUSH_U; ++u)
                if ((wv[u] >> (kv[u] & 31)) & 1u) {
                    acc += lvals[t0 + 32 * u + lane];
                    ++hits;
                }
        }
        if (a.prof) {
            hits = warp_sum_int(hits);
            if (lane == 0) {
                atomicAdd(a.prof + 3, 1ull);
                atomicAdd(a.prof + 4, (unsigned long long)(hi - lo));
                atomicAdd(a.prof + 5, (unsigned long long)hits);
                unsigned long long *pc = a.prof + PROF_BASE + PROF_CLS * pcls;
                atomicAdd(pc + 4, 1ull);
                atomicAdd(pc + 5, (unsigned long long)(hi - lo));
                atomicAdd(pc + 6, (unsigned long long)hits);
            }
        }
    } else {
        // PULL_U row ids in flight per lane: long rows are scanned latency-
        // bound otherwise (one L2 round trip per 64 ids)
        constexpr int PULL_U = 8;
        int fpass = 0, phit = 0;
        const bool blocked = (a.opt & OPT_BLOCKED) != 0, spec = (a.opt & OPT_SPEC) != 0;
        for (long long e0 = lo; e0 < hi; e0 += 32 * PULL_U) {
            int jv[PULL_U];
#pragma unroll
            for (int u = 0; u < PULL_U; ++u) {
                const long long e = e0 + 32 * u + lane;
                jv[u] = e < hi ? __ldg(a.csc_rows + e) : -1;
            }
            if (!Table::can_batch || !tab.batched()) {
#pragma unroll
                for (int u = 0; u < PULL_U; ++u) {
                    if (jv[u] < 0) continue;
                    if (filter_test(filt, jv[u], blocked) && tab.maybe(jv[u])) {
                        const long long q = tab.get(jv[u], spec);
                        acc += q;
                        if (a.prof) {
                            ++fpass;
                            phit += q != 0;
                        }
                    }
                }
                continue;
            }
            // global-memory tables: the Bloom-passing ids are probed together,
            // every step of the PULL_U linear-probing chains one batch of
            // independent loads (probing one id after another serialised L2
            // round trips; in shared / distributed shared memory the scalar
            // probe above is faster -- measured)
            if constexpr (Table::can_batch) {
            unsigned pend = 0u, hit = 0u;
            uint32_t sl[PULL_U];
#pragma unroll
            for (int u = 0; u < PULL_U; ++u) {
                sl[u] = 0;
                if (jv[u] < 0) continue;
                if (filter_test(filt, jv[u], blocked) && tab.maybe(jv[u])) {
                    pend |= 1u << u;
                    sl[u] = hash_slot(jv[u], tab.mask);
                }
            }
            if (a.prof) fpass += __popc(pend);
            while (pend) {
                int kv[PULL_U];
#pragma unroll
                for (int u = 0; u < PULL_U; ++u) kv[u] = (pend >> u) & 1u ? tab.key_at(sl[u]) : EMPTY_KEY;
#pragma unroll
                for (int u = 0; u < PULL_U; ++u) {
                    if (!((pend >> u) & 1u)) continue;
                    if (kv[u] == jv[u]) {
                        hit |= 1u << u;
                        pend &= ~(1u << u);
                    } else if (kv[u] == EMPTY_KEY) {
                        pend &= ~(1u << u);
                    } else {
                        sl[u] = (sl[u] + 1) & tab.mask;
                    }
                }
            }
            long long qv[PULL_U];
#pragma unroll
            for (int u = 0; u < PULL_U; ++u) qv[u] = (hit >> u) & 1u ? tab.val_at(sl[u]) : 0;
#pragma unroll
            for (int u = 0; u < PULL_U; ++u) {
                acc += qv[u];
                if (a.prof) phit += qv[u] != 0;
            }
            }
        }
        if (a.prof) {
            fpass = warp_sum_int(fpass);
            phit = warp_sum_int(phit);
            if (lane == 0) {
                atomicAdd(a.prof + 0, 1ull);
                atomicAdd(a.prof + 1, (unsigned long long)(hi - lo));
                atomicAdd(a.prof + 2, (unsigned long long)fpass);
                atomicAdd(a.prof + 12, (unsigned long long)phit);
                unsigned long long *pc = a.prof + PROF_BASE + PROF_CLS * pcls;
                atomicAdd(pc + 0, 1ull);
                atomicAdd(pc + 1, (unsigned long long)(hi - lo));
                atomicAdd(pc + 2, (unsigned long long)fpass);
                atomicAdd(pc + 3, (unsigned long long)phit);
            }
        }
    }
    return warp_sum_ll(acc);
}

// push or pull for the stored entry (i, c), and the length of that work
__device__ __forceinline__ bool use_push(const QArgs &a, int i, long long deg_i, int nsupp) {
    return a.hub_of && 100 * deg_i > (long long)a.push_pct * nsupp && __ldg(a.hub_of + i) >= 0;
}

// Contribution of the stored entry (i, c): a_ic <Q_c, C_i>, one warp.
__device__ __forceinline__ double pair_value(const QArgs &a, const int *keys, const long long *vals, uint32_t mask,
                                             const int *lkeys, const long long *lvals, int nsupp,
                                             const unsigned *filt, int E, int i, double aic, int lane) {
    const long long ilo = a.csc_ptr[i], ihi = a.csc_ptr[i + 1];
    if (a.uniform) {
        const bool push = use_push(a, i, ihi - ilo, nsupp);
        const LocalTable tab{keys, vals, mask, true};  // k_diag_big: pool tables in global memory
        const long long acc = push ? uniform_partial(a, tab, lkeys, lvals, filt, i, true, 0, nsupp, lane, 4)
                                   : uniform_partial(a, tab, lkeys, lvals, filt, i, false, ilo, ihi, lane, 4);
        return aic * (a.value * ldexp((double)acc, -E));
    }
    double acc = 0.0;
    for (long long e = ilo + lane; e < ihi; e += 32) {
        const int j = __ldg(a.csc_rows + e);
        if (filter_test(filt, j, (a.opt & OPT_BLOCKED) != 0))
            acc = fma(__ldg(a.csc_vals + e), ldexp((double)lookup(keys, vals, mask, j), -E), acc);
    }
    return aic * warp_sum(acc);
}

// Q_c is accumulated in fixed point: every weight is scaled by 2^E (E from the
// column's largest |weight| and its emission count, so no sum can exceed
// 2^62) and rounded to int64; integer adds commute, so Q_c -- and therefore d
// -- does not depend on the order in which threads add (deterministic), and
// plain shared-memory atomics replace any ordering barriers.  The quantum is
// 2^-E <= 2^-61 * M * max|w| (M emissions), orders of magnitude below the
// 1e-10 replay tolerance and the Monte Carlo error.
__global__ void __launch_bounds__(Q_THREADS, 1) k_diag_q(QArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    long long *svals = reinterpret_cast<long long *>(smem_raw);
    int *skeys = reinterpret_cast<int *>(svals + SCAP);
    unsigned *filt = reinterpret_cast<unsigned *>(skeys + SCAP);
    __shared__ long long s_col, s_work, s_slot, s_off;
    __shared__ int s_nsupp, s_next, s_nlong, s_nchunk;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    int *gkeys = a.gkeys ? a.gkeys + (long long)blockIdx.x * a.gcap : nullptr;
    long long *gvals = a.gvals ? a.gvals + (long long)blockIdx.x * a.gcap : nullptr;

    while (true) {
        __syncthreads();
        if (tid == 0) {
            s_col = a.col_begin + (long long)atomicAdd(a.counter, 1ull);
        }
        __syncthreads();
        const long long c = s_col;
        if (c >= a.col_end) break;
        const long long g0 = a.walk_pre[c], g1 = a.walk_pre[c + 1];
        if (g0 == g1) continue;
        const long long s0 = slot_of(a, g0), m = slot_of(a, g1) - s0;
        const long long t_start = a.prof ? clock64() : 0;
        long long need = m < a.n ? m : a.n;
        if (a.cl_maxk && cluster_class(need, a.cl_maxk)) continue;  // k_diag_qc builds this Q_c
        uint32_t cap = 32;
        while ((long long)cap < need * 2 && cap < (uint32_t)SCAP) cap <<= 1;  // load factor <= 1/2 if it fits smem
        while ((long long)cap * 3 < need * 4 + 4) cap <<= 1;                 // and <= 3/4 always
        int *keys;
        long long *vals;
        // small graphs (n <= DENSE_N): Q_c is a dense shared array indexed by
        // node id -- no hashing, no probing (keys == nullptr marks it)
        const bool dense = a.n <= DENSE_N && need * 4 > a.n;
        if (dense) {
            cap = (uint32_t)a.n;
            keys = nullptr;
            vals = svals;
        } else if (cap <= (uint32_t)SCAP) {
            keys = skeys;
            vals = svals;
        } else {
            keys = gkeys;
            vals = gvals;
        }
        const uint32_t mask = cap - 1;
        for (uint32_t t = tid; t < cap; t += Q_THREADS) {
            if (keys) keys[t] = EMPTY_KEY;
            vals[t] = 0;
        }
        __syncthreads();
        const double maxw = __longlong_as_double((long long)a.colmax[c]);
        int lg_m = 0;
        while ((1ll << lg_m) < m) ++lg_m;
        const int E = maxw > 0.0 ? 61 - ilogb(maxw) - lg_m : 0;  // sum of m terms < 2^62
        // pass 2: Q_c[j] += round(w 2^E)   (Alg. 2 line "q_{i l_k} += zeta W")
        constexpr int U = 4;  // emissions in flight per thread (streaming loads ahead of the smem work)
        for (long long base = 0; base < m; base += (long long)U * Q_THREADS) {
            int sv[U];
            double wv[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const long long i = base + (long long)u * Q_THREADS + tid;
                sv[u] = i < m ? __ldcs(a.est + s0 + i) : EMPTY_KEY;
                wv[u] = i < m ? __ldcs(a.ewt + s0 + i) : 0.0;
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                if (sv[u] < 0) continue;
                const long long q = __double2ll_rn(ldexp(wv[u], E));
                const int slot = keys ? find_or_insert(keys, mask, sv[u]) : sv[u];
                smem_add_i64(&vals[slot], q);
            }
        }
        __syncthreads();
        // Bloom filter of the keys and the compact support list (push path)
        for (int t = tid; t < FILTER_WORDS; t += Q_THREADS) filt[t] = 0u;
        if (tid == 0) s_nsupp = 0;
        __syncthreads();
        int *lkeys = a.lkeys + (long long)blockIdx.x * a.lcap;
        long long *lvals = a.lvals + (long long)blockIdx.x * a.lcap;
        for (uint32_t t = tid; t < cap; t += Q_THREADS) {
            const int key = keys ? keys[t] : (vals[t] != 0 ? (int)t : EMPTY_KEY);
            if (key != EMPTY_KEY) {
                filter_add(filt, key, (a.opt & OPT_BLOCKED) != 0);
                if (a.uniform) {
                    const int p = atomicAdd(&s_nsupp, 1);
                    if (p < a.lcap) {
                        lkeys[p] = key;
                        lvals[p] = vals[t];
                    }
                }
            }
        }
        __syncthreads();
        const int nsupp = s_nsupp <= a.lcap ? s_nsupp : 0x3fffffff;  // overflow: never push
        const long long t_built = a.prof ? clock64() : 0;
        if (a.prof && tid == 0) {
            atomicAdd(a.prof + 6, (unsigned long long)m);
            atomicAdd(a.prof + 7, (unsigned long long)s_nsupp);
            atomicAdd(a.prof + 8, 1ull);
            atomicAdd(a.prof + 10, (unsigned long long)(t_built - t_start));
        }

        // combine work of this column: sum of deg(i) over the entries (i, c)
        const long long cs = a.csc_ptr[c], cn = a.csc_ptr[c + 1] - cs;
        long long work = 0;
        for (long long t = tid; t < cn; t += Q_THREADS) {
            const int i = a.csc_rows[cs + t];
            work += a.csc_ptr[i + 1] - a.csc_ptr[i];
        }
        work = warp_sum_ll(work);
        if (tid == 0) s_work = 0;
        __syncthreads();
        if (lane == 0) atomicAdd(reinterpret_cast<unsigned long long *>(&s_work), (unsigned long long)work);
        __syncthreads();
        if (s_work > a.big_work && a.big && keys) {
            // hand Q_c to k_diag_big: all warps of the GPU share the combine
            if (tid == 0) {
                s_slot = -1;
                const unsigned long long off = atomicAdd(a.pool_used, 2ull * cap);
                if (off + 2ull * cap <= a.pool_cap) {
                    const unsigned r = atomicAdd(a.n_big, 1u);
                    if (r < a.max_big) {
                        a.big[r] = BigRec{c, (long long)off, cap, (unsigned)cn};
                        a.pool_E[r] = E;
                        s_slot = (long long)r;
                        s_off = (long long)off;
                    }
                }
            }
            __syncthreads();
            if (s_slot >= 0) {
                for (uint32_t t = tid; t < cap; t += Q_THREADS) {
                    a.pool_keys[s_off + t] = keys[t];
                    a.pool_vals[s_off + t] = vals[t];
                }
                // support list after the table (nsupp <= cap / 2 by the load factor)
                for (int t = tid; t < nsupp && nsupp <= (int)cap; t += Q_THREADS) {
                    a.pool_keys[s_off + cap + t] = lkeys[t];
                    a.pool_vals[s_off + cap + t] = lvals[t];
                }
                if (tid == 0) a.pool_nsupp[s_slot] = nsupp <= (int)cap ? nsupp : 0x3fffffff;
                for (int t = tid; t < FILTER_WORDS; t += Q_THREADS)
                    a.pool_filt[s_slot * FILTER_WORDS + t] = filt[t];
                if (a.prof && tid == 0) atomicAdd(a.prof + 9, 1ull);
                continue;  // the loop-top barrier orders these copies before the table is reused
            }
        }

        // Eq. 20: for every stored (i, c): pcol = a_ic <Q_c, C_i>
        if (!a.uniform) {
            for (long long t = warp; t < cn; t += Q_WARPS) {
                const double v = pair_value(a, keys, vals, mask, lkeys, lvals, nsupp, filt, E, a.csc_rows[cs + t],
                                            a.csc_vals[cs + t], lane);
                if (lane == 0) a.pcol[cs + t] = v;
            }
        } else {
            // Uniform values: warps take entries dynamically; an entry whose
            // scan is longer than LONG_WORK is listed with a range of CHUNK-long
            // pieces (a chunk -> entry map), and once every short entry is done
            // all warps share the pieces of every listed entry (one warp per
            // entry left the CTA waiting on its longest scan).  Piece sums are
            // int64 and added atomically: the same exact total as one warp's
            // scan.  A list or map that is full: the warp scans the entry itself.
            const long long rb = (long long)blockIdx.x;
            int *llist = a.llist + rb * a.llcap;
            int *lbase = a.lbase + rb * a.llcap;
            unsigned long long *lacc = a.lacc + rb * a.llcap;
            int *lown = a.lown + rb * a.ocap;
            if (tid == 0) {
                s_next = 0;
                s_nlong = 0;
                s_nchunk = 0;
            }
            __syncthreads();
            // (global tables here: scalar probes measured faster than batched, k_diag_big the reverse)
            const LocalTable tab{keys, vals, mask, false};
            const int pcls = keys == nullptr ? 2 : (keys == gkeys ? 1 : 0);
            while (true) {
                int t = 0;
                if (lane == 0) t = atomicAdd(&s_next, 1);
                t = __shfl_sync(MCF_FULL, t, 0);
                if (t >= cn) break;
                const int i = a.csc_rows[cs + t];
                const long long ilo = a.csc_ptr[i], ihi = a.csc_ptr[i + 1];
                const bool push = use_push(a, i, ihi - ilo, nsupp);
                const long long len = push ? nsupp : ihi - ilo;
                if (len > a.long_work_q) {
                    const int nch = (int)((len + a.chunk_q - 1) / a.chunk_q);
                    int slot = 0, base = 0;
                    if (lane == 0) {
                        slot = atomicAdd(&s_nlong, 1);
                        base = slot < a.llcap ? atomicAdd(&s_nchunk, nch) : 0;
                    }
                    slot = __shfl_sync(MCF_FULL, slot, 0);
                    base = __shfl_sync(MCF_FULL, base, 0);
                    if (slot < a.llcap) {
                        const bool fits = (long long)base + nch <= a.ocap;
                        for (long long k = base + lane; k < base + nch && k < a.ocap; k += 32) lown[k] = fits ? slot : -1;
                        if (lane == 0) {
                            llist[slot] = fits ? (push ? ~t : t) : INT_MAX;  // INT_MAX: scanned here
                            lbase[slot] = base;
                            lacc[slot] = 0ull;
                        }
                        if (fits) continue;
                    }
                }
                const long long acc = uniform_partial(a, tab, lkeys, lvals, filt, i, push, push ? 0 : ilo,
                                                      push ? nsupp : ihi, lane, pcls);
                if (lane == 0) a.pcol[cs + t] = a.csc_vals[cs + t] * (a.value * ldexp((double)acc, -E));
            }
            __syncthreads();
            const int nlong = s_nlong < a.llcap ? s_nlong : (int)a.llcap;
            if (nlong > 0) {
                const long long K = s_nchunk < a.ocap ? s_nchunk : a.ocap;
                if (tid == 0) s_next = 0;
                __syncthreads();
                while (true) {
                    int k = 0;
                    if (lane == 0) k = atomicAdd(&s_next, 1);
                    k = __shfl_sync(MCF_FULL, k, 0);
                    if (k >= K) break;
                    const int j = lown[k];
                    if (j < 0) continue;
                    const int lt = llist[j];
                    const bool push = lt < 0;
                    const int t = push ? ~lt : lt;
                    const int i = a.csc_rows[cs + t];
                    const long long base = push ? 0 : a.csc_ptr[i];
                    const long long end = push ? nsupp : a.csc_ptr[i + 1];
                    const long long lo = base + (long long)(k - lbase[j]) * a.chunk_q;
                    const long long hi = lo + a.chunk_q < end ? lo + a.chunk_q : end;
                    const long long acc = uniform_partial(a, tab, lkeys, lvals, filt, i, push, lo, hi, lane, pcls);
                    if (lane == 0) atomicAdd(lacc + j, (unsigned long long)acc);
                }
                __syncthreads();
                for (int j = tid; j < nlong; j += Q_THREADS) {
                    const int lt = llist[j];
                    if (lt == INT_MAX) continue;
                    const int t = lt < 0 ? ~lt : lt;
                    a.pcol[cs + t] = a.csc_vals[cs + t] * (a.value * ldexp((double)(long long)__ldcg(lacc + j), -E));
                }
            }
        }
        if (a.prof) {
            __syncthreads();
            if (tid == 0) atomicAdd(a.prof + 11, (unsigned long long)(clock64() - t_built));
            if (tid == 0 && keys == gkeys) {
                atomicAdd(a.prof + 13, 1ull);
                atomicAdd(a.prof + 14, (unsigned long long)(clock64() - t_start));
                atomicAdd(a.prof + 15, (unsigned long long)m);
            }
        }
    }
}

// ---------------------------------------------------------------------------
// Q_c wider than one CTA's shared table: a thread-block cluster of K CTAs (K
// SMs) holds it in distributed shared memory -- slot s lives in CTA s / SCAP
// -- instead of a global-memory table (whose random probes went to L2/HBM and
// were ~90% of the combine time on R-MAT 2^22).  Same fixed-point Q_c, same
// Bloom filter (each CTA ORs in the others' parts) and support list, same
// Eq. 20 combine with every warp of the cluster sharing the (i, c) entries;
// the int64 sums are the ones k_diag_q forms, so pcol is bit-identical.
// Uniform-value graphs only (the combine's exact integer path).
// ---------------------------------------------------------------------------
struct ClusterTable {
    const int *keys;  // this CTA's part (the same offset in every CTA of the cluster)
    const long long *vals;
    uint32_t mask;    // K * SCAP - 1
    const unsigned *exact;  // OPT_EXACT: the cluster's membership bitmap (L2), or null
    bool batch;             // OPT_CBATCH: the Bloom-passing ids of a block probed together
    static constexpr bool can_batch = true;
    __device__ __forceinline__ bool batched() const { return batch; }
    // a key the Bloom filter passed is probed remotely only if it is really in
    // Q_c: the filter's false positives (~half the passes on wide columns)
    // would walk the longest linear-probing chains in distributed shared memory
    __device__ __forceinline__ bool maybe(int key) const {
        return !exact || ((__ldcg(exact + (key >> 5)) >> (key & 31)) & 1u);
    }
    int *const *kb;               // kb[r] / vb[r]: CTA r's key / value array (mapped once per kernel)
    long long *const *vb;
    __device__ __forceinline__ long long get(int key, bool spec = false) const {
        uint32_t s = hash_slot(key, mask);
        if (spec) {  // home slot key and value in one round trip
            const unsigned r = s / SCAP, l = s % SCAP;
            const int k = kb[r][l];
            const long long v = vb[r][l];
            if (k == key) return v;
            if (k == EMPTY_KEY) return 0;
            s = (s + 1) & mask;
        }
        while (true) {
            const unsigned r = s / SCAP, l = s % SCAP;
            const int k = kb[r][l];
            if (k == key) return vb[r][l];
            if (k == EMPTY_KEY) return 0;
            s = (s + 1) & mask;
        }
    }
    __device__ __forceinline__ int key_at(uint32_t s) const { return kb[s / SCAP][s % SCAP]; }
    __device__ __forceinline__ long long val_at(uint32_t s) const { return vb[s / SCAP][s % SCAP]; }
};

__device__ __forceinline__ uint32_t cluster_find_or_insert(int *keys, uint32_t mask, int key) {
    cg::cluster_group cl = cg::this_cluster();
    uint32_t s = hash_slot(key, mask);
    while (true) {
        int *kp = cl.map_shared_rank(keys, s / SCAP) + (s % SCAP);
        const int k = *kp;
        if (k == key) return s;
        if (k == EMPTY_KEY) {
            const int old = atomicCAS(kp, EMPTY_KEY, key);
            if (old == EMPTY_KEY || old == key) return s;
        }
        s = (s + 1) & mask;
    }
}

template <int K>
__global__ void __cluster_dims__(K, 1, 1) __launch_bounds__(Q_THREADS, 1)
    k_diag_qc(QArgs a, const int *__restrict__ cols, unsigned ncols, unsigned *__restrict__ next_col) {
    cg::cluster_group cl = cg::this_cluster();
    const unsigned rank = cl.block_rank();
    extern __shared__ __align__(16) unsigned char smem_raw[];
    long long *svals = reinterpret_cast<long long *>(smem_raw);
    int *skeys = reinterpret_cast<int *>(svals + SCAP);
    unsigned *filt = reinterpret_cast<unsigned *>(skeys + SCAP);
    __shared__ long long s_col, s_work, s_slot, s_off;
    __shared__ int s_nsupp, s_next, s_nlong;  // rank 0's are the cluster's
    int *r0_nsupp = cl.map_shared_rank(&s_nsupp, 0), *r0_next = cl.map_shared_rank(&s_next, 0);
    int *r0_nlong = cl.map_shared_rank(&s_nlong, 0);
    const int tid = threadIdx.x, lane = tid & 31;
    const long long lcap = (long long)K * a.lcap;  // the cluster's K consecutive per-CTA list regions
    // per-CTA scratch regions after k_diag_q's (the two kernels run concurrently)
    const long long cta = a.cl_base + blockIdx.x;
    int *lkeys = a.lkeys + (long long)((cta - rank) / K) * lcap;
    long long *lvals = a.lvals + (long long)((cta - rank) / K) * lcap;
    const uint32_t mask = (uint32_t)K * SCAP - 1;
    const long long CT = (long long)K * Q_THREADS, gt = (long long)rank * Q_THREADS + tid;
    unsigned *cbits = (a.opt & OPT_EXACT) && a.cbits ? a.cbits + (long long)(blockIdx.x / K) * a.cwords : nullptr;
    __shared__ int *s_kb[K];
    __shared__ long long *s_vb[K];
    if (tid < K) {
        s_kb[tid] = cl.map_shared_rank(skeys, tid);
        s_vb[tid] = cl.map_shared_rank(svals, tid);
    }
    __syncthreads();
    const ClusterTable tab{skeys, svals, mask, cbits, (a.opt & OPT_CBATCH) != 0, s_kb, s_vb};
    __shared__ int s_nchunk, s_next2, s_done;  // rank 0's: pieces reserved, piece counter, entries done
    int *r0_nchunk = cl.map_shared_rank(&s_nchunk, 0), *r0_next2 = cl.map_shared_rank(&s_next2, 0);
    int *r0_done = cl.map_shared_rank(&s_done, 0);

    long long ph_prev = a.prof ? clock64() : 0;  // phase timestamps (rank 0, thread 0; MCF_DIAG_PROF)
    auto phase = [&](int k) {
        if (a.prof && rank == 0 && tid == 0) {
            const long long t = clock64();
            atomicAdd(a.prof + PROF_PH + k, (unsigned long long)(t - ph_prev));
            ph_prev = t;
        }
    };
    while (true) {
        for (int t = tid; t < SCAP; t += Q_THREADS) {
            skeys[t] = EMPTY_KEY;
            svals[t] = 0;
        }
        for (int t = tid; t < FILTER_WORDS; t += Q_THREADS) filt[t] = 0u;
        if (rank == 0 && tid == 0) {
            const unsigned x = atomicAdd(next_col, 1u);
            const long long c = x < ncols ? (long long)cols[x] : -1;
            for (int r = 0; r < K; ++r) *cl.map_shared_rank(&s_col, r) = c;  // every CTA reads its own copy
            s_nsupp = 0;
            s_next = 0;
            s_nlong = 0;
            s_work = 0;
            s_nchunk = 0;
            s_next2 = 0;
            s_done = 0;
        }
        cl.sync();
        const long long c = s_col;
        if (c < 0) break;
        phase(0);  // zeroing + column fetch
        const long long t_start = a.prof ? clock64() : 0;
        const long long g0 = a.walk_pre[c], g1 = a.walk_pre[c + 1];
        const long long s0 = slot_of(a, g0), m = slot_of(a, g1) - s0;
        const double maxw = __longlong_as_double((long long)a.colmax[c]);
        int lg_m = 0;
        while ((1ll << lg_m) < m) ++lg_m;
        const int E = maxw > 0.0 ? 61 - ilogb(maxw) - lg_m : 0;  // as k_diag_q: sum of m terms < 2^62
        constexpr int U = 4;
        for (long long base = 0; base < m; base += (long long)U * CT) {
            int sv[U];
            double wv[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const long long i = base + (long long)u * CT + gt;
                sv[u] = i < m ? __ldcs(a.est + s0 + i) : EMPTY_KEY;
                wv[u] = i < m ? __ldcs(a.ewt + s0 + i) : 0.0;
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                if (sv[u] < 0) continue;
                const long long q = __double2ll_rn(ldexp(wv[u], E));
                const uint32_t slot = cluster_find_or_insert(skeys, mask, sv[u]);
                atomicAdd(reinterpret_cast<unsigned long long *>(cl.map_shared_rank(svals, slot / SCAP) + slot % SCAP),
                          (unsigned long long)q);
            }
        }
        cl.sync();
        phase(1);  // Q_c build
        // this CTA's part: Bloom bits and its share of the support list
        for (int t = tid; t < SCAP; t += Q_THREADS) {
            const int key = skeys[t];
            if (key != EMPTY_KEY) {
                filter_add(filt, key, (a.opt & OPT_BLOCKED) != 0);
                const int p = atomicAdd(r0_nsupp, 1);
                if (p < lcap) {
                    lkeys[p] = key;
                    lvals[p] = svals[t];
                }
            }
        }
        cl.sync();
        // OR in the other parts' filters.  Only this CTA writes its filter and
        // OR only adds bits, so a CTA reading it meanwhile still sees a superset
        // of this part's keys.
        for (int r = 1; r < K; ++r) {
            const unsigned *rf = cl.map_shared_rank(filt, (rank + r) % K);
            for (int t = tid; t < FILTER_WORDS; t += Q_THREADS) filt[t] |= rf[t];
        }
        __syncthreads();
        const int nsupp_all = *r0_nsupp;
        const int nsupp = nsupp_all <= lcap ? nsupp_all : 0x3fffffff;  // overflow: never push
        const long long t_built = a.prof ? clock64() : 0;
        phase(2);  // filter + support list + filter merge
        const long long cs = a.csc_ptr[c], cn = a.csc_ptr[c + 1] - cs;
        if (a.big) {
            // combine work sum_{i in C_c} deg(i): above BIG_WORK the table goes to
            // the pool and k_diag_big spreads the entries over the whole GPU (as
            // k_diag_q does) instead of K SMs working through it at the tail
            long long work = 0;
            for (long long t = gt; t < cn; t += CT) {
                const int i = a.csc_rows[cs + t];
                work += a.csc_ptr[i + 1] - a.csc_ptr[i];
            }
            work = warp_sum_ll(work);
            if (lane == 0 && work)
                atomicAdd(reinterpret_cast<unsigned long long *>(cl.map_shared_rank(&s_work, 0)),
                          (unsigned long long)work);
            cl.sync();
            if (rank == 0 && tid == 0) {
                long long slot = -1, off = 0;
                const unsigned long long cap = (unsigned long long)K * SCAP;
                if (s_work > a.big_work && nsupp_all <= (int)cap) {
                    const unsigned long long o = atomicAdd(a.pool_used, 2ull * cap);
                    if (o + 2ull * cap <= a.pool_cap) {
                        const unsigned r = atomicAdd(a.n_big, 1u);
                        if (r < a.max_big) {
                            a.big[r] = BigRec{c, (long long)o, (unsigned)cap, (unsigned)cn};
                            a.pool_E[r] = E;
                            a.pool_nsupp[r] = nsupp_all;
                            slot = (long long)r;
                            off = (long long)o;
                        }
                    }
                }
                for (int r = 0; r < K; ++r) {
                    *cl.map_shared_rank(&s_slot, r) = slot;
                    *cl.map_shared_rank(&s_off, r) = off;
                }
            }
            cl.sync();
            if (s_slot >= 0) {
                const long long cap = (long long)K * SCAP, base = s_off + (long long)rank * SCAP;
                for (int t = tid; t < SCAP; t += Q_THREADS) {
                    a.pool_keys[base + t] = skeys[t];
                    a.pool_vals[base + t] = svals[t];
                }
                for (long long t = gt; t < nsupp_all; t += CT) {  // support list after the table
                    a.pool_keys[s_off + cap + t] = lkeys[t];
                    a.pool_vals[s_off + cap + t] = lvals[t];
                }
                if (rank == 0)
                    for (int t = tid; t < FILTER_WORDS; t += Q_THREADS) a.pool_filt[s_slot * FILTER_WORDS + t] = filt[t];
                if (a.prof && rank == 0 && tid == 0) atomicAdd(a.prof + 9, 1ull);
                cl.sync();  // copies done before the next column resets the tables and lists
                continue;
            }
        }
        if (cbits) {  // exact membership bits of this CTA's keys (cleared after the column)
            for (int t = tid; t < SCAP; t += Q_THREADS) {
                const int key = skeys[t];
                if (key != EMPTY_KEY) atomicOr(cbits + (key >> 5), 1u << (key & 31));
            }
            __threadfence();
            cl.sync();
        }
        phase(3);  // big check + exact bits
        // the cluster's (rank 0's) lists: long entries, their first piece and
        // piece sum, and the piece -> entry map (global scratch, read with .cg)
        const long long reg = cta - rank;
        int *llist = a.llist + reg * a.llcap;
        int *lbase = a.lbase + reg * a.llcap;
        unsigned long long *lacc = a.lacc + reg * a.llcap;
        int *lown = a.lown + reg * a.ocap;
        // One phase for the whole (i, c) work: warps take entries; a long entry
        // is listed with a range of pieces (piece -> entry map lown, written
        // before the piece becomes visible); a warp with no entry left takes
        // pieces, waiting for a piece it drew to be published, and leaves once
        // every entry is done and its piece index is past the final count.
        // No barrier between the short entries and the pieces, so warps never
        // idle while one finishes a long entry.  (int64 piece sums: the same
        // total as one warp's scan.)  lown is -1 until written (reset by its
        // consumer), -3 for a piece whose entry did not fit the map.
        bool entries_left = true;
        while (true) {
            if (entries_left) {
                int t = 0;
                if (lane == 0) t = atomicAdd(r0_next, 1);
                t = __shfl_sync(MCF_FULL, t, 0);
                if (t < cn) {
                    const int i = a.csc_rows[cs + t];
                    const long long ilo = a.csc_ptr[i], ihi = a.csc_ptr[i + 1];
                    const bool push = use_push(a, i, ihi - ilo, nsupp);
                    const long long len = push ? nsupp : ihi - ilo;
                    bool listed = false;
                    if (len > a.long_work) {
                        const int nch = (int)((len + a.chunk_c - 1) / a.chunk_c);
                        int slot = 0, base = 0;
                        if (lane == 0) {
                            slot = atomicAdd(r0_nlong, 1);
                            base = slot < a.llcap ? atomicAdd(r0_nchunk, nch) : 0;
                        }
                        slot = __shfl_sync(MCF_FULL, slot, 0);
                        base = __shfl_sync(MCF_FULL, base, 0);
                        if (slot < a.llcap) {
                            const bool fits = (long long)base + nch <= a.ocap;
                            if (lane == 0) {
                                llist[slot] = fits ? (push ? ~t : t) : INT_MAX;  // INT_MAX: scanned here
                                lbase[slot] = base;
                                lacc[slot] = 0ull;
                            }
                            __syncwarp();
                            __threadfence();  // the entry's record before its pieces are published
                            for (long long k = base + lane; k < base + nch && k < a.ocap; k += 32)
                                st_relaxed_i32(lown + k, fits ? slot : -3);
                            listed = fits;
                        }
                    }
                    if (!listed) {
                        const long long acc = uniform_partial(a, tab, lkeys, lvals, filt, i, push, push ? 0 : ilo,
                                                              push ? nsupp : ihi, lane, 3);
                        if (lane == 0) a.pcol[cs + t] = a.csc_vals[cs + t] * (a.value * ldexp((double)acc, -E));
                    }
                    __syncwarp();
                    if (lane == 0) atomicAdd(r0_done, 1);
                    continue;
                }
                entries_left = false;
            }
            int k = 0;
            if (lane == 0) k = atomicAdd(r0_next2, 1);
            k = __shfl_sync(MCF_FULL, k, 0);
            if (k >= a.ocap) break;
            int j = -1;
            bool stop = false;
            if (lane == 0) {
                unsigned ns = 32;
                while (true) {
                    j = ld_relaxed_i32(lown + k);
                    if (j != -1) break;
                    if (ld_volatile_i32(r0_done) == cn && k >= ld_volatile_i32(r0_nchunk)) {
                        stop = true;
                        break;
                    }
                    __nanosleep(ns);
                    if (ns < 256) ns <<= 1;
                }
                if (!stop) st_relaxed_i32(lown + k, -1);  // consumed: the map is clean for the next column
            }
            stop = __shfl_sync(MCF_FULL, stop, 0);
            j = __shfl_sync(MCF_FULL, j, 0);
            if (stop) break;
            if (j < 0) continue;
            __threadfence();  // acquire side of the publication: the entry record is visible
            const int lt = __ldcg(llist + j);
            const bool push = lt < 0;
            const int t = push ? ~lt : lt;
            const int i = a.csc_rows[cs + t];
            const long long base = push ? 0 : a.csc_ptr[i];
            const long long end = push ? nsupp : a.csc_ptr[i + 1];
            const long long lo = base + (long long)(k - __ldcg(lbase + j)) * a.chunk_c;
            const long long hi = lo + a.chunk_c < end ? lo + a.chunk_c : end;
            const long long acc = uniform_partial(a, tab, lkeys, lvals, filt, i, push, lo, hi, lane, 3);
            if (lane == 0 && acc) atomicAdd(lacc + j, (unsigned long long)acc);
        }
        cl.sync();
        phase(4);  // entries and pieces
        const int nlong_all = *r0_nlong;
        const int nlong = nlong_all < a.llcap ? nlong_all : (int)a.llcap;
        for (long long j = gt; j < nlong; j += CT) {
            const int lt = __ldcg(llist + j);
            if (lt == INT_MAX) continue;
            const int t = lt < 0 ? ~lt : lt;
            a.pcol[cs + t] = a.csc_vals[cs + t] * (a.value * ldexp((double)(long long)__ldcg(lacc + j), -E));
        }
        if (a.prof && rank == 0 && tid == 0) {
            atomicAdd(a.prof + 16, 1ull);
            atomicAdd(a.prof + 17, (unsigned long long)(clock64() - t_start));
            atomicAdd(a.prof + 18, (unsigned long long)m);
            atomicAdd(a.prof + 19, (unsigned long long)(t_built - t_start));
        }
        cl.sync();  // every remote access of this column is done before the tables and counters are reset
        phase(5);  // finalize + end barrier
        if (cbits) {  // clear the bitmap words of this CTA's keys before the next column sets its own
            for (int t = tid; t < SCAP; t += Q_THREADS) {
                const int key = skeys[t];
                if (key != EMPTY_KEY) __stcg(cbits + (key >> 5), 0u);
            }
            __threadfence();
        }
    }
}

// columns of [col_begin, col_end) by the cluster size their table needs: list k
// (K = 2 << k) at cols + k * ncol, counts in cnt[k]
__global__ void k_cluster_classify(QArgs a, int *__restrict__ cols, long long ncol, unsigned *__restrict__ cnt) {
    for (long long c = a.col_begin + (long long)blockIdx.x * blockDim.x + threadIdx.x; c < a.col_end;
         c += (long long)gridDim.x * blockDim.x) {
        const long long g0 = a.walk_pre[c], g1 = a.walk_pre[c + 1];
        if (g0 == g1) continue;
        const long long m = slot_of(a, g1) - slot_of(a, g0);
        const int k = cluster_class(m < a.n ? m : a.n, a.cl_maxk);
        if (!k) continue;
        const int li = k == 2 ? 0 : (k == 4 ? 1 : 2);
        const unsigned p = atomicAdd(cnt + li, 1u);
        cols[li * ncol + p] = (int)c;
    }
}

// Combine of the big columns: the (column, entry) pairs of all records are
// flattened (prefix over cn) and spread over every warp of the GPU; each pair
// is still reduced by one warp in a fixed order.
__global__ void __launch_bounds__(256) k_diag_big(QArgs a, const long long *__restrict__ item_pre, unsigned nrec) {
    const int lane = threadIdx.x & 31;
    const long long total = item_pre[nrec];
    const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
    for (long long x = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5; x < total; x += nw) {
        unsigned lo = 0, hi = nrec - 1;  // record b with item_pre[b] <= x < item_pre[b+1]
        while (lo < hi) {
            const unsigned mid = (lo + hi + 1) >> 1;
            if (item_pre[mid] <= x) lo = mid;
            else hi = mid - 1;
        }
        const BigRec r = a.big[lo];
        const long long t = x - item_pre[lo];
        const int *keys = a.pool_keys + r.off;
        const long long *vals = a.pool_vals + r.off;
        const unsigned *filt = a.pool_filt + (long long)lo * FILTER_WORDS;
        const long long cs = a.csc_ptr[r.c];
        const double v = pair_value(a, keys, vals, r.cap - 1, keys + r.cap, vals + r.cap, a.pool_nsupp[lo], filt,
                                    a.pool_E[lo], a.csc_rows[cs + t], a.csc_vals[cs + t], lane);
        if (lane == 0) a.pcol[cs + t] = v;
    }
}

__global__ void k_big_counts(const BigRec *__restrict__ big, unsigned nrec, long long *__restrict__ cnt) {
    unsigned b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b < nrec) cnt[b] = big[b].cn;
}

// ---------------------------------------------------------------------------
// Combine units (uniform-value graphs; the default).  A walked column c whose
// Q_c is too wide for one CTA's shared table is split into K = 2^k units by
// KEY GROUP (key_group, NGROUPS): unit u builds, in its own shared memory,
// the part of Q_c whose keys fall in its group range, and adds
// sum_{j in C_i, group(j) in range} Q_c[j] for every entry (i, c) -- a
// contiguous slice of the group-ordered column C_i (g->ckeys, g->gofs).  The
// K int64 partials of an entry sum to the int64 <Q_c, C_i> the single-table
// kernels form, so pcol is bit-identical to theirs, with every probe in local
// shared memory: no distributed shared memory, no cluster barriers, no global
// tables, no GPU-wide hand-off of big columns.  One persistent kernel takes the
// units of all columns, widest first (K = NGROUPS ... 1).
// Inside a unit: 32 entries per warp-step have their slices located together
// (coalesced metadata loads); slices of <= UNIT_SERIAL ids are scanned by one
// lane each, longer ones (and push entries) are queued and cut into pieces of
// `chunk` ids that all warps share.  Partials of split entries are int64
// atomics into the entry's pcol slot (zeroed by k_unit_classify), converted to
// fp64 when the column's last unit finishes (deterministic: integer sums).
// ---------------------------------------------------------------------------
constexpr int UNIT_SERIAL = 24;  // slice length scanned by one lane
constexpr int UNIT_BUCKETS = GROUP_BITS + 1;  // K = 1, 2, ..., NGROUPS
constexpr int UPROF_SLOTS = 16;

struct UArgs {
    const long long *__restrict__ walk_pre;
    long long wb, slot_len;
    const long long *__restrict__ eoff;
    const long long *__restrict__ walk_off;
    long long off_base;
    const int *__restrict__ est;
    const double *__restrict__ ewt;
    const long long *__restrict__ csc_ptr;
    const int *__restrict__ csc_rows;
    const double *__restrict__ csc_vals;
    const int *__restrict__ ckeys;
    const int *__restrict__ gidx;
    const int *__restrict__ gofs;
    long long n;
    long long c0, ncol;  // the batch's column range [c0, c0 + ncol)
    double *__restrict__ pcol;
    double value;
    const unsigned long long *__restrict__ colmax;
    int push_pct;
    int opt;
    const int *hub_of;
    const unsigned *hub_bits;
    long long hub_words;
    const int *__restrict__ lists;  // bucket k's columns at lists + k * ncol
    const unsigned *__restrict__ bcnt;  // columns per bucket
    unsigned long long *counter;
    int *done;           // per column of the batch: finished units
    int *qt;             // per-CTA queue of long entries: entry (~t: push), slice start, length, piece prefix
    long long *qlo;
    int *qlen;
    long long *qpre;
    long long qcap;
    int *pmap;           // per-CTA piece -> queue entry map (pcap each; wider units binary-search qpre)
    long long pcap;
    long long chunk;
    int dbg_skip;          // MCF_UNIT_DEBUG_SKIP (timing experiments only): 1 = no scans, 2 = no build either
    int serial_small;      // slices scanned by one lane in phase A when the column has < 32 entries per warp
    long long small_need;  // widest table need of a one-unit column
    long long small_cut;   // one-unit columns up to this need go to the small-table kernel (list UNIT_BUCKETS)
    long long mid_cut;     // ... up to this one to the mid-size kernel (list UNIT_BUCKETS + 1)
    long long ucap;        // table need per unit of a split column
    int dense_n;           // n at or below which a one-unit column may use a dense Q_c
    int *err;              // bit 8: a unit table overflowed
    unsigned long long *prof;
    // emissions of the split columns regrouped by unit (k_unit_partition), or
    // null: then every unit scans the whole column and keeps its groups
    int *pest;
    double *pewt;
    int *pofs;                          // per split column: K + 1 unit offsets (relative to its first slot)
    long long pbase[UNIT_BUCKETS];      // bucket k's first offset row in pofs
};

__device__ __forceinline__ long long uslot(const UArgs &a, long long g) {
    if (a.slot_len > 0) return (g - a.wb) * a.slot_len;
    if (a.eoff) return a.eoff[g - a.wb];
    return a.walk_off[g] - a.off_base + (g - a.wb);
}

// units a column's table need takes (power of two; 0: too wide for NGROUPS units)
__device__ __forceinline__ int unit_count(long long need, long long small_need, long long ucap, bool dense_ok) {
    if (dense_ok || need <= small_need) return 1;
    const long long k = (need + ucap - 1) / ucap;
    int K = 2;
    while (K < k) K <<= 1;
    return K <= NGROUPS ? K : 0;
}

// One warp per 32 columns of the batch: unit count, bucket lists (warp-
// aggregated appends), pcol slots of walked columns zeroed, done counters.
// need_max[0] = widest need that did not fit NGROUPS units (host falls back).
__global__ void k_unit_classify(UArgs a, int *__restrict__ lists, unsigned *__restrict__ bcnt,
                                unsigned long long *__restrict__ too_wide) {
    const int lane = threadIdx.x & 31;
    const long long w0 = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
    for (long long base = w0 * 32; base < a.ncol; base += nw * 32) {
        const long long c = a.c0 + base + lane;
        int b = -1;
        if (base + lane < a.ncol) {
            const long long g0 = a.walk_pre[c], g1 = a.walk_pre[c + 1];
            if (g0 != g1) {
                const long long m = uslot(a, g1) - uslot(a, g0);
                const long long need = m < a.n ? m : a.n;
                const bool dense_ok = a.n <= a.dense_n;
                const int K = unit_count(need, a.small_need, a.ucap, dense_ok);
                if (K == 0) {
                    atomicMax(too_wide, (unsigned long long)need);
                } else {
                    b = 31 - __clz(K);
                    if (K == 1 && !dense_ok && need <= a.small_cut) b = UNIT_BUCKETS;           // 4 tables per SM
                    else if (K == 1 && !dense_ok && need <= a.mid_cut) b = UNIT_BUCKETS + 1;  // 2 tables per SM
                }
                a.done[base + lane] = 0;
            }
        }
        for (int k = 0; k <= UNIT_BUCKETS + 1; ++k) {
            const unsigned msk = __ballot_sync(MCF_FULL, b == k);
            if (!msk) continue;
            unsigned p0 = 0;
            // counts: buckets 0..7 at [k]; the small / mid tiers at [16] / [24] (zeros after each)
            const int ci = k < UNIT_BUCKETS ? k : 16 + 8 * (k - UNIT_BUCKETS);
            if (lane == __ffs(msk) - 1) p0 = atomicAdd(bcnt + ci, (unsigned)__popc(msk));
            p0 = __shfl_sync(MCF_FULL, p0, __ffs(msk) - 1);
            if (b == k) lists[k * a.ncol + p0 + __popc(msk & lanemask_lt())] = (int)c;
        }
        // zero the pcol slots of the walked columns (atomics land there)
        unsigned walked = __ballot_sync(MCF_FULL, b >= 0);
        while (walked) {
            const int l = __ffs(walked) - 1;
            walked &= walked - 1;
            const long long cc = a.c0 + base + l;
            const long long lo = a.csc_ptr[cc], hi = a.csc_ptr[cc + 1];
            for (long long e = lo + lane; e < hi; e += 32) a.pcol[e] = 0.0;
        }
    }
}

// Emissions of every split column (K >= 2) regrouped by unit: unit u's
// emissions land in [s0 + pofs[u], s0 + pofs[u + 1]) of pest/pewt (order
// inside a unit is arbitrary: Q_c sums are integers).  One CTA per column,
// widest first; a counting pass, a scan, a scatter pass.
constexpr int PART_TH = 512;
__global__ void __launch_bounds__(PART_TH) k_unit_partition(UArgs a, unsigned *__restrict__ next) {
    __shared__ int cnt[NGROUPS];
    __shared__ long long s_c;
    __shared__ int s_k, s_sidx;
    const int tid = threadIdx.x, lane = tid & 31;
    while (true) {
        __syncthreads();
        if (tid == 0) {
            unsigned x = atomicAdd(next, 1u);
            int k = UNIT_BUCKETS - 1;
            for (; k >= 1; --k) {
                const unsigned nb = __ldcg(a.bcnt + k);
                if (x < nb) break;
                x -= nb;
            }
            s_k = k;
            s_sidx = (int)x;
            s_c = k >= 1 ? (long long)a.lists[k * a.ncol + x] : -1;
        }
        __syncthreads();
        const long long c = s_c;
        if (c < 0) break;
        const int k = s_k, K = 1 << k, shift = GROUP_BITS - k;
        const long long s0 = uslot(a, a.walk_pre[c]), m = uslot(a, a.walk_pre[c + 1]) - s0;
        for (int t = tid; t < K; t += PART_TH) cnt[t] = 0;
        __syncthreads();
        // warp-aggregated per-unit counts (hot keys share a unit)
        for (long long b = 0; b < m; b += 4 * PART_TH) {
            int st[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const long long i = b + q * PART_TH + tid;
                st[q] = i < m ? __ldcs(a.est + s0 + i) : -1;
            }
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int uq = st[q] >= 0 ? (int)(key_group(st[q]) >> shift) : -1;
                const unsigned same = __match_any_sync(MCF_FULL, uq);
                if (uq >= 0 && lane == __ffs(same) - 1) atomicAdd(&cnt[uq], __popc(same));
            }
        }
        __syncthreads();
        int *of = a.pofs + a.pbase[k] + (long long)s_sidx * (K + 1);
        if (tid == 0) {
            int run = 0;
            for (int t = 0; t < K; ++t) {
                const int v = cnt[t];
                of[t] = run;
                cnt[t] = run;
                run += v;
            }
            of[K] = run;
        }
        __syncthreads();
        for (long long b = 0; b < m; b += 4 * PART_TH) {
            int st[4];
            double wt[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const long long i = b + q * PART_TH + tid;
                st[q] = i < m ? __ldcs(a.est + s0 + i) : -1;
            }
#pragma unroll
            for (int q = 0; q < 4; ++q) wt[q] = st[q] >= 0 ? __ldcs(a.ewt + s0 + b + q * PART_TH + tid) : 0.0;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int uq = st[q] >= 0 ? (int)(key_group(st[q]) >> shift) : -1;
                const unsigned same = __match_any_sync(MCF_FULL, uq);
                const int leader = __ffs(same) - 1;
                int p0 = 0;
                if (uq >= 0 && lane == leader) p0 = atomicAdd(&cnt[uq], __popc(same));
                p0 = __shfl_sync(MCF_FULL, p0, leader);
                if (uq >= 0) {
                    const long long p = s0 + p0 + __popc(same & lanemask_lt());
                    a.pest[p] = st[q];
                    a.pewt[p] = wt[q];
                }
            }
        }
    }
}

// The unit kernel's table in shared memory, addressed by 32-bit shared
// addresses (no generic-pointer conversions in the probe loops): keys (int),
// values (int64) and a one-word-per-key Bloom filter (three bits of one
// 32-bit word: one shared load answers most misses).
struct UTab {
    unsigned keys, vals, filt;  // shared-window byte addresses
    uint32_t mask;              // hash table: slots - 1
    bool dense;                 // values indexed by node id (small graphs), no keys
    int fshift;                 // Bloom word of a key: (key * C) >> fshift (the kernel's 2^(32 - fshift) words)
    int tshift;                 // home slot: (key * phi) >> tshift == hash_slot(key, mask) (slots a power of two)
};
__device__ __forceinline__ uint32_t ufilt_word(int key, int fshift) { return ((uint32_t)key * 0x85EBCA6Bu) >> fshift; }
// one bit per key: the 5 hash bits just below the word index (a miss costs a
// multiply, two shifts and one shared load; measured cheaper than three bits)
__device__ __forceinline__ uint32_t ufilt_bit(int key, int fshift) {
    return 1u << ((((uint32_t)key * 0x85EBCA6Bu) >> (fshift - 5)) & 31u);
}
__device__ __forceinline__ unsigned lds32(unsigned addr) {
    unsigned v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
    return v;
}
__device__ __forceinline__ long long lds64(unsigned addr) {
    long long v;
    asm volatile("ld.shared.s64 %0, [%1];" : "=l"(v) : "r"(addr));
    return v;
}
__device__ __forceinline__ bool utab_maybe(const UTab &t, int key) {
    const uint32_t m = ufilt_bit(key, t.fshift);
    return (lds32(t.filt + 4 * ufilt_word(key, t.fshift)) & m) == m;
}
// The unit kernel's dynamic shared memory by name (values at 0, keys at
// 8 CAP): array accesses with constant offsets compile to LDS [reg + imm],
// with no shared-window base to rematerialise per probe.
extern __shared__ __align__(16) unsigned char mcf_usmem[];
// Linear probing from the key's aligned quad of slots: one 16-B shared load
// answers a lookup unless all four slots hold other keys (the table is at
// most half full, so that is rare); the hit's value is read once, after the
// loop, so lanes that needed another quad do not split the value load.
// sb: the dynamic shared window's address (held in a register by the caller).
__device__ __forceinline__ int4 lds128(unsigned addr) {
    int4 v;
    asm volatile("ld.shared.v4.s32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
    return v;
}
// shared-space atomics by 32-bit shared address (the build loop below: no
// generic-pointer address-space checks, reductions where no value returns)
__device__ __forceinline__ int atoms_cas32(unsigned addr, int cmp, int val) {
    int old;
    asm volatile("atom.shared.cas.b32 %0, [%1], %2, %3;" : "=r"(old) : "r"(addr), "r"(cmp), "r"(val) : "memory");
    return old;
}
__device__ __forceinline__ unsigned atoms_add32(unsigned addr, unsigned v) {
    unsigned old;
    asm volatile("atom.shared.add.u32 %0, [%1], %2;" : "=r"(old) : "r"(addr), "r"(v) : "memory");
    return old;
}
__device__ __forceinline__ void reds_add32(unsigned addr, unsigned v) {
    asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}
__device__ __forceinline__ void reds_or32(unsigned addr, unsigned v) {
    asm volatile("red.shared.or.b32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}
// Find or claim `key` in the unit table, with an occupancy guard: a table
// past its limit drops the key and flags the overflow (never expected: need
// per unit has a ~12 sigma margin).  Keys at shared address kb, cap =
// mask + 1 slots.  Scan the quads from the key's home quad, one 16-B load
// each; the key goes to the first slot in probe order that holds it or is
// empty, so utab_get's "an empty slot ends the search" stays true.  A lost
// claim re-reads the same quad.  Returns the slot (fresh: this lane claimed
// it) or -1 when the table is over its limit (error bit 256 set).
__device__ __forceinline__ int unit_claim(unsigned kb, uint32_t mask, int tshift, int key, unsigned nk_addr, int limit,
                                          int *err, bool &fresh) {
    uint32_t s = (((uint32_t)key * 0x9E3779B1u) >> tshift) & ~3u;
    for (uint32_t quads = 0; quads <= (mask >> 2) + 1; ++quads) {
        while (true) {
            const int4 k = lds128(kb + 4u * s);
            const bool h0 = k.x == key || k.x == EMPTY_KEY, h1 = k.y == key || k.y == EMPTY_KEY;
            const bool h2 = k.z == key || k.z == EMPTY_KEY, h3 = k.w == key || k.w == EMPTY_KEY;
            if (!(h0 | h1 | h2 | h3)) break;  // four other keys: next quad
            const int j = h0 ? 0 : (h1 ? 1 : (h2 ? 2 : 3));
            const int kv = h0 ? k.x : (h1 ? k.y : (h2 ? k.z : k.w));
            if (kv == key) return (int)s + j;
            if ((int)lds32(nk_addr) >= limit) {
                atomicOr(err, 256);
                return -1;
            }
            const int old = atoms_cas32(kb + 4u * (s + j), EMPTY_KEY, key);
            if (old == EMPTY_KEY) {
                fresh = true;
                return (int)s + j;
            }
            if (old == key) return (int)s + j;
        }
        s = (s + 4) & mask;
    }
    atomicOr(err, 256);  // every quad full (the key count lags the claims by at most one warp step)
    return -1;
}
template <int CAP>
__device__ __forceinline__ long long utab_get(const UTab &t, unsigned sb, int key) {
    if (t.dense) return lds64(sb + 8u * (unsigned)key);
    uint32_t s = (((uint32_t)key * 0x9E3779B1u) >> t.tshift) & ~3u;
    int slot;
    while (true) {
        const int4 k = lds128(sb + 8u * CAP + 4u * s);
        const bool e0 = k.x == key, e1 = k.y == key, e2 = k.z == key, e3 = k.w == key;
        if (e0 | e1 | e2 | e3) {
            slot = (int)s + (e0 ? 0 : (e1 ? 1 : (e2 ? 2 : 3)));
            break;
        }
        if ((k.x | k.y | k.z | k.w) < 0) {  // an empty slot in the quad: the key is absent
            slot = -1;
            break;
        }
        s = (s + 4) & t.mask;
    }
    return slot >= 0 ? lds64(sb + 8u * (unsigned)slot) : 0ll;
}
// the dynamic shared window's address, in a register the compiler cannot
// rematerialise (recomputing it from the CTA's cluster rank costs 5-6
// instructions per probe at this kernel's 64-register budget)
__device__ __forceinline__ unsigned usmem_base() {
    unsigned b = (unsigned)__cvta_generic_to_shared(mcf_usmem);
    return __shfl_sync(MCF_FULL, b, 0);
}
#ifndef UNIT_PULL_U
#define UNIT_PULL_U 16
#endif
#ifndef UNIT_PUSH_U
#define UNIT_PUSH_U 4
#endif
// jv[u] for a lane-varying u < 8 without local memory (a select tree)
__device__ __forceinline__ int sel8(const int (&v)[8], int u) {
    const int a0 = (u & 1) ? v[1] : v[0], a1 = (u & 1) ? v[3] : v[2];
    const int a2 = (u & 1) ? v[5] : v[4], a3 = (u & 1) ? v[7] : v[6];
    const int b0 = (u & 2) ? a1 : a0, b1 = (u & 2) ? a3 : a2;
    return (u & 4) ? b1 : b0;
}
template <int N>
__device__ __forceinline__ int selu(const int (&v)[N], int u) {
    if constexpr (N == 4) {
        const int a0 = (u & 1) ? v[1] : v[0], a1 = (u & 1) ? v[3] : v[2];
        return (u & 2) ? a1 : a0;
    } else if constexpr (N == 8) {
        return sel8(v, u);
    } else {
        static_assert(N == 16, "4, 8 or 16 ids per lane");
        const int lo8[8] = {v[0], v[1], v[2], v[3], v[4], v[5], v[6], v[7]};
        const int hi8[8] = {v[8], v[9], v[10], v[11], v[12], v[13], v[14], v[15]};
        const int a = sel8(lo8, u & 7), b = sel8(hi8, u & 7);
        return (u & 8) ? b : a;
    }
}

#ifndef UNIT_SHORT_TAIL
#define UNIT_SHORT_TAIL 1
#endif
// One block of the pull scan: NU ids per lane at p[0], p[32], ... (immediate
// offsets; `rem` of the warp's ids are this lane's or later, FULL: all valid),
// a branch-free Bloom stage over all of them, then the passing ids (bit mask)
// probed one after another -- a warp runs the probe code max-over-lanes-of-
// passes times instead of once per id slot.
template <int CAP, int NU, bool FULL>
__device__ __forceinline__ long long pull_block(const UTab &tab, unsigned sb, const int *p, int rem) {
    int jv[NU];
    unsigned pm = 0;
    if (FULL) {  // no bounds predicates, every id valid
#pragma unroll
        for (int u = 0; u < NU; ++u) jv[u] = __ldg(p + 32 * u);
#pragma unroll
        for (int u = 0; u < NU; ++u) {
            const uint32_t h = (uint32_t)jv[u] * 0x85EBCA6Bu;
            const unsigned w = lds32(tab.filt + 4 * (h >> tab.fshift));
            pm |= ((w >> ((h >> (tab.fshift - 5)) & 31u)) & 1u) << u;
        }
    } else {
#pragma unroll
        for (int u = 0; u < NU; ++u) jv[u] = 32 * u < rem ? __ldg(p + 32 * u) : -1;
#pragma unroll
        for (int u = 0; u < NU; ++u) {
            const uint32_t h = (uint32_t)jv[u] * 0x85EBCA6Bu;
            const unsigned w = lds32(tab.filt + 4 * (h >> tab.fshift));
            pm |= ((w >> ((h >> (tab.fshift - 5)) & 31u)) & (unsigned)(jv[u] >= 0)) << u;
        }
    }
    long long acc = 0;
    if (tab.dense) {  // (small graphs) Q_c indexed by node id
        while (pm) {
            const int u = __ffs(pm) - 1;
            pm &= pm - 1;
            acc += lds64(sb + 8u * (unsigned)selu<NU>(jv, u));
        }
    } else {
        while (pm) {
            const int u = __ffs(pm) - 1;
            pm &= pm - 1;
            acc += utab_get<CAP>(tab, sb, selu<NU>(jv, u));
        }
    }
    return acc;
}

// sum of Q_c over the ids ckeys[lo, hi) (warp-cooperative, PULL_U ids per
// lane in flight) or over the unit's support positions [lo, hi) tested
// against hub row i's bitmap (push)
template <int CAP>
__device__ __forceinline__ long long unit_scan(const UArgs &a, const UTab &tab, int i, bool push, long long lo,
                                               long long hi, int lane) {
    long long acc = 0;
    if (push) {
        const unsigned *bits = a.hub_bits + (long long)__ldg(a.hub_of + i) * a.hub_words;
        constexpr int PUSH_U = UNIT_PUSH_U;
        for (long long t0 = lo; t0 < hi; t0 += 32 * PUSH_U) {
            int kv[PUSH_U];
            unsigned wv[PUSH_U];
#pragma unroll
            for (int u = 0; u < PUSH_U; ++u) {
                const long long t = t0 + 32 * u + lane;
                kv[u] = t < hi ? reinterpret_cast<const int *>(mcf_usmem + 8 * CAP)[t] : -1;  // table slot (or empty)
            }
#pragma unroll
            for (int u = 0; u < PUSH_U; ++u) wv[u] = kv[u] >= 0 ? __ldg(bits + (kv[u] >> 5)) : 0u;
#pragma unroll
            for (int u = 0; u < PUSH_U; ++u)
                if ((wv[u] >> (kv[u] & 31)) & 1u) acc += reinterpret_cast<const long long *>(mcf_usmem)[t0 + 32 * u + lane];
        }
    } else {
        // full blocks of 32 PULL_U ids, then the tail with as few ids per lane as cover it
        constexpr int PULL_U = UNIT_PULL_U;
        const unsigned sb = usmem_base();
        const int *p = a.ckeys + lo + lane;
        int remw = (int)(hi - lo);  // ids left for the warp (uniform); a lane's are `remw - lane`
        for (; remw >= 32 * PULL_U; remw -= 32 * PULL_U, p += 32 * PULL_U)
            acc += pull_block<CAP, PULL_U, true>(tab, sb, p, 0);
        if (remw > 0) {
            // (tails of 1, 2 and 12 ids per lane measured no faster than these)
            const int rem = remw - lane;
            if (UNIT_SHORT_TAIL && PULL_U > 4 && remw <= 128) acc += pull_block<CAP, 4, false>(tab, sb, p, rem);
            else if (UNIT_SHORT_TAIL && PULL_U > 8 && remw <= 256) acc += pull_block<CAP, 8, false>(tab, sb, p, rem);
            else acc += pull_block<CAP, PULL_U, false>(tab, sb, p, rem);
        }
    }
    return warp_sum_ll(acc);
}

// A unit and what its CTA needs to start it.  Thread 0 fetches the NEXT unit
// (work counter, bucket lists, walk prefix, slice offsets, column pointers)
// while the current one is combined, and asks the copy engine to pull its
// emission slice into L2.
struct UnitRec {
    long long c, s0, m, e0, e1, cs, cn;
    unsigned long long maxw;
    int u, lg, sidx;
};

__device__ __forceinline__ void l2_prefetch_range(const void *p, long long bytes) {
    const char *b = reinterpret_cast<const char *>((reinterpret_cast<uintptr_t>(p)) & ~(uintptr_t)15);
    long long len = bytes + (reinterpret_cast<const char *>(p) - b);
    if (len > (1ll << 20)) len = 1ll << 20;  // the first MiB: the rest streams in behind the reads
    for (long long o = 0; o < len; o += 32768) {
        const unsigned n = (unsigned)(((len - o < 32768 ? len - o : 32768) + 15) & ~15ll);
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(b + o), "r"(n) : "memory");
    }
}

__device__ __forceinline__ void unit_fetch(const UArgs &a, const unsigned *sbc, UnitRec &r) {
    unsigned long long x = atomicAdd(a.counter, 1ull);
    r.c = -1;
    for (int k = UNIT_BUCKETS - 1; k >= 0; --k) {  // widest columns first
        const unsigned long long nu = (unsigned long long)sbc[k] << k;
        if (x < nu) {
            r.sidx = (int)(x >> k);
            r.c = a.lists[k * a.ncol + r.sidx];
            r.u = (int)(x & ((1ull << k) - 1));
            r.lg = k;
            break;
        }
        x -= nu;
    }
    if (r.c < 0) return;
    const long long c = r.c;
    const long long g0 = a.walk_pre[c], g1 = a.walk_pre[c + 1];
    r.s0 = uslot(a, g0);
    r.m = uslot(a, g1) - r.s0;
    r.cs = a.csc_ptr[c];
    r.cn = a.csc_ptr[c + 1] - r.cs;
    r.maxw = a.colmax[c];
    r.e0 = 0;
    r.e1 = r.m;
    const bool parted = r.lg > 0 && a.pest;
    if (parted) {
        const int *of = a.pofs + a.pbase[r.lg] + (long long)r.sidx * ((1 << r.lg) + 1) + r.u;
        r.e0 = of[0];
        r.e1 = of[1];
    }
    if (r.e1 > r.e0) {
        l2_prefetch_range((parted ? a.pest : a.est) + r.s0 + r.e0, (r.e1 - r.e0) * 4);
        l2_prefetch_range((parted ? a.pewt : a.ewt) + r.s0 + r.e0, (r.e1 - r.e0) * 8);
    }
}

template <int TH, int CAP, int FW>
__global__ void __launch_bounds__(TH, 1024 / TH) k_diag_unit(UArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    long long *svals = reinterpret_cast<long long *>(smem_raw);
    int *skeys = reinterpret_cast<int *>(svals + CAP);
    unsigned *filt = reinterpret_cast<unsigned *>(skeys + CAP);
    constexpr int NWARP = TH / 32;
    static_assert((FW & (FW - 1)) == 0 && FW >= 32, "Bloom filter words: a power of two");
    constexpr int FSHIFT = 32 - __builtin_ctz(FW);
    __shared__ long long s_c, s_np, s_wsum[NWARP];
    __shared__ int s_u, s_lg, s_next, s_nq, s_nsupp, s_nkeys, s_last, s_sidx;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    int *qt = a.qt + (long long)blockIdx.x * a.qcap;
    long long *qlo = a.qlo + (long long)blockIdx.x * a.qcap;
    int *qlen = a.qlen + (long long)blockIdx.x * a.qcap;
    long long *qpre = a.qpre + (long long)blockIdx.x * (a.qcap + 1);
    int *pmap = a.pmap + (long long)blockIdx.x * a.pcap;
    unsigned long long pr[5] = {0, 0, 0, 0, 0};  // MCF_DIAG_PROF: serial entries, serial ids, pieces, pull ids, push tests
    __shared__ unsigned s_bc[UNIT_BUCKETS];
    __shared__ UnitRec s_cur, s_nxt;
    if (tid < UNIT_BUCKETS) s_bc[tid] = __ldcg(a.bcnt + tid);
    __syncthreads();
    if (tid == 0) unit_fetch(a, s_bc, s_nxt);

    while (true) {
        __syncthreads();
        if (tid == 0) {
            s_cur = s_nxt;
            s_c = s_cur.c;
            s_u = s_cur.u;
            s_lg = s_cur.lg;
            s_sidx = s_cur.sidx;
            s_next = 0;
            s_nq = 0;
            s_nsupp = 0;
            s_nkeys = 0;
            s_np = 0;
        }
        __syncthreads();
        const long long c = s_c;
        if (c < 0) break;
        const int u = s_u, lg = s_lg, K = 1 << lg, shift = GROUP_BITS - lg;
        const long long s0 = s_cur.s0, m = s_cur.m;
        const long long need = m < a.n ? m : a.n;
        const long long t_start = a.prof ? clock64() : 0;
        // this unit's emissions: the whole column (filtered by group below), or
        // its regrouped slice [s0 + e0, s0 + e1) of pest / pewt
        const bool parted = K > 1 && a.pest;
        const long long e0 = s_cur.e0, e1 = s_cur.e1;
        const int *__restrict__ est = parted ? a.pest : a.est;
        const double *__restrict__ ewt = parted ? a.pewt : a.ewt;
        // table: one unit -> sized by need (k_diag_q's rule); K units -> need / K
        // plus a 1/8 + 64 margin for the group's share of the support (and at
        // most the unit's emission count when known)
        const bool dense = K == 1 && a.n <= a.dense_n && need * 4 > a.n;
        long long need_u = K == 1 ? need : need / K + need / (8 * K) + 64;
        if (need_u > need) need_u = need;
        if (parted && need_u > e1 - e0) need_u = e1 - e0;
        uint32_t cap = 32;
        while ((long long)cap < need_u * 2 && cap < (uint32_t)CAP) cap <<= 1;
        while ((long long)cap * 3 < need_u * 4 + 4 && cap < (uint32_t)CAP) cap <<= 1;
        int *keys = dense ? nullptr : skeys;
        long long *vals = svals;
        if (dense) cap = (uint32_t)a.n;
        const uint32_t mask = cap - 1;
        const int limit = (int)(cap - cap / 8);
        for (uint32_t t = tid; t < cap; t += TH) {
            if (keys) keys[t] = EMPTY_KEY;
            vals[t] = 0;
        }
        for (int t = tid; t < FW; t += TH) filt[t] = 0u;
        __syncthreads();
        const long long t_zeroed = a.prof ? clock64() : 0;
        const double maxw = __longlong_as_double((long long)s_cur.maxw);
        const int lg_m = m <= 1 ? 0 : 64 - __clzll(m - 1);  // smallest lg with 2^lg >= m
        const int E = maxw > 0.0 ? 61 - ilogb(maxw) - lg_m : 0;  // as k_diag_q: sum of m terms < 2^62
        // w 2^E as one multiply when 2^E is a normal double (exact: a power-of-two
        // scaling rounds like ldexp, subnormal results included)
        const bool escale_ok = E >= -1022 && E <= 1023;
        const double escale = escale_ok ? __longlong_as_double((long long)(E + 1023) << 52) : 0.0;
        // Q_c over this unit's key groups
        constexpr int U = 4;
        for (long long base = e0; base < (a.dbg_skip >= 2 ? e0 : e1); base += (long long)U * TH) {
            int sv[U];
#pragma unroll
            for (int q = 0; q < U; ++q) {  // all U loads issued before any is used
                const long long i = base + (long long)q * TH + tid;
                sv[q] = i < e1 ? __ldcs(est + s0 + i) : EMPTY_KEY;
            }
            if (K > 1 && !parted) {
#pragma unroll
                for (int q = 0; q < U; ++q)
                    if (sv[q] >= 0 && (int)(key_group(sv[q]) >> shift) != u) sv[q] = EMPTY_KEY;
            }
            double wv[U];
#pragma unroll
            for (int q = 0; q < U; ++q) {  // (unfiltered ranges: issued with the key loads, not after them)
                const long long i = base + (long long)q * TH + tid;
                wv[q] = (K == 1 || parted ? i < e1 : sv[q] >= 0) ? __ldcs(ewt + s0 + i) : 0.0;
            }
            // lanes holding the same key add once (step-major slots: a warp's
            // 32 walks share the start state at step 0 and hubs later on); the
            // group's first lane finds or claims the slot, then all such lanes
            // together set the new keys' Bloom bits, count them (one add per
            // warp) and add their sums (two 32-bit atomics with carry)
            const unsigned sbb = (unsigned)__cvta_generic_to_shared(smem_raw);
            const unsigned nk_addr = (unsigned)__cvta_generic_to_shared(&s_nkeys);
            const int tshift_b = 32 - (31 - __clz((int)cap));
#pragma unroll
            for (int q = 0; q < U; ++q) {
                const int key = sv[q];
                if (!__any_sync(MCF_FULL, key >= 0)) continue;  // no key of this unit in the warp's slot (uniform)
                long long qv = key >= 0 ? __double2ll_rn(escale_ok ? wv[q] * escale : ldexp(wv[q], E)) : 0;
                const unsigned same = __match_any_sync(MCF_FULL, key);
                bool lead = key >= 0;
                if (lead && __popc(same) > 1) {
                    qv = group_sum_i64(same, qv);
                    lead = lane == __ffs(same) - 1;
                }
                int slot = -1;
                bool fresh = false;
                if (lead) slot = keys ? unit_claim(sbb + 8u * CAP, mask, tshift_b, key, nk_addr, limit, a.err, fresh) : key;
                const unsigned fm = __ballot_sync(MCF_FULL, fresh);
                if (fm) {
                    if (fresh) {
                        const uint32_t h = (uint32_t)key * 0x85EBCA6Bu;
                        reds_or32(sbb + 12u * CAP + 4u * (h >> FSHIFT), 1u << ((h >> (FSHIFT - 5)) & 31u));
                    }
                    if (lane == 0) reds_add32(nk_addr, (unsigned)__popc(fm));
                }
                if (slot >= 0) {
                    const unsigned long long uq = (unsigned long long)qv;
                    const unsigned lo = (unsigned)uq, hi = (unsigned)(uq >> 32);
                    const unsigned addr = sbb + 8u * (unsigned)slot;
                    const unsigned oldw = atoms_add32(addr, lo);
                    const unsigned up = hi + (oldw + lo < oldw ? 1u : 0u);
                    if (up) reds_add32(addr + 4u, up);
                }
            }
        }
        __syncthreads();
        const long long t_inserted = a.prof ? clock64() : 0;
        // Bloom filter and key count: set by the inserting lanes; a dense Q_c
        // (small graphs) gets its filter from a pass over the node ids (push
        // entries scan the table's slots themselves: no support list)
        if (!keys) {
            for (uint32_t t = tid; t < cap; t += TH)
                if (vals[t] != 0) atomicOr(&filt[ufilt_word((int)t, FSHIFT)], ufilt_bit((int)t, FSHIFT));
            __syncthreads();
        }
        const int nsupp = keys ? s_nkeys : 0x3fffffff;  // dense tables: never push
        const long long t_built = a.prof ? clock64() : 0;
        const long long cs = s_cur.cs, cn = s_cur.cn;
        const UTab tab{(unsigned)__cvta_generic_to_shared(skeys), (unsigned)__cvta_generic_to_shared(svals),
                       (unsigned)__cvta_generic_to_shared(filt), mask, dense, FSHIFT, 32 - (31 - __clz((int)cap))};
        const double scale = a.value;
        // phase A: 32 entries per warp-step.  A column with fewer entries than
        // the CTA has lanes leaves most warps idle here, so it queues its
        // slices longer than a few ids for phase B, where all warps share them
        const int serial_max = cn >= 32 * NWARP ? UNIT_SERIAL : a.serial_small;
        while (!a.dbg_skip) {
            int t0 = 0;
            if (lane == 0) t0 = atomicAdd(&s_next, 32);
            t0 = __shfl_sync(MCF_FULL, t0, 0);
            if (t0 >= cn) break;
            const int t = t0 + lane;
            const bool valid = t < cn;
            int i = 0;
            long long lo = 0, hi = 0;
            bool grp_filter = false, push = false;
            if (valid) {
                i = __ldg(a.csc_rows + cs + t);
                lo = __ldg(a.csc_ptr + i);
                hi = __ldg(a.csc_ptr + i + 1);
                if (K > 1) {
                    if (hi - lo > GROUP_OFS_MIN) {
                        const int *of = a.gofs + (long long)__ldg(a.gidx + i) * (NGROUPS + 1);
                        const int gl = u << shift;
                        const long long b0 = __ldg(of + gl), b1 = __ldg(of + gl + (1 << shift));
                        hi = lo + b1;
                        lo = lo + b0;
                    } else {
                        grp_filter = true;
                    }
                }
                push = !grp_filter && a.hub_of && 100 * (hi - lo) > (long long)a.push_pct * nsupp &&
                       __ldg(a.hub_of + i) >= 0;
            }
            const bool serial = valid && !push && (grp_filter || hi - lo <= serial_max);
            long long acc = 0;
            if (serial) {
                for (long long e = lo; e < hi; e += 4) {
                    int jv[4];
#pragma unroll
                    for (int q = 0; q < 4; ++q) jv[q] = e + q < hi ? __ldg(a.ckeys + e + q) : -1;
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        if (jv[q] < 0) continue;
                        if (grp_filter && (int)(key_group(jv[q]) >> shift) != u) continue;
                        if (utab_maybe(tab, jv[q])) acc += utab_get<CAP>(tab, (unsigned)__cvta_generic_to_shared(mcf_usmem), jv[q]);
                    }
                }
                if (a.prof) {
                    pr[0] += 1;
                    pr[1] += (unsigned long long)(hi - lo);
                }
                if (K == 1) {
                    a.pcol[cs + t] = a.csc_vals[cs + t] * (scale * ldexp((double)acc, -E));
                } else if (acc) {
                    atomicAdd(reinterpret_cast<unsigned long long *>(a.pcol + cs + t), (unsigned long long)acc);
                }
            }
            const bool queued = valid && !serial && nsupp > 0 && (push || hi > lo);
            const unsigned qm = __ballot_sync(MCF_FULL, queued);
            if (qm) {
                int qb = 0;
                if (lane == 0) qb = atomicAdd(&s_nq, __popc(qm));
                qb = __shfl_sync(MCF_FULL, qb, 0);
                if (queued) {
                    const int k = qb + __popc(qm & lanemask_lt());
                    if (k < a.qcap) {
                        qt[k] = push ? ~t : t;
                        qlo[k] = push ? 0 : lo;
                        qlen[k] = (int)(push ? cap : hi - lo);  // push: the table's slots
                    } else {
                        atomicOr(a.err, 512);  // queue overflow (qcap >= max degree: not expected)
                    }
                }
            }
            if (!queued && valid && !serial && K == 1)  // nothing to scan: the zero partial
                a.pcol[cs + t] = a.csc_vals[cs + t] * (scale * ldexp(0.0, -E));
        }
        __syncthreads();
        const int nq = s_nq < a.qcap ? s_nq : (int)a.qcap;
        // piece prefix over the queue (block-wide scan, chunks of TH)
        for (int b0 = 0; b0 < nq; b0 += TH) {
            const int k = b0 + tid;
            long long v = k < nq ? (qlen[k] + a.chunk - 1) / a.chunk : 0;
            long long inc = v;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const long long x = __shfl_up_sync(MCF_FULL, inc, o);
                if (lane >= o) inc += x;
            }
            if (lane == 31) s_wsum[warp] = inc;
            __syncthreads();
            if (warp == 0) {
                long long ws = lane < NWARP ? s_wsum[lane] : 0, wi = ws;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const long long x = __shfl_up_sync(MCF_FULL, wi, o);
                    if (lane >= o) wi += x;
                }
                if (lane < NWARP) s_wsum[lane] = wi - ws;
            }
            __syncthreads();
            const long long carry = s_np;
            if (k < nq) {
                const long long p0 = carry + s_wsum[warp] + inc - v;
                qpre[k] = p0;
                for (long long p = p0; p < p0 + v && p < a.pcap; ++p) pmap[p] = k;
            }
            __syncthreads();
            if (tid == TH - 1) s_np = carry + s_wsum[warp] + inc;
            __syncthreads();
        }
        const long long npieces = s_np;
        if (tid == 0) {
            qpre[nq] = npieces;
            s_next = 0;
        }
        __syncthreads();
        // the next unit, fetched by thread 0 while the other warps take this
        // unit's pieces (phase B has no barrier until all pieces are done)
        if (tid == 0) unit_fetch(a, s_bc, s_nxt);
        // phase B: pieces of the queued entries, all warps.  A warp takes a
        // batch of pieces at a time: lane k resolves piece k's entry and range
        // (coalesced metadata loads, one dependent chain per batch instead of
        // one per piece), the warp scans them one after another, and lane k
        // stores piece k's sum.  The batch shrinks with the unit's piece count
        // so that a unit with few pieces still spreads over all warps.
        const int bsz = npieces >= 32ll * 4 * NWARP ? 32 : (npieces >= 8ll * 4 * NWARP ? 8 : 1);
        while (true) {
            int x0 = 0;
            if (lane == 0) x0 = atomicAdd(&s_next, bsz);
            x0 = __shfl_sync(MCF_FULL, x0, 0);
            if (x0 >= npieces) break;
            const int nb = npieces - x0 < bsz ? (int)(npieces - x0) : bsz;
            long long mb = 0;
            int mlen = 0, mt = 0;  // mlen: bit 30 = the entry has one piece
            if (lane < nb) {
                const int x = x0 + lane;
                int lo_j = 0, hi_j = nq - 1;  // last entry j with qpre[j] <= x
                if (npieces <= a.pcap) lo_j = hi_j = pmap[x];
                while (lo_j < hi_j) {
                    const int mid = (lo_j + hi_j + 1) >> 1;
                    if (qpre[mid] <= x) lo_j = mid;
                    else hi_j = mid - 1;
                }
                const int j = lo_j;
                mt = qt[j];
                const long long pq = x - qpre[j];
                const int len = qlen[j];
                const long long left = len - pq * a.chunk;
                mb = qlo[j] + pq * a.chunk;
                mlen = (int)(left < a.chunk ? left : a.chunk) | (len <= a.chunk ? 1 << 30 : 0);
            }
            long long myacc = 0;
            for (int k = 0; k < nb; ++k) {
                const long long pb = __shfl_sync(MCF_FULL, mb, k);
                const int plen = __shfl_sync(MCF_FULL, mlen, k) & 0x3fffffff;
                const int qtj = __shfl_sync(MCF_FULL, mt, k);
                const bool push = qtj < 0;
                const int i = push ? __ldg(a.csc_rows + cs + ~qtj) : 0;
                const long long acc = unit_scan<CAP>(a, tab, i, push, pb, pb + plen, lane);
                if (lane == k) myacc = acc;
                if (a.prof && lane == 0) {
                    pr[2] += 1;
                    pr[push ? 4 : 3] += (unsigned long long)plen;
                }
            }
            if (lane < nb) {
                const int t = mt < 0 ? ~mt : mt;
                if (K == 1 && (mlen >> 30)) a.pcol[cs + t] = a.csc_vals[cs + t] * (scale * ldexp((double)myacc, -E));
                else if (myacc) atomicAdd(reinterpret_cast<unsigned long long *>(a.pcol + cs + t), (unsigned long long)myacc);
            }
        }
        __syncthreads();
        // int64 sums -> fp64: one-unit columns convert their split entries,
        // a split column's last unit converts all of its entries
        if (K == 1) {
            for (int k = tid; k < nq; k += TH) {
                if (qlen[k] <= a.chunk) continue;
                const int qtj = qt[k], t = qtj < 0 ? ~qtj : qtj;
                const long long v = (long long)__ldcg(reinterpret_cast<const unsigned long long *>(a.pcol + cs + t));
                a.pcol[cs + t] = a.csc_vals[cs + t] * (scale * ldexp((double)v, -E));
            }
        } else {
            if (tid == 0) {
                __threadfence();
                const int old = atomicAdd(a.done + (c - a.c0), 1);
                s_last = old == K - 1;
            }
            __syncthreads();
            if (s_last) {
                __threadfence();
                for (long long t = tid; t < cn; t += TH) {
                    const long long v =
                        (long long)__ldcg(reinterpret_cast<const unsigned long long *>(a.pcol + cs + t));
                    a.pcol[cs + t] = a.csc_vals[cs + t] * (scale * ldexp((double)v, -E));
                }
            }
        }
        if (a.prof && tid == 0) {
            const long long t_end = clock64();
            atomicAdd(a.prof + 0, 1ull);
            atomicAdd(a.prof + 1, (unsigned long long)cn);
            atomicAdd(a.prof + 2, (unsigned long long)nq);
            atomicAdd(a.prof + 3, (unsigned long long)m);
            atomicAdd(a.prof + 4, (unsigned long long)nsupp);
            atomicAdd(a.prof + 5, (unsigned long long)(t_built - t_start));
            atomicAdd(a.prof + 6, (unsigned long long)(t_end - t_built));
            atomicAdd(a.prof + 7 + (lg < 8 ? lg : 7), 1ull);
            atomicAdd(a.prof + 2 * UPROF_SLOTS + (lg < 8 ? lg : 7), (unsigned long long)(t_end - t_start));
            atomicAdd(a.prof + 2 * UPROF_SLOTS + 8 + (lg < 8 ? lg : 7), (unsigned long long)(t_built - t_start));
            const int ph = lg == 0 ? 0 : 4;  // build sub-phases: one-unit columns, split columns
            atomicAdd(a.prof + 3 * UPROF_SLOTS + ph + 0, (unsigned long long)(t_zeroed - t_start));
            atomicAdd(a.prof + 3 * UPROF_SLOTS + ph + 1, (unsigned long long)(t_inserted - t_zeroed));
            atomicAdd(a.prof + 3 * UPROF_SLOTS + ph + 2, (unsigned long long)(t_built - t_inserted));
            atomicAdd(a.prof + 3 * UPROF_SLOTS + ph + 3, (unsigned long long)(e1 - e0));
        }
    }
    if (a.prof) {
#pragma unroll
        for (int k = 0; k < 5; ++k) {
            unsigned long long v = pr[k];
            for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(MCF_FULL, v, o);
            if (lane == 0 && v) atomicAdd(a.prof + UPROF_SLOTS + k, v);
        }
    }
}

// d_i = zeta_0 + zeta_1 a_ii + sum over row i of pcol[csr2csc[e]] (4 lanes per row).
// PEER: pcol[(i, c)] is read from the part (rank) owning column c -- mapped
// peer memory -- and d_i is stored to every output buffer (mcf_diag_combine_peer).
template <bool PEER = false>
__global__ void k_diag_final(const long long *__restrict__ row_ptr, const int *__restrict__ col_ids,
                             const double *__restrict__ vals, const long long *__restrict__ csr2csc,
                             const double *__restrict__ pcol, double z0, double z1, double *__restrict__ d,
                             long long rb, long long re, PeerArgs pa) {
    long long i = rb + (((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 2);
    int sub = threadIdx.x & 3;
    bool in = i < re;
    double s = 0.0, aii = 0.0;
    if (in) {
        for (long long e = row_ptr[i] + sub; e < row_ptr[i + 1]; e += 4) {
            const int c = col_ids[e];
            s += PEER ? __ldg(pa.x[peer_owner(pa, c)] + csr2csc[e]) : pcol[csr2csc[e]];
            if (c == i) aii = vals[e];
        }
    }
#pragma unroll
    for (int o = 2; o > 0; o >>= 1) {
        s += __shfl_xor_sync(MCF_FULL, s, o, 4);
        aii += __shfl_xor_sync(MCF_FULL, aii, o, 4);
    }
    if (in && sub == 0) {
        const double out = (z0 + z1 * aii) + s;
        if (PEER) {
            for (int k = 0; k < pa.nouts; ++k) pa.y[k][i] = out;
        } else {
            d[i] = out;
        }
    }
}

// default emission-buffer budget (slots of 12 B): 2^30 -> 12 GiB of the 180 GB
static long long emission_budget() {  // read per call: tests switch it at run time
    const char *e = getenv("MCF_EMISSION_SLOTS");
    long long v = e ? atoll(e) : (1ll << 30);
    return v < (1ll << 16) ? (1ll << 16) : v;
}

// the push/pull break-even of the combine (see run_q)
static int push_pct_for(const mcf_graph *g) {
    const char *e = getenv("MCF_PUSH_PCT");
    long long pct = (200ll * g->n) / (1ll << 22);
    pct = pct < 200 ? 200 : (pct > 1600 ? 1600 : pct);
    return e ? atoi(e) : (int)pct;
}

template <int TH, int CAP, int FW>
static int launch_units(UArgs &a, int grid, cudaStream_t s) {
    const size_t smem = (size_t)CAP * (sizeof(int) + sizeof(long long)) + FW * sizeof(unsigned);
    MCF_CUDA(cudaFuncSetAttribute(k_diag_unit<TH, CAP, FW>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_diag_unit<TH, CAP, FW><<<grid, TH, smem, s>>>(a);
    mcf::note_launch();
    MCF_LAUNCHED("k_diag_unit");
    return MCF_OK;
}

// The combine by units (uniform-value graphs).  *fallback = true (nothing run)
// when a column's table would need more than NGROUPS units.
// SMs the unit kernels leave free (set by diag() around run_q while the next batch's walk runs beside them)
static thread_local int t_reserve_sms = 0;

static int run_units(bool timed, mcf_graph *g, const unsigned long long *colmax, const long long *walk_pre,
                     long long cb, long long ce, long long wb, long long slot_len, const long long *eoff,
                     const long long *walk_off, long long off_base, const int *est, const double *ewt, double *pcol,
                     int *pest, double *pewt, cudaStream_t s, bool *fallback) {
    *fallback = false;
    const long long ncol = ce - cb;
    if (ncol <= 0) return MCF_OK;
    int rc = ensure_group_keys(g, s);
    if (rc) return rc;
    static const int th = [] {
        const char *e = getenv("MCF_UNIT_THREADS");  // 1024 (one CTA per SM, 16384-slot tables) or 512 (two)
        return e && atoi(e) == 512 ? 512 : 1024;
    }();
    const int cap = th == 1024 ? 16384 : 8192;
    UArgs a{};
    a.walk_pre = walk_pre;
    a.wb = wb;
    a.slot_len = slot_len;
    a.eoff = eoff;
    a.walk_off = walk_off;
    a.off_base = off_base;
    a.est = est;
    a.ewt = ewt;
    a.csc_ptr = (const long long *)g->csc_ptr;
    a.csc_rows = g->csc_rows;
    a.csc_vals = g->csc_vals;
    a.ckeys = g->ckeys;
    a.gidx = g->gidx;
    a.gofs = g->gofs;
    a.n = g->n;
    a.c0 = cb;
    a.ncol = ncol;
    a.pcol = pcol;
    a.value = g->value;
    a.colmax = colmax;
    {
        // push (hub-bitmap tests of the table's slots) when the slice is longer
        // than push_pct/100 x the unit's keys: measured best ~600 at n = 2^22
        // (R-MAT) and ~1200 at 1.6e7 (Chung-Lu) -- a test is a random load into
        // an n-bit bitmap
        const char *e = getenv("MCF_UNIT_PUSH_PCT");
        double pct = 600.0 * sqrt((double)g->n / (double)(1ll << 22));
        pct = pct < 600.0 ? 600.0 : (pct > 4800.0 ? 4800.0 : pct);
        a.push_pct = e ? atoi(e) : (int)pct;
    }
    a.hub_of = g->hub_of;
    a.hub_bits = g->hub_bits;
    a.hub_words = g->hub_words;
    {
        const char *e = getenv("MCF_UNIT_SERIAL_SMALL");
        a.serial_small = e ? atoi(e) : 2;  // measured: config 5 4.27 -> 4.17 s, config 3 unchanged
        e = getenv("MCF_UNIT_DEBUG_SKIP");
        a.dbg_skip = e ? atoi(e) : 0;
    }
    {
        const char *e = getenv("MCF_UNIT_CHUNK");
        a.chunk = e ? atoll(e) : 1536;  // three full pull blocks (measured: 768 4-5% slower, 1024 / 2048 within 1%)
        if (a.chunk < 32) a.chunk = 32;
    }
    a.small_need = (3ll * cap - 4) / 4;
    a.ucap = (long long)cap * 5 / 8;
    a.dense_n = cap * 12 / 8;
    if (const char *e = getenv("MCF_UNIT_SMALL_NEED")) {  // tests: split narrow columns too (no dense tables)
        const long long v = atoll(e);
        if (v >= 1 && v < a.small_need) {
            a.small_need = v;
            a.ucap = v * 5 / 6 > 0 ? v * 5 / 6 : 1;
            a.dense_n = 0;
        }
    }
    AsyncFrees frees(s);
    static const bool prof_on = getenv("MCF_DIAG_PROF") != nullptr;
    // SMs left to the next batch's walk (diag(): walk / combine overlap)
    const int sms = sm_count() - t_reserve_sms > 8 ? sm_count() - t_reserve_sms : sm_count();
    const int grid = sms * (th == 1024 ? 1 : 2);
    // small device block: bucket counts, work counter, too-wide need, error bits, profile
    unsigned char *blk = nullptr;
    const size_t blk_bytes = 256 + sizeof(unsigned long long) * 4 * UPROF_SLOTS;
    MCF_CUDA(cudaMallocAsync(&blk, blk_bytes, s));
    frees.keep(blk);
    MCF_CUDA(cudaMemsetAsync(blk, 0, blk_bytes, s));
    unsigned *bcnt = reinterpret_cast<unsigned *>(blk);                               // 32 x u32 (see classify)
    unsigned long long *counter = reinterpret_cast<unsigned long long *>(blk + 128);  // work counter
    unsigned long long *too_wide = counter + 1;                                       // (+ tier counters at 144, 152)
    int *err = reinterpret_cast<int *>(blk + 160);
    a.bcnt = bcnt;
    a.counter = counter;
    a.err = err;
    a.prof = prof_on ? reinterpret_cast<unsigned long long *>(blk + 256) : nullptr;
    int *lists = nullptr;
    MCF_CUDA(cudaMallocAsync(&lists, sizeof(int) * ((size_t)(UNIT_BUCKETS + 2) * ncol + (size_t)ncol), s));
    frees.keep(lists);
    a.lists = lists;
    a.done = lists + (size_t)(UNIT_BUCKETS + 2) * ncol;
    {
        // narrow one-unit columns (Chung-Lu 1.6e7: 15.7M of 15.8M walked columns,
        // 1-3K emissions each) run 4 CTAs per SM with 4096-slot tables (or 2
        // with 8192), so several columns' latency chains overlap per SM
        const char *e = getenv("MCF_UNIT_SMALL_CUT");
        a.small_cut = e ? atoll(e) : 4096 * 2 / 3;
        e = getenv("MCF_UNIT_MID_CUT");
        a.mid_cut = e ? atoll(e) : 8192 * 2 / 3;
    }
    // per-CTA scratch: the entry queue (one slot per entry of the longest
    // column) and the piece map
    a.qcap = g->max_col_degree > 64 ? g->max_col_degree : 64;
    // carve one per-CTA scratch block for a kernel of `gs` CTAs
    auto carve_scratch = [&](UArgs &t, int gs) -> int {
        const size_t per_cta = (size_t)t.qcap * (sizeof(int) + sizeof(long long) + sizeof(int) + sizeof(long long)) + 8 +
                               (size_t)t.pcap * sizeof(int);
        unsigned char *p = nullptr;
        MCF_CUDA(cudaMallocAsync(&p, per_cta * gs + 64, s));
        frees.keep(p);
        t.qlo = reinterpret_cast<long long *>(p);
        p += sizeof(long long) * t.qcap * gs;
        t.qpre = reinterpret_cast<long long *>(p);
        p += sizeof(long long) * (t.qcap + 1) * gs;
        t.qt = reinterpret_cast<int *>(p);
        p += sizeof(int) * t.qcap * gs;
        t.qlen = reinterpret_cast<int *>(p);
        p += sizeof(int) * t.qcap * gs;
        t.pmap = reinterpret_cast<int *>(p);
        return MCF_OK;
    };
    a.pcap = 1ll << 18;
    rc = carve_scratch(a, grid);
    if (rc) return rc;
    {
        const long long warps = (ncol + 31) / 32;
        const long long blocks = (warps * 32 + 255) / 256;
        k_unit_classify<<<(unsigned)(blocks < 65536 ? blocks : 65536), 256, 0, s>>>(a, lists, bcnt, too_wide);
        mcf::note_launch();
        MCF_LAUNCHED("k_unit_classify");
    }
    unsigned long long hw = 0;
    unsigned hbc[32];
    MCF_CUDA(cudaMemcpyAsync(&hw, too_wide, sizeof(hw), cudaMemcpyDeviceToHost, s));
    MCF_CUDA(cudaMemcpyAsync(hbc, bcnt, sizeof(hbc), cudaMemcpyDeviceToHost, s));
    MCF_CUDA(cudaStreamSynchronize(s));
    const unsigned hbc_small = hbc[16], hbc_mid = hbc[24];
    if (hw) {
        *fallback = true;
        return MCF_OK;
    }
    // regroup the split columns' emissions by unit (when the second buffer exists)
    long long npofs = 0, nsplit = 0;
    for (int k = 0; k < UNIT_BUCKETS; ++k) {
        a.pbase[k] = npofs;
        if (k >= 1) {
            npofs += (long long)hbc[k] * ((1ll << k) + 1);
            nsplit += hbc[k];
        }
    }
    a.pest = nullptr;
    a.pewt = nullptr;
    a.pofs = nullptr;
    if (pest && pewt && nsplit > 0) {
        MCF_CUDA(cudaMallocAsync(&a.pofs, sizeof(int) * (size_t)npofs, s));
        frees.keep(a.pofs);
        a.pest = pest;
        a.pewt = pewt;
        k_unit_partition<<<sm_count() * 4, PART_TH, 0, s>>>(a, reinterpret_cast<unsigned *>(blk + 168));
        mcf::note_launch();
        MCF_LAUNCHED("k_unit_partition");
    }
    // the small- and mid-table kernels' arguments: their list as bucket 0,
    // their own counter and per-CTA scratch
    auto tier_args = [&](int tier, int per_sm, UArgs &t) -> int {
        t = a;
        t.lists = lists + (size_t)(UNIT_BUCKETS + tier) * ncol;
        t.bcnt = bcnt + 16 + 8 * tier;  // bucket 0 = this tier's count, 1..7 = 0
        t.counter = reinterpret_cast<unsigned long long *>(blk + 144 + 8 * tier);
        t.pcap = 1ll << 16;
        return carve_scratch(t, sm_count() * per_sm);
    };
    UArgs as{}, am{};
    if (hbc_small > 0 && (rc = tier_args(0, 4, as))) return rc;
    if (hbc_mid > 0 && (rc = tier_args(1, 2, am))) return rc;
    rc = timed_begin(g, timed, g->ev_q, s);
    if (rc) return rc;
    rc = th == 1024 ? launch_units<1024, 16384, 8192>(a, grid, s) : launch_units<512, 8192, 4096>(a, grid, s);
    if (rc) return rc;
    if (hbc_mid > 0 && (rc = launch_units<512, 8192, 4096>(am, sms * 2, s))) return rc;
    if (hbc_small > 0 && (rc = launch_units<256, 4096, 2048>(as, sms * 4, s))) return rc;
    rc = timed_end(timed, g->ev_q, s);
    if (rc) return rc;
    int herr = 0;
    MCF_CUDA(cudaMemcpyAsync(&herr, err, sizeof(int), cudaMemcpyDeviceToHost, s));
    unsigned long long hp[4 * UPROF_SLOTS];
    if (a.prof) MCF_CUDA(cudaMemcpyAsync(hp, a.prof, sizeof(hp), cudaMemcpyDeviceToHost, s));
    unsigned hb[UNIT_BUCKETS];
    if (a.prof) MCF_CUDA(cudaMemcpyAsync(hb, bcnt, sizeof(hb), cudaMemcpyDeviceToHost, s));
    MCF_CUDA(cudaStreamSynchronize(s));
    if (a.prof) {
        fprintf(stderr,
                "[unit-prof] units %llu visits %llu queued %llu emissions %llu support %llu | cyc build %.3e pairs %.3e |"
                " serial %llu ids %llu | pieces %llu pull ids %llu push tests %llu | cols by K:",
                hp[0], hp[1], hp[2], hp[3], hp[4], (double)hp[5], (double)hp[6], hp[UPROF_SLOTS], hp[UPROF_SLOTS + 1],
                hp[UPROF_SLOTS + 2], hp[UPROF_SLOTS + 3], hp[UPROF_SLOTS + 4]);
        for (int k = 0; k < UNIT_BUCKETS; ++k) fprintf(stderr, " %u", hb[k]);
        fprintf(stderr, " | cycles by K:");
        for (int k = 0; k < UNIT_BUCKETS; ++k) fprintf(stderr, " %.3e", (double)hp[2 * UPROF_SLOTS + k]);
        fprintf(stderr, " | build cycles by K:");
        for (int k = 0; k < UNIT_BUCKETS; ++k) fprintf(stderr, " %.3e", (double)hp[2 * UPROF_SLOTS + 8 + k]);
        fprintf(stderr, " | build phases K=1 zero %.3e insert %.3e filter %.3e emissions %.3e"
                        " K>1 zero %.3e insert %.3e filter %.3e emissions %.3e\n",
                (double)hp[3 * UPROF_SLOTS + 0], (double)hp[3 * UPROF_SLOTS + 1], (double)hp[3 * UPROF_SLOTS + 2],
                (double)hp[3 * UPROF_SLOTS + 3], (double)hp[3 * UPROF_SLOTS + 4], (double)hp[3 * UPROF_SLOTS + 5],
                (double)hp[3 * UPROF_SLOTS + 6], (double)hp[3 * UPROF_SLOTS + 7]);
    }
    if (herr) {
        set_error("diag combine: unit table or queue overflow (code " + std::to_string(herr) + ")");
        return MCF_ERR_CUDA;
    }
    return MCF_OK;
}

static int run_q(bool timed, mcf_graph *g, const unsigned long long *colmax, const long long *walk_pre, long long cb,
                 long long ce, long long wb, long long slot_len, const long long *eoff, const long long *walk_off,
                 long long off_base, const int *est, const double *ewt, double *pcol,
                 long long max_slots_per_col, cudaStream_t s, int *pest = nullptr, double *pewt = nullptr) {
    {
        // uniform-value graphs above the dense-Q size: the unit combine unless
        // MCF_DIAG_UNITS=0 (=1 forces it on small graphs too).  Below it every
        // column's Q_c is one CTA's dense array and k_diag_q is faster (config 1:
        // 4.4 vs 6.2 ms per estimate, measured)
        const char *e = getenv("MCF_DIAG_UNITS");
        const bool on = e ? strcmp(e, "0") != 0 : g->n > DENSE_N;
        if (g->uniform_value && on && (g->n > DENSE_N || (e && !strcmp(e, "1")))) {
            bool fallback = false;
            const int rc = run_units(timed, g, colmax, walk_pre, cb, ce, wb, slot_len, eoff, walk_off, off_base, est,
                                     ewt, pcol, pest, pewt, s, &fallback);
            if (rc || !fallback) return rc;
        }
    }
    // (the single-table / cluster path below uses the side stream itself: inside an overlapped batch loop,
    // diag(), it first lets the walk running there finish)
    if (t_reserve_sms > 0 && g->side) MCF_CUDA(cudaStreamSynchronize(g->side));
    QArgs q;
    q.walk_pre = walk_pre;
    q.wb = wb;
    q.slot_len = slot_len;
    q.eoff = eoff;
    q.walk_off = walk_off;
    q.off_base = off_base;
    q.est = est;
    q.ewt = ewt;
    q.csc_ptr = (const long long *)g->csc_ptr;
    q.csc_rows = g->csc_rows;
    q.csc_vals = g->csc_vals;
    q.n = g->n;
    q.col_begin = cb;
    q.col_end = ce;
    q.pcol = pcol;
    q.hub_of = g->hub_of;
    q.hub_bits = g->hub_bits;
    q.hub_words = g->hub_words;
    q.uniform = g->uniform_value ? 1 : 0;
    {
        // push while a bitmap test is cheaper than scanning C_i: the bitmaps are
        // n bits, so the push/pull break-even moves up with n (measured with the
        // two-bit filter and shared long scans: R-MAT 2^22 best at 2x |supp Q_c|,
        // Chung-Lu 1.6e7 at 8-16x)
        const char *e = getenv("MCF_PUSH_PCT");
        long long pct = (200ll * g->n) / (1ll << 22);
        pct = pct < 200 ? 200 : (pct > 1600 ? 1600 : pct);
        q.push_pct = e ? atoi(e) : (int)pct;
    }
    q.value = g->value;
    q.colmax = colmax;
    q.prof = nullptr;
    {
        const char *e = getenv("MCF_DIAG_BIG_WORK");
        q.big_work = e ? atoll(e) : BIG_WORK;
        e = getenv("MCF_DIAG_LONG_WORK");
        q.long_work = e ? atoll(e) : LONG_WORK;
        e = getenv("MCF_DIAG_LONG_WORK_Q");
        q.long_work_q = e ? atoll(e) : LONG_WORK_Q;
        e = getenv("MCF_DIAG_OPT");
        q.opt = e ? atoi(e) : DIAG_OPT_DEFAULT;
        e = getenv("MCF_DIAG_CHUNK_Q");
        q.chunk_q = e ? atoll(e) : CHUNK;
        e = getenv("MCF_DIAG_CHUNK");
        q.chunk_c = e ? atoll(e) : CHUNK;
        if (q.chunk_q < 32) q.chunk_q = 32;
        if (q.chunk_c < 32) q.chunk_c = 32;
    }
    AsyncFrees frees(s);  // every stream-ordered allocation below, on every return path
    static const bool prof_on = getenv("MCF_DIAG_PROF") != nullptr;
    if (prof_on) {
        MCF_CUDA(cudaMallocAsync(&q.prof, sizeof(unsigned long long) * PROF_SLOTS, s));
        frees.keep(q.prof);
        MCF_CUDA(cudaMemsetAsync(q.prof, 0, sizeof(unsigned long long) * PROF_SLOTS, s));
    }
    q.gkeys = nullptr;
    q.gvals = nullptr;
    q.gcap = 0;
    int grid = sm_count();
    long long need = max_slots_per_col < g->n ? max_slots_per_col : g->n;
    long long cap = 32;
    while (cap * 3 < need * 4 + 4) cap <<= 1;
    unsigned char *gbuf = nullptr;
    if (cap > SCAP) {
        q.gcap = cap;
        MCF_CUDA(cudaMallocAsync(&gbuf, (size_t)grid * cap * (sizeof(int) + sizeof(double)), s));
        frees.keep(gbuf);
        q.gvals = reinterpret_cast<long long *>(gbuf);
        q.gkeys = reinterpret_cast<int *>(q.gvals + (size_t)grid * cap);
    }
    // per-CTA support lists (push path): up to half the largest table
    q.lcap = cap > 2 * SCAP ? cap / 2 : SCAP;  // >= SCAP: a cluster's list spans its CTAs' regions
    unsigned char *lbuf = nullptr;
    // scratch regions: k_diag_q's grid, then as many for the cluster kernels
    // running beside it (uniform-value graphs above the dense size)
    q.cl_base = grid;
    const long long nreg = (q.uniform && g->n > DENSE_N) ? 2ll * grid : grid;
    MCF_CUDA(cudaMallocAsync(&lbuf, (size_t)nreg * q.lcap * (sizeof(int) + sizeof(long long)), s));
    frees.keep(lbuf);
    q.lvals = reinterpret_cast<long long *>(lbuf);
    q.lkeys = reinterpret_cast<int *>(q.lvals + (size_t)nreg * q.lcap);
    // lists of long (i, c) entries: one per CTA, max_degree entries (a column's
    // length on symmetric graphs; longer columns scan the overflow inline)
    q.llcap = g->info.max_degree > 64 ? g->info.max_degree : 64;
    if (q.llcap > (1ll << 24)) q.llcap = 1ll << 24;
    q.ocap = 2 * q.llcap + 2 * (q.big_work / q.chunk_q) + 1024;
    {
        unsigned char *lb = nullptr;
        MCF_CUDA(cudaMallocAsync(&lb, (size_t)nreg * (q.llcap * (8 + 4 + 4) + q.ocap * 4), s));
        frees.keep(lb);
        q.lacc = reinterpret_cast<unsigned long long *>(lb);
        q.llist = reinterpret_cast<int *>(q.lacc + (size_t)nreg * q.llcap);
        q.lbase = q.llist + (size_t)nreg * q.llcap;
        q.lown = q.lbase + (size_t)nreg * q.llcap;
        // the cluster kernels' piece maps (regions after k_diag_q's) start unwritten (-1)
        if (nreg > grid)
            MCF_CUDA(cudaMemsetAsync(q.lown + (size_t)grid * q.ocap, 0xff, sizeof(int) * (size_t)(nreg - grid) * q.ocap, s));
    }
    unsigned long long *counter = nullptr;
    MCF_CUDA(cudaMallocAsync(&counter, sizeof(unsigned long long) * 4, s));
    frees.keep(counter);
    MCF_CUDA(cudaMemsetAsync(counter, 0, sizeof(unsigned long long) * 4, s));
    q.counter = counter;
    q.n_big = reinterpret_cast<unsigned *>(counter + 1);
    q.pool_used = counter + 2;
    // pool for the tables of big columns (shared GPU-wide by k_diag_big)
    const unsigned max_big = 32768;
    const unsigned long long pool_cap = 1ull << 27;  // 1.5 GiB of (key, value) slots
    unsigned char *pool = nullptr;
    const char *pool_env = getenv("MCF_DIAG_POOL");  // "0": no pool (the allocation-failure path; tests)
    if (!(pool_env && !strcmp(pool_env, "0")) && cudaMallocAsync(&pool, pool_cap * (sizeof(int) + sizeof(long long)) + (size_t)max_big * FILTER_WORDS * 4 +
                                       sizeof(BigRec) * max_big + 2 * sizeof(int) * max_big,
                        s) == cudaSuccess) {
        frees.keep(pool);
        q.pool_vals = reinterpret_cast<long long *>(pool);
        q.pool_keys = reinterpret_cast<int *>(q.pool_vals + pool_cap);
        q.pool_filt = reinterpret_cast<unsigned *>(q.pool_keys + pool_cap);
        q.big = reinterpret_cast<BigRec *>(q.pool_filt + (size_t)max_big * FILTER_WORDS);
        q.pool_E = reinterpret_cast<int *>(q.big + max_big);
        q.pool_nsupp = q.pool_E + max_big;
        q.max_big = max_big;
        q.pool_cap = pool_cap;
    } else {
        cudaGetLastError();
        q.big = nullptr;
        q.max_big = 0;
        q.pool_cap = 0;
    }
    size_t smem = (size_t)SCAP * (sizeof(int) + sizeof(long long)) + FILTER_WORDS * sizeof(unsigned);
    MCF_CUDA(cudaFuncSetAttribute(k_diag_q, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    // clusters of 2/4/8 CTAs for tables wider than one CTA's shared memory
    // (uniform-value graphs above the dense size; MCF_DIAG_CLUSTER=0 disables)
    // Measured: R-MAT 2^22 diag 10.1 -> 7.7 s with clusters up to 8; Chung-Lu
    // 1.6e7 10.7 -> 11.5 s (its wide columns are hub columns of 10^4-10^5
    // short entries, each probing remote shared memory).  Default: clusters
    // below n = 2^23, global tables above; MCF_DIAG_CLUSTER=K overrides.
    const char *cl_e = getenv("MCF_DIAG_CLUSTER");
    const int cl_env = cl_e ? atoi(cl_e) : (g->n < (1ll << 23) ? 8 : 0);
    int cl_grid[3] = {0, 0, 0};
    q.cl_maxk = 0;
    if (q.uniform && g->n > DENSE_N && cl_env >= 2) {
        for (int k = 0; k < 3 && (2 << k) <= cl_env; ++k) {
            int nc = 0;
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(2 << k);
            cfg.blockDim = dim3(Q_THREADS);
            cfg.dynamicSmemBytes = smem;
            cudaError_t e;
            if (k == 0) {
                cudaFuncSetAttribute(k_diag_qc<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
                e = cudaOccupancyMaxActiveClusters(&nc, (void *)k_diag_qc<2>, &cfg);
            } else if (k == 1) {
                cudaFuncSetAttribute(k_diag_qc<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
                e = cudaOccupancyMaxActiveClusters(&nc, (void *)k_diag_qc<4>, &cfg);
            } else {
                cudaFuncSetAttribute(k_diag_qc<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
                e = cudaOccupancyMaxActiveClusters(&nc, (void *)k_diag_qc<8>, &cfg);
            }
            if (e != cudaSuccess || nc < 1) {
                cudaGetLastError();
                break;
            }
            cl_grid[k] = nc * (2 << k);
            q.cl_maxk = 2 << k;
        }
    }
    q.cbits = nullptr;
    q.cwords = (g->n + 31) / 32;
    if (q.cl_maxk && (q.opt & OPT_EXACT)) {  // one n-bit bitmap per concurrently resident cluster
        long long ncl = 0;
        for (int k = 0; k < 3; ++k) ncl = ncl > cl_grid[k] / (2 << k) ? ncl : cl_grid[k] / (2 << k);
        if (ncl > 0) {
            MCF_CUDA(cudaMallocAsync(&q.cbits, sizeof(unsigned) * q.cwords * ncl, s));
            frees.keep(q.cbits);
            MCF_CUDA(cudaMemsetAsync(q.cbits, 0, sizeof(unsigned) * q.cwords * ncl, s));
        }
    }
    int *cl_cols = nullptr;
    unsigned *cl_cnt = nullptr;
    const long long ncol = ce - cb;
    if (q.cl_maxk) {
        MCF_CUDA(cudaMallocAsync(&cl_cols, sizeof(int) * 3 * (size_t)ncol + 32, s));
        frees.keep(cl_cols);
        cl_cnt = reinterpret_cast<unsigned *>(cl_cols + 3 * ncol);
        MCF_CUDA(cudaMemsetAsync(cl_cnt, 0, 32, s));
        k_cluster_classify<<<sm_count() * 4, 256, 0, s>>>(q, cl_cols, ncol, cl_cnt);
        mcf::note_launch();
        MCF_LAUNCHED("k_cluster_classify");
    }
    int rc = timed_begin(g, timed, g->ev_q, s);
    if (rc) return rc;
    // MCF_DIAG_PROF: a timeline of the combine's kernels (ms from the start)
    std::vector<std::pair<const char *, cudaEvent_t>> tl;
    auto mark = [&](const char *what, cudaStream_t st) {
        if (!q.prof) return;
        cudaEvent_t e;
        cudaEventCreate(&e);
        cudaEventRecord(e, st);
        tl.emplace_back(what, e);
    };
    mark("start", s);
    if (q.cl_maxk) {
        // The cluster kernels go first and k_diag_q runs beside them on the side
        // stream: clusters of 4/8 CTAs only fit 128-132 of the 148 SMs, and
        // k_diag_q's persistent CTAs take the rest (and every SM a finished
        // cluster kernel frees).  Integer partials: the split does not matter.
        unsigned hc[8];
        MCF_CUDA(cudaMemcpyAsync(hc, cl_cnt, sizeof(hc), cudaMemcpyDeviceToHost, s));
        MCF_CUDA(cudaStreamSynchronize(s));
        rc = ensure_side_stream(g);
        if (rc) return rc;
        MCF_CUDA(cudaEventRecord(g->ev_fork, s));  // before the cluster kernels: k_diag_q does not wait for them
        MCF_CUDA(cudaStreamWaitEvent(g->side, g->ev_fork, 0));
        for (int k = 0; k < 3; ++k) {
            if (!hc[k]) continue;
            const int *lst = cl_cols + k * ncol;
            unsigned *nxt = cl_cnt + 4 + k;
            if (k == 0) k_diag_qc<2><<<cl_grid[0], Q_THREADS, smem, s>>>(q, lst, hc[k], nxt);
            else if (k == 1) k_diag_qc<4><<<cl_grid[1], Q_THREADS, smem, s>>>(q, lst, hc[k], nxt);
            else k_diag_qc<8><<<cl_grid[2], Q_THREADS, smem, s>>>(q, lst, hc[k], nxt);
            mcf::note_launch();
            MCF_LAUNCHED("k_diag_qc");
            mark(k == 0 ? "qc2 end" : (k == 1 ? "qc4 end" : "qc8 end"), s);
        }
        k_diag_q<<<grid, Q_THREADS, smem, g->side>>>(q);
        mcf::note_launch();
        MCF_LAUNCHED("k_diag_q");
        mark("k_diag_q end (side)", g->side);
        MCF_CUDA(cudaEventRecord(g->ev_join, g->side));
        MCF_CUDA(cudaStreamWaitEvent(s, g->ev_join, 0));
    } else {
        k_diag_q<<<grid, Q_THREADS, smem, s>>>(q);
        mcf::note_launch();
        MCF_LAUNCHED("k_diag_q");
    }
    if (q.big) {
        unsigned nrec = 0;
        MCF_CUDA(cudaMemcpyAsync(&nrec, q.n_big, sizeof(unsigned), cudaMemcpyDeviceToHost, s));
        MCF_CUDA(cudaStreamSynchronize(s));
        if (nrec > max_big) nrec = max_big;
        if (nrec > 0) {
            long long *cnt = nullptr;
            MCF_CUDA(cudaMallocAsync(&cnt, sizeof(long long) * (2 * (size_t)nrec + 1), s));
            frees.keep(cnt);
            k_big_counts<<<(nrec + 255) / 256, 256, 0, s>>>(q.big, nrec, cnt);
            mcf::note_launch();
            rc = exclusive_scan_i64(cnt, cnt + nrec, nrec, s);
            if (rc) return rc;
            mark("big start", s);
            k_diag_big<<<sm_count() * 8, 256, 0, s>>>(q, cnt + nrec, nrec);
            mcf::note_launch();
            MCF_LAUNCHED("k_diag_big");
            mark("big end", s);
        }
    }
    rc = timed_end(timed, g->ev_q, s);
    if (rc) return rc;
    if (q.prof) {
        unsigned long long h[PROF_SLOTS];
        MCF_CUDA(cudaMemcpyAsync(h, q.prof, sizeof(h), cudaMemcpyDeviceToHost, s));
        MCF_CUDA(cudaStreamSynchronize(s));
        fprintf(stderr,
                "[diag-prof] cols %llu big %llu emissions %llu support %llu | pull pairs %llu ids %llu filt %llu hits %llu"
                " | push pairs %llu tests %llu hits %llu | cyc build %.3e combine %.3e | gtable cols %llu cycles %llu emissions %llu | cluster cols %llu cycles %llu emissions %llu build %llu\n",
                h[8], h[9], h[6], h[7], h[0], h[1], h[2], h[12], h[3], h[4], h[5], (double)h[10], (double)h[11], h[13], h[14], h[15], h[16], h[17], h[18], h[19]);
        fprintf(stderr, "[diag-phases] zero+fetch %.3e build %.3e filter %.3e big+exact %.3e pairs %.3e final %.3e\n",
                (double)h[PROF_PH + 0], (double)h[PROF_PH + 1], (double)h[PROF_PH + 2], (double)h[PROF_PH + 3],
                (double)h[PROF_PH + 4], (double)h[PROF_PH + 5]);
        std::string line = "[diag-timeline]";
        for (auto &x : tl) {
            float ms = 0.f;
            cudaEventElapsedTime(&ms, tl[0].second, x.second);
            line += std::string(" ") + x.first + "=" + std::to_string(ms);
        }
        for (auto &x : tl) cudaEventDestroy(x.second);
        fprintf(stderr, "%s\n", line.c_str());
        for (int k = 0; k < PROF_NCLS; ++k) {
            const unsigned long long *c = h + PROF_BASE + PROF_CLS * k;
            fprintf(stderr, "[diag-prof-cls] %d pull pairs %llu ids %llu filt %llu hits %llu | push pairs %llu tests %llu hits %llu\n",
                    k, c[0], c[1], c[2], c[3], c[4], c[5], c[6]);
        }
    }
    return MCF_OK;
}

// second emission buffer for the unit combine's regrouped split columns
// (uniform-value graphs, MCF_DIAG_UNITS / MCF_UNIT_PARTITION not "0");
// an allocation failure leaves both null (units then filter by group)
static void alloc_regroup(const mcf_graph *g, long long slots, int **pest, double **pewt, cudaStream_t s) {
    *pest = nullptr;
    *pewt = nullptr;
    const char *e = getenv("MCF_DIAG_UNITS"), *e2 = getenv("MCF_UNIT_PARTITION");
    const bool units = e ? !strcmp(e, "1") || (strcmp(e, "0") && g->n > DENSE_N) : g->n > DENSE_N;
    if (!g->uniform_value || !units || (e2 && !strcmp(e2, "0")) || slots <= 0) return;
    if (cudaMallocAsync(pest, sizeof(int) * slots, s) != cudaSuccess) {
        cudaGetLastError();
        *pest = nullptr;
        return;
    }
    if (cudaMallocAsync(pewt, sizeof(double) * slots, s) != cudaSuccess) {
        cudaGetLastError();
        cudaFreeAsync(*pest, s);
        *pest = nullptr;
        *pewt = nullptr;
    }
}

// SMs reserved for the next batch's walk while a batch is combined.  MCF_DIAG_OVERLAP: 0 = serial batches,
// N > 0 = N SMs; unset = start at 20 and adapt (*adaptive) from the measured durations of each walk / combine
// pair (diag()).  Only where the unit combine runs (uniform-value graphs above the dense-Q size).  Timing
// only: results do not depend on it.
static int overlap_sms(const mcf_graph *g, bool *adaptive) {
    const char *e = getenv("MCF_DIAG_OVERLAP");
    const int v = e ? atoi(e) : 20;
    *adaptive = e == nullptr;
    const char *u = getenv("MCF_DIAG_UNITS");
    if (!g->uniform_value || g->n <= DENSE_N || v <= 0 || (u && !strcmp(u, "0"))) return 0;
    return v < sm_count() - 8 ? v : sm_count() - 8;
}

static int diag(mcf_graph *g, const mcf_walk_params *p, const long long *walk_pre, long long cb, long long ce,
                const long long *walk_off, const int *entries, double *pcol, long long *stats, cudaStream_t s,
                bool replay) {
    int rc = check_params(g, p, walk_pre, cb, ce);
    if (rc) return rc;
    MCF_ARG(pcol && stats, "diag walk: null pcol/stats");
    if (replay) MCF_ARG(walk_off && entries, "replay: null stream");
    MCF_ARG(!(replay && (p->flags & MCF_FLAG_WALK_GROUP)), "walk groups apply to device-RNG walks, not replay");
    rc = ensure_hub_bitmaps(g, s);
    if (rc) return rc;
    // walks of at most 64 steps get fixed slots; longer caps (cutoff-
    // terminated walks, e.g. max_steps = 10^4) use a count pass instead
    const bool fixed = p->max_steps <= 64;
    const long long L = fixed ? p->max_steps : 64;
    // column batches of at most cap_walks walks (+ one column): the emission
    // buffer budget (MCF_EMISSION_SLOTS); replay takes the range in one batch
    std::vector<long long> hb;
    unsigned long long hmax = 0;
    long long cap_walks = replay ? (1ll << 62) : emission_budget() / L;
    rc = column_batches(walk_pre, cb, ce, cap_walks, hb, &hmax, s);
    if (rc) return rc;
    long long wb = 0, we = 0;
    rc = read_walk_range(walk_pre, cb, ce, &wb, &we, s);
    if (rc) return rc;
    if (we == wb) return MCF_OK;
    MCF_ARG(hmax < (1ull << 31), "a column's walk budget must be below 2^31");
    AsyncFrees frees(s);
    int *err = nullptr;
    MCF_CUDA(cudaMallocAsync(&err, 16, s));
    frees.keep(err);
    MCF_CUDA(cudaMemsetAsync(err, 0, 16, s));
    unsigned long long *colmax = nullptr;  // per-column max |emission| for the fixed-point scale
    MCF_CUDA(cudaMallocAsync(&colmax, sizeof(unsigned long long) * g->n, s));
    frees.keep(colmax);
    MCF_CUDA(cudaMemsetAsync(colmax, 0, sizeof(unsigned long long) * g->n, s));
    const bool timed = (p->flags & MCF_FLAG_TIME_KERNELS) != 0;

    if (replay) {
        MCF_ARG(we - wb < WALKS_PER_LAUNCH, "replay: walks per call must be below 2^31 (split the column range)");
        long long hoff[2];
        MCF_CUDA(cudaMemcpyAsync(&hoff[0], walk_off + wb, 8, cudaMemcpyDeviceToHost, s));
        MCF_CUDA(cudaMemcpyAsync(&hoff[1], walk_off + we, 8, cudaMemcpyDeviceToHost, s));
        MCF_CUDA(cudaStreamSynchronize(s));
        const long long slots = hoff[1] - hoff[0] + (we - wb);
        int *est = nullptr;
        double *ewt = nullptr;
        MCF_CUDA(cudaMallocAsync(&est, sizeof(int) * slots, s));
        frees.keep(est);
        MCF_CUDA(cudaMallocAsync(&ewt, sizeof(double) * slots, s));
        frees.keep(ewt);
        rc = launch_walk_emit(g, p, walk_pre, cb, ce, we - wb, EMIT_REPLAY, walk_off, entries, 0, hoff[0], nullptr, est,
                              ewt, colmax, stats, err, s);
        if (rc) return rc;
        int *pest = nullptr;
        double *pewt = nullptr;
        alloc_regroup(g, slots, &pest, &pewt, s);
        frees.keep(pest);
        frees.keep(pewt);
        // table size is bounded by min(slots, n) per column
        rc = run_q(timed, g, colmax, walk_pre, cb, ce, wb, 0, nullptr, walk_off, hoff[0], est, ewt, pcol, slots, s, pest,
                   pewt);
        if (rc) return rc;
        int herr = 0;
        MCF_CUDA(cudaMemcpyAsync(&herr, err, sizeof(int), cudaMemcpyDeviceToHost, s));
        MCF_CUDA(cudaStreamSynchronize(s));
        if (herr) {
            set_error("replay stream inconsistent with the walk (code " + std::to_string(herr) + ")");
            return MCF_ERR_ARGUMENT;
        }
        return MCF_OK;
    }

    long long buf_slots = (cap_walks + (long long)hmax) * L;
    if (buf_slots > (we - wb) * L) buf_slots = (we - wb) * L;
    int *est = nullptr;
    double *ewt = nullptr;
    MCF_CUDA(cudaMallocAsync(&est, sizeof(int) * buf_slots, s));
    {
        const cudaError_t e_ = cudaMallocAsync(&ewt, sizeof(double) * buf_slots, s);
        if (e_ != cudaSuccess) {
            cudaFreeAsync(est, s);
            return cuda_status(e_, "cudaMallocAsync(ewt)");
        }
    }
    int *pest = nullptr;
    double *pewt = nullptr;
    alloc_regroup(g, buf_slots, &pest, &pewt, s);
    long long pslots = pest ? buf_slots : 0;
    // Walk / combine overlap (fixed-slot walks, two or more batches): the walk is bound by DRAM random-access
    // latency and the unit combine by instruction issue, so batch b + 1's walk runs on a few reserved SMs (side
    // stream, second emission buffer) while batch b is combined on the others.  Same kernels, same data:
    // results are bitwise those of the serial loop below.
    bool ov_adapt = false;
    int ov = overlap_sms(g, &ov_adapt);
    if (fixed && ov > 0 && hb.size() > 2 && ensure_side_stream(g) == MCF_OK) {
        int *est2 = nullptr;
        double *ewt2 = nullptr;
        if (cudaMallocAsync(&est2, sizeof(int) * buf_slots, s) == cudaSuccess &&
            cudaMallocAsync(&ewt2, sizeof(double) * buf_slots, s) == cudaSuccess) {
            const size_t nb = hb.size() - 1;
            std::vector<long long> r0(nb), r1(nb);
            for (size_t b = 0; b < nb && !rc; ++b) rc = read_walk_range(walk_pre, hb[b], hb[b + 1], &r0[b], &r1[b], s);
            int *ebuf[2] = {est, est2};
            double *wbuf[2] = {ewt, ewt2};
            // (timing events: the adaptive SM split below reads the walk's and the combine's durations)
            cudaEvent_t ev_w[2] = {nullptr, nullptr}, ev_q[2] = {nullptr, nullptr}, ev_init = nullptr;
            cudaEvent_t ev_ws = nullptr, ev_cs = nullptr;  // start of the side walk / of the combine beside it
            for (int k = 0; k < 2 && !rc; ++k) {
                if (cudaEventCreate(&ev_w[k]) != cudaSuccess || cudaEventCreate(&ev_q[k]) != cudaSuccess)
                    rc = cuda_status(cudaGetLastError(), "cudaEventCreate");
            }
            if (!rc && (cudaEventCreateWithFlags(&ev_init, cudaEventDisableTiming) != cudaSuccess ||
                        cudaEventCreate(&ev_ws) != cudaSuccess || cudaEventCreate(&ev_cs) != cudaSuccess))
                rc = cuda_status(cudaGetLastError(), "cudaEventCreate");
            cudaStream_t side = g->side;
            if (!rc) {  // the side stream starts after this call's setup (err, colmax, buffers) on s
                cudaEventRecord(ev_init, s);
                cudaStreamWaitEvent(side, ev_init, 0);
            }
            // first non-empty batch: its walk has the GPU to itself
            size_t b = 0;
            while (b < nb && r1[b] == r0[b]) ++b;
            if (!rc && b < nb)
                rc = launch_walk_emit(g, p, walk_pre, hb[b], hb[b + 1], r1[b] - r0[b], EMIT_FIXED, nullptr, nullptr, L, 0,
                                      nullptr, ebuf[0], wbuf[0], colmax, stats, err, s);
            int cur = 0;
            while (!rc && b < nb) {
                size_t nx = b + 1;
                while (nx < nb && r1[nx] == r0[nx]) ++nx;
                if (nx < nb) {  // next batch's walk into the other buffer, once its previous combine is done
                    if (ev_q[cur ^ 1]) cudaStreamWaitEvent(side, ev_q[cur ^ 1], 0);
                    cudaEventRecord(ev_ws, side);
                    rc = launch_walk_emit(g, p, walk_pre, hb[nx], hb[nx + 1], r1[nx] - r0[nx], EMIT_FIXED, nullptr,
                                          nullptr, L, 0, nullptr, ebuf[cur ^ 1], wbuf[cur ^ 1], colmax, stats, err, side,
                                          ov);
                    if (rc) break;
                    cudaEventRecord(ev_w[cur ^ 1], side);
                }
                t_reserve_sms = nx < nb ? ov : 0;
                cudaEventRecord(ev_cs, s);
                rc = run_q(timed, g, colmax, walk_pre, hb[b], hb[b + 1], r0[b], L, nullptr, nullptr, 0, ebuf[cur],
                           wbuf[cur], pcol, (long long)hmax * L, s, pest, pewt);
                t_reserve_sms = 0;
                if (rc) break;
                cudaEventRecord(ev_q[cur], s);
                if (nx < nb) {
                    if (ov_adapt) {
                        // Balance the two sides for the next pair from this pair's durations: the walk's time
                        // scales with 1 / W, the combine's with 1 / (SMs - W), so they would have ended together at
                        // W* = SMs tw W / (tw W + tc (SMs - W)); move halfway there.  (Waiting for the walk here
                        // costs nothing: the next walk and the next combine both wait for it anyway.)
                        static const double bias = [] { const char *e = getenv("MCF_OVERLAP_BIAS"); return e ? atof(e) : 1.3; }();
                        float tw = 0.f, tc = 0.f;
                        if (cudaEventSynchronize(ev_q[cur]) == cudaSuccess && cudaEventSynchronize(ev_w[cur ^ 1]) == cudaSuccess &&
                            cudaEventElapsedTime(&tw, ev_ws, ev_w[cur ^ 1]) == cudaSuccess &&
                            cudaEventElapsedTime(&tc, ev_cs, ev_q[cur]) == cudaSuccess && tw > 0.f && tc > 0.f) {
                            const double S = sm_count(), W = ov, twb = bias * tw;  // (bias: a late walk stalls every SM)
                            const double wstar = S * twb * W / (twb * W + tc * (S - W));
                            int nv = (int)(0.5 * (W + wstar) + 0.5);
                            nv = nv < 4 ? 4 : (nv > sm_count() / 2 ? sm_count() / 2 : nv);
                            if (getenv("MCF_DIAG_PROF"))
                                fprintf(stderr, "[overlap] batch %zu: walk %.1f ms on %d SMs, combine %.1f ms -> %d SMs\n", b,
                                        tw, ov, tc, nv);
                            ov = nv;
                        }
                        cudaGetLastError();
                    }
                    cudaStreamWaitEvent(s, ev_w[cur ^ 1], 0);
                }
                b = nx;
                cur ^= 1;
            }
            cudaStreamSynchronize(side);  // (error paths: nothing of this call is left running on the side stream)
            for (int k = 0; k < 2; ++k) {
                if (ev_w[k]) cudaEventDestroy(ev_w[k]);
                if (ev_q[k]) cudaEventDestroy(ev_q[k]);
            }
            if (ev_init) cudaEventDestroy(ev_init);
            if (ev_ws) cudaEventDestroy(ev_ws);
            if (ev_cs) cudaEventDestroy(ev_cs);
            cudaFreeAsync(est2, s);
            cudaFreeAsync(ewt2, s);
            if (est) cudaFreeAsync(est, s);
            if (ewt) cudaFreeAsync(ewt, s);
            if (pest) cudaFreeAsync(pest, s);
            if (pewt) cudaFreeAsync(pewt, s);
            return rc;
        }
        cudaGetLastError();  // no room for a second emission buffer: the serial loop
        if (est2) cudaFreeAsync(est2, s);
    }
    for (size_t b = 0; b + 1 < hb.size(); ++b) {
        const long long c0 = hb[b], c1 = hb[b + 1];
        long long bw0 = 0, bw1 = 0;
        rc = read_walk_range(walk_pre, c0, c1, &bw0, &bw1, s);
        if (rc) break;
        if (bw1 == bw0) continue;
        if (fixed) {
            rc = launch_walk_emit(g, p, walk_pre, c0, c1, bw1 - bw0, EMIT_FIXED, nullptr, nullptr, L, 0, nullptr, est,
                                  ewt, colmax, stats, err, s);
            if (rc) break;
            rc = run_q(timed, g, colmax, walk_pre, c0, c1, bw0, L, nullptr, nullptr, 0, est, ewt, pcol,
                       (long long)hmax * L, s, pest, pewt);
            if (rc) break;
            continue;
        }
        // variable-length walks: count pass, scan, emit at exact offsets
        const long long nwb = bw1 - bw0;
        long long *elen = nullptr;
        cudaError_t ce_ = cudaMallocAsync(&elen, sizeof(long long) * (2 * nwb + 1), s);
        if (ce_ != cudaSuccess) {
            rc = cuda_status(ce_, "cudaMallocAsync(elen)");
            break;
        }
        AsyncFrees batch_frees(s);
        batch_frees.keep(elen);
        long long *eoff = elen + nwb;
        rc = launch_walk_emit(g, p, walk_pre, c0, c1, nwb, EMIT_COUNT, nullptr, nullptr, 0, 0, elen, nullptr, nullptr,
                              nullptr, stats, err, s);
        if (rc) break;
        rc = exclusive_scan_i64(elen, eoff, nwb, s);
        if (rc) break;
        long long total = 0;
        ce_ = cudaMemcpyAsync(&total, eoff + nwb, sizeof(long long), cudaMemcpyDeviceToHost, s);
        if (ce_ == cudaSuccess) ce_ = cudaStreamSynchronize(s);
        if (ce_ != cudaSuccess) {
            rc = cuda_status(ce_, "emission count");
            break;
        }
        if (total > buf_slots) {
            cudaFreeAsync(est, s);
            cudaFreeAsync(ewt, s);
            est = nullptr;
            ewt = nullptr;
            buf_slots = total;
            ce_ = cudaMallocAsync(&est, sizeof(int) * buf_slots, s);
            if (ce_ == cudaSuccess) ce_ = cudaMallocAsync(&ewt, sizeof(double) * buf_slots, s);
            if (ce_ != cudaSuccess) {
                rc = cuda_status(ce_, "cudaMallocAsync(emissions)");
                break;
            }
        }
        rc = launch_walk_emit(g, p, walk_pre, c0, c1, nwb, EMIT_EXPLICIT, nullptr, nullptr, 0, 0, eoff, est, ewt,
                              colmax, stats, err, s);
        if (rc) break;
        if (pest && total > pslots) {  // the regroup buffer follows the emission buffer's size
            cudaFreeAsync(pest, s);
            cudaFreeAsync(pewt, s);
            alloc_regroup(g, total, &pest, &pewt, s);
            pslots = pest ? total : 0;
        }
        rc = run_q(timed, g, colmax, walk_pre, c0, c1, bw0, 0, eoff, nullptr, 0, est, ewt, pcol, total, s,
                   pest && total <= pslots ? pest : nullptr, pest && total <= pslots ? pewt : nullptr);
        if (rc) break;
    }
    if (est) cudaFreeAsync(est, s);
    if (ewt) cudaFreeAsync(ewt, s);
    if (pest) cudaFreeAsync(pest, s);
    if (pewt) cudaFreeAsync(pewt, s);
    return rc;
}

// Dense rows of Q for the full estimator (rand_funm): one
// CTA per column c, Q_c accumulated in a shared dense int64 row in fixed point
// (scale from the walk kernel's per-column max: deterministic), then written
// as fp64 to Q[(c - cb) * ldq + j].
constexpr int QDENSE_MAX_N = 16384;  // 128 KB shared row

__global__ void __launch_bounds__(512) k_qdense(const long long *__restrict__ walk_pre, long long cb, long long ce,
                                                long long wb, const long long *__restrict__ eoff,
                                                const int *__restrict__ est, const double *__restrict__ ewt,
                                                const unsigned long long *__restrict__ colmax, long long n,
                                                double *__restrict__ Q, long long ldq, int trans) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    long long *row = reinterpret_cast<long long *>(smem_raw);
    for (long long c = cb + blockIdx.x; c < ce; c += gridDim.x) {
        for (long long j = threadIdx.x; j < n; j += blockDim.x) row[j] = 0;
        __syncthreads();
        const long long g0 = walk_pre[c], g1 = walk_pre[c + 1];
        const long long s0 = eoff[g0 - wb], m = eoff[g1 - wb] - s0;
        const double maxw = __longlong_as_double((long long)colmax[c]);
        int lg_m = 0;
        while ((1ll << lg_m) < m) ++lg_m;
        const int E = maxw > 0.0 ? 61 - ilogb(maxw) - lg_m : 0;
        for (long long i = threadIdx.x; i < m; i += blockDim.x) {
            const int s = est[s0 + i];
            if (s >= 0)
                smem_add_i64(&row[s], __double2ll_rn(ldexp(ewt[s0 + i], E)));
        }
        __syncthreads();
        if (trans) {  // Q^T: column (c - cb) of an n x (ce - cb) row-major block
            for (long long j = threadIdx.x; j < n; j += blockDim.x) Q[j * ldq + (c - cb)] = ldexp((double)row[j], -E);
        } else {
            double *out = Q + (c - cb) * ldq;
            for (long long j = threadIdx.x; j < n; j += blockDim.x) out[j] = ldexp((double)row[j], -E);
        }
        __syncthreads();
    }
}

static int qdense(mcf_graph *g, const mcf_walk_params *p, const long long *walk_pre, long long cb, long long ce,
                  double *Q, long long ldq, long long *stats, cudaStream_t s, bool trans = false) {
    int rc = check_params(g, p, walk_pre, cb, ce);
    if (rc) return rc;
    MCF_ARG(Q && stats && ldq >= (trans ? ce - cb : g->n), "mcf_walk_qdense: null Q/stats or ldq too small");
    if (g->n > QDENSE_MAX_N) {
        set_error("dense Q rows need n <= 16384 (use rand_funm_diag / rand_funm_action for larger graphs)");
        return MCF_ERR_RESOURCE;
    }
    long long wb = 0, we = 0;
    rc = read_walk_range(walk_pre, cb, ce, &wb, &we, s);
    if (rc) return rc;
    MCF_CUDA(cudaMemsetAsync(Q, 0, sizeof(double) * ldq * (trans ? g->n : ce - cb), s));
    if (we == wb) return MCF_OK;
    const long long nw = we - wb;
    MCF_ARG(nw < WALKS_PER_LAUNCH, "mcf_walk_qdense: walks per call must be below 2^31 (split the column range)");
    AsyncFrees frees(s);
    unsigned long long *colmax = nullptr;
    long long *elen = nullptr;
    int *err = nullptr;
    MCF_CUDA(cudaMallocAsync(&colmax, sizeof(unsigned long long) * g->n, s));
    frees.keep(colmax);
    MCF_CUDA(cudaMemsetAsync(colmax, 0, sizeof(unsigned long long) * g->n, s));
    MCF_CUDA(cudaMallocAsync(&elen, sizeof(long long) * (2 * nw + 1) + 16, s));
    frees.keep(elen);
    long long *eoff = elen + nw;
    err = reinterpret_cast<int *>(eoff + nw + 1);
    MCF_CUDA(cudaMemsetAsync(err, 0, sizeof(int), s));
    rc = launch_walk_emit(g, p, walk_pre, cb, ce, nw, EMIT_COUNT, nullptr, nullptr, 0, 0, elen, nullptr, nullptr,
                          nullptr, stats, err, s);
    if (rc) return rc;
    rc = exclusive_scan_i64(elen, eoff, nw, s);
    if (rc) return rc;
    long long total = 0;
    MCF_CUDA(cudaMemcpyAsync(&total, eoff + nw, sizeof(long long), cudaMemcpyDeviceToHost, s));
    MCF_CUDA(cudaStreamSynchronize(s));
    MCF_ARG(total <= 4 * emission_budget(), "too many emissions for one dense-Q call (split the column range)");
    int *est = nullptr;
    double *ewt = nullptr;
    MCF_CUDA(cudaMallocAsync(&est, sizeof(int) * (total > 0 ? total : 1), s));
    frees.keep(est);
    MCF_CUDA(cudaMallocAsync(&ewt, sizeof(double) * (total > 0 ? total : 1), s));
    frees.keep(ewt);
    rc = launch_walk_emit(g, p, walk_pre, cb, ce, nw, EMIT_EXPLICIT, nullptr, nullptr, 0, 0, eoff, est, ewt, colmax,
                          stats, err, s);
    if (rc) return rc;
    const size_t smem = sizeof(long long) * g->n;
    MCF_CUDA(cudaFuncSetAttribute(k_qdense, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    long long nc = ce - cb;
    int grid = (int)(nc < 4 * sm_count() ? nc : 4 * sm_count());
    k_qdense<<<grid, 512, smem, s>>>(walk_pre, cb, ce, wb, eoff, est, ewt, colmax, g->n, Q, ldq, trans ? 1 : 0);
    mcf::note_launch();
    MCF_LAUNCHED("k_qdense");
    return MCF_OK;
}

// Variance of d_i from G walk-group passes (MCF_FLAG_WALK_GROUP): for every
// entry (i, c), the group partials P_g = pcol_g[(i, c)] (walks w = g mod G of
// column c, W0 = 1/N_c) give group means Y_g = N_c P_g / n_g of the per-walk
// contribution, n_g = |{w < N_c : w = g mod G}|; the between-group sum of
// squares SSB = sum_g n_g (Y_g - Y)^2, Y = sum_g P_g, has expectation
// (G' - 1) sigma_c^2 (G' = min(G, N_c) non-empty groups), so
// Var(pcol) ~ SSB / ((G' - 1) N_c), and Var(d_i) = sum_c Var(pcol[(i, c)])
// (columns are independent).  4 lanes per row, as k_diag_final.
__global__ void k_diag_variance(const long long *__restrict__ row_ptr, const int *__restrict__ col_ids,
                                const long long *__restrict__ csr2csc, const double *__restrict__ pg, long long nnz,
                                int G, const long long *__restrict__ walk_pre, double *__restrict__ var, long long rb,
                                long long re) {
    const long long i = rb + (((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 2);
    const int sub = threadIdx.x & 3;
    double s = 0.0;
    if (i < re) {
        for (long long e = row_ptr[i] + sub; e < row_ptr[i + 1]; e += 4) {
            const int c = col_ids[e];
            const long long nc = walk_pre[c + 1] - walk_pre[c];
            const long long gn = nc < G ? nc : G;
            if (gn < 2) continue;
            const long long p = csr2csc[e];
            double tot = 0.0;
            for (int g = 0; g < G; ++g) tot += pg[(long long)g * nnz + p];
            const double ybar = tot;  // mean per-walk contribution: N_c * pcol / N_c
            double ssb = 0.0;
            for (int g = 0; g < gn; ++g) {
                const double ng = (double)(nc / G + (g < nc % G ? 1 : 0));
                const double yg = (double)nc * pg[(long long)g * nnz + p] / ng;
                ssb += ng * (yg - ybar) * (yg - ybar);
            }
            s += ssb / ((double)(gn - 1) * (double)nc);
        }
    }
#pragma unroll
    for (int o = 2; o > 0; o >>= 1) s += __shfl_xor_sync(MCF_FULL, s, o, 4);
    if (i < re && sub == 0) var[i] = s;
}

// ---------------------------------------------------------------------------
// Full estimate F = zeta_0 I + zeta_1 A + A Q A (Alg. 2 / Eq. 19,
// SPEC.md:347-356) with the sparse A: per block of b walked columns,
//   Q_b^T (n x b)      dense Q rows of the block, written transposed (k_qdense)
//   R^T = A^T Q_b^T     SpMM over the CSC of A: a warp per output row, lanes
//                       over the block's columns, entries in CSC order
//   R   = (R^T)^T       tiled shared-memory transpose
//   F  += A[:, block] R SpMM: a warp per row i of F, the row's entries in
//                       [cb, ce) in CSR order, lanes over F's columns
// Every sum has a fixed order: deterministic.  Dense output, n <= 16384.
// ---------------------------------------------------------------------------
__global__ void k_dense_init(const long long *__restrict__ row_ptr, const int *__restrict__ col_ids,
                             const double *__restrict__ vals, long long n, double z0, double z1,
                             double *__restrict__ F, long long ldf) {
    const long long i = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (i >= n) return;
    double *row = F + i * ldf;
    for (long long j = lane; j < n; j += 32) row[j] = j == i ? z0 : 0.0;
    __syncwarp();
    for (long long e = row_ptr[i] + lane; e < row_ptr[i + 1]; e += 32) {
        const int c = col_ids[e];
        row[c] = (c == i ? z0 : 0.0) + z1 * vals[e];
    }
}

// Y[k, r] = sum over CSC column k of a_jk X[j, r]  (Y = A^T X, X: n x b, Y: n x b)
__global__ void k_spmm_at(const long long *__restrict__ csc_ptr, const int *__restrict__ csc_rows,
                          const double *__restrict__ csc_vals, long long n, const double *__restrict__ X, long long b,
                          double *__restrict__ Y) {
    const long long k = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (k >= n) return;
    for (long long r0 = 0; r0 < b; r0 += 32 * 4) {
        double acc[4] = {0.0, 0.0, 0.0, 0.0};
        for (long long e = csc_ptr[k]; e < csc_ptr[k + 1]; ++e) {
            const long long j = csc_rows[e];
            const double a = csc_vals[e];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const long long r = r0 + u * 32 + lane;
                if (r < b) acc[u] = fma(a, X[j * b + r], acc[u]);
            }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const long long r = r0 + u * 32 + lane;
            if (r < b) Y[k * b + r] = acc[u];
        }
    }
}

// out (cols x rows) = in (rows x cols)^T, 32 x 32 shared-memory tiles
__global__ void k_transpose(const double *__restrict__ in, long long rows, long long cols, double *__restrict__ out) {
    __shared__ double tile[32][33];
    const long long r0 = (long long)blockIdx.y * 32, c0 = (long long)blockIdx.x * 32;
    for (int dy = threadIdx.y; dy < 32; dy += blockDim.y) {
        const long long r = r0 + dy, c = c0 + threadIdx.x;
        if (r < rows && c < cols) tile[dy][threadIdx.x] = in[r * cols + c];
    }
    __syncthreads();
    for (int dy = threadIdx.y; dy < 32; dy += blockDim.y) {
        const long long c = c0 + dy, r = r0 + threadIdx.x;
        if (c < cols && r < rows) out[c * rows + r] = tile[threadIdx.x][dy];
    }
}

// F[i, :] += sum over the entries (i, c) of row i with c in [cb, ce) of a_ic R[c - cb, :]
__global__ void k_spmm_rows_blk(const long long *__restrict__ row_ptr, const int *__restrict__ col_ids,
                                const double *__restrict__ vals, long long n, long long cb, long long ce,
                                const double *__restrict__ R, double *__restrict__ F, long long ldf) {
    const long long i = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (i >= n) return;
    long long lo = row_ptr[i], hi = row_ptr[i + 1];
    {  // first entry with column >= cb (columns sorted within the row)
        long long a = lo, z = hi;
        while (a < z) {
            const long long m = (a + z) >> 1;
            if (col_ids[m] < cb) a = m + 1;
            else z = m;
        }
        lo = a;
    }
    if (lo >= hi || col_ids[lo] >= ce) return;
    double *row = F + i * ldf;
    for (long long k0 = 0; k0 < n; k0 += 32 * 4) {
        double acc[4] = {0.0, 0.0, 0.0, 0.0};
        for (long long e = lo; e < hi && col_ids[e] < ce; ++e) {
            const double a = vals[e];
            const double *rr = R + (long long)(col_ids[e] - cb) * n;
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const long long k = k0 + u * 32 + lane;
                if (k < n) acc[u] = fma(a, rr[k], acc[u]);
            }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const long long k = k0 + u * 32 + lane;
            if (k < n) row[k] += acc[u];
        }
    }
}

static int funm_full(mcf_graph *g, const mcf_walk_params *p, const long long *walk_pre, double z0, double z1,
                     double *F, long long ldf, long long block, long long *stats, cudaStream_t s) {
    MCF_ARG(g && p && walk_pre && F && stats, "mcf_funm_full: null argument");
    MCF_ARG(ldf >= g->n, "mcf_funm_full: ldf < n");
    if (g->n > QDENSE_MAX_N) {
        set_error("the dense estimate needs n <= 16384 (use rand_funm_diag / rand_funm_action for larger graphs)");
        return MCF_ERR_RESOURCE;
    }
    const long long n = g->n;
    if (block < 1 || block > n) block = n < 1024 ? n : 1024;
    AsyncFrees frees(s);
    double *qt = nullptr, *rt = nullptr, *r = nullptr;
    MCF_CUDA(cudaMallocAsync(&qt, sizeof(double) * n * block, s));
    frees.keep(qt);
    MCF_CUDA(cudaMallocAsync(&rt, sizeof(double) * n * block, s));
    frees.keep(rt);
    MCF_CUDA(cudaMallocAsync(&r, sizeof(double) * n * block, s));
    frees.keep(r);
    const unsigned wgrid = (unsigned)((n * 32 + 255) / 256);
    k_dense_init<<<wgrid, 256, 0, s>>>((const long long *)g->row_ptr, g->col_ids, g->vals, n, z0, z1, F, ldf);
    mcf::note_launch();
    MCF_LAUNCHED("k_dense_init");
    for (long long cb = 0; cb < n; cb += block) {
        const long long ce = cb + block < n ? cb + block : n, b = ce - cb;
        int rc = qdense(g, p, walk_pre, cb, ce, qt, b, stats, s, true);  // Q_b^T, n x b
        if (rc) return rc;
        k_spmm_at<<<wgrid, 256, 0, s>>>((const long long *)g->csc_ptr, g->csc_rows, g->csc_vals, n, qt, b, rt);
        mcf::note_launch();
        k_transpose<<<dim3((unsigned)((b + 31) / 32), (unsigned)((n + 31) / 32)), dim3(32, 8), 0, s>>>(rt, n, b, r);
        mcf::note_launch();
        k_spmm_rows_blk<<<wgrid, 256, 0, s>>>((const long long *)g->row_ptr, g->col_ids, g->vals, n, cb, ce, r, F, ldf);
        mcf::note_launch();
        MCF_LAUNCHED("k_spmm_rows_blk");
    }
    return MCF_OK;
}

static int diag_variance(mcf_graph *g, const double *pcol_groups, int groups, const long long *walk_pre, double *var,
                         long long rb, long long re, cudaStream_t s) {
    MCF_ARG(g && pcol_groups && walk_pre && var, "mcf_diag_variance: null argument");
    MCF_ARG(groups >= 2 && groups <= 256, "mcf_diag_variance: groups must be in [2, 256]");
    MCF_ARG(0 <= rb && rb <= re && re <= g->n, "mcf_diag_variance: bad row range");
    int rc = ensure_csr2csc(g, s);
    if (rc) return rc;
    const long long rows = re - rb;
    if (rows == 0) return MCF_OK;
    k_diag_variance<<<(unsigned)((rows * 4 + 255) / 256), 256, 0, s>>>((const long long *)g->row_ptr, g->col_ids,
                                                                       (const long long *)g->csr2csc, pcol_groups,
                                                                       g->nnz, groups, walk_pre, var, rb, re);
    mcf::note_launch();
    MCF_LAUNCHED("k_diag_variance");
    return MCF_OK;
}

static int diag_combine(mcf_graph *g, double z0, double z1, const double *pcol, double *d, long long rb, long long re,
                        cudaStream_t s) {
    MCF_ARG(g && pcol && d, "mcf_diag_combine: null argument");
    MCF_ARG(0 <= rb && rb <= re && re <= g->n, "mcf_diag_combine: bad row range");
    int rc = ensure_csr2csc(g, s);
    if (rc) return rc;
    long long rows = re - rb;
    if (rows == 0) return MCF_OK;
    k_diag_final<<<(unsigned)((rows * 4 + 255) / 256), 256, 0, s>>>((const long long *)g->row_ptr, g->col_ids, g->vals,
                                                                   (const long long *)g->csr2csc, pcol, z0, z1, d, rb, re,
                                                                   PeerArgs{});
    mcf::note_launch();
    MCF_LAUNCHED("k_diag_final");
    return MCF_OK;
}

static int diag_combine_peer(mcf_graph *g, double z0, double z1, const double *const *pcol_parts,
                             const long long *col_bounds, int nparts, double *const *d_outs, int nouts, long long rb,
                             long long re, cudaStream_t s) {
    MCF_ARG(g, "mcf_diag_combine_peer: null graph");
    MCF_ARG(0 <= rb && rb <= re && re <= g->n, "mcf_diag_combine_peer: bad row range");
    PeerArgs pa{};
    int rc = make_peer_args(pcol_parts, col_bounds, nparts, d_outs, nouts, g->n, &pa);
    if (rc) return rc;
    rc = ensure_csr2csc(g, s);
    if (rc) return rc;
    const long long rows = re - rb;
    if (rows == 0) return MCF_OK;
    k_diag_final<true><<<(unsigned)((rows * 4 + 255) / 256), 256, 0, s>>>(
        (const long long *)g->row_ptr, g->col_ids, g->vals, (const long long *)g->csr2csc, nullptr, z0, z1, nullptr, rb,
        re, pa);
    mcf::note_launch();
    MCF_LAUNCHED("k_diag_final_peer");
    return MCF_OK;
}

}  // namespace mcf

extern "C" {

int mcf_walk_diag(mcf_graph *g, const mcf_walk_params *p, const int64_t *walk_pre, int64_t col_begin, int64_t col_end,
                  double *pcol, int64_t *stats, void *stream) {
    return mcf::diag(g, p, (const long long *)walk_pre, col_begin, col_end, nullptr, nullptr, pcol, (long long *)stats,
                     (cudaStream_t)stream, false);
}

int mcf_replay_diag(mcf_graph *g, const mcf_walk_params *p, const int64_t *walk_pre, int64_t col_begin,
                    int64_t col_end, const int64_t *walk_off, const int32_t *entries, double *pcol, int64_t *stats,
                    void *stream) {
    return mcf::diag(g, p, (const long long *)walk_pre, col_begin, col_end, (const long long *)walk_off, entries, pcol,
                     (long long *)stats, (cudaStream_t)stream, true);
}

int mcf_walk_qdense(mcf_graph *g, const mcf_walk_params *p, const int64_t *walk_pre, int64_t col_begin,
                    int64_t col_end, double *Q, int64_t ldq, int64_t *stats, void *stream) {
    return mcf::qdense(g, p, (const long long *)walk_pre, col_begin, col_end, Q, ldq, (long long *)stats,
                       (cudaStream_t)stream);
}

int mcf_funm_full(mcf_graph *g, const mcf_walk_params *p, const int64_t *walk_pre, double zeta0, double zeta1,
                  double *F, int64_t ldf, int64_t block, int64_t *stats, void *stream) {
    return mcf::funm_full(g, p, (const long long *)walk_pre, zeta0, zeta1, F, ldf, block, (long long *)stats,
                          (cudaStream_t)stream);
}

int mcf_diag_variance(mcf_graph *g, const double *pcol_groups, int groups, const int64_t *walk_pre, double *var,
                      int64_t row_begin, int64_t row_end, void *stream) {
    return mcf::diag_variance(g, pcol_groups, groups, (const long long *)walk_pre, var, row_begin, row_end,
                              (cudaStream_t)stream);
}

int mcf_diag_combine(mcf_graph *g, double zeta0, double zeta1, const double *pcol, double *d, int64_t row_begin,
                     int64_t row_end, void *stream) {
    return mcf::diag_combine(g, zeta0, zeta1, pcol, d, row_begin, row_end, (cudaStream_t)stream);
}

int mcf_diag_combine_peer(mcf_graph *g, double zeta0, double zeta1, const double *const *pcol_parts,
                          const int64_t *col_bounds, int n_parts, double *const *d_outs, int n_outs,
                          int64_t row_begin, int64_t row_end, void *stream) {
    return mcf::diag_combine_peer(g, zeta0, zeta1, pcol_parts, (const long long *)col_bounds, n_parts, d_outs, n_outs,
                                  (long long)row_begin, (long long)row_end, (cudaStream_t)stream);
}

}  // extern "C"
