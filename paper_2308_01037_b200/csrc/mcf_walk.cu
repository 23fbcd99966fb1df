// Action walks (Alg. 3, :337-367) and the SpMV combine.
//
// Replaces the reference hot loop: the estimator's per-column Python loop
// around walker.run_walks_batch (walker.py:245-290) whose on_step callback
// accumulates q_c += zeta_{k+2} W r[l_k].
//
// Work decomposition: every walk is one lane.  A warp refills idle lanes from
// a global walk counter with one aggregated atomic, so walks of different
// columns and different lengths share a warp without waiting for each other
// (Katz walks end at the weight cutoff after 1..60 steps).  Per step a lane
// touches two random 32-byte sectors: the node header of its state and the
// sampled CSR entry -- the 64 B/step algorithmic traffic of DESIGN.md.
//
// Per-walk contributions are written to a buffer and summed per column in a
// fixed order, so q does not depend on scheduling, on the number of GPUs or on
// how the column range is split.
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <tuple>

#include "mcf_internal.cuh"

namespace mcf {

constexpr uint32_t PHILOX_SALT = 0x6d636621u;  // "mcf!"

struct WalkCommon {
    const NodeHdr *__restrict__ hdr;
    const NodeHdr *__restrict__ went;  // fat layout (nullptr: compact)
    const int *__restrict__ ecol;
    const double *__restrict__ cdf;
    const unsigned long long *__restrict__ alias;  // Vose alias entries of non-uniform rows (or null: cdf)
    int alias_tbits;
    const double *__restrict__ zeta;
    const long long *__restrict__ walk_pre;
    const int *__restrict__ blk_col;
    long long col_begin, col_end;  // walk range = [walk_pre[col_begin], walk_pre[col_end]), read on the device
    long long capacity;            // walks the per-walk buffers hold (a larger range is clamped and flagged)
    int col_last;
    long long max_steps;
    double cutoff;
    uint32_t key0, key1;
    const long long *__restrict__ walk_off;  // replay only
    const int *__restrict__ entries;          // replay only
    unsigned *counter;  // walks handed out (chunked, relative to the range start)
    unsigned long long *colmax;  // diag: per-column max |emission| (IEEE bits), or null
    int return_only;             // MCF_FLAG_RETURN_ONLY
    unsigned grp_n, grp_i;       // MCF_FLAG_WALK_GROUP: run only walks w = grp_i mod grp_n (0: all)
    long long *stats;
    int *err;
    const uint2 *__restrict__ lean;         // v = 1 on uniform-value graphs (else null)
    const uint32_t *__restrict__ lean4;     // compact 4-B variant (nnz < 2^25), preferred when built
    const unsigned long long *__restrict__ lean_id;  // diag: {start, id, degree} of col[e] in 8 B (or null)
    int li_sbits, li_ibits, li_dbits;
    const long long *__restrict__ row_ptr;  // lean walks: start state of a column
    const double *__restrict__ rsum_by_deg;
    // L2 bulk prefetch of the walk tables at kernel start (bytes 0: none)
    const char *pf[3];
    long long pf_bytes[3];
};

// Alternative (MCF_L2_PREFETCH=2): a streaming read of the tables by a
// separate kernel (16-B loads cached in L2 only) right before the walk.
__global__ void k_l2_touch(const uint4 *__restrict__ p, long long n16, unsigned *sink) {
    uint32_t acc = 0;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += (long long)gridDim.x * blockDim.x) {
        const uint4 v = __ldcg(p + i);
        acc ^= v.x ^ v.w;
    }
    if (acc == 0x9e3779b9u && sink) *sink = acc;
}

// Each CTA streams its share of the walk tables into L2 with TMA bulk
// prefetches (cp.async.bulk.prefetch.L2: no registers, no shared memory, the
// copy engine does the sequential read) before its lanes start walking.
__device__ __forceinline__ void l2_prefetch_tables(const WalkCommon &a) {
    if (threadIdx.x >= 3 || a.pf_bytes[threadIdx.x] <= 0) return;
    const long long bytes = a.pf_bytes[threadIdx.x];
    const long long share = ((bytes + gridDim.x - 1) / gridDim.x + 15) & ~15ll;
    const long long lo = share * blockIdx.x;
    const long long hi = lo + share < bytes ? lo + share : bytes;
    for (long long o = lo; o < hi; o += 32768) {
        const unsigned len = (unsigned)((hi - o < 32768 ? hi - o : 32768) & ~15ll);
        if (len) asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a.pf[threadIdx.x] + o), "r"(len) : "memory");
    }
}

// Inverse-CDF draw inside one non-uniform row: first t with cdf[t] > u.
__device__ __forceinline__ int cdf_pick(const double *__restrict__ cdf, int deg, double u) {
    int lo = 0, hi = deg - 1;
    while (lo < hi) {
        int mid = (lo + hi) >> 1;
        if (__ldg(cdf + mid) > u) hi = mid;
        else lo = mid + 1;
    }
    return lo;
}

// Walk statistics: warp sums into shared counters, then one global atomic
// per CTA and counter (per-warp atomics on the same 4 words contended at the
// end of the kernel).  Called once by every thread of the CTA.
__device__ __forceinline__ void flush_stats(long long *stats, unsigned walks_, unsigned em_, unsigned tr_,
                                            unsigned ab_) {
    __shared__ unsigned long long cta[4];
    if (threadIdx.x < 4) cta[threadIdx.x] = 0;
    __syncthreads();
    long long walks = walks_, em = em_, tr = tr_, ab = ab_;
    walks = warp_sum_ll(walks);
    em = warp_sum_ll(em);
    tr = warp_sum_ll(tr);
    ab = warp_sum_ll(ab);
    if ((threadIdx.x & 31) == 0) {
        if (walks) atomicAdd(&cta[0], (unsigned long long)walks);
        if (em) atomicAdd(&cta[1], (unsigned long long)em);
        if (tr) atomicAdd(&cta[2], (unsigned long long)tr);
        if (ab) atomicAdd(&cta[3], (unsigned long long)ab);
    }
    __syncthreads();
    if (threadIdx.x < 4 && cta[threadIdx.x]) atomicAdd((unsigned long long *)&stats[threadIdx.x], cta[threadIdx.x]);
}

// Walk state of one lane (one walk slot).
struct Lane {
    int rel;               // walk index relative to the range start; -1 wants a walk, -2 none left
    int k, c;              // step, start column
    unsigned wl;           // walk index inside its column
    double w, thr, x;      // weight, cutoff threshold, per-walk accumulator
    NodeHdr h;             // header of the current state; h.pad = the state's node id
    uint32_t r0, r1;       // second half of the Philox block (odd steps)
    long long epos, eend;  // replay cursor
};

// Warp-level walk pool: a warp takes `chunk` consecutive walks from the
// global counter at a time and hands them to its lanes as they finish, so the
// single counter sees one atomic per chunk (a per-refill atomic serialised
// short Katz walks on the counter's L2 slice).  pool/pool_end are warp-uniform.
struct WarpPool {
    int next, end, chunk;
};

__device__ __forceinline__ WarpPool make_pool(int nw_total) {
    const int warps = (gridDim.x * blockDim.x) >> 5;
    int c = nw_total / (warps * 8);
    c = c < 32 ? 32 : (c > 256 ? 256 : c);
    return WarpPool{0, 0, c & ~31};
}

// Walks of the launch: the range read from walk_pre, clamped to the buffers'
// capacity (budgets summing past the caller's walk_capacity would otherwise
// write past them); a clamp sets error bit 8, which the host reports.
__device__ __forceinline__ int clamp_walks(const WalkCommon &a, long long nw) {
    if (nw > a.capacity) {
        if (blockIdx.x == 0 && threadIdx.x == 0 && a.err) atomicOr(a.err, 8);
        nw = a.capacity;
    }
    return (int)nw;
}

template <bool REPLAY, bool LEAN = false>
__device__ __forceinline__ bool refill(const WalkCommon &a, long long wb, int nw, Lane &L, unsigned &n_walks,
                                       WarpPool &P) {
    const unsigned need = __ballot_sync(MCF_FULL, L.rel == -1);
    if (need) {
        const int rank = __popc(need & lanemask_lt());
        const int cnt = __popc(need);
        const int avail = P.end - P.next;
        int rel = P.next + rank;
        if (cnt > avail) {  // pool runs dry: one atomic for the next chunk
            unsigned base = 0;
            if ((threadIdx.x & 31) == 0) base = atomicAdd(a.counter, (unsigned)P.chunk);
            base = __shfl_sync(MCF_FULL, base, 0);
            if (rank >= avail) rel = (int)base + (rank - avail);
            P.next = (int)base + (cnt - avail);
            P.end = (int)base + P.chunk;
        } else {
            P.next += cnt;
        }
        if (L.rel == -1) {
            const long long g = wb + rel;
            if (rel < nw) {
                int c = column_of_walk(g, rel, nw, a.walk_pre, a.blk_col, a.col_last);
                long long pre = __ldg(a.walk_pre + c);
                long long nc = __ldg(a.walk_pre + c + 1) - pre;
                L.rel = (int)rel;
                L.c = c;
                L.wl = (unsigned)(g - pre);
                L.k = 0;
                if (LEAN) {  // start state from row_ptr (8 B per node, column-contiguous) and the degree table
                    const long long rs = __ldg(a.row_ptr + c), re = __ldg(a.row_ptr + c + 1);
                    L.h.start = (int)rs;
                    L.h.deg = (int)(re - rs);
                    L.h.flags = HDR_UNIFORM;
                    L.h.rsum = __ldg(a.rsum_by_deg + (re - rs));
                    L.h.aux = L.h.rsum;
                } else {
                    L.h = load_hdr(a.hdr + c);
                }
                L.h.pad = (uint32_t)c;
                L.w = 1.0 / (double)nc;       // W0 = 1/N_c (walker.py:263)
                L.thr = a.cutoff * L.w;       // strict cutoff W_c * W0 (walker.py:264)
                L.x = 0.0;
                if (REPLAY) {
                    L.epos = __ldg(a.walk_off + g);
                    L.eend = __ldg(a.walk_off + g + 1);
                }
                ++n_walks;
            } else {
                L.rel = -2;
            }
        }
    }
    return !__all_sync(MCF_FULL, L.rel == -2);
}

constexpr long long PICK_END = -1;   // walk ends at this emission (absorbed, or bad replay stream)
constexpr long long PICK_LAST = -2;  // final draw: only |W| matters, and |a/t| = row sum for every entry

// First half of a step (walker.py:274-281): choose the CSR entry to take from
// the current row.  Philox-4x32-10 yields 128 bits per (step pair, walk,
// column): even steps use the first 64, odd steps the second.
template <bool REPLAY, bool LEAN = false>
__device__ __forceinline__ long long pick(const WalkCommon &a, Lane &L, unsigned &ab) {
    const NodeHdr &h = L.h;
    if (h.deg == 0) {  // absorbing row (walker.py:274-278)
        ++ab;
        return PICK_END;
    }
    if (REPLAY) {
        if (L.epos >= L.eend) {
            atomicOr(a.err, 1);
            return PICK_END;
        }
        long long e = __ldg(a.entries + L.epos);
        ++L.epos;
        if (e < h.start || e >= (long long)h.start + h.deg) {
            atomicOr(a.err, 2);
            return PICK_END;
        }
        return e;
    }
    if (L.k + 1 >= a.max_steps) return PICK_LAST;
    uint64_t r;
    if ((L.k & 1) == 0) {
        U4 p = philox4x32_10(U4{(uint32_t)(L.k >> 1), L.wl, (uint32_t)L.c, PHILOX_SALT}, a.key0, a.key1);
        r = ((uint64_t)p.x << 32) | p.y;
        L.r0 = p.z;
        L.r1 = p.w;
    } else {
        r = ((uint64_t)L.r0 << 32) | L.r1;
    }
    if (LEAN || (h.flags & HDR_UNIFORM)) return h.start + (long long)__umul64hi(r, (uint64_t)h.deg);
    if (a.alias) {  // slot k = floor(u deg); keep it if the fraction of u deg is below its threshold
        const uint64_t k = __umul64hi(r, (uint64_t)h.deg), frac = r * (uint64_t)h.deg;
        const unsigned long long t = __ldg(a.alias + h.start + k);
        const unsigned long long tq = t & ((1ull << a.alias_tbits) - 1);
        const uint64_t f = frac >> (64 - a.alias_tbits);
        return h.start + (long long)(f < tq ? k : (t >> a.alias_tbits));
    }
    return h.start + cdf_pick(a.cdf + h.start, h.deg, (double)(r >> 11) * 0x1.0p-53);
}

// The header of the entry's target, with pad = target id and HDR_NEG_EDGE =
// sign of a_e.  Fat layout: one 32-B sector; compact: the entry's packed
// column id, then the target's header (two dependent sectors).
template <bool FAT, bool LEAN = false, bool WITH_ID = false>
__device__ __forceinline__ NodeHdr fetch_next(const WalkCommon &a, long long e) {
    if (LEAN) {  // {start, degree} of the target; |a| row sum (= r for v = 1) by degree
        NodeHdr h;
        if (WITH_ID && a.lean_id) {  // one 8-B entry: start, target id and degree together
            const unsigned long long t = __ldg(a.lean_id + e);
            const unsigned long long smask = (1ull << a.li_sbits) - 1, imask = (1ull << a.li_ibits) - 1;
            const unsigned long long dmax = (1ull << a.li_dbits) - 1;
            h.start = (int)(t & smask);
            h.pad = (uint32_t)((t >> a.li_sbits) & imask);
            const unsigned long long d = t >> (a.li_sbits + a.li_ibits);
            h.deg = d < dmax ? (int)d : (int)(__ldg(a.row_ptr + h.pad + 1) - h.start);  // hub target: row_ptr
            h.flags = HDR_UNIFORM;
            h.rsum = __ldg(a.rsum_by_deg + h.deg);
            h.aux = h.rsum;
            return h;
        }
        // the target id (diag emissions): issued together with the entry load,
        // consumed only at the end, so the two round trips overlap (measured:
        // reading it after decoding the entry stalled the diag walk a second time)
        const int idv = WITH_ID ? __ldg(a.ecol + e) : 0;
        if (a.lean4) {  // 4-B entries: [0 | deg:6 | start:25], or [1 | target id] for degree >= 63
            const uint32_t t = __ldg(a.lean4 + e);
            if (t & 0x80000000u) {
                const long long s0 = __ldg(a.row_ptr + (t & 0x7fffffffu)), s1 = __ldg(a.row_ptr + (t & 0x7fffffffu) + 1);
                h.start = (int)s0;
                h.deg = (int)(s1 - s0);
            } else {
                h.start = (int)(t & 0x1ffffffu);
                h.deg = (int)((t >> 25) & 63u);
            }
        } else {
            const uint2 t = __ldg(a.lean + e);
            h.start = (int)t.x;
            h.deg = (int)t.y;
        }
        h.flags = HDR_UNIFORM;
        h.pad = WITH_ID ? (uint32_t)(idv & 0x7fffffff) : 0u;
        h.rsum = __ldg(a.rsum_by_deg + h.deg);
        h.aux = h.rsum;
        return h;
    }
    if (FAT) return load_hdr(a.went + e);
    const int pc = __ldg(a.ecol + e);
    const int nxt = pc & 0x7fffffff;
    NodeHdr h = load_hdr(a.hdr + nxt);
    h.pad = (uint32_t)nxt;
    if (pc < 0) h.flags |= HDR_NEG_EDGE;
    return h;
}

// Second half (walker.py:282-288): weight update a/t = copysign(rowsum, a_e)
// of the CURRENT row (walker.py:124-125), move, then the strict cutoff and
// the step cap.  Returns true when the walk ended.
__device__ __forceinline__ bool apply(const WalkCommon &a, Lane &L, long long e, const NodeHdr &nh, unsigned &tr) {
    if (e == PICK_LAST) {
        L.w *= L.h.rsum;
    } else {
        L.w *= (nh.flags & HDR_NEG_EDGE) ? -L.h.rsum : L.h.rsum;
        L.h = nh;
    }
    ++L.k;
    if (!(fabs(L.w) > L.thr)) return true;  // walker.py:286-288
    if (L.k >= a.max_steps) {               // step cap: truncated (walker.py:270, :289)
        ++tr;
        return true;
    }
    return false;
}

template <int NW, int OCC>
struct WalkOcc {  // resident CTAs per SM the register budget is tuned for
    static constexpr int v = NW == 1 ? OCC : (NW == 2 ? (OCC == 4 ? 4 : 3) : 2);
};

// NW walks per lane, stepped together so their dependent loads overlap.
// OCC: CTAs per SM the one-walk variant is register-tuned for (4: no spills,
// 5: more warps with a few spilled registers).
template <bool REPLAY, bool FAT, int NW, int OCC = 5, bool LEAN = false>
__global__ void __launch_bounds__(256, (WalkOcc<NW, OCC>::v)) k_walk_action(WalkCommon a, double *__restrict__ xw) {
    l2_prefetch_tables(a);
    const long long wb = __ldg(a.walk_pre + a.col_begin);
    const int nw = clamp_walks(a, __ldg(a.walk_pre + a.col_end) - wb);
    Lane L[NW];
#pragma unroll
    for (int s = 0; s < NW; ++s) L[s].rel = -1;
    WarpPool P = make_pool(nw);
    unsigned n_walks = 0, em = 0, tr = 0, ab = 0;
    while (true) {
        bool more = false;
#pragma unroll
        for (int s = 0; s < NW; ++s) more |= refill<REPLAY, LEAN>(a, wb, nw, L[s], n_walks, P);
        if (!more) break;
        long long e[NW];
        NodeHdr nh[NW];
#pragma unroll
        for (int s = 0; s < NW; ++s) {
            if (L[s].rel < 0) continue;
            if (a.grp_n && L[s].k == 0 && L[s].wl % a.grp_n != a.grp_i) {  // walk outside the group
                xw[L[s].rel] = 0.0;
                L[s].rel = -1;
                --n_walks;
                continue;
            }
            // q_c += zeta W r[l]; classic MC diagonal: only back at the start (Alg. 1)
            // lean walks (v = 1, uniform values): the payload r = A 1 is the row sum itself
            const double pay = LEAN ? L[s].h.rsum
                                    : (a.return_only ? ((int)L[s].h.pad == L[s].c ? 1.0 : 0.0) : L[s].h.aux);
            L[s].x = fma(__ldg(a.zeta + L[s].k + 2) * L[s].w, pay, L[s].x);
            ++em;
            e[s] = pick<REPLAY, LEAN>(a, L[s], ab);
        }
#pragma unroll
        for (int s = 0; s < NW; ++s)
            if (L[s].rel >= 0 && e[s] >= 0) nh[s] = fetch_next<FAT, LEAN>(a, e[s]);
#pragma unroll
        for (int s = 0; s < NW; ++s) {
            if (L[s].rel < 0) continue;
            if (e[s] == PICK_END || apply(a, L[s], e[s], nh[s], tr)) {
                if (REPLAY && L[s].epos != L[s].eend) atomicOr(a.err, 4);
                xw[L[s].rel] = L[s].x;
                L[s].rel = -1;
            }
        }
    }
    flush_stats(a.stats, n_walks, em, tr, ab);
}

// Diagonal-mode walks.  Slot layout of the emission buffer per MODE:
//   EMIT_FIXED     column c owns slots [(pre_c - wb) L, (pre_{c+1} - wb) L),
//                  step-major inside: emission k of the column's walk w is at
//                  + k N_c + w, so lanes holding consecutive walks write
//                  consecutive addresses
//   EMIT_REPLAY    walk g owns walk_off[g]-off_base+rel .. + draws+1
//   EMIT_COUNT     no emission written; elen[rel] = number of emissions
//   EMIT_EXPLICIT  walk rel owns [eoff[rel], eoff[rel+1]) (exclusive scan of a
//                  previous EMIT_COUNT pass over the same Philox stream)
// Each emission is (state, zeta_{k+2} W_k); unused slots of a walk hold -1.
enum { EMIT_FIXED = 0, EMIT_REPLAY = 1, EMIT_COUNT = 2, EMIT_EXPLICIT = 3 };

// TH: threads per CTA (1024 with OCC 1: one CTA owns an SM -- the walks that run beside a combine, diag())
template <int MODE, bool FAT, int OCC = 4, bool LEAN = false, int TH = 256>
__global__ void __launch_bounds__(TH, OCC) k_walk_emit(WalkCommon a, long long slot_len, long long off_base,
                                                   long long *__restrict__ eaux, int *__restrict__ est,
                                                   double *__restrict__ ewt) {
    constexpr bool REPLAY = MODE == EMIT_REPLAY;
    if (MODE != EMIT_COUNT) l2_prefetch_tables(a);
    const long long wb = __ldg(a.walk_pre + a.col_begin);
    const int nw = clamp_walks(a, __ldg(a.walk_pre + a.col_end) - wb);
    Lane L;
    L.rel = -1;
    WarpPool P = make_pool(nw);
    unsigned n_walks = 0, em = 0, tr = 0, ab = 0;
    long long sb = 0, scap = 0, stride = 1;
    double wmax = 0.0;  // this walk's largest |emission| -> per-column max (fixed-point scale of k_diag_q)
    while (refill<REPLAY, LEAN>(a, wb, nw, L, n_walks, P)) {
        if (L.rel < 0) continue;
        const long long rel = L.rel;
        if (L.k == 0) {
            wmax = 0.0;
            if (MODE == EMIT_REPLAY) {
                sb = L.epos - off_base + rel;
                scap = L.eend - L.epos + 1;
            } else if (MODE == EMIT_FIXED) {
                const long long pre = __ldg(a.walk_pre + L.c);
                stride = __ldg(a.walk_pre + L.c + 1) - pre;
                sb = (pre - wb) * slot_len + L.wl;
                scap = slot_len;
            } else if (MODE == EMIT_EXPLICIT) {
                sb = eaux[rel];
                scap = eaux[rel + 1] - sb;
            }
            if (!REPLAY && a.grp_n && L.wl % a.grp_n != a.grp_i) {  // walk outside the group: no emission
                if (MODE == EMIT_COUNT) eaux[rel] = 0;
                else
                    for (long long t = 0; t < scap; ++t) __stcs(est + sb + t * stride, -1);
                --n_walks;
                L.rel = -1;
                continue;
            }
        }
        if (MODE != EMIT_COUNT) {
            const double om = __ldg(a.zeta + L.k + 2) * L.w;
            // streaming stores: the emission buffer (GBs) must not evict the walk tables from L2
            __stcs(est + sb + L.k * stride, (int)L.h.pad);
            __stcs(ewt + sb + L.k * stride, om);
            wmax = fmax(wmax, fabs(om));
        }
        ++em;
        const long long emitted = L.k + 1;
        const long long e = pick<REPLAY, LEAN>(a, L, ab);
        NodeHdr nh;
        if (e >= 0) nh = fetch_next<FAT, LEAN, true>(a, e);
        if (e == PICK_END || apply(a, L, e, nh, tr)) {
            if (REPLAY && L.epos != L.eend) atomicOr(a.err, 4);
            if (MODE == EMIT_COUNT) {
                eaux[rel] = emitted;
            } else {
                for (long long t = emitted; t < scap; ++t) __stcs(est + sb + t * stride, -1);
                if (wmax > 0.0) atomicMax(a.colmax + L.c, (unsigned long long)__double_as_longlong(wmax));
            }
            L.rel = -1;
        }
    }
    if (MODE != EMIT_COUNT) flush_stats(a.stats, n_walks, em, tr, ab);
}

// hdr[i].aux = r[i]
__global__ void k_set_aux(NodeHdr *__restrict__ hdr, const double *__restrict__ r, long long n) {
    long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) hdr[i].aux = r[i];
}

// fat layout: went[e].aux = r[target of e]
__global__ void k_set_aux_fat(NodeHdr *__restrict__ went, const double *__restrict__ r, long long nnz) {
    long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e < nnz) went[e].aux = __ldg(r + went[e].pad);
}

// q[c] = sum of the per-walk contributions of column c, fixed order; optional
// variance of that mean from the per-walk spread (SE for the z-tests).
// One warp per 32 consecutive columns: a lane sums a small column serially,
// the warp cooperates on large ones.
constexpr int SMALL_COL = 32;

__global__ void k_col_reduce(const long long *__restrict__ walk_pre, long long col_begin, long long col_end,
                             const double *__restrict__ xw, double *__restrict__ q, double *__restrict__ qvar) {
    const long long walk_begin = __ldg(walk_pre + col_begin);
    long long wid = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    int lane = threadIdx.x & 31;
    long long c = col_begin + wid * 32 + lane;
    bool in = c < col_end;
    long long lo = 0, hi = 0;
    if (in) {
        lo = walk_pre[c] - walk_begin;
        hi = walk_pre[c + 1] - walk_begin;
    }
    long long nc = hi - lo;
    if (in && nc <= SMALL_COL) {
        double s = 0.0;
        for (long long i = lo; i < hi; ++i) s += xw[i];
        q[c] = s;
        if (qvar) {
            double m2 = 0.0;
            for (long long i = lo; i < hi; ++i) {
                double d = (double)nc * xw[i] - s;
                m2 += d * d;
            }
            qvar[c] = nc > 1 ? m2 / ((double)(nc - 1) * (double)nc) : 0.0;
        }
    }
    unsigned big = __ballot_sync(MCF_FULL, in && nc > SMALL_COL);
    while (big) {
        int src = __ffs(big) - 1;
        big &= big - 1;
        long long blo = __shfl_sync(MCF_FULL, lo, src), bhi = __shfl_sync(MCF_FULL, hi, src);
        long long bc = __shfl_sync(MCF_FULL, c, src);
        double s = 0.0;
        for (long long i = blo + lane; i < bhi; i += 32) s += xw[i];
        s = warp_sum(s);
        if (lane == 0) q[bc] = s;
        if (qvar) {
            double bn = (double)(bhi - blo), m2 = 0.0;
            for (long long i = blo + lane; i < bhi; i += 32) {
                double d = bn * xw[i] - s;
                m2 += d * d;
            }
            m2 = warp_sum(m2);
            if (lane == 0) qvar[bc] = m2 / ((bn - 1.0) * bn);
        }
    }
}

// y = alpha v + beta r + A x, rows binned by length so hub rows do not
// serialise a few lanes: rows with degree <= LONG_ROW use G lanes each,
// longer rows (graph->long_rows) one warp each (one CTA above HUGE_ROW).
// UNI: every stored value equals `uval` (0/1 graph times gamma), so the value
// array is not read: y = h + uval * sum_j x_j.  Fixed reduction order.
constexpr int HUGE_ROW = 1024;

// Short rows (<= LONG_ROW entries): a warp takes 32 consecutive rows and walks
// their entries as one flat, coalesced segment, up to SEG_CAP entries per pass
// with every load of a pass in flight at once (the latency chain per row is
// row_ptr -> col_ids -> x, paid once per warp instead of once per entry).
// The products land in shared memory and each lane then sums its own row in
// CSR order with separate multiply and add, so y matches a sequential CSR
// matvec (scipy's) bit for bit on these rows.  Long rows take the blocks
// in front of the grid (a warp each, or the whole CTA past HUGE_ROW).
constexpr int SEG_CAP = 256;
constexpr int SPMV_WARPS = 8;

// v == V_ONES stands for the all-ones vector (total communicability)
#define V_ONES (reinterpret_cast<const double *>(1))

__device__ __forceinline__ double combine_exact(double alpha, const double *v, double beta, bool has_r, double ri,
                                                long long i, double s) {
    // ((alpha v) + (beta r)) + s, each operation rounded: the numpy expression
    // z0 * v + z1 * r + A @ q evaluated elementwise
    double h = 0.0;
    if (v) h = v == V_ONES ? alpha : __dmul_rn(alpha, v[i]);
    if (has_r) h = v ? __dadd_rn(h, __dmul_rn(beta, ri)) : __dmul_rn(beta, ri);
    return (v || has_r) ? __dadd_rn(h, s) : s;
}

// r for the combine: r[i], or (lean v = 1 path) the row sum by degree, also
// stored to rt.out -- r = A 1 is then produced here, after the walks, instead
// of before them.
struct RowSumR {
    const double *tab;  // rsum_by_deg, or null
    double *out;
};

__device__ __forceinline__ double r_of(const double *r, const RowSumR &rt, long long i, long long deg) {
    if (rt.tab) {
        const double ri = __ldg(rt.tab + deg);
        rt.out[i] = ri;
        return ri;
    }
    return r ? r[i] : 0.0;
}

// r = A 1 for v = 1: the sequential CSR row sum of a_ij, which for a row
// without negative entries is exactly the |a| row sum already in the header
// (same additions, same order, a * 1.0 == a); rows with a negative entry are
// summed again with their signs.  r also lands in hdr.aux for the walk.
__global__ void k_r_ones(NodeHdr *__restrict__ hdr, const double *__restrict__ vals, long long n, double *__restrict__ r,
                         long long *__restrict__ stats) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < 4 && stats) stats[i] = 0;
    if (i >= n) return;
    const NodeHdr h = load_hdr(hdr + i);
    double s = h.rsum;
    if (h.flags & HDR_HAS_NEG) {
        s = 0.0;
        for (int t = 0; t < h.deg; ++t) s = __dadd_rn(s, vals[h.start + t]);
    }
    if (h.deg == 0) s = 0.0;
    r[i] = s;
    hdr[i].aux = s;
}

// Multi-GPU action without a separate collective (mcf_spmv_peer): x (= q) is
// gathered straight from the rank that owns each column -- its buffer mapped
// into this process over NVLink (CUDA IPC) -- and every result row is stored
// to every rank's y buffer, so the SpMV itself is the exchange.
template <bool PEER>
__device__ __forceinline__ double xload(const double *__restrict__ x, const PeerArgs &pa, int c) {
    if (!PEER) return __ldg(x + c);
    return __ldg(pa.x[peer_owner(pa, c)] + c);
}

template <bool PEER>
__device__ __forceinline__ void ystore(double *__restrict__ y, const PeerArgs &pa, long long i, double out) {
    if (!PEER) {
        y[i] = out;
        return;
    }
    for (int k = 0; k < pa.nouts; ++k) pa.y[k][i] = out;
}

template <bool UNI, bool PEER = false>
__global__ void __launch_bounds__(256, 4) k_spmv(const long long *__restrict__ row_ptr, const int *__restrict__ col_ids,
                                              const double *__restrict__ vals, double uval, double alpha,
                                              const double *__restrict__ v, double beta, const double *__restrict__ r,
                                              const double *__restrict__ x, double *__restrict__ y, long long row_begin,
                                              long long row_end, NodeHdr *__restrict__ aux,
                                              const int *__restrict__ long_rows, long long n_long, int long_blocks,
                                              RowSumR rt, PeerArgs pa) {
    __shared__ double prod[SPMV_WARPS][SEG_CAP];
    const bool has_r = r || rt.tab;
    __shared__ double part[SPMV_WARPS];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if ((int)blockIdx.x < long_blocks) {
        // ---- long rows: a warp per row up to HUGE_ROW, the CTA beyond -------
        const long long gw = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
        const long long nw = ((long long)long_blocks * blockDim.x) >> 5;
        for (long long li = gw; li < n_long; li += nw) {
            const long long i = long_rows[li];
            const long long e0 = row_ptr[i], e1 = row_ptr[i + 1];
            if (i < row_begin || i >= row_end || e1 - e0 > HUGE_ROW) continue;
            double s = 0.0;
            for (long long e = e0 + lane; e < e1; e += 32)
                s += __dmul_rn(UNI ? uval : __ldg(vals + e), xload<PEER>(x, pa, __ldg(col_ids + e)));
            s = warp_sum(s);
            if (lane == 0) {
                const double out = combine_exact(alpha, v, beta, has_r, r_of(r, rt, i, e1 - e0), i, s);
                ystore<PEER>(y, pa, i, out);
                if (aux) aux[i].aux = out;
            }
        }
        for (long long li = blockIdx.x; li < n_long; li += long_blocks) {
            const long long i = long_rows[li];
            const long long e0 = row_ptr[i], e1 = row_ptr[i + 1];
            if (i < row_begin || i >= row_end || e1 - e0 <= HUGE_ROW) continue;
            double s = 0.0;
            for (long long e = e0 + threadIdx.x; e < e1; e += blockDim.x)
                s += __dmul_rn(UNI ? uval : __ldg(vals + e), xload<PEER>(x, pa, __ldg(col_ids + e)));
            s = warp_sum(s);
            if (lane == 0) part[w] = s;
            __syncthreads();
            if (threadIdx.x < 32) {
                const double t = warp_sum(threadIdx.x < SPMV_WARPS ? part[threadIdx.x] : 0.0);
                if (threadIdx.x == 0) {
                    const double out = combine_exact(alpha, v, beta, has_r, r_of(r, rt, i, e1 - e0), i, t);
                    ystore<PEER>(y, pa, i, out);
                    if (aux) aux[i].aux = out;
                }
            }
            __syncthreads();
        }
        return;
    }
    // ---- short rows: 32 consecutive rows per warp ---------------------------
    // The warp's short rows form runs of consecutive rows between long rows;
    // each run's entries are one contiguous CSR range, walked SEG_CAP at a time.
    const long long i0 = row_begin + ((long long)(blockIdx.x - long_blocks) * SPMV_WARPS + w) * 32;
    if (i0 >= row_end) return;
    const long long i = i0 + lane;
    const bool in = i < row_end;
    long long e0 = 0, e1 = 0;
    if (in) {
        e0 = row_ptr[i];
        e1 = row_ptr[i + 1];
    }
    const bool mine = in && e1 - e0 <= LONG_ROW;
    const int nl = row_end - i0 < 32 ? (int)(row_end - i0) : 32;  // valid lanes (warp-uniform)
    unsigned longm = __ballot_sync(MCF_FULL, in && !mine);
    double s = 0.0;
    int first = 0;
    while (first < nl) {
        const int stop = longm ? __ffs(longm) - 1 : nl;  // run = lanes [first, stop)
        if (stop > first) {
            const long long run_lo = __shfl_sync(MCF_FULL, e0, first);
            const long long run_hi = __shfl_sync(MCF_FULL, e1, stop - 1);
            const bool member = lane >= first && lane < stop;
            const long long rs = e0 - run_lo, re = e1 - run_lo;  // my row inside the run
            for (long long P = 0; P < run_hi - run_lo; P += SEG_CAP) {
                const int cnt = (int)(run_hi - run_lo - P < SEG_CAP ? run_hi - run_lo - P : SEG_CAP);
                int c[SEG_CAP / 32];
                double av[SEG_CAP / 32];
#pragma unroll
                for (int k = 0; k < SEG_CAP / 32; ++k) {
                    const int t = lane + 32 * k;
                    if (t < cnt) {
                        const long long e = run_lo + P + t;
                        c[k] = __ldg(col_ids + e);
                        av[k] = UNI ? uval : __ldg(vals + e);
                    }
                }
#pragma unroll
                for (int k = 0; k < SEG_CAP / 32; ++k) {
                    const int t = lane + 32 * k;
                    if (t < cnt) prod[w][t] = __dmul_rn(av[k], xload<PEER>(x, pa, c[k]));
                }
                __syncwarp();
                if (member) {
                    const long long lo = rs > P ? rs : P, hi = re < P + cnt ? re : P + cnt;
                    for (long long t = lo; t < hi; ++t) s = __dadd_rn(s, prod[w][t - P]);
                }
                __syncwarp();
            }
        }
        if (!longm) break;
        first = stop + 1;
        longm &= longm - 1;
    }
    if (mine) {
        const double out = combine_exact(alpha, v, beta, has_r, r_of(r, rt, i, e1 - e0), i, s);
        ystore<PEER>(y, pa, i, out);
        if (aux) aux[i].aux = out;
    }
}

// y_i = (A 1)_i for rows [rb, re): the row sums in CSR order, bit-identical
// to the reference's A @ ones (scipy's sequential CSR matvec, walker.py /
// PAPER.md:345 with v = 1): |a| sums from the headers, signed rows re-summed
__global__ void k_row_sums(const NodeHdr *__restrict__ hdr, const double *__restrict__ vals, long long rb,
                           long long re, double *__restrict__ y) {
    const long long i = rb + (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= re) return;
    const NodeHdr h = load_hdr(hdr + i);
    double s = h.rsum;
    if (h.flags & HDR_HAS_NEG) {
        s = 0.0;
        for (int t = 0; t < h.deg; ++t) s = __dadd_rn(s, vals[h.start + t]);
    }
    y[i] = h.deg ? s : 0.0;
}

int spmv(mcf_graph *g, double alpha, const double *v, double beta, const double *r, const double *x, double *y,
         long long rb, long long re, cudaStream_t s, NodeHdr *aux = nullptr, RowSumR rt = RowSumR{nullptr, nullptr}) {
    MCF_ARG(g && y, "mcf_spmv: null argument");
    MCF_ARG(0 <= rb && rb <= re && re <= g->n, "mcf_spmv: bad row range");
    if (re == rb) return MCF_OK;
    if (!x) {  // x = 1: the row sums (alpha = beta = 0 only)
        MCF_ARG(alpha == 0.0 && beta == 0.0 && !aux, "mcf_spmv: x = NULL (row sums) takes alpha = beta = 0");
        k_row_sums<<<(unsigned)((re - rb + 255) / 256), 256, 0, s>>>(g->hdr, g->vals, rb, re, y);
        mcf::note_launch();
        MCF_LAUNCHED("k_row_sums");
        return MCF_OK;
    }
    const long long *rp = (const long long *)g->row_ptr;
    long long lb = g->n_long_rows > 0 ? (g->n_long_rows + SPMV_WARPS - 1) / SPMV_WARPS : 0;
    if (lb > 2 * sm_count()) lb = 2 * sm_count();
    const long long sb = (re - rb + 32 * SPMV_WARPS - 1) / (32 * SPMV_WARPS);
    const unsigned grid = (unsigned)(lb + sb);
    if (g->uniform_value)
        k_spmv<true><<<grid, 32 * SPMV_WARPS, 0, s>>>(rp, g->col_ids, g->vals, g->value, alpha, v, beta, r, x, y, rb,
                                                      re, aux, g->long_rows, g->n_long_rows, (int)lb, rt, PeerArgs{});
    else
        k_spmv<false><<<grid, 32 * SPMV_WARPS, 0, s>>>(rp, g->col_ids, g->vals, g->value, alpha, v, beta, r, x, y, rb,
                                                       re, aux, g->long_rows, g->n_long_rows, (int)lb, rt, PeerArgs{});
    mcf::note_launch();
    MCF_LAUNCHED("k_spmv");
    return MCF_OK;
}

int spmv_peer(mcf_graph *g, double alpha, const double *v, double beta, const double *r,
              const double *const *x_parts, const long long *bounds, int nparts, double *const *y_outs, int nouts,
              long long rb, long long re, cudaStream_t s) {
    MCF_ARG(g, "mcf_spmv_peer: null graph");
    MCF_ARG(0 <= rb && rb <= re && re <= g->n, "mcf_spmv_peer: bad row range");
    PeerArgs pa{};
    int rc = make_peer_args(x_parts, bounds, nparts, y_outs, nouts, g->n, &pa);
    if (rc) return rc;
    if (re == rb) return MCF_OK;
    const long long *rp = (const long long *)g->row_ptr;
    long long lb = g->n_long_rows > 0 ? (g->n_long_rows + SPMV_WARPS - 1) / SPMV_WARPS : 0;
    if (lb > 2 * sm_count()) lb = 2 * sm_count();
    const long long sb = (re - rb + 32 * SPMV_WARPS - 1) / (32 * SPMV_WARPS);
    const unsigned grid = (unsigned)(lb + sb);
    const RowSumR rt{nullptr, nullptr};
    if (g->uniform_value)
        k_spmv<true, true><<<grid, 32 * SPMV_WARPS, 0, s>>>(rp, g->col_ids, g->vals, g->value, alpha, v, beta, r,
                                                            nullptr, nullptr, rb, re, nullptr, g->long_rows,
                                                            g->n_long_rows, (int)lb, rt, pa);
    else
        k_spmv<false, true><<<grid, 32 * SPMV_WARPS, 0, s>>>(rp, g->col_ids, g->vals, g->value, alpha, v, beta, r,
                                                             nullptr, nullptr, rb, re, nullptr, g->long_rows,
                                                             g->n_long_rows, (int)lb, rt, pa);
    mcf::note_launch();
    MCF_LAUNCHED("k_spmv_peer");
    return MCF_OK;
}

// ---------------------------------------------------------------------------
// host drivers
// ---------------------------------------------------------------------------
int check_params(const mcf_graph *g, const mcf_walk_params *p, const long long *walk_pre, long long cb,
                 long long ce) {
    MCF_ARG(g && p && walk_pre, "walk call: null argument");
    MCF_ARG(p->max_steps >= 1, "max_steps must be at least 1");                          // walker.py:66-67
    MCF_ARG(p->weight_cutoff > 0.0 && p->weight_cutoff < 1.0,
            "weight_cutoff must lie strictly between 0 and 1");                         // walker.py:64-65
    MCF_ARG(p->max_steps < (1ll << 31), "max_steps must be below 2^31");
    MCF_ARG(p->zeta, "zeta coefficients missing");
    MCF_ARG(!(p->flags & MCF_FLAG_WALK_GROUP) || MCF_GROUP_INDEX(p->flags) < MCF_GROUP_COUNT(p->flags),
            "walk group index must be below the group count");
    MCF_ARG(0 <= cb && cb <= ce && ce <= g->n, "bad column range");
    return MCF_OK;
}

// Kernel arguments for a column range.  No host synchronisation: the walk
// range is read by the kernels from walk_pre, buffers are sized by the
// caller's upper bound `capacity` (so the whole call can be captured in a
// CUDA graph).
int setup_common(mcf_graph *g, const mcf_walk_params *p, const long long *walk_pre, long long cb, long long ce,
                 long long capacity, WalkCommon &a, int **blk, cudaStream_t s, int *blk_ready = nullptr) {
    if (blk_ready) {
        *blk = blk_ready;  // filled by the budget scan (funm_action)
    } else {
        int rc = build_blk_col(walk_pre, cb, ce, capacity, blk, s);
        if (rc) return rc;
    }
    a.hdr = g->hdr;
    a.went = g->went;
    a.ecol = g->ecol;
    a.cdf = g->cdf;
    a.alias = g->alias;
    a.alias_tbits = g->alias_tbits;
    a.zeta = p->zeta;
    a.walk_pre = walk_pre;
    a.blk_col = *blk;
    a.col_begin = cb;
    a.col_end = ce;
    a.capacity = capacity;
    a.err = nullptr;
    a.col_last = (int)(ce > cb ? ce - 1 : cb);
    a.max_steps = p->max_steps;
    a.cutoff = p->weight_cutoff;
    a.key0 = (uint32_t)(p->seed & 0xffffffffu);
    a.key1 = (uint32_t)(p->seed >> 32);
    a.walk_off = nullptr;
    a.entries = nullptr;
    a.colmax = nullptr;
    a.lean = nullptr;
    a.lean4 = nullptr;
    a.lean_id = nullptr;
    a.li_sbits = a.li_ibits = a.li_dbits = 0;
    a.rsum_by_deg = nullptr;
    a.row_ptr = (const long long *)g->row_ptr;
    a.return_only = (p->flags & MCF_FLAG_RETURN_ONLY) ? 1 : 0;
    a.grp_n = (p->flags & MCF_FLAG_WALK_GROUP) ? (unsigned)MCF_GROUP_COUNT(p->flags) : 0u;
    a.grp_i = (p->flags & MCF_FLAG_WALK_GROUP) ? (unsigned)MCF_GROUP_INDEX(p->flags) : 0u;
    for (int k = 0; k < 3; ++k) {
        a.pf[k] = nullptr;
        a.pf_bytes[k] = 0;
    }
    if (g->l2_prefetch) {
        a.pf[0] = (const char *)g->hdr;
        a.pf_bytes[0] = (long long)sizeof(NodeHdr) * g->n;
        a.pf[1] = (const char *)g->ecol;
        a.pf_bytes[1] = 4ll * g->nnz;
        if (g->cdf) {
            a.pf[2] = (const char *)g->cdf;
            a.pf_bytes[2] = 8ll * g->nnz;
        }
        for (int k = 0; k < 3; ++k)  // bulk prefetch wants 16-B aligned ranges
            if ((uintptr_t)a.pf[k] & 15) a.pf_bytes[k] = 0;
        const char *mode = getenv("MCF_L2_PREFETCH");
        if (mode && !strcmp(mode, "2")) {
            for (int k = 0; k < 3; ++k) {
                if (a.pf_bytes[k] > 0) {
                    k_l2_touch<<<sm_count() * 4, 512, 0, s>>>((const uint4 *)a.pf[k], a.pf_bytes[k] / 16, nullptr);
                    mcf::note_launch();
                }
                a.pf_bytes[k] = 0;
            }
        }
    }
    return MCF_OK;
}

// Upper bound on the walks of [cb, ce): the caller's hint, else read (sync).
int walk_capacity(const mcf_walk_params *p, const long long *walk_pre, long long cb, long long ce, long long *cap,
                  cudaStream_t s) {
    if (p->walk_capacity > 0) {
        *cap = p->walk_capacity;
        return MCF_OK;
    }
    long long wb = 0, we = 0;
    int rc = read_walk_range(walk_pre, cb, ce, &wb, &we, s);
    *cap = we - wb;
    return rc;
}

// walks stepped together per lane (MCF_WALKS_PER_LANE = 1, 2 or 4; 14 = one
// walk at 4 CTAs/SM).  Measured on B200 (r01): one walk per lane at 4 CTAs/SM
// is fastest on both the L2-resident config 2 and the HBM-bound config 4 --
// the walk is bound by the random-sector rate, not by per-lane latency.
static int walks_per_lane() {
    static int v = 0;
    if (!v) {
        const char *e = getenv("MCF_WALKS_PER_LANE");
        v = e ? atoi(e) : 0;  // 0: each kernel's default
        // 1/2/4 walks per lane; 14/15/16 = one walk at 4/5/6 CTAs per SM;
        // 24 = two walks at 4.  -1: the kernel's measured default
        if (v != 1 && v != 2 && v != 4 && v != 14 && v != 15 && v != 16 && v != 24) v = -1;
    }
    return v;
}

template <typename K>
int walk_grid(K kernel, int threads, size_t smem) {
    // occupancy queries cost a few microseconds each: cache per (kernel, shape)
    static std::mutex mu;
    static std::map<std::tuple<const void *, int, size_t>, int> cache;
    const auto key = std::make_tuple(reinterpret_cast<const void *>(kernel), threads, smem);
    {
        std::lock_guard<std::mutex> lock(mu);
        auto it = cache.find(key);
        if (it != cache.end()) return it->second;
    }
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, smem);
    if (per_sm < 1) per_sm = 1;
    const int grid = per_sm * sm_count();
    std::lock_guard<std::mutex> lock(mu);
    cache[key] = grid;
    return grid;
}

// lean[e] = {start, degree} of col[e]
__global__ void k_build_lean(const long long *__restrict__ row_ptr, const int *__restrict__ col_ids, long long nnz,
                             uint2 *__restrict__ lean) {
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= nnz) return;
    const int c = col_ids[e];
    const long long s0 = row_ptr[c], s1 = row_ptr[c + 1];
    lean[e] = make_uint2((unsigned)s0, (unsigned)(s1 - s0));
}

// lean4[e]: [0 | degree:6 | start:25] of col[e] when the degree is below 63,
// else [1 | col[e]] (the walk then reads row_ptr): half the bytes of lean[]
// for graphs with nnz < 2^25, so the table stays L2-resident far longer
__global__ void k_build_lean4(const long long *__restrict__ row_ptr, const int *__restrict__ col_ids, long long nnz,
                              uint32_t *__restrict__ lean4) {
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= nnz) return;
    const int c = col_ids[e];
    const long long s0 = row_ptr[c], d = row_ptr[c + 1] - s0;
    lean4[e] = d < 63 ? ((uint32_t)d << 25) | (uint32_t)s0 : 0x80000000u | (uint32_t)c;
}

// rsum_by_deg[deg(i)] = rsum(i): with every |a| equal, rows of equal degree add
// the same values in the same order, so every writer stores the same bits
__global__ void k_rsum_by_deg(const NodeHdr *__restrict__ hdr, long long n, double *__restrict__ tab) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const NodeHdr h = load_hdr(hdr + i);
    tab[h.deg] = h.deg ? h.rsum : 0.0;
}

// lean_id[e] = [deg : dbits | col[e] : ibits | row start : sbits] of col[e]
__global__ void k_build_lean_id(const long long *__restrict__ row_ptr, const int *__restrict__ col_ids, long long nnz,
                                int sbits, int ibits, int dbits, unsigned long long *__restrict__ out) {
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= nnz) return;
    const int c = col_ids[e];
    const long long s0 = row_ptr[c], d = row_ptr[c + 1] - s0;
    const unsigned long long dmax = (1ull << dbits) - 1;
    const unsigned long long dd = (unsigned long long)d < dmax ? (unsigned long long)d : dmax;
    out[e] = (dd << (sbits + ibits)) | ((unsigned long long)c << sbits) | (unsigned long long)s0;
}

static int bits_for(long long v) {  // bits to hold values 0..v
    int b = 1;
    while (b < 63 && (1ll << b) <= v) ++b;
    return b;
}

static bool lean_eligible(const mcf_graph *g) {
    const char *env = getenv("MCF_LEAN_WALK");
    if (env && !strcmp(env, "0")) return false;
    return g->uniform_value && g->nnz < (1ll << 31) && g->info.max_degree < (1ll << 31);
}

// The diag walk's one-load table (MCF_LEAN_ID=0 disables: ecol[e] beside the lean entry)
static int ensure_lean_id(mcf_graph *g, cudaStream_t s) {
    if (g->lean_id) return MCF_OK;
    const char *env = getenv("MCF_LEAN_ID");
    if (env && !strcmp(env, "0")) return MCF_OK;
    const int sb = bits_for(g->nnz), ib = bits_for(g->n - 1), db = 64 - sb - ib;
    if (db < 6) return MCF_OK;  // too few degree bits: keep the two-array walk
    unsigned long long *t = nullptr;
    MCF_CUDA(cudaMallocAsync(&t, sizeof(unsigned long long) * g->nnz, s));
    k_build_lean_id<<<(unsigned)((g->nnz + 255) / 256), 256, 0, s>>>((const long long *)g->row_ptr, g->col_ids,
                                                                       g->nnz, sb, ib, db, t);
    mcf::note_launch();
    MCF_LAUNCHED("k_build_lean_id");
    g->lean_id = t;
    g->li_sbits = sb;
    g->li_ibits = ib;
    g->li_dbits = db;
    return MCF_OK;
}

static int ensure_lean(mcf_graph *g, cudaStream_t s) {
    if (g->lean || g->lean4) return MCF_OK;
    double *tab = nullptr;
    MCF_CUDA(cudaMallocAsync(&tab, sizeof(double) * (g->info.max_degree + 1), s));
    MCF_CUDA(cudaMemsetAsync(tab, 0, sizeof(double) * (g->info.max_degree + 1), s));
    const char *env = getenv("MCF_LEAN4");
    if (g->nnz < (1ll << 25) && !(env && !strcmp(env, "0"))) {
        uint32_t *lean4 = nullptr;
        MCF_CUDA(cudaMallocAsync(&lean4, sizeof(uint32_t) * g->nnz, s));
        k_build_lean4<<<(unsigned)((g->nnz + 255) / 256), 256, 0, s>>>((const long long *)g->row_ptr, g->col_ids,
                                                                        g->nnz, lean4);
        g->lean4 = lean4;
    } else {
        uint2 *lean = nullptr;
        MCF_CUDA(cudaMallocAsync(&lean, sizeof(uint2) * g->nnz, s));
        k_build_lean<<<(unsigned)((g->nnz + 255) / 256), 256, 0, s>>>((const long long *)g->row_ptr, g->col_ids,
                                                                      g->nnz, lean);
        g->lean = lean;
    }
    mcf::note_launch();
    k_rsum_by_deg<<<(unsigned)((g->n + 255) / 256), 256, 0, s>>>(g->hdr, g->n, tab);
    mcf::note_launch();
    MCF_LAUNCHED("k_build_lean");
    g->rsum_by_deg = tab;
    return MCF_OK;
}

int launch_walk_emit(mcf_graph *g, const mcf_walk_params *p, const long long *walk_pre, long long cb, long long ce,
                     long long nwalks, int mode, const long long *walk_off, const int *entries, long long slot_len,
                     long long off_base, long long *eaux, int *est, double *ewt, unsigned long long *colmax,
                     long long *stats, int *err, cudaStream_t s, int max_sms) {
    MCF_ARG(nwalks < WALKS_PER_LAUNCH, "walks per launch must be below 2^31 - 4096");
    // max_sms > 0: a grid sized for that many SMs (the walk pools take any grid), for walks that run beside
    // the previous batch's combine
    auto grid_for = [&](int full) { return max_sms > 0 && max_sms < sm_count() ? full / sm_count() * max_sms : full; };
    AsyncFrees frees(s);
    WalkCommon a;
    int *blk = nullptr;
    int rc = setup_common(g, p, walk_pre, cb, ce, nwalks, a, &blk, s);
    if (rc) return rc;
    frees.keep(blk);
    unsigned *counter = nullptr;
    MCF_CUDA(cudaMallocAsync(&counter, sizeof(unsigned long long), s));
    frees.keep(counter);
    MCF_CUDA(cudaMemsetAsync(counter, 0, sizeof(unsigned long long), s));
    a.counter = counter;
    a.err = err;
    a.stats = stats;
    a.walk_off = walk_off;
    a.entries = entries;
    a.colmax = colmax;
    const bool timed = (p->flags & MCF_FLAG_TIME_KERNELS) != 0 && mode != EMIT_COUNT;
    rc = timed_begin(g, timed, g->ev_walk, s);
    if (rc) return rc;
    // uniform-value graphs: {start, degree} entries + row sums by degree (one
    // dependent load per step; the emitted id comes from ecol alongside)
    const bool lean = mode != EMIT_REPLAY && lean_eligible(g);
    if (lean) {
        rc = ensure_lean(g, s);
        if (rc) return rc;
        rc = ensure_lean_id(g, s);
        if (rc) return rc;
        a.lean = g->lean;
        a.lean4 = g->lean4;
        a.lean_id = g->lean_id;
        a.li_sbits = g->li_sbits;
        a.li_ibits = g->li_ibits;
        a.li_dbits = g->li_dbits;
        a.rsum_by_deg = g->rsum_by_deg;
        for (int k = 0; k < 3; ++k) a.pf_bytes[k] = 0;
        switch (mode) {
            case EMIT_FIXED:
                if (max_sms > 0 && max_sms < sm_count()) {
                    // one 1024-thread CTA per reserved SM: no other CTA fits beside it, so the walk and the
                    // combine split the SMs cleanly.  (More walks per lane on fewer threads -- 2 x 1024, 4 x 512,
                    // 8 x 256 -- measured 1.2-3x slower: on a few SMs the walk is bound by issue, the Philox
                    // rounds, not by load latency.)
                    k_walk_emit<EMIT_FIXED, false, 1, true, 1024><<<max_sms, 1024, 0, s>>>(a, slot_len, 0, eaux, est, ewt);
                } else
                    k_walk_emit<EMIT_FIXED, false, 4, true><<<walk_grid(k_walk_emit<EMIT_FIXED, false, 4, true>, 256, 0), 256, 0, s>>>(a, slot_len, 0, eaux, est, ewt);
                break;
            case EMIT_COUNT: k_walk_emit<EMIT_COUNT, false, 4, true><<<grid_for(walk_grid(k_walk_emit<EMIT_COUNT, false, 4, true>, 256, 0)), 256, 0, s>>>(a, 0, 0, eaux, est, ewt); break;
            default: k_walk_emit<EMIT_EXPLICIT, false, 4, true><<<grid_for(walk_grid(k_walk_emit<EMIT_EXPLICIT, false, 4, true>, 256, 0)), 256, 0, s>>>(a, 0, 0, eaux, est, ewt);
        }
    } else if (g->went) {
        switch (mode) {
            case EMIT_FIXED: k_walk_emit<EMIT_FIXED, true><<<grid_for(walk_grid(k_walk_emit<EMIT_FIXED, true>, 256, 0)), 256, 0, s>>>(a, slot_len, 0, eaux, est, ewt); break;
            case EMIT_REPLAY: k_walk_emit<EMIT_REPLAY, true><<<grid_for(walk_grid(k_walk_emit<EMIT_REPLAY, true>, 256, 0)), 256, 0, s>>>(a, 0, off_base, eaux, est, ewt); break;
            case EMIT_COUNT: k_walk_emit<EMIT_COUNT, true><<<grid_for(walk_grid(k_walk_emit<EMIT_COUNT, true>, 256, 0)), 256, 0, s>>>(a, 0, 0, eaux, est, ewt); break;
            default: k_walk_emit<EMIT_EXPLICIT, true><<<grid_for(walk_grid(k_walk_emit<EMIT_EXPLICIT, true>, 256, 0)), 256, 0, s>>>(a, 0, 0, eaux, est, ewt);
        }
    } else {
        switch (mode) {
            case EMIT_FIXED: k_walk_emit<EMIT_FIXED, false><<<grid_for(walk_grid(k_walk_emit<EMIT_FIXED, false>, 256, 0)), 256, 0, s>>>(a, slot_len, 0, eaux, est, ewt); break;
            case EMIT_REPLAY: k_walk_emit<EMIT_REPLAY, false><<<grid_for(walk_grid(k_walk_emit<EMIT_REPLAY, false>, 256, 0)), 256, 0, s>>>(a, 0, off_base, eaux, est, ewt); break;
            case EMIT_COUNT: k_walk_emit<EMIT_COUNT, false><<<grid_for(walk_grid(k_walk_emit<EMIT_COUNT, false>, 256, 0)), 256, 0, s>>>(a, 0, 0, eaux, est, ewt); break;
            default: k_walk_emit<EMIT_EXPLICIT, false><<<grid_for(walk_grid(k_walk_emit<EMIT_EXPLICIT, false>, 256, 0)), 256, 0, s>>>(a, 0, 0, eaux, est, ewt);
        }
    }
    mcf::note_launch();
    MCF_LAUNCHED("k_walk_emit");
    return timed_end(timed, g->ev_walk, s);
}

static int action(mcf_graph *g, const mcf_walk_params *p, const long long *walk_pre, long long cb, long long ce,
                  const long long *walk_off, const int *entries, const double *r, double *q, double *qvar,
                  long long *stats, cudaStream_t s, bool replay, bool aux_ready = false, int *blk_ready = nullptr,
                  bool lean = false, double *xw_ready = nullptr, unsigned *counter_ready = nullptr,
                  bool capacity_exact = false) {
    int rc = check_params(g, p, walk_pre, cb, ce);
    if (rc) return rc;
    MCF_ARG(r && q && stats, "action walk: null r/q/stats");
    MCF_ARG(!(replay && (p->flags & MCF_FLAG_WALK_GROUP)), "walk groups apply to device-RNG walks, not replay");
    if (replay) MCF_ARG(walk_off && entries, "replay: null stream");
    long long nw = 0;
    rc = walk_capacity(p, walk_pre, cb, ce, &nw, s);
    if (rc) return rc;
    if (nw >= WALKS_PER_LAUNCH && !blk_ready) {
        // more walks than one launch indexes (int lanes): read the exact count
        // and, if it is still too large, run the range in column batches of at
        // most 2^30 walks (+ one column) -- q per column is the same either way
        long long wb = 0, we = 0;
        rc = read_walk_range(walk_pre, cb, ce, &wb, &we, s);
        if (rc) return rc;
        nw = we - wb;
        if (nw >= WALKS_PER_LAUNCH) {
            std::vector<long long> hb;
            unsigned long long hmax = 0;
            rc = column_batches(walk_pre, cb, ce, 1ll << 30, hb, &hmax, s);
            if (rc) return rc;
            MCF_ARG(hmax < (1ull << 30), "a column's walk budget must be below 2^30");
            mcf_walk_params pb = *p;
            pb.walk_capacity = 0;  // each batch reads its exact range
            for (size_t b = 0; b + 1 < hb.size(); ++b) {
                rc = action(g, &pb, walk_pre, hb[b], hb[b + 1], walk_off, entries, r, q, qvar, stats, s, replay,
                            b > 0 || aux_ready, nullptr, lean);
                if (rc) return rc;
            }
            return MCF_OK;
        }
    }
    MCF_ARG(nw < WALKS_PER_LAUNCH, "walks per call must be below 2^31 - 4096 (split the column range)");
    AsyncFrees frees(s);
    WalkCommon a;
    int *blk = nullptr;
    rc = setup_common(g, p, walk_pre, cb, ce, nw, a, &blk, s, blk_ready);
    if (rc) return rc;
    if (!blk_ready) frees.keep(blk);
    double *xw = xw_ready;
    unsigned *counter = counter_ready;  // preallocated: already zero (funm_action's one memset)
    int *err = nullptr;
    if (!xw) {
        MCF_CUDA(cudaMallocAsync(&xw, sizeof(double) * (nw > 0 ? nw : 1), s));
        frees.keep(xw);
    }
    if (!counter) {
        MCF_CUDA(cudaMallocAsync(&counter, sizeof(unsigned long long) + sizeof(int) * 2, s));
        frees.keep(counter);
        MCF_CUDA(cudaMemsetAsync(counter, 0, sizeof(unsigned long long) + sizeof(int) * 2, s));
    }
    err = (int *)(counter + 2);
    a.counter = counter;
    a.err = err;
    a.stats = stats;
    a.walk_off = walk_off;
    a.entries = entries;
    if (!aux_ready) {
        k_set_aux<<<(unsigned)((g->n + 255) / 256), 256, 0, s>>>(g->hdr, r, g->n);
        mcf::note_launch();
    }
    if (lean) {
        rc = ensure_lean(g, s);
        if (rc) return rc;
        a.lean = g->lean;
        a.lean4 = g->lean4;
        a.rsum_by_deg = g->rsum_by_deg;
        for (int k = 0; k < 3; ++k) a.pf_bytes[k] = 0;  // the L2 prefetch covers the compact tables only
    } else if (g->went) {
        k_set_aux_fat<<<(unsigned)((g->nnz + 255) / 256), 256, 0, s>>>(g->went, r, g->nnz);
        mcf::note_launch();
    }
    MCF_LAUNCHED("k_set_aux");
    const bool timed = (p->flags & MCF_FLAG_TIME_KERNELS) != 0;
    if (nw > 0) {
        rc = timed_begin(g, timed, g->ev_walk, s);
        if (rc) return rc;
        if (lean) {
            // one walk per lane at 5 CTAs/SM (no spills): measured best for the
            // one-load chain (4: -12%, 6: equal with spills, 2 walks/lane: -45%)
            switch (walks_per_lane()) {
                case 14: k_walk_action<false, false, 1, 4, true><<<walk_grid(k_walk_action<false, false, 1, 4, true>, 256, 0), 256, 0, s>>>(a, xw); break;
                case 16: k_walk_action<false, false, 1, 6, true><<<walk_grid(k_walk_action<false, false, 1, 6, true>, 256, 0), 256, 0, s>>>(a, xw); break;
                case 24: k_walk_action<false, false, 2, 4, true><<<walk_grid(k_walk_action<false, false, 2, 4, true>, 256, 0), 256, 0, s>>>(a, xw); break;
                default: k_walk_action<false, false, 1, 5, true><<<walk_grid(k_walk_action<false, false, 1, 5, true>, 256, 0), 256, 0, s>>>(a, xw);
            }
        } else if (g->went) {
            if (replay) {
                k_walk_action<true, true, 1><<<walk_grid(k_walk_action<true, true, 1>, 256, 0), 256, 0, s>>>(a, xw);
            } else {
                switch (walks_per_lane() < 0 ? 14 : walks_per_lane()) {  // header walk: 4 CTAs/SM
                    case 2: k_walk_action<false, true, 2><<<walk_grid(k_walk_action<false, true, 2>, 256, 0), 256, 0, s>>>(a, xw); break;
                    case 4: k_walk_action<false, true, 4><<<walk_grid(k_walk_action<false, true, 4>, 256, 0), 256, 0, s>>>(a, xw); break;
                    case 14: k_walk_action<false, true, 1, 4><<<walk_grid(k_walk_action<false, true, 1, 4>, 256, 0), 256, 0, s>>>(a, xw); break;
                    case 16: k_walk_action<false, true, 1, 6><<<walk_grid(k_walk_action<false, true, 1, 6>, 256, 0), 256, 0, s>>>(a, xw); break;
                    case 24: k_walk_action<false, true, 2, 4><<<walk_grid(k_walk_action<false, true, 2, 4>, 256, 0), 256, 0, s>>>(a, xw); break;
                    default: k_walk_action<false, true, 1><<<walk_grid(k_walk_action<false, true, 1>, 256, 0), 256, 0, s>>>(a, xw);
                }
            }
        } else {
            if (replay) {
                k_walk_action<true, false, 1><<<walk_grid(k_walk_action<true, false, 1>, 256, 0), 256, 0, s>>>(a, xw);
            } else {
                switch (walks_per_lane() < 0 ? 14 : walks_per_lane()) {  // header walk: 4 CTAs/SM
                    case 2: k_walk_action<false, false, 2><<<walk_grid(k_walk_action<false, false, 2>, 256, 0), 256, 0, s>>>(a, xw); break;
                    case 4: k_walk_action<false, false, 4><<<walk_grid(k_walk_action<false, false, 4>, 256, 0), 256, 0, s>>>(a, xw); break;
                    case 14: k_walk_action<false, false, 1, 4><<<walk_grid(k_walk_action<false, false, 1, 4>, 256, 0), 256, 0, s>>>(a, xw); break;
                    case 16: k_walk_action<false, false, 1, 6><<<walk_grid(k_walk_action<false, false, 1, 6>, 256, 0), 256, 0, s>>>(a, xw); break;
                    case 24: k_walk_action<false, false, 2, 4><<<walk_grid(k_walk_action<false, false, 2, 4>, 256, 0), 256, 0, s>>>(a, xw); break;
                    default: k_walk_action<false, false, 1><<<walk_grid(k_walk_action<false, false, 1>, 256, 0), 256, 0, s>>>(a, xw);
                }
            }
        }
        mcf::note_launch();
        MCF_LAUNCHED("k_walk_action");
        rc = timed_end(timed, g->ev_walk, s);
        if (rc) return rc;
    }
    long long ncol = ce - cb;
    if (ncol > 0) {
        long long warps = (ncol + 31) / 32;
        k_col_reduce<<<(unsigned)((warps * 32 + 255) / 256), 256, 0, s>>>(walk_pre, cb, ce, xw, q, qvar);
        mcf::note_launch();
        MCF_LAUNCHED("k_col_reduce");
    }
    int herr = 0;
    // replay streams are always checked; a caller-supplied walk_capacity (an
    // upper bound the device cannot verify without a sync) is checked whenever
    // the stream is not being captured into a CUDA graph
    cudaStreamCaptureStatus cap_st = cudaStreamCaptureStatusNone;
    MCF_CUDA(cudaStreamIsCapturing(s, &cap_st));
    if (replay || (p->walk_capacity > 0 && !capacity_exact && cap_st == cudaStreamCaptureStatusNone)) {
        MCF_CUDA(cudaMemcpyAsync(&herr, err, sizeof(int), cudaMemcpyDeviceToHost, s));
        MCF_CUDA(cudaStreamSynchronize(s));
    }
    if (herr & 8) {
        set_error("walk budgets of the column range exceed walk_capacity (" + std::to_string(p->walk_capacity) +
                  "): pass the exact walk count or 0");
        return MCF_ERR_ARGUMENT;
    }
    if (herr) {
        set_error("replay stream inconsistent with the walk (code " + std::to_string(herr) +
                  "): entries missing, surplus, or outside the current row");
        return MCF_ERR_ARGUMENT;
    }
    return MCF_OK;
}

// One side stream per device, shared by every graph (created once), and the
// graph's fork/join events: budgets beside r = A v in the action path, the
// global-table combine beside the cluster kernels in the diag path.
int ensure_side_stream(mcf_graph *g) {
    if (g->side) return MCF_OK;
    static std::mutex mu;
    static std::map<int, cudaStream_t> streams;
    std::lock_guard<std::mutex> lock(mu);
    auto it = streams.find(g->device);
    if (it == streams.end()) {
        cudaStream_t st;
        MCF_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
        it = streams.emplace(g->device, st).first;
    }
    MCF_CUDA(cudaEventCreateWithFlags(&g->ev_fork, cudaEventDisableTiming));
    MCF_CUDA(cudaEventCreateWithFlags(&g->ev_join, cudaEventDisableTiming));
    g->side = it->second;
    return MCF_OK;
}

// The whole RandFunmAction estimate for one process (Alg. 3): the walk
// budgets (largest remainder) on a side stream concurrently with r = A v (the
// SpMV writes r into the walk headers directly; v = NULL means v = 1, whose
// r is the row sums), then walks, per-column reduction, y = z0 v + z1 r + A q.  No host synchronisation; the fork/join
// uses events, so the whole call captures into one CUDA graph.
static int funm_action(mcf_graph *g, const mcf_walk_params *p, long long n_walks, long long *ni, long long *walk_pre,
                       const double *v, double z0, double z1, double *r, double *q, double *qvar, double *y,
                       long long *stats, cudaStream_t s) {
    MCF_ARG(g && r && q && y && walk_pre, "mcf_funm_action: null argument");  // ni optional
    int rc0 = ensure_side_stream(g);
    if (rc0) return rc0;
    MCF_ARG(p && n_walks >= 1, "mcf_funm_action: n_walks must be at least 1");
    if (n_walks >= WALKS_PER_LAUNCH) {
        // more walks than one launch indexes: budgets, r = A v, then the walks
        // in column batches (mcf_walk_action's path), then y -- not capturable
        AsyncFrees frees(s);
        long long *ni_ = ni;
        if (!ni_) {
            MCF_CUDA(cudaMallocAsync(&ni_, sizeof(long long) * g->n, s));
            frees.keep(ni_);
        }
        int rc = allocate_walks(g, n_walks, ni_, walk_pre, nullptr, s);
        if (rc) return rc;
        MCF_CUDA(cudaMemsetAsync(stats, 0, sizeof(long long) * 4, s));
        if (v) {
            rc = spmv(g, 0.0, nullptr, 0.0, nullptr, v, r, 0, g->n, s, g->hdr);
            if (rc) return rc;
        } else {
            k_r_ones<<<(unsigned)((g->n + 255) / 256), 256, 0, s>>>(g->hdr, g->vals, g->n, r, stats);
            mcf::note_launch();
            MCF_LAUNCHED("k_r_ones");
        }
        mcf_walk_params pp = *p;
        pp.walk_capacity = 0;
        const bool lean = !v && !(p->flags & MCF_FLAG_RETURN_ONLY) && lean_eligible(g);
        rc = action(g, &pp, walk_pre, 0, g->n, nullptr, nullptr, r, q, qvar, stats, s, false, true, nullptr, lean);
        if (rc) return rc;
        return spmv(g, z0, v ? v : V_ONES, z1, r, q, y, 0, g->n, s);
    }
    // one scratch block, one memset: [walk counter + error flags | budget-kernel state | blk | xw]
    const bool fused = fused_alloc_applies(g);
    const size_t ctl = 256, fz = fused ? fused_scratch_zero_bytes() : 0, fb = fused ? fused_scratch_bytes() : 0;
    const size_t fb_al = (fb + 255) & ~size_t(255);
    const long long nblk = (n_walks + (1ll << WALK_BLK_SHIFT) - 1) >> WALK_BLK_SHIFT;
    const size_t blk_bytes = ((size_t)nblk * sizeof(int) + 255) & ~size_t(255);
    char *scratch = nullptr;
    MCF_CUDA(cudaMallocAsync(&scratch, ctl + fb_al + blk_bytes + sizeof(double) * (size_t)n_walks, s));
    unsigned *counter = reinterpret_cast<unsigned *>(scratch);
    void *F = fused ? scratch + ctl : nullptr;
    int *blk = reinterpret_cast<int *>(scratch + ctl + fb_al);
    double *xw = reinterpret_cast<double *>(scratch + ctl + fb_al + blk_bytes);
    // MCF_FLAG_TIME_KERNELS: the span up to the walks (budgets, r) goes to the
    // graph's second timer (mcf_graph_kernel_times' q_ms on the action path)
    const bool timed = (p->flags & MCF_FLAG_TIME_KERNELS) != 0;
    int rc = timed_begin(g, timed, g->ev_q, s);
    if (rc) return rc;
    MCF_CUDA(cudaMemsetAsync(scratch, 0, ctl + fz, s));
    // v = 1 on a uniform-value graph: the lean walk needs neither r nor
    // hdr.aux, so r = A 1 (row sums by degree) is written by the final SpMV
    const bool lean_ones = !v && !(p->flags & MCF_FLAG_RETURN_ONLY) && lean_eligible(g);
    if (!v && fused) {  // v = 1: ONE kernel computes the budgets (and r = A 1 unless lean), zeroes stats
        rc = allocate_walks(g, n_walks, ni, walk_pre, blk, s, F, lean_ones ? nullptr : r, stats);
        if (rc) return rc;
        v = V_ONES;
    } else {  // budgets on the side stream, concurrently with r = A v
        MCF_CUDA(cudaEventRecord(g->ev_fork, s));
        MCF_CUDA(cudaStreamWaitEvent(g->side, g->ev_fork, 0));
        rc = allocate_walks(g, n_walks, ni, walk_pre, blk, g->side, F);
        if (rc) return rc;
        MCF_CUDA(cudaEventRecord(g->ev_join, g->side));
        if (v) {
            MCF_CUDA(cudaMemsetAsync(stats, 0, sizeof(long long) * 4, s));
            rc = spmv(g, 0.0, nullptr, 0.0, nullptr, v, r, 0, g->n, s, g->hdr);
            if (rc) return rc;
        } else {  // v = 1 (the same kernel zeroes the statistics)
            k_r_ones<<<(unsigned)((g->n + 255) / 256), 256, 0, s>>>(g->hdr, g->vals, g->n, r, stats);
            mcf::note_launch();
            MCF_LAUNCHED("k_r_ones");
            v = V_ONES;
        }
        MCF_CUDA(cudaStreamWaitEvent(s, g->ev_join, 0));
    }
    rc = timed_end(timed, g->ev_q, s);
    if (rc) return rc;
    mcf_walk_params pp = *p;
    pp.walk_capacity = n_walks;  // exact: the budgets sum to n_walks
    const bool lean = v == V_ONES && !(p->flags & MCF_FLAG_RETURN_ONLY) && lean_eligible(g);
    rc = action(g, &pp, walk_pre, 0, g->n, nullptr, nullptr, r, q, qvar, stats, s, false, true, blk, lean, xw, counter,
                true);
    if (rc) return rc;
    if (lean_ones && fused)
        rc = spmv(g, z0, v, z1, nullptr, q, y, 0, g->n, s, nullptr, RowSumR{g->rsum_by_deg, r});
    else
        rc = spmv(g, z0, v, z1, r, q, y, 0, g->n, s);
    if (rc) return rc;
    MCF_CUDA(cudaFreeAsync(scratch, s));
    return MCF_OK;
}



}  // namespace mcf

extern "C" {

int mcf_funm_action(mcf_graph *g, const mcf_walk_params *p, int64_t n_walks, int64_t *ni, int64_t *walk_pre,
                    const double *v, double zeta0, double zeta1, double *r, double *q, double *q_var, double *y,
                    int64_t *stats, void *stream) {
    return mcf::funm_action(g, p, (long long)n_walks, (long long *)ni, (long long *)walk_pre, v, zeta0, zeta1, r, q,
                            q_var, y, (long long *)stats, (cudaStream_t)stream);
}

int mcf_spmv_peer(mcf_graph *g, double alpha, const double *v, double beta, const double *r,
                  const double *const *x_parts, const int64_t *part_bounds, int n_parts, double *const *y_outs,
                  int n_outs, int64_t row_begin, int64_t row_end, void *stream) {
    return mcf::spmv_peer(g, alpha, v, beta, r, x_parts, (const long long *)part_bounds, n_parts, y_outs, n_outs,
                          (long long)row_begin, (long long)row_end, (cudaStream_t)stream);
}

int mcf_spmv(mcf_graph *g, double alpha, const double *v, double beta, const double *r, const double *x, double *y,
             int64_t row_begin, int64_t row_end, void *stream) {
    return mcf::spmv(g, alpha, v, beta, r, x, y, row_begin, row_end, (cudaStream_t)stream);
}

int mcf_walk_action(mcf_graph *g, const mcf_walk_params *p, const int64_t *walk_pre, int64_t col_begin,
                    int64_t col_end, const double *r, double *q, double *q_var, int64_t *stats, void *stream) {
    return mcf::action(g, p, (const long long *)walk_pre, col_begin, col_end, nullptr, nullptr, r, q, q_var,
                       (long long *)stats, (cudaStream_t)stream, false);
}

int mcf_replay_action(mcf_graph *g, const mcf_walk_params *p, const int64_t *walk_pre, int64_t col_begin,
                      int64_t col_end, const int64_t *walk_off, const int32_t *entries, const double *r, double *q,
                      int64_t *stats, void *stream) {
    return mcf::action(g, p, (const long long *)walk_pre, col_begin, col_end, (const long long *)walk_off, entries,
                       r, q, nullptr, (long long *)stats, (cudaStream_t)stream, true);
}

}  // extern "C"
