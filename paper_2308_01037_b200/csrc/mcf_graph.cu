// Graph ingest: device transition tables (replaces walker.build_transition_model,
// /root/reference/pkg/src/mcfunm/walker.py:97-145).
//
// Layout in HBM (all owned by the handle except the caller's CSR/CSC arrays):
//   hdr[n]      32 B per node {row start, degree, flags, row |a| sum, aux}
//   ecol[nnz]   int32 column id with the value's sign in bit 31 (only when the
//               matrix holds negative values; otherwise aliases col_ids)
//   cdf[nnz]    within-row CDF of |a| (only when some row is not uniform)
//   col_norm[n], init_prob[n]  start distribution, bit-identical to the
//               reference (numpy pairwise summation order reproduced).
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "mcf_internal.cuh"

namespace mcf {

struct BuildCounters {
    unsigned long long n_uniform, n_empty, n_negative;
    unsigned long long max_degree;
    unsigned long long max_rsum_bits;  // rsum >= 0: IEEE bits order like the values
    unsigned long long n_long_rows, n_long_cols;
    unsigned long long min_abs_bits, max_abs_bits;  // over all stored |a| (uniform-value graphs)
};

constexpr int LONG_COL = 256;   // columns longer than this get a warp in k_colnorm_long
constexpr int LEAFCAP = 2048;   // leaves of the pairwise tree a warp keeps in smem

// Graph statistics: per-thread accumulators, reduced per warp, merged per CTA
// in shared memory, then one global atomic per CTA and counter (per-warp
// atomics on the same few words serialised the table build).
struct RowStats {
    unsigned long long uni = 0, emp = 0, neg = 0, maxdeg = 0, maxr = 0, minb = ~0ull, maxb = 0;
};

__device__ __forceinline__ void stats_init(unsigned long long *sh) {
    if (threadIdx.x < 7) sh[threadIdx.x] = threadIdx.x == 5 ? ~0ull : 0ull;
}

// every thread of the CTA calls it once, after stats_init + a barrier
__device__ __forceinline__ void stats_flush(RowStats r, unsigned long long *sh, BuildCounters *cnt) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        r.uni += __shfl_xor_sync(MCF_FULL, r.uni, o);
        r.emp += __shfl_xor_sync(MCF_FULL, r.emp, o);
        r.neg += __shfl_xor_sync(MCF_FULL, r.neg, o);
        unsigned long long a = __shfl_xor_sync(MCF_FULL, r.maxdeg, o), b = __shfl_xor_sync(MCF_FULL, r.maxr, o);
        r.maxdeg = a > r.maxdeg ? a : r.maxdeg;
        r.maxr = b > r.maxr ? b : r.maxr;
        a = __shfl_xor_sync(MCF_FULL, r.minb, o);
        b = __shfl_xor_sync(MCF_FULL, r.maxb, o);
        r.minb = a < r.minb ? a : r.minb;
        r.maxb = b > r.maxb ? b : r.maxb;
    }
    if ((threadIdx.x & 31) == 0) {
        if (r.uni) atomicAdd(&sh[0], r.uni);
        if (r.emp) atomicAdd(&sh[1], r.emp);
        if (r.neg) atomicAdd(&sh[2], r.neg);
        atomicMax(&sh[3], r.maxdeg);
        atomicMax(&sh[4], r.maxr);
        atomicMin(&sh[5], r.minb);
        atomicMax(&sh[6], r.maxb);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        if (sh[0]) atomicAdd(&cnt->n_uniform, sh[0]);
        if (sh[1]) atomicAdd(&cnt->n_empty, sh[1]);
        if (sh[2]) atomicAdd(&cnt->n_negative, sh[2]);
        if (sh[3]) atomicMax(&cnt->max_degree, sh[3]);
        if (sh[4]) atomicMax(&cnt->max_rsum_bits, sh[4]);
        if (sh[5] != ~0ull) atomicMin(&cnt->min_abs_bits, sh[5]);
        if (sh[6]) atomicMax(&cnt->max_abs_bits, sh[6]);
    }
}

__device__ __forceinline__ NodeHdr make_hdr(long long s, long long e, double acc, bool uniform, bool neg) {
    NodeHdr h;
    h.start = (int)s;
    h.deg = (int)(e - s);
    h.pad = 0;
    h.flags = (uniform ? HDR_UNIFORM : 0u) | (neg ? HDR_HAS_NEG : 0u);
    h.rsum = acc;
    h.aux = 0.0;
    return h;
}

// Rows (or columns) longer than `thr`, compacted (order irrelevant).
__global__ void k_mark_long(const long long *__restrict__ ptr, long long n, long long thr, int *__restrict__ out,
                            unsigned long long *count) {
    long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n && ptr[i + 1] - ptr[i] > thr) out[atomicAdd(count, 1ull)] = (int)i;
}

// One thread per row of degree <= LONG_ROW.  Row |a| sums are accumulated
// sequentially in CSR order, which is what np.add.at does for row_abs_sums
// (sparsemat.py:355-360), so the weight ratios a/t = copysign(rsum, a)
// (walker.py:124-125) match bit for bit.  Loads are batched 8 at a time.
__global__ void k_rows(const long long *__restrict__ row_ptr, const double *__restrict__ vals, long long n,
                       NodeHdr *__restrict__ hdr, BuildCounters *__restrict__ cnt) {
    __shared__ unsigned long long sh[7];
    stats_init(sh);
    __syncthreads();
    RowStats st;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const long long s = row_ptr[i], e = row_ptr[i + 1];
        if (e - s > LONG_ROW) continue;
        double acc = 0.0, mn = INFINITY, mx = 0.0;
        bool uniform = true;
        unsigned long long neg = 0;
        const double first = (e > s) ? fabs(vals[s]) : 0.0;
        for (long long j = s; j < e; j += 8) {
            double v[8];
#pragma unroll
            for (int t = 0; t < 8; ++t) v[t] = (j + t < e) ? vals[j + t] : 0.0;
#pragma unroll
            for (int t = 0; t < 8; ++t) {
                if (j + t < e) {
                    const double a = fabs(v[t]);
                    acc = __dadd_rn(acc, a);
                    uniform &= (a == first);
                    neg += (v[t] < 0.0);
                    mn = fmin(mn, a);
                    mx = fmax(mx, a);
                }
            }
        }
        hdr[i] = make_hdr(s, e, acc, uniform, neg != 0);
        if (e > s) {
            const unsigned long long lo = (unsigned long long)__double_as_longlong(mn);
            const unsigned long long hi = (unsigned long long)__double_as_longlong(mx);
            st.minb = lo < st.minb ? lo : st.minb;
            st.maxb = hi > st.maxb ? hi : st.maxb;
        }
        st.uni += (uniform && e > s);
        st.emp += (e == s);
        st.neg += neg;
        st.maxdeg = (unsigned long long)(e - s) > st.maxdeg ? (unsigned long long)(e - s) : st.maxdeg;
        const unsigned long long rb = (unsigned long long)__double_as_longlong(acc);
        st.maxr = rb > st.maxr ? rb : st.maxr;
    }
    stats_flush(st, sh, cnt);
}

// One warp per long row: 32 coalesced loads, then the sequential sum in CSR
// order through shuffles (same bits as the one-thread loop).
__global__ void k_rows_long(const int *__restrict__ rows, const unsigned long long *count,
                            const long long *__restrict__ row_ptr, const double *__restrict__ vals,
                            NodeHdr *__restrict__ hdr, BuildCounters *__restrict__ cnt) {
    __shared__ unsigned long long sh[7];
    __shared__ __align__(16) double stage[8][256];  // per warp: 256 values in CSR order
    stats_init(sh);
    __syncthreads();
    RowStats st;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    double *buf = stage[w];
    const long long nl = (long long)*count;
    const long long warps = ((long long)gridDim.x * blockDim.x) >> 5;
    for (long long li = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5; li < nl; li += warps) {
        const int i = rows[li];
        const long long s = row_ptr[i], e = row_ptr[i + 1];
        const double first = fabs(vals[s]);
        double acc = 0.0, mn = INFINITY, mx = 0.0;
        bool uniform = true;
        unsigned long long neg = 0;
        for (long long j = s; j < e; j += 256) {
            const int m = (int)(e - j < 256 ? e - j : 256);
#pragma unroll
            for (int t = 0; t < 8; ++t) {  // coalesced: 8 loads in flight per lane
                const int o = t * 32 + lane;
                const double v = o < m ? vals[j + o] : 0.0;
                const double a = fabs(v);
                uniform &= (o >= m || a == first);
                if (o < m) {
                    mn = fmin(mn, a);
                    mx = fmax(mx, a);
                    neg += (v < 0.0);
                }
                buf[o] = a;
            }
            __syncwarp();
            if (lane == 0) {  // the sequential CSR-order sum, from shared memory
                const double2 *b2 = reinterpret_cast<const double2 *>(buf);
                int t = 0;
                for (; t + 2 <= m; t += 2) {
                    const double2 x = b2[t >> 1];
                    acc = __dadd_rn(__dadd_rn(acc, x.x), x.y);
                }
                if (t < m) acc = __dadd_rn(acc, buf[t]);
            }
            __syncwarp();
        }
        uniform = __all_sync(MCF_FULL, uniform);
        neg = warp_sum_ll((long long)neg);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            mn = fmin(mn, __shfl_xor_sync(MCF_FULL, mn, o));
            mx = fmax(mx, __shfl_xor_sync(MCF_FULL, mx, o));
        }
        if (lane == 0) {
            hdr[i] = make_hdr(s, e, acc, uniform, neg != 0);
            const unsigned long long lo = (unsigned long long)__double_as_longlong(mn);
            const unsigned long long hi = (unsigned long long)__double_as_longlong(mx);
            st.minb = lo < st.minb ? lo : st.minb;
            st.maxb = hi > st.maxb ? hi : st.maxb;
            st.uni += uniform ? 1 : 0;
            st.neg += neg;
            st.maxdeg = (unsigned long long)(e - s) > st.maxdeg ? (unsigned long long)(e - s) : st.maxdeg;
            const unsigned long long rb = (unsigned long long)__double_as_longlong(acc);
            st.maxr = rb > st.maxr ? rb : st.maxr;
        }
    }
    stats_flush(st, sh, cnt);
}

// Fat walk entries: went[e] = hdr[col[e]], pad = col[e], sign of a_e in flags.
__global__ void k_build_went(const NodeHdr *__restrict__ hdr, const int *__restrict__ col_ids,
                             const double *__restrict__ vals, long long nnz, NodeHdr *__restrict__ went) {
    long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= nnz) return;
    const int c = col_ids[e];
    NodeHdr h = hdr[c];
    h.pad = (uint32_t)c;
    if (vals[e] < 0.0) h.flags |= HDR_NEG_EDGE;
    went[e] = h;
}

// Packed column ids with the sign of a in bit 31 (only built if some a < 0).
__global__ void k_ecol(const int *__restrict__ col_ids, const double *__restrict__ vals, long long nnz,
                       int *__restrict__ ecol) {
    long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e < nnz) ecol[e] = (int)((unsigned)col_ids[e] | (vals[e] < 0.0 ? 0x80000000u : 0u));
}

// Within-row CDF for non-uniform rows (inverse-CDF sampling, walker.py:183-189
// semantics: first entry whose CDF exceeds u).  Last entry pinned to 1.
__global__ void k_cdf(const NodeHdr *__restrict__ hdr, const double *__restrict__ vals, long long n,
                      double *__restrict__ cdf) {
    long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    NodeHdr h = hdr[i];
    if (h.deg == 0 || (h.flags & HDR_UNIFORM)) return;
    double run = 0.0;
    for (int t = 0; t < h.deg; ++t) {
        run = __dadd_rn(run, fabs(vals[h.start + t]));
        cdf[h.start + t] = fmin(__ddiv_rn(run, h.rsum), 1.0);
    }
    cdf[h.start + h.deg - 1] = 1.0;
}

// Vose's alias method per non-uniform row (one thread per row; scratch p and
// the two work stacks live at the row's own CSR range): p_t = |a_t| deg /
// rowsum, small (< 1) entries paired with large ones.  The draw (walk pick())
// takes slot k = floor(u deg) and keeps it when the fractional part of u deg
// is below threshold k, else its alias -- the within-row distribution of
// walker.py:112-125 (|a| / row sum), up to the 2^-tbits threshold quantum.
__global__ void k_alias(const NodeHdr *__restrict__ hdr, const double *__restrict__ vals, long long n, int tbits,
                        double *__restrict__ p, int *__restrict__ stk, unsigned long long *__restrict__ out) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const NodeHdr h = hdr[i];
    if (h.deg == 0 || (h.flags & HDR_UNIFORM)) return;
    const long long s0 = h.start;
    const int d = h.deg;
    double *pp = p + s0;
    int *st = stk + s0;
    const unsigned long long one = 1ull << tbits;
    int ns = 0, nl = 0;  // small stack grows from the front, large from the back
    for (int t = 0; t < d; ++t) {
        pp[t] = fabs(vals[s0 + t]) * (double)d / h.rsum;
        if (pp[t] < 1.0) st[ns++] = t;
        else st[d - 1 - nl++] = t;
    }
    while (ns > 0 && nl > 0) {
        const int sm = st[--ns];
        const int lg = st[d - nl];  // top of the large stack
        double th = pp[sm] * (double)one;
        unsigned long long q = th >= (double)one ? one - 1 : (unsigned long long)th;
        out[s0 + sm] = ((unsigned long long)lg << tbits) | q;
        pp[lg] = (pp[lg] + pp[sm]) - 1.0;
        if (pp[lg] < 1.0) {  // the large entry became small: move it
            --nl;
            st[ns++] = lg;
        }
    }
    for (int k = 0; k < ns; ++k) out[s0 + st[k]] = ((unsigned long long)st[k] << tbits) | (one - 1);
    for (int k = 0; k < nl; ++k) out[s0 + st[d - 1 - k]] = ((unsigned long long)st[d - 1 - k] << tbits) | (one - 1);
}

// numpy's pairwise summation (numpy/_core/src/umath/loops_utils.h.src,
// pairwise_sum): < 8 terms sequential from 0; <= 128 terms eight strided
// accumulators combined as ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) then the tail;
// otherwise split at n/2 rounded down to a multiple of 8 and recurse.
template <bool SQUARE>
__device__ __forceinline__ double term(const double *a, long long i) {
    double v = a[i];
    return SQUARE ? __dmul_rn(v, v) : v;
}

template <bool SQUARE>
__device__ double pw_block(const double *a, long long n) {
    if (n < 8) {
        double r = 0.0;
        for (long long i = 0; i < n; ++i) r = __dadd_rn(r, term<SQUARE>(a, i));
        return r;
    }
    double r[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = term<SQUARE>(a, j);
    long long i = 8;
    for (; i < n - (n % 8); i += 8) {
#pragma unroll
        for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], term<SQUARE>(a, i + j));
    }
    double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                           __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
    for (; i < n; ++i) res = __dadd_rn(res, term<SQUARE>(a, i));
    return res;
}

// The recursion of pairwise_sum evaluated with an explicit stack (no device
// recursion): frame state 0 = descend left, 1 = left done -> descend right,
// 2 = both done -> combine and pop.  `ret` carries the value of the child that
// just finished.  leaf(k, off, len) supplies the value of the k-th leaf
// (<= 128 terms) in recursion order.
template <class LeafFn>
__device__ double pw_eval(long long n, LeafFn leaf) {
    if (n <= 128) return leaf(0, 0ll, n);
    long long off[28], len[28];  // depth <= 25 for n < 2^31
    double left[28];
    unsigned char st[28];
    int sp = 0, k = 0;
    off[0] = 0;
    len[0] = n;
    st[0] = 0;
    double ret = 0.0;
    while (sp >= 0) {
        const long long L = len[sp];
        if (L <= 128) {
            ret = leaf(k++, off[sp], L);
            --sp;
            continue;
        }
        long long n2 = L / 2;
        n2 -= n2 % 8;
        if (st[sp] == 0) {
            st[sp] = 1;
            off[sp + 1] = off[sp];
            len[sp + 1] = n2;
            st[sp + 1] = 0;
            ++sp;
        } else if (st[sp] == 1) {
            left[sp] = ret;
            st[sp] = 2;
            off[sp + 1] = off[sp] + n2;
            len[sp + 1] = L - n2;
            st[sp + 1] = 0;
            ++sp;
        } else {
            ret = __dadd_rn(left[sp], ret);
            --sp;
        }
    }
    return ret;
}

template <bool SQUARE>
__device__ double pw_sum(const double *a, long long n) {
    return pw_eval(n, [&](int, long long off, long long len) { return pw_block<SQUARE>(a + off, len); });
}

__device__ long long pw_leaf_count(long long n) {
    long long c = 0;
    pw_eval(n, [&](int, long long, long long) { ++c; return 0.0; });
    return c;
}

// ||C_j||_2 exactly as scipy computes csc.multiply(csc).sum(axis=0) then sqrt
// (walker.py:127): np.add.reduceat over the column = first + pairwise(rest).
__global__ void k_colnorm(const long long *__restrict__ csc_ptr, const double *__restrict__ csc_vals, long long n,
                          double *__restrict__ col_norm) {
    long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    long long s = csc_ptr[j], e = csc_ptr[j + 1];
    if (e - s > LONG_COL) return;  // k_colnorm_long
    double sq = 0.0;
    if (e > s) {
        sq = __dmul_rn(csc_vals[s], csc_vals[s]);
        const long long m = e - s - 1;
        const double *a = csc_vals + s + 1;
        if (m > 128) {  // pairwise_sum for m < LONG_COL = 256: left <= 127, right <= 135 (maybe split once more)
            long long n2 = m / 2;
            n2 -= n2 % 8;
            const long long r = m - n2;
            double right;
            if (r <= 128) {
                right = pw_block<true>(a + n2, r);
            } else {
                long long n3 = r / 2;
                n3 -= n3 % 8;
                right = __dadd_rn(pw_block<true>(a + n2, n3), pw_block<true>(a + n2 + n3, r - n3));
            }
            sq = __dadd_rn(sq, __dadd_rn(pw_block<true>(a, n2), right));
        } else if (m > 0) {
            sq = __dadd_rn(sq, pw_block<true>(a, m));
        }
    }
    col_norm[j] = __dsqrt_rn(sq);
}

// One warp (one CTA) per long column.  Lane 0 enumerates the leaves of the
// pairwise tree once (offsets into shared memory); rounds of 32 consecutive
// leaves -- one contiguous value range -- are staged into shared memory with
// coalesced loads and summed one leaf per lane; lane 0 combines the leaf sums
// in the recursion order -> the same bits as the sequential evaluation.
constexpr int LEAFCAP_L = 1024;  // leaves held per column (columns up to ~131k entries; beyond: lane 0 alone)

__global__ void __launch_bounds__(32) k_colnorm_long(const int *__restrict__ cols, const unsigned long long *count,
                                                     const long long *__restrict__ csc_ptr,
                                                     const double *__restrict__ csc_vals, double *__restrict__ col_norm) {
    __shared__ __align__(16) double stage[32 * 128];
    __shared__ double buf[LEAFCAP_L];
    __shared__ int lofs[LEAFCAP_L + 1];
    const int lane = threadIdx.x;
    const long long nl = (long long)*count;
    for (long long li = blockIdx.x; li < nl; li += gridDim.x) {
        const int j = cols[li];
        const long long s = csc_ptr[j], e = csc_ptr[j + 1];
        const double *a = csc_vals + s + 1;
        const long long m = e - s - 1;
        int nleaf = 0;
        if (lane == 0) {
            pw_eval(m, [&](int k, long long off, long long) {
                if (k < LEAFCAP_L) lofs[k] = (int)off;
                nleaf = k + 1;
                return 0.0;
            });
            if (nleaf <= LEAFCAP_L) lofs[nleaf] = (int)m;
        }
        nleaf = __shfl_sync(MCF_FULL, nleaf, 0);
        __syncwarp();
        double tail = 0.0;
        if (nleaf > LEAFCAP_L) {
            if (lane == 0) tail = pw_sum<true>(a, m);
        } else {
            for (int r0 = 0; r0 < nleaf; r0 += 32) {
                const int r1 = r0 + 32 < nleaf ? r0 + 32 : nleaf;
                const int lo = lofs[r0], hi = lofs[r1];
                for (int o = lane; o < hi - lo; o += 32) stage[o] = a[lo + o];
                __syncwarp();
                if (r0 + lane < r1) {
                    const int k = r0 + lane;
                    buf[k] = pw_block<true>(stage + (lofs[k] - lo), lofs[k + 1] - lofs[k]);
                }
                __syncwarp();
            }
            if (lane == 0) tail = pw_eval(m, [&](int k, long long, long long) { return buf[k]; });
        }
        if (lane == 0) col_norm[j] = __dsqrt_rn(__dadd_rn(__dmul_rn(csc_vals[s], csc_vals[s]), tail));
        __syncwarp();
    }
}

__global__ void k_leaf_sums(const double *__restrict__ a, const long long *__restrict__ leaf_off,
                            const int *__restrict__ leaf_len, int nleaf, double *__restrict__ out) {
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t < nleaf) out[t] = pw_block<false>(a + leaf_off[t], leaf_len[t]);
}

__global__ void k_divide(const double *__restrict__ a, double denom, long long n, double *__restrict__ out) {
    long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (j < n) out[j] = __ddiv_rn(a[j], denom);
}

// host side of np.sum(x) for a device vector: enumerate the recursion leaves,
// sum them on the device, combine in the same tree on the host.
static void pw_leaves(long long off, long long n, std::vector<long long> &lo, std::vector<int> &ln) {
    if (n <= 128) {
        lo.push_back(off);
        ln.push_back((int)n);
        return;
    }
    long long n2 = n / 2;
    n2 -= n2 % 8;
    pw_leaves(off, n2, lo, ln);
    pw_leaves(off + n2, n - n2, lo, ln);
}

static double pw_combine(long long n, const double *leaf, size_t &k) {
    if (n <= 128) return leaf[k++];
    long long n2 = n / 2;
    n2 -= n2 % 8;
    double a = pw_combine(n2, leaf, k);
    double b = pw_combine(n - n2, leaf, k);
    return a + b;
}

static void release(mcf_graph *g) {
    if (!g) return;
    cudaDeviceSynchronize();
    if (g->hdr) cudaFreeAsync(g->hdr, 0);
    if (g->ecol_owned) cudaFreeAsync(g->ecol, 0);
    if (g->cdf) cudaFreeAsync(g->cdf, 0);
    if (g->alias) cudaFreeAsync(g->alias, 0);
    if (g->col_norm) cudaFreeAsync(g->col_norm, 0);
    if (g->csr2csc) cudaFreeAsync(g->csr2csc, 0);
    if (g->long_rows) cudaFreeAsync(g->long_rows, 0);
    if (g->went) cudaFreeAsync(g->went, 0);
    if (g->lean) cudaFreeAsync(g->lean, 0);
    if (g->lean4) cudaFreeAsync(g->lean4, 0);
    if (g->lean_id) cudaFreeAsync(g->lean_id, 0);
    if (g->rsum_by_deg) cudaFreeAsync(g->rsum_by_deg, 0);
    if (g->hub_of) cudaFreeAsync(g->hub_of, 0);
    if (g->hub_bits) cudaFreeAsync(g->hub_bits, 0);
    if (g->ckeys) cudaFreeAsync(g->ckeys, 0);
    if (g->gidx) cudaFreeAsync(g->gidx, 0);
    if (g->gofs) cudaFreeAsync(g->gofs, 0);
    if (g->scratch) cudaFreeAsync(g->scratch, 0);
    // g->side is the per-device stream shared by all graphs: not destroyed here
    if (g->ev_fork) cudaEventDestroy(g->ev_fork);
    if (g->ev_join) cudaEventDestroy(g->ev_join);
    for (auto &p : g->ev_walk) { cudaEventDestroy(p.first); cudaEventDestroy(p.second); }
    for (auto &p : g->ev_q) { cudaEventDestroy(p.first); cudaEventDestroy(p.second); }
    delete g;
}

// keep freed stream-ordered memory in the pool (graph handles come and go)
static void tune_pool() {
    static bool done = false;
    if (done) return;
    int dev = 0;
    cudaGetDevice(&dev);
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t thr = ~0ull;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    done = true;
}

// Device tables in one pass with a single host synchronisation (counters +
// the leaves of sum_j ||C_j|| come back together; the host finishes numpy's
// pairwise tree over the leaves and the rest is launched asynchronously).
static int create(const mcf_csr *c, cudaStream_t s, mcf_graph **out) {
    MCF_ARG(c && out, "mcf_graph_create: null argument");
    MCF_ARG(c->n > 0, "matrix dimension must be positive");
    MCF_ARG(c->n < (1ll << 31) && c->nnz < (1ll << 31), "n and nnz must be below 2^31");
    if (c->nnz == 0) {
        set_error("all columns are zero: the initial distribution is undefined");
        return MCF_ERR_DEGENERATE;  // walker.py:100-103
    }
    MCF_ARG(c->row_ptr && c->col_ids && c->vals && c->csc_ptr && c->csc_rows && c->csc_vals,
            "mcf_graph_create: null CSR/CSC array");
    tune_pool();
    mcf_graph *g = new mcf_graph();
    g->n = c->n;
    g->nnz = c->nnz;
    g->row_ptr = c->row_ptr;
    g->col_ids = c->col_ids;
    g->vals = c->vals;
    g->csc_ptr = c->csc_ptr;
    g->csc_rows = c->csc_rows;
    g->csc_vals = c->csc_vals;
    cudaGetDevice(&g->device);
    const long long n = g->n;
    auto fail = [&](int code) {
        release(g);
        return code;
    };
    cudaError_t e;
    // leaves of the pairwise tree over the n column norms (host-enumerated)
    std::vector<long long> lo;
    std::vector<int> ln;
    pw_leaves(0, n, lo, ln);
    const int nl = (int)lo.size();
    // one scratch block: counters | long-col list | leaf offsets | leaf lengths | leaf sums
    size_t sz = sizeof(BuildCounters) + sizeof(int) * n + sizeof(long long) * nl + sizeof(int) * nl +
                sizeof(double) * nl + 64;
    char *scr = nullptr;
    if ((e = cudaMallocAsync(&g->hdr, sizeof(NodeHdr) * n, s)) != cudaSuccess) return fail(cuda_status(e, "hdr"));
    if ((e = cudaMallocAsync(&g->col_norm, sizeof(double) * 2 * n, s)) != cudaSuccess)
        return fail(cuda_status(e, "col_norm"));
    g->init_prob = g->col_norm + n;
    const long long n_even = (n + 1) & ~1ll;  // 8-byte aligned counter after the list
    if ((e = cudaMallocAsync(&g->long_rows, sizeof(int) * n_even + sizeof(unsigned long long), s)) != cudaSuccess)
        return fail(cuda_status(e, "long_rows"));
    if ((e = cudaMallocAsync(&scr, sz, s)) != cudaSuccess) return fail(cuda_status(e, "scratch"));
    BuildCounters *cnt = reinterpret_cast<BuildCounters *>(scr);
    int *long_cols = reinterpret_cast<int *>(scr + sizeof(BuildCounters));
    long long *d_lo = reinterpret_cast<long long *>(((uintptr_t)(long_cols + n) + 15) & ~(uintptr_t)15);
    int *d_ln = reinterpret_cast<int *>(d_lo + nl);
    double *d_leaf = reinterpret_cast<double *>(((uintptr_t)(d_ln + nl) + 15) & ~(uintptr_t)15);
    unsigned long long *lr_count = reinterpret_cast<unsigned long long *>(g->long_rows + n_even);
    cudaMemsetAsync(cnt, 0, sizeof(BuildCounters), s);
    cudaMemsetAsync(&cnt->min_abs_bits, 0xff, sizeof(unsigned long long), s);
    cudaMemsetAsync(lr_count, 0, sizeof(unsigned long long), s);
    cudaMemcpyAsync(d_lo, lo.data(), sizeof(long long) * nl, cudaMemcpyHostToDevice, s);
    cudaMemcpyAsync(d_ln, ln.data(), sizeof(int) * nl, cudaMemcpyHostToDevice, s);
    const unsigned nb = (unsigned)((n + 255) / 256);
    const int wgrid = sm_count() * 8;
    const long long *rp = (const long long *)g->row_ptr, *cp = (const long long *)g->csc_ptr;
    k_mark_long<<<nb, 256, 0, s>>>(rp, n, LONG_ROW, g->long_rows, lr_count);
    mcf::note_launch();
    k_mark_long<<<nb, 256, 0, s>>>(cp, n, LONG_COL, long_cols, &cnt->n_long_cols);
    mcf::note_launch();
    k_rows<<<(unsigned)(nb < (unsigned)wgrid ? nb : (unsigned)wgrid), 256, 0, s>>>(rp, g->vals, n, g->hdr, cnt);
    mcf::note_launch();
    k_rows_long<<<wgrid, 256, 0, s>>>(g->long_rows, lr_count, rp, g->vals, g->hdr, cnt);
    mcf::note_launch();
    k_colnorm<<<nb, 256, 0, s>>>(cp, g->csc_vals, n, g->col_norm);
    mcf::note_launch();
    k_colnorm_long<<<wgrid * 2, 32, 0, s>>>(long_cols, &cnt->n_long_cols, cp, g->csc_vals, g->col_norm);
    mcf::note_launch();
    k_leaf_sums<<<(nl + 255) / 256, 256, 0, s>>>(g->col_norm, d_lo, d_ln, nl, d_leaf);
    mcf::note_launch();
    if ((e = cudaGetLastError()) != cudaSuccess) return fail(cuda_status(e, "graph build kernels"));
    BuildCounters hc;
    std::vector<double> leaf(nl);
    cudaMemcpyAsync(&hc, cnt, sizeof(hc), cudaMemcpyDeviceToHost, s);
    cudaMemcpyAsync(&g->n_long_rows, lr_count, sizeof(long long), cudaMemcpyDeviceToHost, s);
    cudaMemcpyAsync(leaf.data(), d_leaf, sizeof(double) * nl, cudaMemcpyDeviceToHost, s);
    if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return fail(cuda_status(e, "graph build"));
    size_t k = 0;
    const double total = pw_combine(n, leaf.data(), k);  // np.sum(col_norms) (walker.py:128)
    g->info.n = n;
    g->info.nnz = g->nnz;
    g->info.n_uniform_rows = (int64_t)hc.n_uniform;
    g->info.n_empty_rows = (int64_t)hc.n_empty;
    g->info.n_negative = (int64_t)hc.n_negative;
    g->info.max_degree = (int64_t)hc.max_degree;
    memcpy(&g->info.max_row_abs_sum, &hc.max_rsum_bits, sizeof(double));
    g->info.col_norm_total = total;
    if (hc.n_negative == 0 && hc.min_abs_bits == hc.max_abs_bits) {  // every stored value equal
        g->uniform_value = true;
        memcpy(&g->value, &hc.min_abs_bits, sizeof(double));
    }
    if (hc.n_negative) {
        if ((e = cudaMallocAsync(&g->ecol, sizeof(int) * g->nnz, s)) != cudaSuccess) return fail(cuda_status(e, "ecol"));
        g->ecol_owned = true;
        k_ecol<<<(unsigned)((g->nnz + 255) / 256), 256, 0, s>>>(g->col_ids, g->vals, g->nnz, g->ecol);
        mcf::note_launch();
    } else {
        g->ecol = const_cast<int32_t *>(g->col_ids);
    }
    if (hc.n_uniform + hc.n_empty < (unsigned long long)n) {
        if ((e = cudaMallocAsync(&g->cdf, sizeof(double) * g->nnz, s)) != cudaSuccess) return fail(cuda_status(e, "cdf"));
        k_cdf<<<nb, 256, 0, s>>>(g->hdr, g->vals, n, g->cdf);
        mcf::note_launch();
        const char *aenv = getenv("MCF_ALIAS");  // "0": inverse-CDF search for device-RNG draws
        if (!(aenv && !strcmp(aenv, "0"))) {
            int dbits = 1;
            while (dbits < 40 && (1ll << dbits) <= g->info.max_degree) ++dbits;
            const int tbits = 64 - dbits;  // >= 24 even for degree ~2^40
            double *p = nullptr;
            int *stk = nullptr;
            if ((e = cudaMallocAsync(&g->alias, sizeof(unsigned long long) * g->nnz, s)) != cudaSuccess)
                return fail(cuda_status(e, "alias"));
            if ((e = cudaMallocAsync(&p, sizeof(double) * g->nnz, s)) != cudaSuccess) return fail(cuda_status(e, "alias p"));
            if ((e = cudaMallocAsync(&stk, sizeof(int) * g->nnz, s)) != cudaSuccess) {
                cudaFreeAsync(p, s);
                return fail(cuda_status(e, "alias stack"));
            }
            k_alias<<<nb, 256, 0, s>>>(g->hdr, g->vals, n, tbits, p, stk, g->alias);
            mcf::note_launch();
            cudaFreeAsync(p, s);
            cudaFreeAsync(stk, s);
            g->alias_tbits = tbits;
        }
    }
    // walk layout: fat entries when the compact tables (32 n + 4 nnz bytes)
    // would not stay resident in L2 (MCF_WALK_LAYOUT=fat|compact overrides)
    {
        int l2 = 0;
        cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, g->device);
        const double compact_bytes = 32.0 * n + 4.0 * g->nnz;
        bool fat = compact_bytes > 0.75 * (double)l2;
        const char *env = getenv("MCF_WALK_LAYOUT");
        if (env && !strcmp(env, "fat")) fat = true;
        if (env && !strcmp(env, "compact")) fat = false;
        if (fat && cudaMallocAsync(&g->went, sizeof(NodeHdr) * g->nnz, s) == cudaSuccess) {
            k_build_went<<<(unsigned)((g->nnz + 255) / 256), 256, 0, s>>>(g->hdr, g->col_ids, g->vals, g->nnz,
                                                                          g->went);
            mcf::note_launch();
        } else {
            cudaGetLastError();  // no room for 32 B x nnz: stay compact
            g->went = nullptr;
        }
        g->info.walk_layout = g->went ? 1 : 0;
        // L2-resident compact tables: the walk kernels stream them into L2
        // with TMA bulk prefetches before walking (sequential HBM reads instead
        // of one random sector fetch per first touch; MCF_L2_PREFETCH=0 off)
        const double walk_bytes = compact_bytes + (g->cdf ? 8.0 * g->nnz : 0.0);
        const char *pf = getenv("MCF_L2_PREFETCH");
        g->l2_prefetch = !g->went && walk_bytes <= 0.6 * (double)l2 && !(pf && !strcmp(pf, "0"));
    }
    k_divide<<<nb, 256, 0, s>>>(g->col_norm, total, n, g->init_prob);  // p_j (walker.py:129)
    mcf::note_launch();
    cudaFreeAsync(scr, s);
    if ((e = cudaGetLastError()) != cudaSuccess) return fail(cuda_status(e, "graph build tail"));
    *out = g;
    return MCF_OK;
}

}  // namespace mcf

extern "C" {

int mcf_graph_create(const mcf_csr *csr, void *stream, mcf_graph **out) {
    // MCF_L2_FETCH=<bytes>: the L2 fetch-granularity hint (cudaLimitMaxL2FetchGranularity)
    // for this process's device -- the walks' random 8-B entry loads want 32-B fills
    if (const char *e = getenv("MCF_L2_FETCH")) {
        if (cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, (size_t)atoll(e)) != cudaSuccess) cudaGetLastError();
    }
    return mcf::create(csr, (cudaStream_t)stream, out);
}

int mcf_graph_destroy(mcf_graph *g) {
    mcf::release(g);
    return MCF_OK;
}

int mcf_graph_get_info(const mcf_graph *g, mcf_graph_info *info) {
    MCF_ARG(g && info, "mcf_graph_get_info: null argument");
    *info = g->info;
    return MCF_OK;
}

int mcf_graph_tables(const mcf_graph *g, double *row_abs_sum, double *col_norms, double *init_prob,
                     void *stream) {
    MCF_ARG(g, "mcf_graph_tables: null graph");
    cudaStream_t s = (cudaStream_t)stream;
    if (row_abs_sum)  // strided copy of hdr[i].rsum
        MCF_CUDA(cudaMemcpy2DAsync(row_abs_sum, sizeof(double), &g->hdr[0].rsum, sizeof(mcf::NodeHdr),
                                   sizeof(double), g->n, cudaMemcpyDeviceToDevice, s));
    if (col_norms)
        MCF_CUDA(cudaMemcpyAsync(col_norms, g->col_norm, sizeof(double) * g->n, cudaMemcpyDeviceToDevice, s));
    if (init_prob)
        MCF_CUDA(cudaMemcpyAsync(init_prob, g->init_prob, sizeof(double) * g->n, cudaMemcpyDeviceToDevice, s));
    return MCF_OK;
}

}  // extern "C"
