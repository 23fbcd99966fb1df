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
#include <cstring>
#include <vector>

#include "mcf_internal.cuh"

namespace mcf {

struct BuildCounters {
    unsigned long long n_uniform, n_empty, n_negative;
    unsigned long long max_degree;
    unsigned long long max_rsum_bits;  // rsum >= 0: IEEE bits order like the values
};

// One thread per row.  Row |a| sums are accumulated sequentially in CSR order,
// which is what np.add.at does for row_abs_sums (sparsemat.py:355-360), so the
// weight ratios a/t = copysign(rsum, a) (walker.py:124-125) match bit for bit.
__global__ void k_rows(const long long *__restrict__ row_ptr, const double *__restrict__ vals, long long n,
                       NodeHdr *__restrict__ hdr, BuildCounters *__restrict__ cnt) {
    long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    unsigned long long uni = 0, emp = 0, neg = 0, maxdeg = 0, maxr = 0;
    if (i < n) {
        long long s = row_ptr[i], e = row_ptr[i + 1];
        double acc = 0.0;
        bool uniform = true;
        double first = (e > s) ? fabs(vals[s]) : 0.0;
        for (long long j = s; j < e; ++j) {
            double v = vals[j];
            double a = fabs(v);
            acc = __dadd_rn(acc, a);
            uniform &= (a == first);
            neg += (v < 0.0);
        }
        uint32_t flags = 0;
        if (uniform) flags |= HDR_UNIFORM;
        if (neg) flags |= HDR_HAS_NEG;
        NodeHdr h;
        h.start = s;
        h.deg = (int)(e - s);
        h.flags = flags;
        h.rsum = acc;
        h.aux = 0.0;
        hdr[i] = h;
        uni = (uniform && e > s);
        emp = (e == s);
        maxdeg = (unsigned long long)(e - s);
        maxr = (unsigned long long)__double_as_longlong(acc);
    }
    // block-aggregate then one atomic per warp
    uni = warp_sum_ll((long long)uni);
    emp = warp_sum_ll((long long)emp);
    neg = warp_sum_ll((long long)neg);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        unsigned long long a = __shfl_xor_sync(MCF_FULL, maxdeg, o);
        unsigned long long b = __shfl_xor_sync(MCF_FULL, maxr, o);
        maxdeg = a > maxdeg ? a : maxdeg;
        maxr = b > maxr ? b : maxr;
    }
    if ((threadIdx.x & 31) == 0) {
        if (uni) atomicAdd(&cnt->n_uniform, uni);
        if (emp) atomicAdd(&cnt->n_empty, emp);
        if (neg) atomicAdd(&cnt->n_negative, neg);
        atomicMax(&cnt->max_degree, maxdeg);
        atomicMax(&cnt->max_rsum_bits, maxr);
    }
}

// Rows longer than LONG_ROW, compacted (order irrelevant: each is reduced alone).
__global__ void k_long_rows(const long long *__restrict__ row_ptr, long long n, int *__restrict__ out,
                            unsigned long long *count) {
    long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n && row_ptr[i + 1] - row_ptr[i] > LONG_ROW) out[atomicAdd(count, 1ull)] = (int)i;
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

// The recursion of pairwise_sum evaluated with an explicit stack (device
// recursion is avoided): frame state 0 = descend left, 1 = left done -> descend
// right, 2 = both done -> combine and pop.  `ret` carries the value of the
// child that just finished.
template <bool SQUARE>
__device__ double pw_sum(const double *a, long long n) {
    if (n <= 128) return pw_block<SQUARE>(a, n);
    long long off[28], len[28];  // depth <= 25 for n < 2^31
    double left[28];
    unsigned char st[28];
    int sp = 0;
    off[0] = 0;
    len[0] = n;
    st[0] = 0;
    double ret = 0.0;
    while (sp >= 0) {
        const long long L = len[sp];
        if (L <= 128) {
            ret = pw_block<SQUARE>(a + off[sp], L);
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

// ||C_j||_2 exactly as scipy computes csc.multiply(csc).sum(axis=0) then sqrt
// (walker.py:127): np.add.reduceat over the column = first + pairwise(rest).
__global__ void k_colnorm(const long long *__restrict__ csc_ptr, const double *__restrict__ csc_vals, long long n,
                          double *__restrict__ col_norm) {
    long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    long long s = csc_ptr[j], e = csc_ptr[j + 1];
    double sq = 0.0;
    if (e > s) {
        sq = __dmul_rn(csc_vals[s], csc_vals[s]);
        if (e - s > 1) sq = __dadd_rn(sq, pw_sum<true>(csc_vals + s + 1, e - s - 1));
    }
    col_norm[j] = __dsqrt_rn(sq);
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

static int numpy_sum(const double *dev, long long n, cudaStream_t s, double *out) {
    std::vector<long long> lo;
    std::vector<int> ln;
    pw_leaves(0, n, lo, ln);
    int nl = (int)lo.size();
    long long *d_lo = nullptr;
    int *d_ln = nullptr;
    double *d_sum = nullptr;
    MCF_CUDA(cudaMallocAsync(&d_lo, sizeof(long long) * nl, s));
    MCF_CUDA(cudaMallocAsync(&d_ln, sizeof(int) * nl, s));
    MCF_CUDA(cudaMallocAsync(&d_sum, sizeof(double) * nl, s));
    MCF_CUDA(cudaMemcpyAsync(d_lo, lo.data(), sizeof(long long) * nl, cudaMemcpyHostToDevice, s));
    MCF_CUDA(cudaMemcpyAsync(d_ln, ln.data(), sizeof(int) * nl, cudaMemcpyHostToDevice, s));
    k_leaf_sums<<<(nl + 255) / 256, 256, 0, s>>>(dev, d_lo, d_ln, nl, d_sum);
    mcf::note_launch();
    MCF_LAUNCHED("k_leaf_sums");
    std::vector<double> h(nl);
    MCF_CUDA(cudaMemcpyAsync(h.data(), d_sum, sizeof(double) * nl, cudaMemcpyDeviceToHost, s));
    MCF_CUDA(cudaStreamSynchronize(s));
    size_t k = 0;
    *out = pw_combine(n, h.data(), k);
    cudaFreeAsync(d_lo, s);
    cudaFreeAsync(d_ln, s);
    cudaFreeAsync(d_sum, s);
    return MCF_OK;
}

static void release(mcf_graph *g) {
    if (!g) return;
    cudaFree(g->hdr);
    if (g->ecol_owned) cudaFree(g->ecol);
    cudaFree(g->cdf);
    cudaFree(g->col_norm);
    cudaFree(g->init_prob);
    cudaFree(g->csr2csc);
    cudaFree(g->long_rows);
    delete g;
}

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
    int rc = MCF_OK;
    auto fail = [&](int code) {
        release(g);
        return code;
    };
    BuildCounters *cnt = nullptr;
    cudaError_t e;
    if ((e = cudaMalloc(&g->hdr, sizeof(NodeHdr) * g->n)) != cudaSuccess) return fail(cuda_status(e, "hdr"));
    if ((e = cudaMalloc(&g->col_norm, sizeof(double) * g->n)) != cudaSuccess) return fail(cuda_status(e, "col_norm"));
    if ((e = cudaMalloc(&g->init_prob, sizeof(double) * g->n)) != cudaSuccess) return fail(cuda_status(e, "init_prob"));
    if ((e = cudaMallocAsync(&cnt, sizeof(BuildCounters), s)) != cudaSuccess) return fail(cuda_status(e, "counters"));
    cudaMemsetAsync(cnt, 0, sizeof(BuildCounters), s);
    unsigned nb = (unsigned)((g->n + 255) / 256);
    k_rows<<<nb, 256, 0, s>>>((const long long *)g->row_ptr, g->vals, g->n, g->hdr, cnt);
    mcf::note_launch();
    k_colnorm<<<nb, 256, 0, s>>>((const long long *)g->csc_ptr, g->csc_vals, g->n, g->col_norm);
    mcf::note_launch();
    if ((e = cudaGetLastError()) != cudaSuccess) return fail(cuda_status(e, "k_rows/k_colnorm"));
    BuildCounters hc;
    cudaMemcpyAsync(&hc, cnt, sizeof(hc), cudaMemcpyDeviceToHost, s);
    if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return fail(cuda_status(e, "graph build"));
    cudaFreeAsync(cnt, s);
    g->info.n = g->n;
    g->info.nnz = g->nnz;
    g->info.n_uniform_rows = (int64_t)hc.n_uniform;
    g->info.n_empty_rows = (int64_t)hc.n_empty;
    g->info.n_negative = (int64_t)hc.n_negative;
    g->info.max_degree = (int64_t)hc.max_degree;
    memcpy(&g->info.max_row_abs_sum, &hc.max_rsum_bits, sizeof(double));
    if (hc.max_degree > (unsigned long long)LONG_ROW) {  // hub rows get their own SpMV bin
        unsigned long long *lc = nullptr, nl = 0;
        if ((e = cudaMalloc(&lc, sizeof(unsigned long long))) != cudaSuccess) return fail(cuda_status(e, "long"));
        cudaMemsetAsync(lc, 0, sizeof(unsigned long long), s);
        int *tmp = nullptr;
        if ((e = cudaMalloc(&tmp, sizeof(int) * g->n)) != cudaSuccess) return fail(cuda_status(e, "long rows"));
        k_long_rows<<<nb, 256, 0, s>>>((const long long *)g->row_ptr, g->n, tmp, lc);
        mcf::note_launch();
        cudaMemcpyAsync(&nl, lc, sizeof(nl), cudaMemcpyDeviceToHost, s);
        if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return fail(cuda_status(e, "long rows"));
        g->n_long_rows = (long long)nl;
        if ((e = cudaMalloc(&g->long_rows, sizeof(int) * (nl ? nl : 1))) != cudaSuccess)
            return fail(cuda_status(e, "long rows"));
        cudaMemcpyAsync(g->long_rows, tmp, sizeof(int) * nl, cudaMemcpyDeviceToDevice, s);
        cudaStreamSynchronize(s);
        cudaFree(tmp);
        cudaFree(lc);
    }
    if (hc.n_negative) {
        if ((e = cudaMalloc(&g->ecol, sizeof(int) * g->nnz)) != cudaSuccess) return fail(cuda_status(e, "ecol"));
        g->ecol_owned = true;
        k_ecol<<<(unsigned)((g->nnz + 255) / 256), 256, 0, s>>>(g->col_ids, g->vals, g->nnz, g->ecol);
        mcf::note_launch();
    } else {
        g->ecol = const_cast<int32_t *>(g->col_ids);
    }
    if (hc.n_uniform + hc.n_empty < (unsigned long long)g->n) {
        if ((e = cudaMalloc(&g->cdf, sizeof(double) * g->nnz)) != cudaSuccess) return fail(cuda_status(e, "cdf"));
        k_cdf<<<nb, 256, 0, s>>>(g->hdr, g->vals, g->n, g->cdf);
        mcf::note_launch();
    }
    if ((e = cudaGetLastError()) != cudaSuccess) return fail(cuda_status(e, "k_ecol/k_cdf"));
    double total = 0.0;
    rc = numpy_sum(g->col_norm, g->n, s, &total);
    if (rc) return fail(rc);
    g->info.col_norm_total = total;
    k_divide<<<nb, 256, 0, s>>>(g->col_norm, total, g->n, g->init_prob);
    mcf::note_launch();
    if ((e = cudaGetLastError()) != cudaSuccess) return fail(cuda_status(e, "k_divide"));
    if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return fail(cuda_status(e, "graph build"));
    *out = g;
    return MCF_OK;
}

}  // namespace mcf

extern "C" {

int mcf_graph_create(const mcf_csr *csr, void *stream, mcf_graph **out) {
    return mcf::create(csr, (cudaStream_t)stream, out);
}

int mcf_graph_destroy(mcf_graph *g) {
    if (g) cudaDeviceSynchronize();
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
