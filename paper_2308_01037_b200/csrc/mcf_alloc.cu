// Per-column walk budgets (replaces walker.allocate_walks / largest_remainder,
// /root/reference/pkg/src/mcfunm/walker.py:148-170) without a sort:
//   N_i = floor(p_i N_s); the residue R = N_s - sum N_i goes to the R largest
//   remainders, ties to the lowest index (the reference's stable argsort of
//   -remainder), p_i = 0 never selected ahead of p_i > 0.
// The R-th largest remainder is found by an 8-pass MSB-first radix select on
// the remainder's IEEE bits (non-negative doubles order like their bits).
#include "mcf_internal.cuh"

namespace mcf {

struct SelectState {
    unsigned long long total_floor;  // sum of floor(p N)
    unsigned long long prefix, mask;
    long long k;     // still to select inside the current prefix bucket
    long long left;  // residue R
    unsigned long long hist[256];
};

__global__ void k_floor(const double *__restrict__ p, long long n, double total, long long *__restrict__ ni,
                        unsigned long long *__restrict__ key, SelectState *st) {
    long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    long long got = 0;
    if (i < n) {
        double pi = p[i];
        double want = __dmul_rn(pi, total);
        double fl = floor(want);
        got = (long long)fl;
        ni[i] = got;
        key[i] = (pi == 0.0) ? 0ull : (unsigned long long)__double_as_longlong(__dsub_rn(want, fl)) + 1ull;
    }
    got = warp_sum_ll(got);
    if ((threadIdx.x & 31) == 0 && got) atomicAdd(&st->total_floor, (unsigned long long)got);
}

__global__ void k_select_init(SelectState *st, long long n_walks) {
    st->left = n_walks - (long long)st->total_floor;
    st->k = st->left;
    st->prefix = 0;
    st->mask = 0;
    for (int b = 0; b < 256; ++b) st->hist[b] = 0;
}

__global__ void k_hist(const unsigned long long *__restrict__ key, long long n, int shift, SelectState *st) {
    __shared__ unsigned int h[256];
    if (st->k <= 0) return;
    for (int b = threadIdx.x; b < 256; b += blockDim.x) h[b] = 0;
    __syncthreads();
    unsigned long long pre = st->prefix, msk = st->mask;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        unsigned long long k = key[i];
        if ((k & msk) == pre) atomicAdd(&h[(k >> shift) & 255u], 1u);
    }
    __syncthreads();
    for (int b = threadIdx.x; b < 256; b += blockDim.x)
        if (h[b]) atomicAdd(&st->hist[b], (unsigned long long)h[b]);
}

__global__ void k_pick(int shift, SelectState *st) {
    if (st->k <= 0) return;
    long long k = st->k;
    for (int b = 255; b >= 0; --b) {
        long long c = (long long)st->hist[b];
        if (k <= c) {
            st->prefix |= (unsigned long long)b << shift;
            st->mask |= 255ull << shift;
            break;
        }
        k -= c;
    }
    st->k = k;
    for (int b = 0; b < 256; ++b) st->hist[b] = 0;
}

__global__ void k_tie_flags(const unsigned long long *__restrict__ key, long long n, const SelectState *st,
                            long long *__restrict__ flag) {
    long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) flag[i] = (st->left > 0 && key[i] == st->prefix) ? 1 : 0;
}

__global__ void k_final(const unsigned long long *__restrict__ key, long long n, const SelectState *st,
                        const long long *__restrict__ tie_rank, long long *__restrict__ ni) {
    long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n || st->left <= 0) return;
    unsigned long long k = key[i], t = st->prefix;
    if (k > t || (k == t && tie_rank[i] < st->k)) ni[i] += 1;
}

static int allocate(mcf_graph *g, long long n_walks, long long *ni, long long *walk_pre, cudaStream_t s) {
    MCF_ARG(g && ni && walk_pre, "mcf_allocate_walks: null argument");
    MCF_ARG(n_walks >= 1, "n_walks must be at least 1");  // walker.py:168-169
    MCF_ARG(n_walks < (1ll << 53), "n_walks must be below 2^53");
    long long n = g->n;
    SelectState *st = nullptr;
    unsigned long long *key = nullptr;
    long long *tmp = nullptr;
    MCF_CUDA(cudaMallocAsync(&st, sizeof(SelectState), s));
    MCF_CUDA(cudaMallocAsync(&key, sizeof(unsigned long long) * n, s));
    MCF_CUDA(cudaMallocAsync(&tmp, sizeof(long long) * (2 * n + 1), s));
    MCF_CUDA(cudaMemsetAsync(st, 0, sizeof(SelectState), s));
    unsigned nb = (unsigned)((n + 255) / 256);
    k_floor<<<nb, 256, 0, s>>>(g->init_prob, n, (double)n_walks, ni, key, st);
    mcf::note_launch();
    k_select_init<<<1, 1, 0, s>>>(st, n_walks);
    mcf::note_launch();
    int hb = sm_count() * 4;
    for (int pass = 0; pass < 8; ++pass) {
        int shift = 56 - 8 * pass;
        k_hist<<<hb, 256, 0, s>>>(key, n, shift, st);
        mcf::note_launch();
        k_pick<<<1, 1, 0, s>>>(shift, st);
        mcf::note_launch();
    }
    k_tie_flags<<<nb, 256, 0, s>>>(key, n, st, tmp);
    mcf::note_launch();
    MCF_LAUNCHED("allocate");
    int rc = exclusive_scan_i64(tmp, tmp + n, n, s);
    if (rc) return rc;
    k_final<<<nb, 256, 0, s>>>(key, n, st, tmp + n, ni);
    mcf::note_launch();
    MCF_LAUNCHED("k_final");
    rc = exclusive_scan_i64(ni, walk_pre, n, s);
    if (rc) return rc;
    MCF_CUDA(cudaFreeAsync(st, s));
    MCF_CUDA(cudaFreeAsync(key, s));
    MCF_CUDA(cudaFreeAsync(tmp, s));
    return MCF_OK;
}

}  // namespace mcf

extern "C" int mcf_allocate_walks(mcf_graph *g, int64_t n_walks, int64_t *ni, int64_t *walk_pre, void *stream) {
    return mcf::allocate(g, (long long)n_walks, (long long *)ni, (long long *)walk_pre, (cudaStream_t)stream);
}
