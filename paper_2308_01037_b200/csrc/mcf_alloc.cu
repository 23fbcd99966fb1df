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
    unsigned int done;
    unsigned int hist[256];
};

// floor(p N), remainder keys, sum of floors; the last block to finish also
// initialises the selection (residue R = N - sum floor).
__global__ void k_floor(const double *__restrict__ p, long long n, double total, long long n_walks,
                        long long *__restrict__ ni, unsigned long long *__restrict__ key, SelectState *st) {
    __shared__ bool last;
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
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(&st->done, 1u) == gridDim.x - 1;
    __syncthreads();
    if (last && threadIdx.x == 0) {
        __threadfence();
        st->left = n_walks - (long long)atomicAdd(&st->total_floor, 0ull);
        st->k = st->left;
        st->prefix = 0;
        st->mask = 0;
        st->done = 0;
    }
}

// One radix-select pass: histogram of the 8-bit digit at `shift` over keys
// that match the current prefix; the last block picks the bucket holding the
// k-th largest key (parallel suffix scan over the 256 bins).
__global__ void __launch_bounds__(256) k_select_pass(const unsigned long long *__restrict__ key, long long n,
                                                     int shift, SelectState *st) {
    __shared__ unsigned int h[256];
    __shared__ bool last;
    if (st->k <= 0) return;  // uniform across the grid
    h[threadIdx.x] = 0;
    __syncthreads();
    const unsigned long long pre = st->prefix, msk = st->mask;
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long base = (long long)blockIdx.x * blockDim.x; base < n; base += stride) {  // warp-uniform trip count
        const long long i = base + threadIdx.x;
        const unsigned long long k = i < n ? key[i] : ~0ull;
        const bool in = i < n && (k & msk) == pre;
        const unsigned dig = in ? (unsigned)((k >> shift) & 255u) : 256u;
        // ties are common (equal-degree nodes share p): a warp whose keys all
        // fall in one bin adds once
        const unsigned d0 = __shfl_sync(MCF_FULL, dig, 0);
        if (__all_sync(MCF_FULL, dig == d0)) {
            if ((threadIdx.x & 31) == 0 && d0 < 256u) atomicAdd(&h[d0], 32u);
        } else if (in) {
            atomicAdd(&h[dig], 1u);
        }
    }
    __syncthreads();
    if (h[threadIdx.x]) atomicAdd(&st->hist[threadIdx.x], h[threadIdx.x]);
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(&st->done, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!last) return;
    __threadfence();
    // thread t looks at bin 255 - t: inclusive scan of counts from the top
    const int b = 255 - threadIdx.x;
    const long long c = (long long)atomicAdd(&st->hist[b], 0u);
    __shared__ long long wsum[8];
    long long x = c;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        long long y = __shfl_up_sync(MCF_FULL, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) wsum[w] = x;
    __syncthreads();
    long long before = 0;
    for (int j = 0; j < w; ++j) before += wsum[j];
    const long long incl = before + x;
    const long long k = st->k;
    __syncthreads();
    if (incl - c < k && k <= incl) {
        st->prefix = pre | ((unsigned long long)b << shift);
        st->mask = msk | (255ull << shift);
        st->k = k - (incl - c);
    }
    st->hist[b] = 0;
    if (threadIdx.x == 0) st->done = 0;
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
    long long *rank = nullptr;
    MCF_CUDA(cudaMallocAsync(&st, sizeof(SelectState), s));
    MCF_CUDA(cudaMallocAsync(&key, sizeof(unsigned long long) * n, s));
    MCF_CUDA(cudaMallocAsync(&rank, sizeof(long long) * (n + 1), s));
    MCF_CUDA(cudaMemsetAsync(st, 0, sizeof(SelectState), s));
    unsigned nb = (unsigned)((n + 255) / 256);
    k_floor<<<nb, 256, 0, s>>>(g->init_prob, n, (double)n_walks, n_walks, ni, key, st);
    mcf::note_launch();
    long long want_blocks = (n + 2047) / 2048;
    int hb = (int)(want_blocks < sm_count() * 2 ? (want_blocks > 0 ? want_blocks : 1) : sm_count() * 2);
    for (int pass = 0; pass < 8; ++pass) {
        k_select_pass<<<hb, 256, 0, s>>>(key, n, 56 - 8 * pass, st);
        mcf::note_launch();
    }
    MCF_LAUNCHED("allocate");
    // rank of each tied key among the ties (index order) = the stable argsort tie-break
    ScanSrc ties{nullptr, key, &st->prefix};
    int rc = scan_src(ties, rank, n, s);
    if (rc) return rc;
    k_final<<<nb, 256, 0, s>>>(key, n, st, rank, ni);
    mcf::note_launch();
    MCF_LAUNCHED("k_final");
    rc = exclusive_scan_i64(ni, walk_pre, n, s);
    if (rc) return rc;
    MCF_CUDA(cudaFreeAsync(st, s));
    MCF_CUDA(cudaFreeAsync(key, s));
    MCF_CUDA(cudaFreeAsync(rank, s));
    return MCF_OK;
}

}  // namespace mcf

extern "C" int mcf_allocate_walks(mcf_graph *g, int64_t n_walks, int64_t *ni, int64_t *walk_pre, void *stream) {
    return mcf::allocate(g, (long long)n_walks, (long long *)ni, (long long *)walk_pre, (cudaStream_t)stream);
}
