// Graph generation and ingest on the device: the R-MAT and
// Chung-Lu edge generators (graphgen.py:124-156 quadrant rule; the BASELINE
// configs 3-5 graphs) and the cleanup filters of simple_graph_from_edges
// (sparsemat.py:243-290: self loops, undirected expansion, duplicates,
// isolated-node compaction) as kernels.
//
// Edges travel as 64-bit keys (u << 32) | v.  mcf_edges_to_csr removes loops,
// optionally adds the reverse of every edge, removes duplicates with a
// device hash set, counts rows, scatters the columns and sorts every row
// (a thread per short row, a CTA bitonic sort for mid rows, an n-bit bitmap
// per hub row: set bits, then compact in order).  mcf_csr_compact drops the
// nodes with no incident edge and renumbers the rest in order.
#include <climits>
#include <cstring>

#include "mcf_internal.cuh"

namespace mcf {

constexpr unsigned long long KEY_EMPTY = ~0ull;

// ---------------------------------------------------------------------------
// generators
// ---------------------------------------------------------------------------
// R-MAT: draw d takes `scale` uniforms, one per level (graphgen.py:138-143):
// row bit = r >= a + b, column bit = a <= r < a + b or r >= a + b + c.
// Philox-4x32-10 keyed by the seed, counter (level pair, draw): 2 uniforms per call.
__global__ void k_rmat_keys(int scale, long long draws, double pa, double pb, double pc, uint32_t k0, uint32_t k1,
                            unsigned long long *__restrict__ keys) {
    const long long d = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (d >= draws) return;
    const double ab = pa + pb, abc = pa + pb + pc;
    unsigned long long u = 0, v = 0;
    for (int l = 0; l < scale; l += 2) {
        const U4 r = philox4x32_10(U4{(uint32_t)(l >> 1), (uint32_t)d, (uint32_t)(d >> 32), 0x524d4154u}, k0, k1);
        for (int h = 0; h < 2 && l + h < scale; ++h) {
            const double x = u53(h ? r.z : r.x, h ? r.w : r.y);
            const bool rb = x >= ab;
            const bool cb = (x >= pa && !rb) || x >= abc;
            u = (u << 1) | (rb ? 1ull : 0ull);
            v = (v << 1) | (cb ? 1ull : 0ull);
        }
    }
    keys[d] = (u << 32) | v;
}

// Chung-Lu: both endpoints of edge d drawn from the expected-degree
// distribution (cdf = normalised prefix of the weights): first index with
// cdf > x (numpy searchsorted 'right' on the uniform)
__device__ __forceinline__ long long cdf_search(const double *__restrict__ cdf, long long n, double x) {
    long long lo = 0, hi = n - 1;
    while (lo < hi) {
        const long long mid = (lo + hi) >> 1;
        if (__ldg(cdf + mid) > x) hi = mid;
        else lo = mid + 1;
    }
    return lo;
}

__global__ void k_chung_lu_keys(const double *__restrict__ cdf, long long n, long long m, uint32_t k0, uint32_t k1,
                                unsigned long long *__restrict__ keys) {
    const long long d = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (d >= m) return;
    const U4 r = philox4x32_10(U4{0u, (uint32_t)d, (uint32_t)(d >> 32), 0x43484c55u}, k0, k1);
    const unsigned long long u = (unsigned long long)cdf_search(cdf, n, u53(r.x, r.y));
    const unsigned long long v = (unsigned long long)cdf_search(cdf, n, u53(r.z, r.w));
    keys[d] = (u << 32) | v;
}

// ---------------------------------------------------------------------------
// edges -> CSR
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned long long mix64(unsigned long long z) {
    z ^= z >> 33;
    z *= 0xff51afd7ed558ccdull;
    z ^= z >> 33;
    z *= 0xc4ceb9fe1a85ec53ull;
    return z ^ (z >> 33);
}

// insert key (and its reverse); loops dropped first if asked; counts how many
// insertions found the key already present (duplicates)
__global__ void k_edge_insert(const unsigned long long *__restrict__ keys, long long m, int flags,
                              unsigned long long *__restrict__ table, unsigned long long mask,
                              unsigned long long *__restrict__ dups, unsigned long long *__restrict__ loops) {
    const long long d = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    unsigned long long ndup = 0, nloop = 0;
    if (d < m) {
        const unsigned long long key = keys[d];
        const unsigned long long u = key >> 32, v = key & 0xffffffffull;
        if (u == v && (flags & MCF_EDGES_DROP_LOOPS)) {
            nloop = 1;
        } else {
            for (int rep = 0; rep < ((flags & MCF_EDGES_ADD_REVERSE) && u != v ? 2 : 1); ++rep) {
                const unsigned long long kk = rep ? ((v << 32) | u) : key;
                unsigned long long s = mix64(kk) & mask;
                while (true) {
                    const unsigned long long old = atomicCAS(table + s, KEY_EMPTY, kk);
                    if (old == KEY_EMPTY) break;
                    if (old == kk) {
                        ++ndup;
                        break;
                    }
                    s = (s + 1) & mask;
                }
            }
        }
    }
    ndup = warp_sum_ll((long long)ndup);
    nloop = warp_sum_ll((long long)nloop);
    if ((threadIdx.x & 31) == 0) {
        if (ndup) atomicAdd(dups, ndup);
        if (nloop) atomicAdd(loops, nloop);
    }
}

__global__ void k_edge_degrees(const unsigned long long *__restrict__ table, unsigned long long size,
                               unsigned long long *__restrict__ deg) {
    for (unsigned long long s = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; s < size;
         s += (unsigned long long)gridDim.x * blockDim.x) {
        const unsigned long long k = table[s];
        if (k != KEY_EMPTY) atomicAdd(deg + (k >> 32), 1ull);
    }
}

__global__ void k_edge_scatter(const unsigned long long *__restrict__ table, unsigned long long size,
                               unsigned long long *__restrict__ cursor, int *__restrict__ col_ids) {
    for (unsigned long long s = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; s < size;
         s += (unsigned long long)gridDim.x * blockDim.x) {
        const unsigned long long k = table[s];
        if (k != KEY_EMPTY) col_ids[atomicAdd(cursor + (k >> 32), 1ull)] = (int)(k & 0xffffffffull);
    }
}

constexpr int SORT_SHORT = 32, SORT_MID = 4096;

// rows of <= SORT_SHORT entries: insertion sort by the row's thread; longer
// rows are listed for the CTA sorts
__global__ void k_sort_short(const long long *__restrict__ row_ptr, long long n, int *__restrict__ col_ids,
                             int *__restrict__ mid, unsigned *__restrict__ nmid, int *__restrict__ big,
                             unsigned *__restrict__ nbig) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const long long lo = row_ptr[i], d = row_ptr[i + 1] - lo;
    if (d > SORT_MID) {
        big[atomicAdd(nbig, 1u)] = (int)i;
        return;
    }
    if (d > SORT_SHORT) {
        mid[atomicAdd(nmid, 1u)] = (int)i;
        return;
    }
    int *c = col_ids + lo;
    for (long long t = 1; t < d; ++t) {
        const int x = c[t];
        long long j = t - 1;
        while (j >= 0 && c[j] > x) {
            c[j + 1] = c[j];
            --j;
        }
        c[j + 1] = x;
    }
}

// rows of (SORT_SHORT, SORT_MID] entries: bitonic sort in shared memory, a CTA per row
__global__ void __launch_bounds__(512) k_sort_mid(const long long *__restrict__ row_ptr, const int *__restrict__ rows,
                                                  unsigned nrows, int *__restrict__ col_ids) {
    __shared__ int sh[SORT_MID];
    for (unsigned r = blockIdx.x; r < nrows; r += gridDim.x) {
        const long long i = rows[r], lo = row_ptr[i], d = row_ptr[i + 1] - lo;
        int P = 64;
        while (P < d) P <<= 1;
        for (int t = threadIdx.x; t < P; t += blockDim.x) sh[t] = t < d ? col_ids[lo + t] : INT_MAX;
        __syncthreads();
        for (int k = 2; k <= P; k <<= 1)
            for (int j = k >> 1; j > 0; j >>= 1) {
                for (int t = threadIdx.x; t < P; t += blockDim.x) {
                    const int p = t ^ j;
                    if (p > t) {
                        const bool up = (t & k) == 0;
                        const int a = sh[t], b = sh[p];
                        if ((a > b) == up) {
                            sh[t] = b;
                            sh[p] = a;
                        }
                    }
                }
                __syncthreads();
            }
        for (int t = threadIdx.x; t < d; t += blockDim.x) col_ids[lo + t] = sh[t];
        __syncthreads();
    }
}

// rows above SORT_MID (hub rows): the row's ids as bits of an n-bit bitmap
// (this CTA's scratch), then compacted in order with a CTA prefix over the
// words' population counts; the bitmap is cleared behind the scan
__global__ void __launch_bounds__(1024) k_sort_big(const long long *__restrict__ row_ptr, const int *__restrict__ rows,
                                                   unsigned nrows, long long words, unsigned *__restrict__ scratch,
                                                   int *__restrict__ col_ids) {
    __shared__ long long s_base;
    __shared__ int s_warp[32];
    unsigned *bits = scratch + (long long)blockIdx.x * words;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (unsigned r = blockIdx.x; r < nrows; r += gridDim.x) {
        const long long i = rows[r], lo = row_ptr[i], d = row_ptr[i + 1] - lo;
        for (long long t = threadIdx.x; t < d; t += blockDim.x) {
            const int c = col_ids[lo + t];
            atomicOr(bits + (c >> 5), 1u << (c & 31));
        }
        if (threadIdx.x == 0) s_base = lo;
        __syncthreads();
        for (long long w0 = 0; w0 < words; w0 += blockDim.x) {
            const long long wi = w0 + threadIdx.x;
            unsigned x = wi < words ? bits[wi] : 0u;
            if (wi < words && x) bits[wi] = 0u;
            int cnt = __popc(x), incl = cnt;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(MCF_FULL, incl, o);
                if (lane >= o) incl += y;
            }
            if (lane == 31) s_warp[w] = incl;
            __syncthreads();
            if (w == 0) {
                int v = lane < (int)(blockDim.x >> 5) ? s_warp[lane] : 0, iv = v;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int y = __shfl_up_sync(MCF_FULL, iv, o);
                    if (lane >= o) iv += y;
                }
                s_warp[lane] = iv - v;
            }
            __syncthreads();
            long long pos = s_base + s_warp[w] + incl - cnt;
            while (x) {
                const int b = __ffs(x) - 1;
                x &= x - 1;
                col_ids[pos++] = (int)(wi * 32 + b);
            }
            __syncthreads();
            if (threadIdx.x == blockDim.x - 1) s_base = pos;
            __syncthreads();
        }
    }
}

static int edges_to_csr(const unsigned long long *keys, long long m, long long n, int flags, long long *row_ptr,
                        int *col_ids, long long col_cap, long long *nnz_out, cudaStream_t s) {
    MCF_ARG(keys && row_ptr && col_ids && nnz_out, "mcf_edges_to_csr: null argument");
    MCF_ARG(n >= 1 && n < (1ll << 31) && m >= 0, "mcf_edges_to_csr: need 1 <= n < 2^31 and m >= 0");
    AsyncFrees frees(s);
    const long long mm = (flags & MCF_EDGES_ADD_REVERSE) ? 2 * m : m;
    unsigned long long P = 64;
    while ((long long)P < 2 * mm) P <<= 1;
    unsigned long long *table = nullptr, *cnt = nullptr, *deg = nullptr;
    MCF_CUDA(cudaMallocAsync(&table, sizeof(unsigned long long) * P, s));
    frees.keep(table);
    MCF_CUDA(cudaMemsetAsync(table, 0xff, sizeof(unsigned long long) * P, s));
    MCF_CUDA(cudaMallocAsync(&cnt, sizeof(unsigned long long) * 4, s));
    frees.keep(cnt);
    MCF_CUDA(cudaMemsetAsync(cnt, 0, sizeof(unsigned long long) * 4, s));
    MCF_CUDA(cudaMallocAsync(&deg, sizeof(unsigned long long) * (n + 1), s));
    frees.keep(deg);
    MCF_CUDA(cudaMemsetAsync(deg, 0, sizeof(unsigned long long) * (n + 1), s));
    if (m > 0) {
        k_edge_insert<<<(unsigned)((m + 255) / 256), 256, 0, s>>>(keys, m, flags, table, P - 1, cnt, cnt + 1);
        note_launch();
    }
    const unsigned g = (unsigned)(sm_count() * 8);
    k_edge_degrees<<<g, 256, 0, s>>>(table, P, deg);
    note_launch();
    int rc = exclusive_scan_i64((const long long *)deg, row_ptr, n, s);
    if (rc) return rc;
    unsigned long long h[2];
    long long nnz = 0;
    MCF_CUDA(cudaMemcpyAsync(h, cnt, sizeof(h), cudaMemcpyDeviceToHost, s));
    MCF_CUDA(cudaMemcpyAsync(&nnz, row_ptr + n, sizeof(long long), cudaMemcpyDeviceToHost, s));
    MCF_CUDA(cudaStreamSynchronize(s));
    *nnz_out = nnz;
    if ((flags & MCF_EDGES_FAIL_ON_DUPLICATES) && h[0]) {
        set_error("duplicate (row, col) entries");  // the reference's SparseMatrix.from_coo check
        return MCF_ERR_ARGUMENT;
    }
    MCF_ARG(nnz <= col_cap, "mcf_edges_to_csr: col_ids capacity below the edge count");
    // scatter through per-row cursors (deg reused), then sort every row
    MCF_CUDA(cudaMemcpyAsync(deg, row_ptr, sizeof(long long) * n, cudaMemcpyDeviceToDevice, s));
    k_edge_scatter<<<g, 256, 0, s>>>(table, P, deg, col_ids);
    note_launch();
    int *lists = nullptr;
    unsigned *ncnt = nullptr;
    MCF_CUDA(cudaMallocAsync(&lists, sizeof(int) * 2 * n + 16, s));
    frees.keep(lists);
    ncnt = reinterpret_cast<unsigned *>(lists + 2 * n);
    MCF_CUDA(cudaMemsetAsync(ncnt, 0, 16, s));
    k_sort_short<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(row_ptr, n, col_ids, lists, ncnt, lists + n, ncnt + 1);
    note_launch();
    unsigned hn[2];
    MCF_CUDA(cudaMemcpyAsync(hn, ncnt, sizeof(hn), cudaMemcpyDeviceToHost, s));
    MCF_CUDA(cudaStreamSynchronize(s));
    if (hn[0]) {
        k_sort_mid<<<(unsigned)(hn[0] < (unsigned)g ? hn[0] : (unsigned)g), 512, 0, s>>>(row_ptr, lists, hn[0], col_ids);
        note_launch();
    }
    if (hn[1]) {
        const long long words = (n + 31) / 32;
        const unsigned gb = hn[1] < (unsigned)sm_count() ? hn[1] : (unsigned)sm_count();
        unsigned *scratch = nullptr;
        MCF_CUDA(cudaMallocAsync(&scratch, sizeof(unsigned) * words * gb, s));
        frees.keep(scratch);
        MCF_CUDA(cudaMemsetAsync(scratch, 0, sizeof(unsigned) * words * gb, s));
        k_sort_big<<<gb, 1024, 0, s>>>(row_ptr, lists + n, hn[1], words, scratch, col_ids);
        note_launch();
    }
    MCF_LAUNCHED("mcf_edges_to_csr");
    return MCF_OK;
}

// ---------------------------------------------------------------------------
// isolated-node compaction (sparsemat.py:271-278): keep the nodes with an
// incident edge (as row or column), renumber them in order
// ---------------------------------------------------------------------------
__global__ void k_mark_present(const long long *__restrict__ row_ptr, const int *__restrict__ col_ids, long long n,
                               long long nnz, long long *__restrict__ flag) {
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < nnz; e += (long long)gridDim.x * blockDim.x)
        flag[col_ids[e]] = 1;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        if (row_ptr[i + 1] > row_ptr[i]) flag[i] = 1;
}

__global__ void k_compact_rows(const long long *__restrict__ row_ptr, long long n, const long long *__restrict__ flag,
                               const long long *__restrict__ newid, long long *__restrict__ new_row_ptr,
                               long long *__restrict__ old_ids) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    if (flag[i]) {
        new_row_ptr[newid[i]] = row_ptr[i];
        old_ids[newid[i]] = i;
    }
    if (i == n - 1) new_row_ptr[newid[n]] = row_ptr[n];
}

__global__ void k_remap_cols(int *__restrict__ col_ids, long long nnz, const long long *__restrict__ newid) {
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < nnz; e += (long long)gridDim.x * blockDim.x)
        col_ids[e] = (int)newid[col_ids[e]];
}

static int csr_compact(long long n, const long long *row_ptr, int *col_ids, long long nnz, long long *new_row_ptr,
                       long long *old_ids, long long *n_out, cudaStream_t s) {
    MCF_ARG(row_ptr && col_ids && new_row_ptr && old_ids && n_out && n >= 1, "mcf_csr_compact: null argument");
    AsyncFrees frees(s);
    long long *flag = nullptr;
    MCF_CUDA(cudaMallocAsync(&flag, sizeof(long long) * (2 * n + 1), s));
    frees.keep(flag);
    long long *newid = flag + n;
    MCF_CUDA(cudaMemsetAsync(flag, 0, sizeof(long long) * n, s));
    const unsigned g = (unsigned)(sm_count() * 8);
    k_mark_present<<<g, 256, 0, s>>>(row_ptr, col_ids, n, nnz, flag);
    note_launch();
    int rc = exclusive_scan_i64(flag, newid, n, s);
    if (rc) return rc;
    k_compact_rows<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(row_ptr, n, flag, newid, new_row_ptr, old_ids);
    note_launch();
    k_remap_cols<<<g, 256, 0, s>>>(col_ids, nnz, newid);
    note_launch();
    MCF_LAUNCHED("mcf_csr_compact");
    MCF_CUDA(cudaMemcpyAsync(n_out, newid + n, sizeof(long long), cudaMemcpyDeviceToHost, s));
    MCF_CUDA(cudaStreamSynchronize(s));
    return MCF_OK;
}

}  // namespace mcf

extern "C" {

int mcf_gen_rmat_keys(int scale, int64_t draws, double a, double b, double c, uint64_t seed, uint64_t *keys,
                      void *stream) {
    MCF_ARG(keys && scale >= 1 && scale <= 31 && draws >= 0, "mcf_gen_rmat_keys: need 1 <= scale <= 31");
    MCF_ARG(a >= 0 && b >= 0 && c >= 0 && a + b + c <= 1.0, "mcf_gen_rmat_keys: quadrant probabilities");
    if (draws == 0) return MCF_OK;
    mcf::k_rmat_keys<<<(unsigned)((draws + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
        scale, (long long)draws, a, b, c, (uint32_t)seed, (uint32_t)(seed >> 32), (unsigned long long *)keys);
    mcf::note_launch();
    MCF_LAUNCHED("k_rmat_keys");
    return MCF_OK;
}

int mcf_gen_chung_lu_keys(const double *cdf, int64_t n, int64_t m, uint64_t seed, uint64_t *keys, void *stream) {
    MCF_ARG(cdf && keys && n >= 1 && m >= 0, "mcf_gen_chung_lu_keys: bad argument");
    if (m == 0) return MCF_OK;
    mcf::k_chung_lu_keys<<<(unsigned)((m + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
        cdf, (long long)n, (long long)m, (uint32_t)seed, (uint32_t)(seed >> 32), (unsigned long long *)keys);
    mcf::note_launch();
    MCF_LAUNCHED("k_chung_lu_keys");
    return MCF_OK;
}

int mcf_edges_to_csr(const uint64_t *keys, int64_t m, int64_t n, int flags, int64_t *row_ptr, int32_t *col_ids,
                     int64_t col_cap, int64_t *nnz, void *stream) {
    return mcf::edges_to_csr((const unsigned long long *)keys, (long long)m, (long long)n, flags,
                             (long long *)row_ptr, col_ids, (long long)col_cap, (long long *)nnz,
                             (cudaStream_t)stream);
}

int mcf_csr_compact(int64_t n, const int64_t *row_ptr, int32_t *col_ids, int64_t nnz, int64_t *new_row_ptr,
                    int64_t *old_ids, int64_t *n_out, void *stream) {
    return mcf::csr_compact((long long)n, (const long long *)row_ptr, col_ids, (long long)nnz,
                            (long long *)new_row_ptr, (long long *)old_ids, (long long *)n_out, (cudaStream_t)stream);
}

}  // extern "C"
