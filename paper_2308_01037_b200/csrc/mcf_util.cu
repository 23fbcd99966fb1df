// Shared host/device utilities: error state, prefix scans, walk -> column
// index, coefficient upload, CSR -> CSC entry map.
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <string>

#include "mcf_internal.cuh"

namespace mcf {

static thread_local std::string g_last_error;
static std::atomic<long long> g_launches{0};

void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
long long launches() { return g_launches.load(); }

// Inside stream capture a plain cudaEventRecord only expresses a dependency;
// an external record makes the event a node that fires on every graph replay.
static cudaError_t record_event(cudaEvent_t e, cudaStream_t s) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    cudaError_t err = cudaStreamIsCapturing(s, &cs);
    if (err != cudaSuccess) return err;
    if (cs == cudaStreamCaptureStatusActive) return cudaEventRecordWithFlags(e, s, cudaEventRecordExternal);
    return cudaEventRecord(e, s);
}

int timed_begin(mcf_graph *, bool on, std::vector<std::pair<cudaEvent_t, cudaEvent_t>> &v, cudaStream_t s) {
    if (!on) return MCF_OK;
    cudaEvent_t a, b;
    MCF_CUDA(cudaEventCreate(&a));
    MCF_CUDA(cudaEventCreate(&b));
    MCF_CUDA(record_event(a, s));
    v.emplace_back(a, b);
    return MCF_OK;
}

int timed_end(bool on, std::vector<std::pair<cudaEvent_t, cudaEvent_t>> &v, cudaStream_t s) {
    if (!on || v.empty()) return MCF_OK;
    MCF_CUDA(record_event(v.back().second, s));
    return MCF_OK;
}

void set_error(const std::string &msg) { g_last_error = msg; }
const char *last_error() { return g_last_error.c_str(); }

int cuda_status(cudaError_t e, const char *what) {
    set_error(std::string(what) + ": " + cudaGetErrorString(e));
    if (e == cudaErrorMemoryAllocation) {
        cudaGetLastError();  // clear the sticky-free allocation error
        return MCF_ERR_RESOURCE;
    }
    return MCF_ERR_CUDA;
}

int sm_count() {
    static int cached = 0;
    if (!cached) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&cached, cudaDevAttrMultiProcessorCount, dev);
        if (cached <= 0) cached = 148;
    }
    return cached;
}

// ---------------------------------------------------------------------------
// exclusive scan of int64, single pass (decoupled look-back, mcf_internal.cuh):
// out[0..n] with out[n] = total.  Tiles take ids from a counter so every
// predecessor a tile waits on has already started.
// ---------------------------------------------------------------------------
__device__ __forceinline__ long long scan_item(const ScanSrc &src, long long j) {
    if (src.in) return src.in[j];
    return src.key[j] == *src.match ? 1 : 0;
}

__global__ void __launch_bounds__(SCAN_T, 2) k_scan(ScanSrc src, long long n, long long *__restrict__ out,
                                                    unsigned long long *status, unsigned int *tile_ctr) {
    __shared__ unsigned int s_tile;
    if (threadIdx.x == 0) s_tile = atomicAdd(tile_ctr, 1u);
    __syncthreads();
    const long long tile = s_tile;
    const long long base = tile * SCAN_TILE + (long long)(threadIdx.x >> 5) * 32 * SCAN_I + (threadIdx.x & 31);
    long long v[SCAN_I], e[SCAN_I], none[SCAN_I], none2[SCAN_I];
#pragma unroll
    for (int k = 0; k < SCAN_I; ++k) {
        const long long j = base + 32 * k;
        v[k] = j < n ? scan_item(src, j) : 0;
        none[k] = 0;
    }
    tile_scan<false>(tile, v, none, e, none2, status, nullptr);
#pragma unroll
    for (int k = 0; k < SCAN_I; ++k) {
        const long long j = base + 32 * k;
        if (j < n) out[j] = e[k];
        if (j == n - 1) out[n] = e[k] + v[k];
    }
}

int scan_src(ScanSrc src, long long *out, long long n, cudaStream_t s) {
    if (n <= 0) {
        MCF_CUDA(cudaMemsetAsync(out, 0, sizeof(long long), s));
        return MCF_OK;
    }
    long long nb = (n + SCAN_TILE - 1) / SCAN_TILE;
    unsigned long long *status = nullptr;
    MCF_CUDA(cudaMallocAsync(&status, sizeof(unsigned long long) * nb + 16, s));
    unsigned int *ctr = reinterpret_cast<unsigned int *>(status + nb);
    MCF_CUDA(cudaMemsetAsync(status, 0, sizeof(unsigned long long) * nb + 16, s));
    k_scan<<<(unsigned)nb, SCAN_T, 0, s>>>(src, n, out, status, ctr);
    mcf::note_launch();
    MCF_LAUNCHED("k_scan");
    MCF_CUDA(cudaFreeAsync(status, s));
    return MCF_OK;
}

int exclusive_scan_i64(const long long *in, long long *out, long long n, cudaStream_t s) {
    ScanSrc src{in, nullptr, nullptr};
    return scan_src(src, out, n, s);
}

// ---------------------------------------------------------------------------
// walk-block -> column index for a column range
// ---------------------------------------------------------------------------
__global__ void k_blk_col(const long long *__restrict__ walk_pre, long long col_begin, long long col_end,
                          long long capacity, int *__restrict__ blk_col) {
    long long c = col_begin + (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= col_end) return;
    const long long walk_begin = __ldg(walk_pre + col_begin);
    long long a = walk_pre[c] - walk_begin, b = walk_pre[c + 1] - walk_begin;
    if (b > capacity) b = capacity;  // walks past the capacity are never run (the walk kernels clamp)
    if (b <= a) return;
    const long long B = 1ll << WALK_BLK_SHIFT;
    for (long long blk = (a + B - 1) >> WALK_BLK_SHIFT; blk * B < b; ++blk) blk_col[blk] = (int)c;
}

int build_blk_col(const long long *walk_pre, long long col_begin, long long col_end, long long capacity,
                  int **blk_col, cudaStream_t s) {
    long long nb = (capacity + (1ll << WALK_BLK_SHIFT) - 1) >> WALK_BLK_SHIFT;
    if (nb < 1) nb = 1;
    MCF_CUDA(cudaMallocAsync(blk_col, sizeof(int) * nb, s));
    long long nc = col_end - col_begin;
    if (nc > 0 && capacity > 0) {
        k_blk_col<<<(unsigned)((nc + 255) / 256), 256, 0, s>>>(walk_pre, col_begin, col_end, capacity, *blk_col);
        mcf::note_launch();
        MCF_LAUNCHED("k_blk_col");
    }
    return MCF_OK;
}

__global__ void k_batch_bounds(const long long *__restrict__ walk_pre, long long cb, long long ce, long long wb,
                               long long cap_walks, long long nb, long long *__restrict__ bounds) {
    long long b = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (b > nb) return;
    if (b == 0) { bounds[0] = cb; return; }
    if (b == nb) { bounds[nb] = ce; return; }
    long long target = wb + b * cap_walks;  // largest c in [cb, ce] with walk_pre[c] <= target
    long long lo = cb, hi = ce;
    while (lo < hi) {
        long long mid = (lo + hi + 1) >> 1;
        if (walk_pre[mid] <= target) lo = mid;
        else hi = mid - 1;
    }
    bounds[b] = lo;
}

__global__ void k_max_walks(const long long *__restrict__ walk_pre, long long cb, long long ce,
                            unsigned long long *out) {
    long long c = cb + (long long)blockIdx.x * blockDim.x + threadIdx.x;
    unsigned long long v = (c < ce) ? (unsigned long long)(walk_pre[c + 1] - walk_pre[c]) : 0ull;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        unsigned long long x = __shfl_xor_sync(MCF_FULL, v, o);
        v = x > v ? x : v;
    }
    if ((threadIdx.x & 31) == 0 && v) atomicMax(out, v);
}

// Column batches of [cb, ce) with at most cap_walks + max N_c walks each
// (bounds[b] .. bounds[b+1]); *max_walks = the largest N_c of the range.
// Synchronises the stream.
int column_batches(const long long *walk_pre, long long cb, long long ce, long long cap_walks,
                   std::vector<long long> &bounds, unsigned long long *max_walks, cudaStream_t s) {
    bounds.assign(1, cb);
    if (ce <= cb) {
        bounds.push_back(ce);
        if (max_walks) *max_walks = 0;
        return MCF_OK;
    }
    long long wb = 0, we = 0;
    int rc = read_walk_range(walk_pre, cb, ce, &wb, &we, s);
    if (rc) return rc;
    if (cap_walks < 1) cap_walks = 1;
    const long long nb = (we - wb + cap_walks - 1) / cap_walks > 0 ? (we - wb + cap_walks - 1) / cap_walks : 1;
    unsigned long long *d = nullptr;
    MCF_CUDA(cudaMallocAsync(&d, sizeof(long long) * (nb + 2), s));
    MCF_CUDA(cudaMemsetAsync(d, 0, sizeof(long long), s));
    const long long ncol = ce - cb;
    k_max_walks<<<(unsigned)((ncol + 255) / 256), 256, 0, s>>>(walk_pre, cb, ce, d);
    mcf::note_launch();
    long long *db = reinterpret_cast<long long *>(d + 1);
    k_batch_bounds<<<(unsigned)((nb + 1 + 255) / 256), 256, 0, s>>>(walk_pre, cb, ce, wb, cap_walks, nb, db);
    mcf::note_launch();
    MCF_LAUNCHED("k_batch_bounds");
    std::vector<unsigned long long> h((size_t)nb + 2);
    MCF_CUDA(cudaMemcpyAsync(h.data(), d, sizeof(long long) * (nb + 2), cudaMemcpyDeviceToHost, s));
    MCF_CUDA(cudaStreamSynchronize(s));
    MCF_CUDA(cudaFreeAsync(d, s));
    if (max_walks) *max_walks = h[0];
    bounds.clear();
    for (long long b = 0; b <= nb; ++b) {
        const long long v = (long long)h[1 + b];
        if (bounds.empty() || v != bounds.back()) bounds.push_back(v);
    }
    return MCF_OK;
}

int read_walk_range(const long long *walk_pre, long long col_begin, long long col_end, long long *wb,
                    long long *we, cudaStream_t s) {
    long long h[2];
    MCF_CUDA(cudaMemcpyAsync(&h[0], walk_pre + col_begin, sizeof(long long), cudaMemcpyDeviceToHost, s));
    MCF_CUDA(cudaMemcpyAsync(&h[1], walk_pre + col_end, sizeof(long long), cudaMemcpyDeviceToHost, s));
    MCF_CUDA(cudaStreamSynchronize(s));
    *wb = h[0];
    *we = h[1];
    return MCF_OK;
}

// ---------------------------------------------------------------------------
// CSR entry e = (i, c) -> position of (i, c) inside CSC column c
// ---------------------------------------------------------------------------
__global__ void k_csr2csc(const long long *__restrict__ row_ptr, const int *__restrict__ col_ids,
                          const long long *__restrict__ csc_ptr, const int *__restrict__ csc_rows,
                          long long n, long long *__restrict__ out) {
    long long i = (long long)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
    if (i >= n) return;
    int lane = threadIdx.x & 31;
    for (long long e = row_ptr[i] + lane; e < row_ptr[i + 1]; e += 32) {
        int c = col_ids[e];
        long long lo = csc_ptr[c], hi = csc_ptr[c + 1];  // search row id i in column c
        while (lo < hi) {
            long long mid = (lo + hi) >> 1;
            if (csc_rows[mid] < i) lo = mid + 1;
            else hi = mid;
        }
        out[e] = lo;
    }
}

int ensure_csr2csc(mcf_graph *g, cudaStream_t s) {
    if (g->csr2csc) return MCF_OK;
    MCF_CUDA(cudaMalloc(&g->csr2csc, sizeof(long long) * (g->nnz > 0 ? g->nnz : 1)));
    long long blocks = (g->n + 7) / 8;
    k_csr2csc<<<(unsigned)blocks, 256, 0, s>>>((const long long *)g->row_ptr, g->col_ids,
                                               (const long long *)g->csc_ptr, g->csc_rows, g->n,
                                               (long long *)g->csr2csc);
    mcf::note_launch();
    MCF_LAUNCHED("k_csr2csc");
    return MCF_OK;
}

}  // namespace mcf

// ---------------------------------------------------------------------------
// hub-row bitmaps (diag combine push path; uniform-value graphs)
// ---------------------------------------------------------------------------
namespace mcf {

__global__ void k_deg_hist(const long long *__restrict__ row_ptr, long long n, unsigned long long *hist) {
    long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    long long d = row_ptr[i + 1] - row_ptr[i];
    if (d > 0) atomicAdd(&hist[63 - __clzll(d)], 1ull);  // bin b: 2^b <= deg < 2^(b+1)
}

__global__ void k_mark_hubs(const long long *__restrict__ row_ptr, long long n, long long min_deg, int max_hubs,
                            int *__restrict__ hub_of, unsigned *count) {
    long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    int h = -1;
    if (row_ptr[i + 1] - row_ptr[i] >= min_deg) {
        unsigned k = atomicAdd(count, 1u);
        if ((int)k < max_hubs) h = (int)k;
    }
    hub_of[i] = h;
}

__global__ void k_hub_bits(const long long *__restrict__ row_ptr, const int *__restrict__ col_ids,
                           const int *__restrict__ hub_of, long long n, long long words, unsigned *__restrict__ bits) {
    for (long long i = blockIdx.x; i < n; i += gridDim.x) {
        const int h = hub_of[i];
        if (h < 0) continue;
        unsigned *b = bits + (long long)h * words;
        for (long long e = row_ptr[i] + threadIdx.x; e < row_ptr[i + 1]; e += blockDim.x) {
            const int c = col_ids[e];
            atomicOr(b + (c >> 5), 1u << (c & 31));
        }
    }
}

int make_peer_args(const double *const *x_parts, const long long *bounds, int nparts, double *const *y_outs,
                   int nouts, long long ncols, PeerArgs *pa) {
    MCF_ARG(x_parts && bounds && y_outs && pa, "peer exchange: null argument");
    MCF_ARG(nparts >= 1 && nparts <= MAX_PEERS && nouts >= 1 && nouts <= MAX_PEERS,
            "peer exchange: 1..8 parts and outputs");
    MCF_ARG(bounds[0] == 0 && bounds[nparts] == ncols, "peer exchange: the parts must cover [0, n)");
    for (int k = 0; k < nparts; ++k) {
        MCF_ARG(x_parts[k] && bounds[k] <= bounds[k + 1], "peer exchange: bad part");
        pa->x[k] = x_parts[k];
        pa->bounds[k] = bounds[k];
    }
    pa->bounds[nparts] = bounds[nparts];
    pa->nparts = nparts;
    for (int k = 0; k < nouts; ++k) {
        MCF_ARG(y_outs[k], "peer exchange: null output");
        pa->y[k] = y_outs[k];
    }
    pa->nouts = nouts;
    return MCF_OK;
}

int ensure_hub_bitmaps(mcf_graph *g, cudaStream_t s) {
    if (g->hubs_ready) return MCF_OK;
    g->hubs_ready = true;
    static const long long HUB_MIN_DEG = [] {
        const char *e = getenv("MCF_HUB_MIN_DEG");
        return e ? atoll(e) : 2048ll;
    }();
    if (!g->uniform_value || g->info.max_degree < HUB_MIN_DEG) return MCF_OK;
    const char *env = getenv("MCF_HUB_BITMAP_MB");
    const long long budget = (env ? atoll(env) : 4096ll) << 20;
    const long long words = (g->n + 31) / 32;
    const long long max_hubs = budget / (words * 4);
    if (max_hubs < 1) return MCF_OK;
    unsigned long long *hist = nullptr;
    MCF_CUDA(cudaMallocAsync(&hist, sizeof(unsigned long long) * 64 + 16, s));
    MCF_CUDA(cudaMemsetAsync(hist, 0, sizeof(unsigned long long) * 64 + 16, s));
    const unsigned nb = (unsigned)((g->n + 255) / 256);
    // C_i is column i of A: the bitmaps (and the hub degree) come from the CSC
    // (== the CSR on symmetric graphs)
    k_deg_hist<<<nb, 256, 0, s>>>((const long long *)g->csc_ptr, g->n, hist);
    mcf::note_launch();
    unsigned long long h[64];
    MCF_CUDA(cudaMemcpyAsync(h, hist, sizeof(h), cudaMemcpyDeviceToHost, s));
    MCF_CUDA(cudaStreamSynchronize(s));
    // smallest power-of-two threshold >= HUB_MIN_DEG whose hub count fits the budget
    int b0 = 63 - __builtin_clzll((unsigned long long)HUB_MIN_DEG);
    long long above = 0;
    int bsel = 64;
    for (int b = 63; b >= b0; --b) {
        if (above + (long long)h[b] > max_hubs) break;
        above += (long long)h[b];
        bsel = b;
    }
    if (bsel == 64 || above == 0) {
        cudaFreeAsync(hist, s);
        return MCF_OK;
    }
    MCF_CUDA(cudaMallocAsync(&g->hub_of, sizeof(int) * g->n, s));
    MCF_CUDA(cudaMallocAsync(&g->hub_bits, sizeof(unsigned) * words * above, s));
    MCF_CUDA(cudaMemsetAsync(g->hub_bits, 0, sizeof(unsigned) * words * above, s));
    unsigned *cnt = reinterpret_cast<unsigned *>(hist + 64);
    k_mark_hubs<<<nb, 256, 0, s>>>((const long long *)g->csc_ptr, g->n, 1ll << bsel, (int)above, g->hub_of, cnt);
    mcf::note_launch();
    k_hub_bits<<<sm_count() * 4, 256, 0, s>>>((const long long *)g->csc_ptr, g->csc_rows, g->hub_of, g->n, words,
                                            g->hub_bits);
    mcf::note_launch();
    MCF_LAUNCHED("hub bitmaps");
    g->hub_words = words;
    cudaFreeAsync(hist, s);
    return MCF_OK;
}

// ---------------------------------------------------------------------------
// Group-ordered CSC row ids for the diag combine units (mcf_diag.cu): column
// c's ids reordered by (key_group(id), CSC position), a stable counting sort
// by one warp per column; columns longer than GROUP_OFS_MIN also keep the
// NGROUPS + 1 group slice offsets, so a unit owning a group range reads one
// contiguous slice of every C_i it scans.
// ---------------------------------------------------------------------------
__global__ void k_mark_long_cols(const long long *__restrict__ csc_ptr, long long n, int *__restrict__ gidx,
                                 unsigned *count) {
    const long long c = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= n) return;
    int o = -1;
    const long long d = csc_ptr[c + 1] - csc_ptr[c];
    if (d > GROUP_OFS_MIN) o = (int)atomicAdd(count, 1u);
    gidx[c] = o;
    if (d > 0) atomicMax(reinterpret_cast<unsigned long long *>(count + 2), (unsigned long long)d);  // longest column
}

constexpr int GK_WARPS = 8;

__global__ void __launch_bounds__(GK_WARPS * 32) k_group_keys(const long long *__restrict__ csc_ptr,
                                                              const int *__restrict__ csc_rows, long long n,
                                                              const int *__restrict__ gidx, int *__restrict__ gofs,
                                                              int *__restrict__ ckeys) {
    __shared__ int cnt[GK_WARPS][NGROUPS];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int *wc = cnt[w];
    for (long long c = (long long)blockIdx.x * GK_WARPS + w; c < n; c += (long long)gridDim.x * GK_WARPS) {
        const long long lo = csc_ptr[c], hi = csc_ptr[c + 1], deg = hi - lo;
        if (deg == 0) continue;
        if (deg <= 32) {  // one chunk: rank = ids of smaller group + same group at lower lanes
            const bool v = lane < deg;
            const int j = v ? csc_rows[lo + lane] : 0;
            const int gj = v ? (int)key_group(j) : NGROUPS;
            int pos = 0;
            for (int l = 0; l < 32; ++l) {
                const int gl = __shfl_sync(MCF_FULL, gj, l);
                pos += (gl < gj) || (gl == gj && l < lane);
            }
            if (v) ckeys[lo + pos] = j;
            continue;  // deg <= GROUP_OFS_MIN: no offsets
        }
        for (int k = lane; k < NGROUPS; k += 32) wc[k] = 0;
        __syncwarp();
        for (long long e = lo + lane; e < hi; e += 32) atomicAdd(&wc[key_group(csc_rows[e])], 1);
        __syncwarp();
        // exclusive scan of the NGROUPS counts (NGROUPS / 32 per lane)
        constexpr int PER = NGROUPS / 32;
        int v[PER], s = 0;
#pragma unroll
        for (int k = 0; k < PER; ++k) {
            v[k] = wc[lane * PER + k];
            s += v[k];
        }
        int inc = s;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(MCF_FULL, inc, o);
            if (lane >= o) inc += t;
        }
        int run = inc - s;
        const int o = gidx[c];
        int *of = o >= 0 ? gofs + (long long)o * (NGROUPS + 1) : nullptr;
        __syncwarp();
#pragma unroll
        for (int k = 0; k < PER; ++k) {
            wc[lane * PER + k] = run;
            if (of) of[lane * PER + k] = run;
            run += v[k];
        }
        if (of && lane == 31) of[NGROUPS] = run;
        __syncwarp();
        // stable scatter, chunk by chunk in CSC order
        for (long long e0 = lo; e0 < hi; e0 += 32) {
            const long long e = e0 + lane;
            const bool ok = e < hi;
            const int j = ok ? csc_rows[e] : 0;
            const int gj = ok ? (int)key_group(j) : NGROUPS + lane;  // invalid lanes: unique dummy groups
            const unsigned same = __match_any_sync(MCF_FULL, gj);
            const int rank = __popc(same & lanemask_lt());
            const int base = ok ? wc[gj] : 0;
            __syncwarp();
            if (ok && rank == 0) wc[gj] += __popc(same);
            __syncwarp();
            if (ok) ckeys[lo + base + rank] = j;
        }
        __syncwarp();
    }
}

int ensure_group_keys(mcf_graph *g, cudaStream_t s) {
    if (g->ckeys) return MCF_OK;
    MCF_CUDA(cudaMallocAsync(&g->gidx, sizeof(int) * (g->n > 0 ? g->n : 1), s));
    unsigned *cnt = nullptr;  // [0]: long columns, [2..3]: the longest column (u64)
    MCF_CUDA(cudaMallocAsync(&cnt, 16, s));
    MCF_CUDA(cudaMemsetAsync(cnt, 0, 16, s));
    k_mark_long_cols<<<(unsigned)((g->n + 255) / 256), 256, 0, s>>>((const long long *)g->csc_ptr, g->n, g->gidx, cnt);
    mcf::note_launch();
    unsigned hc[4] = {0, 0, 0, 0};
    MCF_CUDA(cudaMemcpyAsync(hc, cnt, 16, cudaMemcpyDeviceToHost, s));
    MCF_CUDA(cudaStreamSynchronize(s));
    cudaFreeAsync(cnt, s);
    const unsigned nl = hc[0];
    g->max_col_degree = (long long)(((unsigned long long)hc[3] << 32) | hc[2]);
    g->n_gofs = nl;
    MCF_CUDA(cudaMallocAsync(&g->gofs, sizeof(int) * (size_t)(nl > 0 ? nl : 1) * (NGROUPS + 1), s));
    MCF_CUDA(cudaMallocAsync(&g->ckeys, sizeof(int) * (size_t)(g->nnz > 0 ? g->nnz : 1), s));
    const long long blocks = (g->n + GK_WARPS - 1) / GK_WARPS;
    k_group_keys<<<(unsigned)(blocks < 65536 ? blocks : 65536), GK_WARPS * 32, 0, s>>>(
        (const long long *)g->csc_ptr, g->csc_rows, g->n, g->gidx, g->gofs, g->ckeys);
    mcf::note_launch();
    MCF_LAUNCHED("k_group_keys");
    return MCF_OK;
}

}  // namespace mcf

// ---------------------------------------------------------------------------
// Per-column work estimates for cost-balanced column shards (SURVEY 8(e):
// "contiguous column ranges balanced by the prefix sum of N_i x expected
// length").  Action: N_c walks.  Diag: the walk emissions N_c (L + 1)
// weighted by DIAG_WALK_WEIGHT plus the Eq. 20 combine's probes
// sum_{i in C_c} min(deg i, N_c (L + 1)) (one warp per column, CSC order).
// ---------------------------------------------------------------------------
namespace mcf {

constexpr long long DIAG_WALK_WEIGHT = 3;  // measured: a walk emission costs ~2.5 combine probes (R-MAT 2^22)

__global__ void k_column_costs(const long long *__restrict__ walk_pre, const long long *__restrict__ csc_ptr,
                               const int *__restrict__ csc_rows, const long long *__restrict__ row_ptr, long long n,
                               long long steps, int mode, long long *__restrict__ cost) {
    const long long c = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (c >= n) return;
    const long long nc = walk_pre[c + 1] - walk_pre[c];
    if (mode == 0 || nc == 0) {
        if (lane == 0) cost[c] = nc;
        return;
    }
    const long long m = nc * steps;
    long long acc = 0;
    for (long long e = csc_ptr[c] + lane; e < csc_ptr[c + 1]; e += 32) {
        const int i = __ldg(csc_rows + e);
        const long long d = __ldg(row_ptr + i + 1) - __ldg(row_ptr + i);
        acc += d < m ? d : m;
    }
    acc = warp_sum_ll(acc);
    if (lane == 0) cost[c] = DIAG_WALK_WEIGHT * m + acc;
}

}  // namespace mcf

extern "C" int mcf_column_costs(mcf_graph *g, const int64_t *walk_pre, int64_t max_steps, int mode, int64_t *cost,
                                void *stream) {
    MCF_ARG(g && walk_pre && cost, "mcf_column_costs: null argument");
    MCF_ARG(mode == 0 || mode == 1, "mcf_column_costs: mode must be 0 (action) or 1 (diag)");
    MCF_ARG(max_steps >= 1, "mcf_column_costs: max_steps must be at least 1");
    if (g->n == 0) return MCF_OK;
    const long long steps = max_steps + 1;
    mcf::k_column_costs<<<(unsigned)((g->n * 32 + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
        (const long long *)walk_pre, (const long long *)g->csc_ptr, g->csc_rows, (const long long *)g->row_ptr, g->n,
        steps, mode, (long long *)cost);
    mcf::note_launch();
    MCF_LAUNCHED("k_column_costs");
    return MCF_OK;
}
