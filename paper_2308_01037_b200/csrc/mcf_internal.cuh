// Internal definitions shared by the libmcfunm_cuda kernels (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdlib>
#include <string>
#include <utility>
#include <vector>

#include "../../include/mcfunm_cuda.h"

#define MCF_FULL 0xffffffffu

// ---------------------------------------------------------------------------
// error plumbing (C ABI returns codes; message in a thread-local string)
// ---------------------------------------------------------------------------
namespace mcf {

void set_error(const std::string &msg);
int cuda_status(cudaError_t e, const char *what);
void note_launch();  // counts kernel launches (mcf_kernel_launches)

// Stream-ordered allocations released on every return path of a host driver
// (error returns included): frees run in reverse order on the stream.
struct AsyncFrees {
    cudaStream_t s;
    std::vector<void *> p;
    explicit AsyncFrees(cudaStream_t st) : s(st) {}
    template <class T>
    T *keep(T *x) {
        p.push_back((void *)x);
        return x;
    }
    ~AsyncFrees() {
        for (auto it = p.rbegin(); it != p.rend(); ++it)
            if (*it) cudaFreeAsync(*it, s);
    }
};

}  // namespace mcf

#define MCF_CUDA(call)                                                  \
    do {                                                                \
        cudaError_t e__ = (call);                                       \
        if (e__ != cudaSuccess) return mcf::cuda_status(e__, #call);    \
    } while (0)

#define MCF_LAUNCHED(what)                                              \
    do {                                                                \
        cudaError_t e__ = cudaGetLastError();                           \
        if (e__ != cudaSuccess) return mcf::cuda_status(e__, what);     \
    } while (0)

#define MCF_ARG(cond, msg)                                              \
    do {                                                                \
        if (!(cond)) {                                                  \
            mcf::set_error(msg);                                        \
            return MCF_ERR_ARGUMENT;                                    \
        }                                                               \
    } while (0)

// ---------------------------------------------------------------------------
// device graph
// ---------------------------------------------------------------------------
namespace mcf {

// Per-node header: one 32-byte sector holds everything a walk step needs
// about the current state besides the sampled entry itself.
enum : uint32_t {
    HDR_UNIFORM = 1u,   // all |a_ij| of the row equal -> sample by index
    HDR_HAS_NEG = 2u,   // row holds a negative value -> sign packed in ecol
    HDR_NEG_EDGE = 4u,  // walk-entry copy only: the entry's own value a_e < 0
};

struct __align__(32) NodeHdr {
    int start;        // row_ptr[i]  (nnz < 2^31)
    int deg;          // row_ptr[i+1] - row_ptr[i]
    uint32_t flags;
    uint32_t pad;     // walk-entry copy: the node id itself
    double rsum;      // sum_j |a_ij| in CSR order (= a/t magnitude, walker.py:124-125)
    double aux;       // per-call payload: r_i = (A v)_i for action walks
};
static_assert(sizeof(NodeHdr) == 32, "NodeHdr must be one sector");

}  // namespace mcf

struct mcf_graph {
    int64_t n = 0, nnz = 0;
    // caller-owned inputs
    const int64_t *row_ptr = nullptr;
    const int32_t *col_ids = nullptr;
    const double *vals = nullptr;
    const int64_t *csc_ptr = nullptr;
    const int32_t *csc_rows = nullptr;
    const double *csc_vals = nullptr;
    // owned device tables
    mcf::NodeHdr *hdr = nullptr;     // n
    int32_t *ecol = nullptr;         // nnz; col | (a<0)<<31 (aliases col_ids if no negatives)
    bool ecol_owned = false;
    double *cdf = nullptr;           // nnz within-row CDF (only if some row is non-uniform)
    // Walker/Vose alias tables of the non-uniform rows (device-RNG draws: one
    // dependent load per step instead of a log2(deg)-deep CDF search):
    // alias[e] = (alias index within the row << alias_tbits) | acceptance
    // threshold (alias_tbits-bit fixed point); alias index == own index: always taken
    unsigned long long *alias = nullptr;
    int alias_tbits = 0;
    bool l2_prefetch = false;        // compact tables fit L2: walk kernels bulk-prefetch them first
    double *col_norm = nullptr;      // n
    double *init_prob = nullptr;     // n
    int64_t *csr2csc = nullptr;      // nnz, lazily built for diag
    // "fat" walk layout: went[e] = hdr[col[e]] with pad = col[e] and the
    // entry's sign in flags, so a step reads ONE random 32-B sector instead of
    // two (entry, then the target's header).  32 B x nnz; used when the
    // compact tables would not stay in L2.
    mcf::NodeHdr *went = nullptr;
    // "lean" walk entries for v = 1 on uniform-value graphs: lean[e] = {start,
    // degree} of col[e].  With every |a| equal, a row's |a| sum -- the weight
    // factor, and for v = 1 also the payload r -- depends only on its degree
    // (rsum_by_deg), so a step is ONE dependent random 8-B load.  Built lazily.
    uint2 *lean = nullptr;
    uint32_t *lean4 = nullptr;       // 4-B variant for nnz < 2^25 (used instead of lean when built)
    // diag walks (the emitted state id is needed too): lean_id[e] packs
    // [deg : li_dbits | col[e] : li_ibits | start : li_sbits] of col[e] in 8 B,
    // so a step is one random load instead of the lean entry plus ecol[e];
    // deg = 2^li_dbits - 1 escapes to row_ptr (hub targets).  Built lazily.
    unsigned long long *lean_id = nullptr;
    int li_sbits = 0, li_ibits = 0, li_dbits = 0;
    double *rsum_by_deg = nullptr;   // max_degree + 1
    int *long_rows = nullptr;        // rows with degree > LONG_ROW (SpMV / table build bins)
    long long n_long_rows = 0;
    void *scratch = nullptr;
    // hub-row bitmaps for the diag combine (uniform-value graphs, built lazily)
    int *hub_of = nullptr;           // n: bitmap index of row i, or -1
    unsigned *hub_bits = nullptr;    // n_hubs x hub_words
    long long hub_words = 0;
    bool hubs_ready = false;
    // diag combine units (uniform-value graphs, built lazily): every CSC
    // column's row ids reordered by (key_group(id), id), so the unit that owns
    // a range of key groups finds its ids as one contiguous slice; columns
    // longer than GROUP_OFS_MIN keep their NGROUPS + 1 slice offsets
    int32_t *ckeys = nullptr;        // nnz
    int32_t *gidx = nullptr;         // n: offset-table row of a long column, or -1
    int32_t *gofs = nullptr;         // n_long x (NGROUPS + 1), relative to csc_ptr[c]
    long long n_gofs = 0;
    long long max_col_degree = 0;    // longest CSC column (set with ckeys): a unit's entry queue capacity
    bool uniform_value = false;      // all stored values equal `value` (0/1 graphs scaled by gamma)
    double value = 0.0;
    mcf_graph_info info{};
    int device = 0;
    // optional per-launch timing of the dominant kernels (MCF_FLAG_TIME_KERNELS)
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev_walk, ev_q;
    // side stream (per device, shared) + fork/join events (budgets computed concurrently with r = A v)
    cudaStream_t side = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
};

namespace mcf {

// ---------------------------------------------------------------------------
// Philox-4x32-10 counter-based RNG
// ---------------------------------------------------------------------------
struct U4 {
    uint32_t x, y, z, w;
};

__device__ __forceinline__ U4 philox4x32_10(U4 c, uint32_t k0, uint32_t k1) {
    const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
    const uint32_t W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        uint32_t hi0 = __umulhi(M0, c.x), lo0 = M0 * c.x;
        uint32_t hi1 = __umulhi(M1, c.z), lo1 = M1 * c.z;
        c = U4{hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0};
        k0 += W0;
        k1 += W1;
    }
    return c;
}

// 53-bit uniform in [0, 1)
__device__ __forceinline__ double u53(uint32_t hi, uint32_t lo) {
    uint64_t v = ((uint64_t)hi << 32) | lo;
    return (double)(v >> 11) * 0x1.0p-53;
}

// ---------------------------------------------------------------------------
// small device helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(MCF_FULL, v, o);
    return v;
}

__device__ __forceinline__ long long warp_sum_ll(long long v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(MCF_FULL, v, o);
    return v;
}

__device__ __forceinline__ int warp_sum_int(int v) { return __reduce_add_sync(MCF_FULL, v); }

__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// One 256-bit load (sm_100 LDG.E.ENL2.256): a random 32-B record costs one
// L1 wavefront instead of two for a pair of 128-bit loads -- the walk kernels
// are bound by L1 wavefronts per step.
__device__ __forceinline__ NodeHdr load_hdr(const NodeHdr *h) {
    int4 a, b;
    asm("ld.global.nc.L2::evict_normal.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
        : "=r"(a.x), "=r"(a.y), "=r"(a.z), "=r"(a.w), "=r"(b.x), "=r"(b.y), "=r"(b.z), "=r"(b.w)
        : "l"(h));
    NodeHdr r;
    r.start = a.x;
    r.deg = a.y;
    r.flags = (uint32_t)a.z;
    r.pad = (uint32_t)a.w;
    r.rsum = __hiloint2double(b.y, b.x);
    r.aux = __hiloint2double(b.w, b.z);
    return r;
}

// Key groups of the diag combine units: a node id's group is the top GROUP_BITS
// bits of a full-avalanche hash (independent of the table slot and Bloom
// hashes, which are multiplicative), so every group holds ~1/NGROUPS of any
// support set.  A column split into K units gives unit u the groups
// [u NGROUPS / K, (u + 1) NGROUPS / K).
constexpr int GROUP_BITS = 7;
constexpr int NGROUPS = 1 << GROUP_BITS;
constexpr int GROUP_OFS_MIN = 32;  // columns longer than this keep their group slice offsets
__device__ __forceinline__ uint32_t key_group(int key) {
    uint32_t h = (uint32_t)key;  // lowbias32
    h ^= h >> 16;
    h *= 0x7feb352du;
    h ^= h >> 15;
    h *= 0x846ca68bu;
    h ^= h >> 16;
    return h >> (32 - GROUP_BITS);
}

// rows longer than this get a CTA each in SpMV (load balance on hub rows)
constexpr int LONG_ROW = 64;

// column of global walk g: blk_col[g >> WALK_BLK_SHIFT] brackets the search
constexpr int WALK_BLK_SHIFT = 6;

// g is the global walk index, g_rel = g - walk_begin of the call, nw the
// number of walks in the call's range.
__device__ __forceinline__ int column_of_walk(long long g, long long g_rel, long long nw,
                                              const long long *__restrict__ walk_pre,
                                              const int *__restrict__ blk_col, int col_last) {
    long long b = g_rel >> WALK_BLK_SHIFT;
    int lo = __ldg(blk_col + b);
    int hi = ((b + 1) << WALK_BLK_SHIFT) < nw ? __ldg(blk_col + b + 1) : col_last;
    // find largest c in [lo, hi] with walk_pre[c] <= g
    while (lo < hi) {
        int mid = (lo + hi + 1) >> 1;
        if (__ldg(walk_pre + mid) <= g) lo = mid;
        else hi = mid - 1;
    }
    return lo;
}

// ---------------------------------------------------------------------------
// single-pass scans (decoupled look-back) without fences: each component of a
// tile's state is one 64-bit word flag | value (62 bits), ST_AGG = the tile's
// own total, ST_PRE = its inclusive prefix.  With two components (sa, sb) a
// reader accepts a pair only when both flags agree -- flags only move
// 0 -> AGG -> PRE and the value for each flag is fixed, so an agreeing pair is
// consistent without any release/acquire ordering.  One warp looks back 32
// tiles per round.  Tiles are warp-striped: element k of lane l
// in warp w is item tile * SCAN_TILE + w * 32 * SCAN_I + k * 32 + l, so every
// load and store is coalesced.
// ---------------------------------------------------------------------------
constexpr unsigned long long ST_AGG = 1ull << 62, ST_PRE = 2ull << 62, ST_VAL = (1ull << 62) - 1;
constexpr int SCAN_T = 512, SCAN_I = 8, SCAN_TILE = SCAN_T * SCAN_I, SCAN_W = SCAN_T / 32;

__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void st_relaxed_u64(unsigned long long *p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// inclusive warp scan
__device__ __forceinline__ long long warp_incl_scan(long long x) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const long long y = __shfl_up_sync(MCF_FULL, x, o);
        if (lane >= o) x += y;
    }
    return x;
}

// warp 0 of tile `tile` (> 0): exclusive prefix (pa, pb) over tiles < tile.
// 32 tiles per round (one per lane); a lane whose tile has not published yet
// polls it with a short back-off, so the status words (a few L2 lines every
// tile polls) are not flooded.
template <bool HAS_B>
__device__ __forceinline__ void lookback(long long tile, const unsigned long long *sa, const unsigned long long *sb,
                                         long long &pa, long long &pb) {
    const int lane = threadIdx.x & 31;
    pa = 0;
    pb = 0;
    for (long long t = tile - 1;; t -= 32) {
        const long long idx = t - lane;
        unsigned long long xa = ST_PRE, xb = ST_PRE;  // idx < 0: nothing
        if (idx >= 0) {
            unsigned ns = 32;
            while (true) {
                xa = ld_relaxed_u64(sa + idx);
                if (HAS_B) xb = ld_relaxed_u64(sb + idx);
                if ((xa & ~ST_VAL) && (!HAS_B || (xa & ~ST_VAL) == (xb & ~ST_VAL))) break;
                __nanosleep(ns);
                if (ns < 512) ns <<= 1;
            }
        }
        const unsigned pre = __ballot_sync(MCF_FULL, idx >= 0 && (xa & ST_PRE));
        const int f = pre ? __ffs(pre) - 1 : 32;  // nearest tile holding an inclusive prefix
        long long a = (idx >= 0 && lane <= f) ? (long long)(xa & ST_VAL) : 0;
        long long b = (HAS_B && idx >= 0 && lane <= f) ? (long long)(xb & ST_VAL) : 0;
        pa += warp_sum_ll(a);
        if (HAS_B) pb += warp_sum_ll(b);
        if (pre || t - 32 < 0) break;
    }
}

// Tile-level exclusive scan of one or two components held warp-striped
// (a[k], b[k] for k < SCAN_I).  On return ea[k] / eb[k] are the exclusive
// prefixes of the item over the whole array.  Two barriers; every thread of
// the SCAN_T-thread block calls it.
template <bool HAS_B>
__device__ __forceinline__ void tile_scan(long long tile, const long long (&a)[SCAN_I], const long long (&b)[SCAN_I],
                                          long long (&ea)[SCAN_I], long long (&eb)[SCAN_I], unsigned long long *sa,
                                          unsigned long long *sb) {
    __shared__ long long s_wa[SCAN_W], s_wb[SCAN_W];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    long long ca = 0, cb = 0;
#pragma unroll
    for (int k = 0; k < SCAN_I; ++k) {
        const long long xa = warp_incl_scan(a[k]);
        ea[k] = ca + xa - a[k];
        ca += __shfl_sync(MCF_FULL, xa, 31);
        if (HAS_B) {
            const long long xb = warp_incl_scan(b[k]);
            eb[k] = cb + xb - b[k];
            cb += __shfl_sync(MCF_FULL, xb, 31);
        }
    }
    if (lane == 0) {
        s_wa[w] = ca;
        if (HAS_B) s_wb[w] = cb;
    }
    __syncthreads();
    if (w == 0) {
        const long long va = lane < SCAN_W ? s_wa[lane] : 0, vb = (HAS_B && lane < SCAN_W) ? s_wb[lane] : 0;
        const long long ia = warp_incl_scan(va), ib = HAS_B ? warp_incl_scan(vb) : 0;
        const long long ta = __shfl_sync(MCF_FULL, ia, 31), tb = HAS_B ? __shfl_sync(MCF_FULL, ib, 31) : 0;
        long long pa = 0, pb = 0;
        if (tile == 0) {
            if (lane == 0) {
                st_relaxed_u64(sa, ST_PRE | (unsigned long long)ta);
                if (HAS_B) st_relaxed_u64(sb, ST_PRE | (unsigned long long)tb);
            }
        } else {
            if (lane == 0) {
                st_relaxed_u64(sa + tile, ST_AGG | (unsigned long long)ta);
                if (HAS_B) st_relaxed_u64(sb + tile, ST_AGG | (unsigned long long)tb);
            }
            lookback<HAS_B>(tile, sa, sb, pa, pb);
            if (lane == 0) {
                st_relaxed_u64(sa + tile, ST_PRE | (unsigned long long)(pa + ta));
                if (HAS_B) st_relaxed_u64(sb + tile, ST_PRE | (unsigned long long)(pb + tb));
            }
        }
        __syncwarp();
        if (lane < SCAN_W) {  // exclusive warp offsets, including the tile prefix
            s_wa[lane] = pa + ia - va;
            if (HAS_B) s_wb[lane] = pb + ib - vb;
        }
    }
    __syncthreads();
    const long long oa = s_wa[w], ob = HAS_B ? s_wb[w] : 0;
#pragma unroll
    for (int k = 0; k < SCAN_I; ++k) {
        ea[k] += oa;
        if (HAS_B) eb[k] += ob;
    }
}

// ---------------------------------------------------------------------------
// Peer-memory exchange (mcf_spmv_peer, mcf_diag_combine_peer): per-rank
// input buffers (local or mapped peer memory), each valid on the index range
// of the columns its rank owns, and the output buffers every result goes to.
// ---------------------------------------------------------------------------
constexpr int MAX_PEERS = 8;
struct PeerArgs {
    const double *x[MAX_PEERS];       // x[k]: valid where the column is in [bounds[k], bounds[k+1])
    long long bounds[MAX_PEERS + 1];  // column ranges of the parts
    int nparts;
    double *y[MAX_PEERS];             // every output buffer receives every row
    int nouts;
};

__device__ __forceinline__ int peer_owner(const PeerArgs &pa, long long col) {
    int k = 0;
#pragma unroll
    for (int t = 1; t < MAX_PEERS; ++t) k += (t < pa.nparts && col >= pa.bounds[t]) ? 1 : 0;
    return k;
}

// host: validate and pack the pointer lists (rc != 0 on bad arguments)
int make_peer_args(const double *const *x_parts, const long long *bounds, int nparts, double *const *y_outs,
                   int nouts, long long ncols, PeerArgs *pa);

// ---------------------------------------------------------------------------
// host helpers implemented in mcf_util.cu
// ---------------------------------------------------------------------------
int exclusive_scan_i64(const long long *in, long long *out, long long n, cudaStream_t s);
// single-pass scan over a device functor: out[i] = sum_{j<i} f(j), out[n] = total
struct ScanSrc {
    const long long *in;                       // plain input, or
    const unsigned long long *key;             // key[j] == *match ? 1 : 0
    const unsigned long long *match;
};
int scan_src(ScanSrc src, long long *out, long long n, cudaStream_t s);
int build_blk_col(const long long *walk_pre, long long col_begin, long long col_end, long long capacity,
                  int **blk_col, cudaStream_t s);
int ensure_csr2csc(mcf_graph *g, cudaStream_t s);
int ensure_hub_bitmaps(mcf_graph *g, cudaStream_t s);
int ensure_group_keys(mcf_graph *g, cudaStream_t s);
int ensure_side_stream(mcf_graph *g);
// r_ones/stats_zero (fused path only, see fused_alloc_applies): also write
// r = A 1 into r_ones and the headers, and zero stats_zero[4]
int allocate_walks(mcf_graph *g, long long n_walks, long long *ni, long long *walk_pre, int *blk_col,
                   cudaStream_t s, void *fused_scratch = nullptr, double *r_ones = nullptr,
                   long long *stats_zero = nullptr);
size_t fused_scratch_bytes();       // scratch of the one-kernel budget path
size_t fused_scratch_zero_bytes();  // its prefix that must be zero
bool fused_alloc_applies(const mcf_graph *g);
int column_batches(const long long *walk_pre, long long cb, long long ce, long long cap_walks,
                   std::vector<long long> &bounds, unsigned long long *max_walks, cudaStream_t s);
// largest walk count one walk launch takes (lane walk indices are int)
constexpr long long WALKS_PER_LAUNCH = (1ll << 31) - 4096;
int read_walk_range(const long long *walk_pre, long long col_begin, long long col_end,
                    long long *wb, long long *we, cudaStream_t s);
int sm_count();
// event pair around one launch of a timed kernel (no-op unless flag set)
int timed_begin(mcf_graph *g, bool on, std::vector<std::pair<cudaEvent_t, cudaEvent_t>> &v, cudaStream_t s);
int timed_end(bool on, std::vector<std::pair<cudaEvent_t, cudaEvent_t>> &v, cudaStream_t s);

}  // namespace mcf
