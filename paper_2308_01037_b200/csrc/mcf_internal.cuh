// Internal definitions shared by the libmcfunm_cuda kernels (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

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
    double *col_norm = nullptr;      // n
    double *init_prob = nullptr;     // n
    int64_t *csr2csc = nullptr;      // nnz, lazily built for diag
    // "fat" walk layout: went[e] = hdr[col[e]] with pad = col[e] and the
    // entry's sign in flags, so a step reads ONE random 32-B sector instead of
    // two (entry, then the target's header).  32 B x nnz; used when the
    // compact tables would not stay in L2.
    mcf::NodeHdr *went = nullptr;
    int *long_rows = nullptr;        // rows with degree > LONG_ROW (SpMV / table build bins)
    long long n_long_rows = 0;
    void *scratch = nullptr;
    // hub-row bitmaps for the diag combine (uniform-value graphs, built lazily)
    int *hub_of = nullptr;           // n: bitmap index of row i, or -1
    unsigned *hub_bits = nullptr;    // n_hubs x hub_words
    long long hub_words = 0;
    bool hubs_ready = false;
    bool uniform_value = false;      // all stored values equal `value` (0/1 graphs scaled by gamma)
    double value = 0.0;
    mcf_graph_info info{};
    int device = 0;
    // optional per-launch timing of the dominant kernels (MCF_FLAG_TIME_KERNELS)
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev_walk, ev_q;
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

__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

__device__ __forceinline__ NodeHdr load_hdr(const NodeHdr *h) {
    const int4 *p = reinterpret_cast<const int4 *>(h);
    int4 a = __ldg(p), b = __ldg(p + 1);
    NodeHdr r;
    r.start = a.x;
    r.deg = a.y;
    r.flags = (uint32_t)a.z;
    r.pad = (uint32_t)a.w;
    r.rsum = __hiloint2double(b.y, b.x);
    r.aux = __hiloint2double(b.w, b.z);
    return r;
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
int read_walk_range(const long long *walk_pre, long long col_begin, long long col_end,
                    long long *wb, long long *we, cudaStream_t s);
int sm_count();
// event pair around one launch of a timed kernel (no-op unless flag set)
int timed_begin(mcf_graph *g, bool on, std::vector<std::pair<cudaEvent_t, cudaEvent_t>> &v, cudaStream_t s);
int timed_end(bool on, std::vector<std::pair<cudaEvent_t, cudaEvent_t>> &v, cudaStream_t s);

}  // namespace mcf
