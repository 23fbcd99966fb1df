// Phase timing of the single-pass scan structure (variants of k_alloc_scan's
// body): full / no look-back / no loads / no stores.
#include "../paper_2308_01037_b200/csrc/mcf_alloc.cu"
#include <cstdio>
using namespace mcf;

template <int V>  // 0 full, 1 no lookback, 2 no loads, 3 no stores
__global__ void __launch_bounds__(SCAN_T, 2) k_var(const unsigned long long *__restrict__ key, long long n,
                                                   const long long *__restrict__ ni_in, long long *__restrict__ ni,
                                                   long long *__restrict__ walk_pre, unsigned long long *sa,
                                                   unsigned long long *sb, unsigned *tile_ctr) {
    __shared__ unsigned s_tile;
    if (threadIdx.x == 0) s_tile = atomicAdd(tile_ctr, 1u);
    __syncthreads();
    const long long tile = s_tile;
    const unsigned long long T = 1002;
    const long long I = 7;
    const long long base = tile * SCAN_TILE + (long long)(threadIdx.x >> 5) * 32 * SCAN_I + (threadIdx.x & 31);
    long long a[SCAN_I], b[SCAN_I], ea[SCAN_I], eb[SCAN_I];
#pragma unroll
    for (int k = 0; k < SCAN_I; ++k) {
        const long long j = base + 32 * k;
        a[k] = b[k] = 0;
        if (j < n) {
            const unsigned long long kj = V == 2 ? (unsigned long long)j : key[j];
            a[k] = (V == 2 ? 1 : ni_in[j]) + (kj > T ? 1 : 0);
            b[k] = kj == T ? 1 : 0;
        }
    }
    tile_scan<true>(V == 1 ? 0 : tile, a, b, ea, eb, sa + (V == 1 ? tile : 0), sb + (V == 1 ? tile : 0));
    if (V == 3 && ea[0] != -5) return;
#pragma unroll
    for (int k = 0; k < SCAN_I; ++k) {
        const long long j = base + 32 * k;
        if (j < n) {
            ni[j] = a[k] + ((b[k] && eb[k] < I) ? 1 : 0);
            walk_pre[j] = ea[k] + (eb[k] < I ? eb[k] : I);
        }
    }
}

template <int V>
float run(long long n, const unsigned long long *key, const long long *nin, long long *ni, long long *wp,
          unsigned long long *status, cudaStream_t s) {
    const long long tiles = (n + SCAN_TILE - 1) / SCAN_TILE;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float best = 1e9;
    for (int rep = 0; rep < 5; ++rep) {
        cudaMemsetAsync(status, 0, 8 * (2 * tiles + 2), s);
        cudaEventRecord(a, s);
        k_var<V><<<(unsigned)tiles, SCAN_T, 0, s>>>(key, n, nin, ni, wp, status, status + tiles,
                                                   (unsigned *)(status + 2 * tiles));
        cudaEventRecord(b, s);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        best = ms < best ? ms : best;
    }
    return best * 1e3;
}

int main() {
    cudaStream_t s;
    cudaStreamCreate(&s);
    for (long long n : {1ll << 12, 1000000ll, 1ll << 24}) {
        long long *ni, *nin, *wp;
        unsigned long long *key, *status;
        cudaMalloc(&ni, 8 * (n + 1));
        cudaMalloc(&nin, 8 * (n + 1));
        cudaMalloc(&wp, 8 * (n + 1));
        cudaMalloc(&key, 8 * (n + 1));
        cudaMemset(nin, 0, 8 * n);
        cudaMemset(key, 0, 8 * n);
        const long long tiles = (n + SCAN_TILE - 1) / SCAN_TILE;
        cudaMalloc(&status, 8 * (2 * tiles + 2));
        printf("n=%lld: full %.1f  no-lookback %.1f  no-loads %.1f  no-stores %.1f us  (%s)\n", n,
               run<0>(n, key, nin, ni, wp, status, s), run<1>(n, key, nin, ni, wp, status, s),
               run<2>(n, key, nin, ni, wp, status, s), run<3>(n, key, nin, ni, wp, status, s),
               cudaGetErrorString(cudaGetLastError()));
        cudaFree(ni); cudaFree(nin); cudaFree(wp); cudaFree(key); cudaFree(status);
    }
    return 0;
}
