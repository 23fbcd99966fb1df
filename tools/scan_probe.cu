// Timing probe for the single-pass scans (k_scan, k_alloc_scan) in isolation.
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -rdc=true -o tools/scan_probe \
//   tools/scan_probe.cu paper_2308_01037_b200/csrc/mcf_util.cu paper_2308_01037_b200/csrc/mcf_graph.cu \
//   paper_2308_01037_b200/csrc/mcf_walk.cu paper_2308_01037_b200/csrc/mcf_diag.cu paper_2308_01037_b200/csrc/mcf_capi.cu
#include "../paper_2308_01037_b200/csrc/mcf_alloc.cu"
#include <cstdio>
#include <vector>

using namespace mcf;

__global__ void k_empty() {}

int main() {
    cudaStream_t s;
    cudaStreamCreate(&s);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    {  // event overhead
        float me = 1e9, ms;
        for (int r = 0; r < 5; ++r) {
            cudaEventRecord(a, s);
            k_empty<<<1, 32, 0, s>>>();
            cudaEventRecord(b, s);
            cudaEventSynchronize(b);
            cudaEventElapsedTime(&ms, a, b);
            me = ms < me ? ms : me;
        }
        printf("empty kernel %.1f us\n", me * 1e3);
    }
    for (long long n : {1ll << 12, 1ll << 16, 1ll << 20, 1000000ll, 1ll << 22, 1ll << 24}) {
        long long *in, *out, *ni, *wp;
        unsigned long long *key;
        AllocState *st;
        cudaMalloc(&in, 8 * (n + 1));
        cudaMalloc(&out, 8 * (n + 1));
        cudaMalloc(&ni, 8 * (n + 1));
        cudaMalloc(&wp, 8 * (n + 1));
        cudaMalloc(&key, 8 * (n + 1));
        cudaMalloc(&st, sizeof(AllocState));
        std::vector<long long> h(n);
        std::vector<unsigned long long> hk(n);
        for (long long i = 0; i < n; ++i) {
            h[i] = i % 7;
            hk[i] = 1000 + (i * 2654435761ull) % 5;
        }
        cudaMemcpy(in, h.data(), 8 * n, cudaMemcpyHostToDevice);
        cudaMemcpy(key, hk.data(), 8 * n, cudaMemcpyHostToDevice);
        AllocState hs{};
        hs.bstar = 3;
        hs.T = 1002;
        hs.I = n / 10;
        cudaMemcpy(st, &hs, sizeof(hs), cudaMemcpyHostToDevice);
        const long long tiles = (n + SCAN_TILE - 1) / SCAN_TILE;
        unsigned long long *status;
        cudaMalloc(&status, 8 * (2 * tiles + 2));
        float ms1 = 1e9, ms2 = 1e9, ms;
        for (int rep = 0; rep < 5; ++rep) {
            cudaMemcpyAsync(ni, in, 8 * n, cudaMemcpyDeviceToDevice, s);
            cudaEventRecord(a, s);
            exclusive_scan_i64(in, out, n, s);
            cudaEventRecord(b, s);
            cudaEventSynchronize(b);
            cudaEventElapsedTime(&ms, a, b);
            ms1 = ms < ms1 ? ms : ms1;
            cudaMemsetAsync(status, 0, 8 * (2 * tiles + 2), s);
            cudaEventRecord(a, s);
            k_alloc_scan<<<(unsigned)tiles, SCAN_T, 0, s>>>(key, n, st, ni, wp, nullptr, status, status + tiles,
                                                           (unsigned *)(status + 2 * tiles));
            cudaEventRecord(b, s);
            cudaEventSynchronize(b);
            cudaEventElapsedTime(&ms, a, b);
            ms2 = ms < ms2 ? ms : ms2;
        }
        std::vector<long long> hw(n + 1), ho(n + 1);
        cudaMemcpy(hw.data(), wp, 8 * (n + 1), cudaMemcpyDeviceToHost);
        cudaMemcpy(ho.data(), out, 8 * (n + 1), cudaMemcpyDeviceToHost);
        // check both against the host
        long long run = 0, ties = 0, runa = 0;
        bool ok1 = true, ok2 = true;
        for (long long i = 0; i < n; ++i) {
            ok1 &= ho[i] == run;
            run += h[i];
            const bool t = hk[i] == 1002;
            const long long aa = h[i] + (hk[i] > 1002 ? 1 : 0);
            ok2 &= hw[i] == runa + std::min(ties, (long long)hs.I);
            runa += aa;
            ties += t;
        }
        printf("n=%lld tiles=%lld  k_scan %.1f us (%s)  k_alloc_scan %.1f us (%s)  err=%s\n", n, tiles, ms1 * 1e3,
               ok1 ? "ok" : "BAD", ms2 * 1e3, ok2 ? "ok" : "BAD", cudaGetErrorString(cudaGetLastError()));
        cudaFree(in); cudaFree(out); cudaFree(ni); cudaFree(wp); cudaFree(key); cudaFree(st); cudaFree(status);
    }
    return 0;
}
