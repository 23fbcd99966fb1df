// Phase timing of k_alloc_fused (CTA 0's view, %globaltimer) on a synthetic
// power-law p with many ties.  Build:
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -rdc=true -DMCF_ALLOC_TRACE \
//     -o tools/alloc_probe tools/alloc_probe.cu paper_2308_01037_b200/csrc/mcf_{util,graph,walk,diag,capi}.cu
#include "../paper_2308_01037_b200/csrc/mcf_alloc.cu"
#include <cmath>
#include <cstdio>
#include <random>
#include <vector>
using namespace mcf;

int main(int argc, char **argv) {
    long long n = 1000000;
    const long long nw = 640000;
    std::mt19937_64 rng(1);
    std::vector<double> p(n);
    double tot = 0;
    for (long long i = 0; i < n; ++i) {
        const double u = std::uniform_real_distribution<double>(0, 1)(rng);
        const int deg = 4 + (int)(4.0 / (u * u + 1e-6) > 5000 ? 5000 : 4.0 / (u * u + 1e-6)) - 4;
        p[i] = std::sqrt((double)(deg < 4 ? 4 : deg));
        tot += p[i];
    }
    for (auto &x : p) x /= tot;
    if (argc > 1) {  // p from a file (float64, e.g. a graph's init_prob)
        FILE *f = fopen(argv[1], "rb");
        fseek(f, 0, SEEK_END);
        n = ftell(f) / 8;
        fseek(f, 0, SEEK_SET);
        p.resize(n);
        if (fread(p.data(), 8, n, f) != (size_t)n) return 1;
        fclose(f);
    }
    double *dp;
    long long *ni, *wp;
    AllocFused *F;
    cudaMalloc(&dp, 8 * n);
    cudaMalloc(&ni, 8 * n);
    cudaMalloc(&wp, 8 * (n + 1));
    cudaMalloc(&F, sizeof(AllocFused));
    cudaMemcpy(dp, p.data(), 8 * n, cudaMemcpyHostToDevice);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const long long K = (n + (long long)sms * AF_T - 1) / ((long long)sms * AF_T);
    for (int rep = 0; rep < 3; ++rep) {
        cudaMemset(F, 0, sizeof(AllocFused));
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        cudaEventRecord(a);
        k_alloc_fused<<<sms, AF_T>>>(dp, n, (double)nw, nw, (int)K, F, ni, wp, nullptr, OnesR{nullptr, nullptr, nullptr, nullptr});
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        unsigned long long tr[32];
        cudaMemcpy(tr, F->trace, sizeof(tr), cudaMemcpyDeviceToHost);
        printf("last CTA level-1 done +%.1f, ", (tr[27] - tr[0]) / 1e3);
        printf("last CTA start +%.1f, last shared hist done +%.1f, last flush done +%.1f | ", (tr[28] - tr[0]) / 1e3,
               (tr[29] - tr[0]) / 1e3, (tr[30] - tr[0]) / 1e3);
        printf("K=%lld event %.1f us | phase1 %.1f  bar1 %.1f", K, ms * 1e3, (tr[1] - tr[0]) / 1e3, (tr[2] - tr[1]) / 1e3);
        unsigned long long prev = tr[2];
        for (int l = 1; l < 8; ++l)
            if (tr[2 + 2 * l]) {
                printf("  lvl%d %.1f bar %.1f", l, (tr[2 + 2 * l - 1] - prev) / 1e3, (tr[2 + 2 * l] - tr[2 + 2 * l - 1]) / 1e3);
                prev = tr[2 + 2 * l];
            }
        printf("  ->T %.1f  scan-local %.1f  bar %.1f  out %.1f  total %.1f us (%s)\n", (tr[20] - prev) / 1e3,
               (tr[21] - tr[20]) / 1e3, (tr[22] - tr[21]) / 1e3, (tr[23] - tr[22]) / 1e3, (tr[23] - tr[0]) / 1e3,
               cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
