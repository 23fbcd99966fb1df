// Random-sector micro-benchmark: the practical ceiling
// for the walk kernel's access pattern on this GPU.
//   indep : every thread issues K independent random 32-B sector loads
//   chain : every thread follows a dependent chain through a random
//           permutation of 32-B records (a walk step is such a dependency)
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/gups tools/gups.cu
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t mix(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

struct __align__(32) Rec {
    unsigned next;
    unsigned pad[7];
};

__global__ void k_init(Rec *r, unsigned long long n, unsigned long long mult, unsigned long long add) {
    for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < n;
         i += (unsigned long long)gridDim.x * blockDim.x) {
        // affine permutation of [0, n) (n power of two, mult odd) -> random-looking successor
        r[i].next = (unsigned)((i * mult + add) & (n - 1));
        for (int k = 1; k < 8; ++k) r[i].pad[k - 1] = (unsigned)i;
    }
}

enum { LD_NC = 0, LD_CA = 1, LD_CG = 2, LD_CS = 3, LD_V4NC = 4, LD_V4CG = 5 };

template <int MODE>
__device__ __forceinline__ unsigned ld(const Rec *p) {
    unsigned v;
    if (MODE == LD_NC) return __ldg(&p->next);
    if (MODE == LD_CA) asm volatile("ld.global.ca.u32 %0, [%1];" : "=r"(v) : "l"(&p->next));
    if (MODE == LD_CG) asm volatile("ld.global.cg.u32 %0, [%1];" : "=r"(v) : "l"(&p->next));
    if (MODE == LD_CS) asm volatile("ld.global.cs.u32 %0, [%1];" : "=r"(v) : "l"(&p->next));
    if (MODE == LD_V4NC) { int4 a = __ldg(reinterpret_cast<const int4 *>(p)); int4 b = __ldg(reinterpret_cast<const int4 *>(p) + 1); v = a.x + b.w; }
    if (MODE == LD_V4CG) {
        int4 a, b;
        asm volatile("ld.global.cg.v4.s32 {%0,%1,%2,%3}, [%4];" : "=r"(a.x), "=r"(a.y), "=r"(a.z), "=r"(a.w) : "l"(p));
        asm volatile("ld.global.cg.v4.s32 {%0,%1,%2,%3}, [%4+16];" : "=r"(b.x), "=r"(b.y), "=r"(b.z), "=r"(b.w) : "l"(p));
        v = a.x + b.w;
    }
    return v;
}

template <int MODE>
__global__ void k_chain_mode(const Rec *r, unsigned long long n, int steps, unsigned *out) {
    unsigned long long t = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x;
    unsigned p = (unsigned)(mix(t) & (n - 1));
    for (int s = 0; s < steps; ++s) p = ld<MODE>(&r[p]) & (unsigned)(n - 1);
    if (p == 0x12345678u) out[0] = p;
}

template <int K>
__global__ void k_indep(const Rec *r, unsigned long long n, int iters, unsigned *out) {
    unsigned long long t = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x;
    unsigned acc = 0;
    for (int it = 0; it < iters; ++it) {
        unsigned v[K];
#pragma unroll
        for (int k = 0; k < K; ++k) v[k] = __ldg(&r[mix(t * 1315423911ull + it * K + k) & (n - 1)].next);
#pragma unroll
        for (int k = 0; k < K; ++k) acc += v[k];
    }
    if (acc == 0x12345678u) out[0] = acc;
}

template <int NW>
__global__ void k_chain(const Rec *r, unsigned long long n, int steps, unsigned *out) {
    unsigned long long t = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x;
    unsigned p[NW];
#pragma unroll
    for (int w = 0; w < NW; ++w) p[w] = (unsigned)(mix(t * NW + w) & (n - 1));
    for (int s = 0; s < steps; ++s) {
#pragma unroll
        for (int w = 0; w < NW; ++w) p[w] = __ldg(&r[p[w]].next);
    }
    unsigned acc = 0;
#pragma unroll
    for (int w = 0; w < NW; ++w) acc += p[w];
    if (acc == 0x12345678u) out[0] = acc;
}

template <class F>
float timeit(F f) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    f();
    cudaDeviceSynchronize();
    cudaEventRecord(a);
    f();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    return ms;
}

int main(int argc, char **argv) {
    if (argc > 1) {  // L2 fetch granularity hint in bytes (32, 64, 128)
        size_t gran = (size_t)atoi(argv[1]);
        cudaError_t e = cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, gran);
        size_t got = 0;
        cudaDeviceGetLimit(&got, cudaLimitMaxL2FetchGranularity);
        printf("L2 fetch granularity: requested %zu -> %s, now %zu\n", gran, cudaGetErrorString(e), got);
    }
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    unsigned *out;
    cudaMalloc(&out, 4);
    for (unsigned long long bytes : {64ull << 20, 4ull << 30, 16ull << 30}) {
        unsigned long long n = bytes / sizeof(Rec);
        Rec *r;
        if (cudaMalloc(&r, n * sizeof(Rec)) != cudaSuccess) { printf("alloc failed\n"); return 1; }
        k_init<<<sms * 8, 256>>>(r, n, 0x9E3779B97F4A7C15ull | 1ull, 12345);
        cudaDeviceSynchronize();
        int threads = sms * 2048;
        int iters = 64;
        float ms = timeit([&] { k_indep<8><<<threads / 256, 256>>>(r, n, iters, out); });
        double loads = (double)threads * iters * 8;
        printf("%6llu MB indep  : %7.2f G sectors/s  (%7.1f GB/s of 32-B sectors)\n", bytes >> 20,
               loads / ms / 1e6, loads * 32 / ms / 1e6);
        for (int occ : {2048, 1024}) {
            int th = sms * occ;
            int steps = 256;
            float m1 = timeit([&] { k_chain<1><<<th / 256, 256>>>(r, n, steps, out); });
            float m2 = timeit([&] { k_chain<2><<<th / 256, 256>>>(r, n, steps, out); });
            float m4 = timeit([&] { k_chain<4><<<th / 256, 256>>>(r, n, steps, out); });
            double st = (double)th * steps;
            printf("%6llu MB chain thr/SM=%d: NW=1 %6.2f  NW=2 %6.2f  NW=4 %6.2f  G dependent loads/s\n", bytes >> 20,
                   occ, st / m1 / 1e6, 2 * st / m2 / 1e6, 4 * st / m4 / 1e6);
        }
        {
            int th = sms * 2048, steps = 256;
            double st = (double)th * steps;
            float a0 = timeit([&] { k_chain_mode<LD_NC><<<th / 256, 256>>>(r, n, steps, out); });
            float a1 = timeit([&] { k_chain_mode<LD_CA><<<th / 256, 256>>>(r, n, steps, out); });
            float a2 = timeit([&] { k_chain_mode<LD_CG><<<th / 256, 256>>>(r, n, steps, out); });
            float a3 = timeit([&] { k_chain_mode<LD_CS><<<th / 256, 256>>>(r, n, steps, out); });
            float a4 = timeit([&] { k_chain_mode<LD_V4NC><<<th / 256, 256>>>(r, n, steps, out); });
            float a5 = timeit([&] { k_chain_mode<LD_V4CG><<<th / 256, 256>>>(r, n, steps, out); });
            printf("%6llu MB chain by load kind (G loads/s): nc %.2f  ca %.2f  cg %.2f  cs %.2f  2xv4.nc %.2f  2xv4.cg %.2f\n",
                   bytes >> 20, st / a0 / 1e6, st / a1 / 1e6, st / a2 / 1e6, st / a3 / 1e6, st / a4 / 1e6, st / a5 / 1e6);
        }
        cudaFree(r);
    }
    return 0;
}
