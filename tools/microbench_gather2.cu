// Gather tuning microbench: items per thread, cache hints, u32/f64, window sizes.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <random>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

template <class T, int ITEMS, int HINT>
__global__ void __launch_bounds__(256) gatherN(const T* __restrict__ in, const uint32_t* __restrict__ idx, T* __restrict__ out, uint64_t n) {
    const uint64_t base = (blockIdx.x * 256ull) * ITEMS + threadIdx.x;
    uint32_t d[ITEMS];
    T v[ITEMS];
#pragma unroll
    for (int k = 0; k < ITEMS; ++k) { uint64_t i = base + k * 256ull; d[k] = i < n ? __ldcs(idx + i) : 0; }
#pragma unroll
    for (int k = 0; k < ITEMS; ++k) {
        uint64_t i = base + k * 256ull;
        if (i < n) v[k] = HINT == 0 ? in[d[k]] : (HINT == 1 ? __ldg(in + d[k]) : __ldcg(in + d[k]));
    }
#pragma unroll
    for (int k = 0; k < ITEMS; ++k) { uint64_t i = base + k * 256ull; if (i < n) __stcs(out + i, v[k]); }
}

int main() {
    const uint64_t n = 134217728ull;
    std::vector<uint32_t> h(n);
    std::mt19937_64 rng(1);
    double* din; double* dout; uint32_t* didx;
    CK(cudaMalloc(&din, n * 8)); CK(cudaMalloc(&dout, n * 8)); CK(cudaMalloc(&didx, n * 4));
    CK(cudaMemset(din, 1, n * 8));
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    auto timeit = [&](auto launch, const char* name, double bytes) {
        launch(); cudaDeviceSynchronize();
        float best = 1e9;
        for (int r = 0; r < 5; ++r) {
            cudaEventRecord(a); launch(); cudaEventRecord(b); cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b); best = std::min(best, ms);
        }
        printf("%-55s %8.3f ms  %7.1f GB/s(useful)\n", name, best, bytes / best / 1e6);
    };
    for (uint64_t W : std::vector<uint64_t>{1ull << 20, 1ull << 21, 1ull << 23, 1ull << 24, n}) {
        for (uint64_t s = 0; s < n; s += W) {
            uint64_t e = std::min(n, s + W);
            for (uint64_t i = s; i < e; ++i) h[i] = (uint32_t)i;
            std::shuffle(h.begin() + s, h.begin() + e, rng);
        }
        CK(cudaMemcpy(didx, h.data(), n * 4, cudaMemcpyHostToDevice));
        char nm[128];
#define RUN(T, IT, HI, BYTES) \
        snprintf(nm, sizeof nm, "gather %s items=%d hint=%d window %llu", #T, IT, HI, (unsigned long long)W); \
        timeit([&] { gatherN<T, IT, HI><<<(unsigned)((n + 256 * IT - 1) / (256 * IT)), 256>>>((const T*)din, didx, (T*)dout, n); }, nm, BYTES * n);
        RUN(double, 1, 0, 20.0) RUN(double, 4, 0, 20.0) RUN(double, 8, 0, 20.0) RUN(double, 8, 1, 20.0) RUN(double, 8, 2, 20.0)
        RUN(uint32_t, 1, 0, 12.0) RUN(uint32_t, 8, 0, 12.0) RUN(uint32_t, 8, 2, 12.0)
    }
    return 0;
}
