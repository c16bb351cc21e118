// Floor for the recompose gather: out[i] = fl(K16[node[i]] * b1) + fl(i * b2)
// with node[i] uniform random over 16.7M grid nodes (33 MB int16 table, L2
// resident), vs. the same with 2-byte and 4-byte tables, items per thread 8/16.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>
#include <algorithm>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ uint64_t pol_last() { uint64_t p; asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p)); return p; }
__device__ __forceinline__ uint64_t pol_first() { uint64_t p; asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p)); return p; }

template <class T, int ITEMS, bool HINT>
__global__ void __launch_bounds__(256) rec(const T* __restrict__ tab, const uint32_t* __restrict__ node, double* __restrict__ out, uint64_t n, double b1, double b2) {
    const uint64_t base = (blockIdx.x * 256ull) * ITEMS + threadIdx.x;
    const uint64_t pl = pol_last(), pf = pol_first();
    uint32_t d[ITEMS];
    int32_t g[ITEMS];
#pragma unroll
    for (int k = 0; k < ITEMS; ++k) { uint64_t i = base + k * 256ull; d[k] = i < n ? __ldcs(node + i) : 0; }
#pragma unroll
    for (int k = 0; k < ITEMS; ++k) {
        uint64_t i = base + k * 256ull;
        if (i < n) {
            if (HINT) {
                if (sizeof(T) == 2) { int16_t v; asm volatile("ld.global.nc.L2::cache_hint.s16 %0, [%1], %2;" : "=h"(v) : "l"(tab + d[k]), "l"(pl)); g[k] = v; }
                else { int32_t v; asm volatile("ld.global.nc.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(v) : "l"(tab + d[k]), "l"(pl)); g[k] = v; }
            } else g[k] = (int32_t)__ldg(tab + d[k]);
        }
    }
#pragma unroll
    for (int k = 0; k < ITEMS; ++k) {
        uint64_t i = base + k * 256ull;
        if (i < n) {
            double v = __dadd_rn(__dmul_rn((double)g[k], b1), __dmul_rn((double)(int32_t)i, b2));
            if (HINT) asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(out + i), "d"(v), "l"(pf) : "memory");
            else __stcs(out + i, v);
        }
    }
}

int main() {
    const uint64_t n = 134217728ull, n1 = 16777216ull;
    std::vector<uint32_t> h(n);
    std::mt19937_64 rng(1);
    for (uint64_t i = 0; i < n; ++i) h[i] = (uint32_t)(rng() % n1);
    void* tab; double* dout; uint32_t* dnode;
    CK(cudaMalloc(&tab, n1 * 4)); CK(cudaMalloc(&dout, n * 8)); CK(cudaMalloc(&dnode, n * 4));
    CK(cudaMemset(tab, 1, n1 * 4));
    CK(cudaMemcpy(dnode, h.data(), n * 4, cudaMemcpyHostToDevice));
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    auto timeit = [&](auto launch, const char* name) {
        launch(); cudaDeviceSynchronize();
        float best = 1e9;
        for (int r = 0; r < 5; ++r) {
            cudaEventRecord(a); launch(); cudaEventRecord(b); cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b); best = std::min(best, ms);
        }
        printf("%-40s %8.3f ms  %7.1f GB/s (12 B/item)\n", name, best, 12.0 * n / best / 1e6);
    };
#define RUN(T, IT, HI) timeit([&] { rec<T, IT, HI><<<(unsigned)((n + 256 * IT - 1) / (256 * IT)), 256>>>((const T*)tab, dnode, dout, n, 1e-3, 1e-5); }, #T " items=" #IT " hint=" #HI);
    RUN(int16_t, 4, false) RUN(int16_t, 8, false) RUN(int16_t, 16, false) RUN(int16_t, 8, true) RUN(int16_t, 16, true)
    RUN(int32_t, 8, false) RUN(int32_t, 8, true)
    // sorted nodes (perfectly local) for comparison
    std::sort(h.begin(), h.end());
    CK(cudaMemcpy(dnode, h.data(), n * 4, cudaMemcpyHostToDevice));
    RUN(int16_t, 8, true)
    return 0;
}
