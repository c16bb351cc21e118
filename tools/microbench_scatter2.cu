// Residual-code transposition microbench (k_resid_codes design question):
// int16 lattice indices KE in layout E (epochs of 2^22 vertices, random
// permutation inside each epoch) -> vertex-order codes q_i = K_i - K_{i-1}.
//   A  gather  : codes[i] = zz(KE[dst[i]] - KE[dst[i-1]])  (the current kernel's access pattern)
//   B  scatter : Kv[src[p]] = KE[p] (window-local 2-byte stores), then a coalesced pass over Kv
//   B2 scatter with 4-byte stores of pairs is impossible (random), so B also tries .cs stores
// Prints the best of 5 for each.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <random>
#include <vector>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ uint16_t zz16(int32_t v) { return (uint16_t)((v << 1) ^ (v >> 31)); }

__global__ void __launch_bounds__(256) k_gather(const int16_t* __restrict__ KE, const uint32_t* __restrict__ dst,
                                               uint16_t* __restrict__ codes, uint64_t n) {
    const uint64_t first = (blockIdx.x * 256ull + threadIdx.x) * 8;
    if (first >= n) return;
    uint32_t d[8];
    for (int k = 0; k < 8; ++k) d[k] = first + k < n ? dst[first + k] : 0;
    int32_t prev = first ? (int32_t)__ldcg(&KE[dst[first - 1]]) : 0;
    int32_t K[8];
    for (int k = 0; k < 8; ++k) K[k] = (int32_t)__ldcg(&KE[d[k]]);
    uint16_t v[8];
    for (int k = 0; k < 8; ++k) { v[k] = zz16(K[k] - prev); prev = K[k]; }
    *reinterpret_cast<uint4*>(codes + first) = make_uint4(v[0] | (v[1] << 16), v[2] | (v[3] << 16), v[4] | (v[5] << 16),
                                                          v[6] | (v[7] << 16));
}

template <int CS>
__global__ void __launch_bounds__(256) k_scatter(const int16_t* __restrict__ KE, const uint32_t* __restrict__ src,
                                                int16_t* __restrict__ Kv, uint64_t n) {
    const uint64_t base = (blockIdx.x * 256ull) * 8 + threadIdx.x;
    uint32_t s[8];
    int16_t k[8];
    for (int j = 0; j < 8; ++j) {
        const uint64_t p = base + j * 256ull;
        s[j] = p < n ? __ldcs(src + p) : 0;
        k[j] = p < n ? __ldcs(KE + p) : 0;
    }
    for (int j = 0; j < 8; ++j) {
        const uint64_t p = base + j * 256ull;
        if (p < n) {
            if (CS) __stcg(Kv + s[j], k[j]);
            else Kv[s[j]] = k[j];
        }
    }
}

__global__ void __launch_bounds__(256) k_stream(const int16_t* __restrict__ Kv, uint16_t* __restrict__ codes, uint64_t n) {
    const uint64_t first = (blockIdx.x * 256ull + threadIdx.x) * 8;
    if (first >= n) return;
    const uint4 a = *reinterpret_cast<const uint4*>(Kv + first);
    int32_t prev = first ? (int32_t)Kv[first - 1] : 0;
    const int16_t* K = reinterpret_cast<const int16_t*>(&a);
    uint16_t v[8];
    for (int k = 0; k < 8; ++k) { v[k] = zz16((int32_t)K[k] - prev); prev = K[k]; }
    *reinterpret_cast<uint4*>(codes + first) = make_uint4(v[0] | (v[1] << 16), v[2] | (v[3] << 16), v[4] | (v[5] << 16),
                                                          v[6] | (v[7] << 16));
}

int main() {
    const uint64_t n = 134217728ull, W = 1ull << 22;
    std::vector<uint32_t> src(n), dst(n);
    std::mt19937_64 rng(7);
    for (uint64_t s = 0; s < n; s += W) {
        for (uint64_t i = s; i < s + W; ++i) src[i] = (uint32_t)i;
        std::shuffle(src.begin() + s, src.begin() + s + W, rng);
    }
    for (uint64_t p = 0; p < n; ++p) dst[src[p]] = (uint32_t)p;
    int16_t *KE, *Kv;
    uint32_t *dsrc, *ddst;
    uint16_t *c1, *c2;
    CK(cudaMalloc(&KE, n * 2)); CK(cudaMalloc(&Kv, n * 2)); CK(cudaMalloc(&dsrc, n * 4)); CK(cudaMalloc(&ddst, n * 4));
    CK(cudaMalloc(&c1, n * 2)); CK(cudaMalloc(&c2, n * 2));
    std::vector<int16_t> hk(n);
    for (uint64_t i = 0; i < n; ++i) hk[i] = (int16_t)((rng() % 20001) - 10000);
    CK(cudaMemcpy(KE, hk.data(), n * 2, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dsrc, src.data(), n * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(ddst, dst.data(), n * 4, cudaMemcpyHostToDevice));
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    auto timeit = [&](auto launch, const char* name) {
        launch();
        cudaDeviceSynchronize();
        float best = 1e9;
        for (int r = 0; r < 5; ++r) {
            cudaEventRecord(a);
            launch();
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            best = std::min(best, ms);
        }
        printf("%-48s %8.3f ms\n", name, best);
    };
    const unsigned g8 = (unsigned)(n / 8 / 256);
    timeit([&] { k_gather<<<g8, 256>>>(KE, ddst, c1, n); }, "A gather KE[dst[i]] (current pattern)");
    timeit([&] { k_scatter<0><<<g8, 256>>>(KE, dsrc, Kv, n); }, "B1 scatter Kv[src[p]] = KE[p]");
    timeit([&] { k_scatter<1><<<g8, 256>>>(KE, dsrc, Kv, n); }, "B1 scatter .cg");
    timeit([&] { k_stream<<<g8, 256>>>(Kv, c2, n); }, "B2 stream Kv -> codes");
    timeit([&] { k_scatter<0><<<g8, 256>>>(KE, dsrc, Kv, n); k_stream<<<g8, 256>>>(Kv, c2, n); }, "B total");
    std::vector<uint16_t> h1(n), h2(n);
    CK(cudaMemcpy(h1.data(), c1, n * 2, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(h2.data(), c2, n * 2, cudaMemcpyDeviceToHost));
    printf("codes equal: %d\n", (int)(h1 == h2));
    return 0;
}
