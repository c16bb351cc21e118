// Microbenchmark: scattered reads/writes on B200 under different locality
// windows (design input for the partitioned compress path).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb tools/microbench_scatter.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <random>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

template <class T>
__global__ void gather(const T* __restrict__ in, const uint32_t* __restrict__ idx, T* __restrict__ out, uint64_t n) {
    uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i < n) out[i] = in[idx[i]];
}
template <class T>
__global__ void scatter(const T* __restrict__ in, const uint32_t* __restrict__ idx, T* __restrict__ out, uint64_t n) {
    uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i < n) out[idx[i]] = in[i];
}
template <class T>
__global__ void copyk(const T* __restrict__ in, T* __restrict__ out, uint64_t n) {
    uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i < n) out[i] = in[i];
}
// scatter with streaming hints on the read side
template <class T>
__global__ void scatter_hint(const T* __restrict__ in, const uint32_t* __restrict__ idx, T* __restrict__ out, uint64_t n) {
    uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i < n) {
        T v = __ldcs(in + i);
        uint32_t d = __ldcs(idx + i);
        out[d] = v;
    }
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
        printf("%-50s %8.3f ms  %7.1f GB/s(useful)\n", name, best, bytes / best / 1e6);
    };
    const unsigned G = (unsigned)((n + 255) / 256);
    timeit([&] { copyk<double><<<G, 256>>>(din, dout, n); }, "copy f64", 16.0 * n);
    // windows: permutation within blocks of W elements
    for (uint64_t W : std::vector<uint64_t>{1ull << 12, 1ull << 16, 1ull << 20, 1ull << 22, 1ull << 24, n}) {
        for (uint64_t s = 0; s < n; s += W) {
            uint64_t e = std::min(n, s + W);
            for (uint64_t i = s; i < e; ++i) h[i] = (uint32_t)i;
            std::shuffle(h.begin() + s, h.begin() + e, rng);
        }
        CK(cudaMemcpy(didx, h.data(), n * 4, cudaMemcpyHostToDevice));
        char nm[128];
        snprintf(nm, sizeof nm, "gather  f64 window %llu", (unsigned long long)W);
        timeit([&] { gather<double><<<G, 256>>>(din, didx, dout, n); }, nm, 20.0 * n);
        snprintf(nm, sizeof nm, "scatter f64 window %llu", (unsigned long long)W);
        timeit([&] { scatter<double><<<G, 256>>>(din, didx, dout, n); }, nm, 20.0 * n);
        snprintf(nm, sizeof nm, "scatter f64 window %llu (ldcs)", (unsigned long long)W);
        timeit([&] { scatter_hint<double><<<G, 256>>>(din, didx, dout, n); }, nm, 20.0 * n);
        snprintf(nm, sizeof nm, "gather  u32 window %llu", (unsigned long long)W);
        timeit([&] { gather<uint32_t><<<G, 256>>>((uint32_t*)din, didx, (uint32_t*)dout, n); }, nm, 12.0 * n);
        snprintf(nm, sizeof nm, "scatter u32 window %llu", (unsigned long long)W);
        timeit([&] { scatter<uint32_t><<<G, 256>>>((uint32_t*)din, didx, (uint32_t*)dout, n); }, nm, 12.0 * n);
    }
    // bucket-major scatter: vertex i -> bucket b (random), position = rank within bucket (B buckets)
    for (uint64_t B : std::vector<uint64_t>{32768ull, 256ull * 1024}) {
        std::vector<uint32_t> cnt(B, 0), start(B + 1, 0);
        std::vector<uint32_t> bk(n);
        for (uint64_t i = 0; i < n; ++i) { bk[i] = (uint32_t)(rng() % B); cnt[bk[i]]++; }
        for (uint64_t q = 0; q < B; ++q) start[q + 1] = start[q] + cnt[q];
        std::fill(cnt.begin(), cnt.end(), 0);
        for (uint64_t i = 0; i < n; ++i) h[i] = start[bk[i]] + cnt[bk[i]]++;
        CK(cudaMemcpy(didx, h.data(), n * 4, cudaMemcpyHostToDevice));
        char nm[128];
        snprintf(nm, sizeof nm, "scatter f64 bucket-major B=%llu", (unsigned long long)B);
        timeit([&] { scatter<double><<<G, 256>>>(din, didx, dout, n); }, nm, 20.0 * n);
        // transposed: position = rank * B + bucket (row-major [k][b])
        std::fill(cnt.begin(), cnt.end(), 0);
        uint64_t kmax = 0;
        for (uint64_t q = 0; q < B; ++q) kmax = std::max<uint64_t>(kmax, start[q + 1] - start[q]);
        if (kmax * B <= n * 2) {
            double* dT; CK(cudaMalloc(&dT, kmax * B * 8));
            for (uint64_t i = 0; i < n; ++i) h[i] = (uint32_t)(cnt[bk[i]]++ * B + bk[i]);
            CK(cudaMemcpy(didx, h.data(), n * 4, cudaMemcpyHostToDevice));
            snprintf(nm, sizeof nm, "scatter f64 transposed [k][b] B=%llu", (unsigned long long)B);
            timeit([&] { scatter<double><<<G, 256>>>(din, didx, dT, n); }, nm, 20.0 * n);
            cudaFree(dT);
        }
        // epoch-blocked: E epochs of n/E vertices; within epoch bucket-major
        for (uint64_t E : std::vector<uint64_t>{16ull, 64ull}) {
            std::vector<uint32_t> ec(B);
            uint64_t per = (n + E - 1) / E;
            for (uint64_t e = 0; e < E; ++e) {
                uint64_t s = e * per, t = std::min(n, s + per);
                std::fill(ec.begin(), ec.end(), 0);
                for (uint64_t i = s; i < t; ++i) ec[bk[i]]++;
                std::vector<uint32_t> es(B + 1, 0);
                for (uint64_t q = 0; q < B; ++q) es[q + 1] = es[q] + ec[q];
                std::fill(ec.begin(), ec.end(), 0);
                for (uint64_t i = s; i < t; ++i) h[i] = (uint32_t)(s + es[bk[i]] + ec[bk[i]]++);
            }
            CK(cudaMemcpy(didx, h.data(), n * 4, cudaMemcpyHostToDevice));
            snprintf(nm, sizeof nm, "scatter f64 epoch-blocked E=%llu B=%llu", (unsigned long long)E, (unsigned long long)B);
            timeit([&] { scatter<double><<<G, 256>>>(din, didx, dout, n); }, nm, 20.0 * n);
            snprintf(nm, sizeof nm, "scatter u32 epoch-blocked E=%llu B=%llu", (unsigned long long)E, (unsigned long long)B);
            timeit([&] { scatter<uint32_t><<<G, 256>>>((uint32_t*)din, didx, (uint32_t*)dout, n); }, nm, 12.0 * n);
            snprintf(nm, sizeof nm, "gather  f64 epoch-blocked E=%llu B=%llu", (unsigned long long)E, (unsigned long long)B);
            timeit([&] { gather<double><<<G, 256>>>(din, didx, dout, n); }, nm, 20.0 * n);
        }
    }
    return 0;
}
