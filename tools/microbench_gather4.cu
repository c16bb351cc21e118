// Random 2-byte gathers from a 16.7M-entry (L2-resident) int16 table with a
// streamed u32 index: LDG (one L1 tag lookup per element) vs TMA
// tile::gather4 (four 32-byte table rows per instruction into shared memory,
// element picked from its row). nvcc -gencode arch=compute_100a,code=sm_100a
// -O3 -o tools/mb_gather4 tools/microbench_gather4.cu
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                              \
    do {                                                                                   \
        cudaError_t e_ = (x);                                                              \
        if (e_ != cudaSuccess) {                                                           \
            std::printf("CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
            std::exit(1);                                                                  \
        }                                                                                  \
    } while (0)

__global__ void k_ldg(const int16_t* __restrict__ tab, const uint32_t* __restrict__ idx, uint64_t n,
                      int16_t* __restrict__ out) {
    constexpr int U = 8;
    const uint64_t base = (uint64_t)blockIdx.x * 256 * U + threadIdx.x;
    uint32_t d[U];
#pragma unroll
    for (int u = 0; u < U; ++u) d[u] = base + 256 * u < n ? __ldcs(idx + base + 256 * u) : 0;
    int16_t v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = __ldg(tab + d[u]);
#pragma unroll
    for (int u = 0; u < U; ++u)
        if (base + 256 * u < n) out[base + 256 * u] = v[u];
}

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// Persistent CTAs; chunk = CH elements, rows staged as 16 B each, NB buffers.
template <int CH, int NB, int ISSUE_WARPS>
__global__ void __launch_bounds__(256) k_g4(const __grid_constant__ CUtensorMap tmap, const uint32_t* __restrict__ idx,
                                            uint64_t n, int16_t* __restrict__ out) {
    extern __shared__ __align__(128) unsigned char sm[];
    __shared__ __align__(8) uint64_t bar[NB];
    __shared__ uint32_t sidx[NB][CH];
    const uint64_t nch = (n + CH - 1) / CH;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0)
        for (int b = 0; b < NB; ++b)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[b])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncthreads();
    auto issue = [&](uint64_t c, int b) {
        // indices of chunk c -> sidx[b]
        for (int e = threadIdx.x; e < CH; e += 256) {
            const uint64_t i = c * CH + e;
            sidx[b][e] = i < n ? __ldcs(idx + i) : 0u;
        }
        __syncthreads();
        if (warp < ISSUE_WARPS) {
            if (threadIdx.x == 0)
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar[b])),
                             "r"((uint32_t)CH * 32)
                             : "memory");
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            for (int g = threadIdx.x; g < CH / 4; g += 32 * ISSUE_WARPS) {
                const int r0 = (int)(sidx[b][4 * g] >> 4), r1 = (int)(sidx[b][4 * g + 1] >> 4),
                          r2 = (int)(sidx[b][4 * g + 2] >> 4), r3 = (int)(sidx[b][4 * g + 3] >> 4);
                unsigned char* dst = sm + ((size_t)b * CH + 4 * g) * 32;
                asm volatile(
                    "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
                    " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(su32(dst)),
                    "l"(&tmap), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(su32(&bar[b]))
                    : "memory");
            }
        }
    };
    uint32_t ph[NB] = {};
    uint64_t c = blockIdx.x;
    // prologue: NB - 1 chunks in flight
    for (int b = 0; b < NB - 1; ++b)
        if (c + (uint64_t)b * gridDim.x < nch) issue(c + (uint64_t)b * gridDim.x, b);
    for (int it = 0; c < nch; ++it, c += gridDim.x) {
        const int b = it % NB;
        const uint64_t cn = c + (uint64_t)(NB - 1) * gridDim.x;
        if (cn < nch) issue(cn, (it + NB - 1) % NB);
        // wait chunk c
        uint32_t ok = 0;
        while (!ok)
            asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
                         : "=r"(ok)
                         : "r"(su32(&bar[b])), "r"(ph[b])
                         : "memory");
        ph[b] ^= 1;
        const int16_t* rows = reinterpret_cast<const int16_t*>(sm + (size_t)b * CH * 32);
        for (int e = threadIdx.x; e < CH; e += 256) {
            const uint64_t i = c * CH + e;
            if (i < n) out[i] = rows[e * 16 + (sidx[b][e] & 15)];
        }
        __syncthreads();
    }
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main(int argc, char** argv) {
    const uint64_t n = 1ull << 27, n1 = 1ull << 24;
    std::vector<uint32_t> hidx(n);
    uint64_t s = 0x9E3779B97F4A7C15ull;
    for (uint64_t i = 0; i < n; ++i) {
        s ^= s << 13; s ^= s >> 7; s ^= s << 17;
        hidx[i] = (uint32_t)(s % n1);
    }
    std::vector<int16_t> htab(n1);
    for (uint64_t j = 0; j < n1; ++j) htab[j] = (int16_t)(j * 2654435761u >> 7);
    int16_t *tab, *o1, *o2;
    uint32_t* idx;
    CK(cudaMalloc(&tab, n1 * 2));
    CK(cudaMalloc(&idx, n * 4));
    CK(cudaMalloc(&o1, n * 2));
    CK(cudaMalloc(&o2, n * 2));
    CK(cudaMemcpy(tab, htab.data(), n1 * 2, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(idx, hidx.data(), n * 4, cudaMemcpyHostToDevice));

    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
    CUtensorMap tm;
    const cuuint64_t gdim[2] = {16, n1 / 16};
    const cuuint64_t gstr[1] = {32};
    const cuuint32_t box[2] = {16, 1};
    const cuuint32_t es[2] = {1, 1};
    CUresult r = ((EncodeFn)fn)(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, tab, gdim, gstr, box, es,
                                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) { std::printf("encode failed %d\n", (int)r); return 1; }
    int sms = 148;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    auto time = [&](const char* name, auto&& launch) {
        for (int w = 0; w < 3; ++w) launch();
        CK(cudaDeviceSynchronize());
        CK(cudaEventRecord(a));
        for (int w = 0; w < 10; ++w) launch();
        CK(cudaEventRecord(b));
        CK(cudaEventSynchronize(b));
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, a, b));
        CK(cudaGetLastError());
        std::printf("%-28s %.3f ms\n", name, ms / 10);
    };
    time("ldg", [&] { k_ldg<<<(unsigned)((n + 2047) / 2048), 256>>>(tab, idx, n, o1); });
    std::vector<int16_t> r1(n), r2(n);
    CK(cudaMemcpy(r1.data(), o1, n * 2, cudaMemcpyDeviceToHost));
#define G4(CH, NB, IW, BPS)                                                                                  \
    {                                                                                                        \
        auto k = k_g4<CH, NB, IW>;                                                                           \
        const int smem = CH * NB * 32;                                                                       \
        CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));                      \
        CK(cudaMemset(o2, 0, n * 2));                                                                        \
        time("g4 CH" #CH " NB" #NB " IW" #IW " BPS" #BPS,                                                   \
             [&] { k<<<sms * BPS, 256, smem>>>(tm, idx, n, o2); });                                          \
        CK(cudaMemcpy(r2.data(), o2, n * 2, cudaMemcpyDeviceToHost));                                        \
        uint64_t bad = 0;                                                                                    \
        for (uint64_t i = 0; i < n; ++i) bad += r1[i] != r2[i];                                              \
        std::printf("   mismatches %llu\n", (unsigned long long)bad);                                        \
    }
    G4(1024, 2, 1, 2)
    G4(1024, 2, 8, 2)
    G4(1024, 3, 8, 2)
    G4(1024, 2, 8, 4)
    G4(512, 4, 8, 4)
    // Mixed: LDG on the first f*n elements (stream s1) beside TMA gather4 on the
    // rest (stream s2) -- is TMA a second path to L2 next to L1TEX?
    {
        cudaStream_t s1, s2;
        CK(cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking));
        CK(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
        auto k = k_g4<1024, 2, 8>;
        const int smem = 1024 * 2 * 32;
        CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        for (double f : {1.0, 0.85, 0.75, 0.65}) {
            for (int bps : {1, 2}) {
                const uint64_t n1s = (uint64_t)(f * n) & ~2047ull, n2s = n - n1s;
                CK(cudaMemset(o2, 0, n * 2));
                auto launch = [&] {
                    CK(cudaEventRecord(a, 0));
                    CK(cudaStreamWaitEvent(s1, a));
                    CK(cudaStreamWaitEvent(s2, a));
                    k_ldg<<<(unsigned)((n1s + 2047) / 2048), 256, 0, s1>>>(tab, idx, n1s, o2);
                    if (n2s) k<<<sms * bps, 256, smem, s2>>>(tm, idx + n1s, n2s, o2 + n1s);
                    cudaEvent_t e1, e2;
                    cudaEventCreate(&e1); cudaEventCreate(&e2);
                    cudaEventRecord(e1, s1); cudaEventRecord(e2, s2);
                    cudaStreamWaitEvent(0, e1); cudaStreamWaitEvent(0, e2);
                    cudaEventDestroy(e1); cudaEventDestroy(e2);
                };
                for (int w = 0; w < 3; ++w) launch();
                CK(cudaDeviceSynchronize());
                cudaEvent_t t0, t1;
                cudaEventCreate(&t0); cudaEventCreate(&t1);
                cudaEventRecord(t0, 0);
                for (int w = 0; w < 10; ++w) launch();
                cudaEventRecord(t1, 0);
                CK(cudaEventSynchronize(t1));
                float ms = 0;
                cudaEventElapsedTime(&ms, t0, t1);
                CK(cudaMemcpy(r2.data(), o2, n * 2, cudaMemcpyDeviceToHost));
                uint64_t bad = 0;
                for (uint64_t i = 0; i < n; ++i) bad += r1[i] != r2[i];
                std::printf("mixed ldg %.2f + g4 bps%d        %.3f ms  (mismatches %llu)\n", f, bps, ms / 10,
                            (unsigned long long)bad);
            }
        }
    }
    return 0;
}
