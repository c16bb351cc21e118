// Random-gather paths on B200 (round 2 A/B): LDG vs the texture path
// (tex1Dfetch) for window-local 8-byte and 2-byte gathers, and a run-sorted
// variant of the layout-E -> vertex-order gather that k_resid_codes does.
//
// Layout E is simulated the way plan.cu builds it: epochs of 2^22 consecutive
// vertices, inside an epoch vertices grouped by bucket (random bucket per
// vertex, ~4096 vertices per bucket over the whole field), ascending vertex
// inside a bucket chunk.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <random>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

constexpr int IT = 8;

// xE[p] = x[srcE[p]] via LDG (.cg) / tex1Dfetch / half and half
template <int MODE>
__global__ void __launch_bounds__(256) g8(const double* __restrict__ x, cudaTextureObject_t tx,
                                          const uint32_t* __restrict__ src, double* __restrict__ out, uint64_t n) {
    const uint64_t base = (uint64_t)blockIdx.x * 256 * IT + threadIdx.x;
    uint32_t s[IT];
#pragma unroll
    for (int k = 0; k < IT; ++k) s[k] = __ldcs(src + base + k * 256);
    double v[IT];
#pragma unroll
    for (int k = 0; k < IT; ++k) {
        const bool tex = MODE == 1 || (MODE == 2 && (k & 1));
        if (tex) {
            const int2 t = tex1Dfetch<int2>(tx, (int)s[k]);
            v[k] = __hiloint2double(t.y, t.x);
        } else {
            v[k] = __ldcg(x + s[k]);
        }
    }
#pragma unroll
    for (int k = 0; k < IT; ++k) __stcs(out + base + k * 256, v[k]);
}

// codes_i = K[dst[i]] - K[dst[i-1]] (2-byte gathers) via LDG / tex / mixed
template <int MODE>
__global__ void __launch_bounds__(256) g2(const int16_t* __restrict__ K, cudaTextureObject_t tk,
                                          const uint32_t* __restrict__ dst, uint16_t* __restrict__ out, uint64_t n) {
    const uint64_t first = ((uint64_t)blockIdx.x * 256 + threadIdx.x) * IT;
    uint32_t d[IT];
    const uint4 a = __ldg(reinterpret_cast<const uint4*>(dst + first));
    const uint4 c = __ldg(reinterpret_cast<const uint4*>(dst + first) + 1);
    d[0] = a.x; d[1] = a.y; d[2] = a.z; d[3] = a.w; d[4] = c.x; d[5] = c.y; d[6] = c.z; d[7] = c.w;
    int32_t prev = first ? K[dst[first - 1]] : 0;
    int32_t v[IT];
#pragma unroll
    for (int k = 0; k < IT; ++k) {
        const bool tex = MODE == 1 || (MODE == 2 && (k & 1));
        v[k] = tex ? (int32_t)tex1Dfetch<short>(tk, (int)d[k]) : (int32_t)__ldcg(K + d[k]);
    }
    uint32_t w[IT / 2];
#pragma unroll
    for (int k = 0; k < IT; k += 2) {
        const int32_t q0 = v[k] - prev, q1 = v[k + 1] - v[k];
        prev = v[k + 1];
        w[k / 2] = ((uint32_t)((q0 << 1) ^ (q0 >> 31)) & 0xffffu) | ((uint32_t)((q1 << 1) ^ (q1 >> 31)) << 16);
    }
    *reinterpret_cast<uint4*>(out + first) = make_uint4(w[0], w[1], w[2], w[3]);
}

// Run-sorted variant: one CTA per tile of T vertices. Pt = the tile's layout-E
// positions in ascending order (runs of consecutive positions), Lt = the
// tile-local vertex of each. K staged in shared memory in vertex order, then
// codes written coalesced.
template <int T, int NT>
__global__ void __launch_bounds__(NT) g2sorted(const int16_t* __restrict__ K, const uint32_t* __restrict__ Pt,
                                              const uint16_t* __restrict__ Lt, const uint32_t* __restrict__ dst,
                                              uint16_t* __restrict__ out, uint64_t n) {
    extern __shared__ int16_t ks[];
    const uint64_t t0 = (uint64_t)blockIdx.x * T;
    constexpr int PERT = T / NT;
    static_assert(PERT % 8 == 0, "");
    // lane-contiguous: one warp instruction covers 32 consecutive sorted positions
    for (int k = threadIdx.x; k < T; k += NT * 4) {
        uint32_t p[4];
        uint16_t l[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            p[u] = __ldcs(Pt + t0 + k + u * NT);
            l[u] = __ldcs(Lt + t0 + k + u * NT);
        }
        int16_t v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) v[u] = __ldcg(K + p[u]);
#pragma unroll
        for (int u = 0; u < 4; ++u) ks[l[u]] = v[u];
    }
    __syncthreads();
    const int32_t prev0 = t0 ? (int32_t)__ldg(K + __ldg(dst + t0 - 1)) : 0;
    for (int i0 = threadIdx.x * 8; i0 < T; i0 += NT * 8) {
        int32_t prev = i0 ? (int32_t)ks[i0 - 1] : prev0;
        uint32_t w[4];
#pragma unroll
        for (int k = 0; k < 8; k += 2) {
            const int32_t a = ks[i0 + k], b = ks[i0 + k + 1];
            const int32_t q0 = a - prev, q1 = b - a;
            prev = b;
            w[k / 2] = ((uint32_t)((q0 << 1) ^ (q0 >> 31)) & 0xffffu) | ((uint32_t)((q1 << 1) ^ (q1 >> 31)) << 16);
        }
        __stcs(reinterpret_cast<uint4*>(out + t0 + i0), make_uint4(w[0], w[1], w[2], w[3]));
    }
}


// Synthetic: gather in runs of R consecutive elements (random run starts),
// lane-contiguous, element type V: the cost of a random permutation as a
// function of its run length.
template <class V>
__global__ void __launch_bounds__(256) grun(const V* __restrict__ in, const uint32_t* __restrict__ idx,
                                            V* __restrict__ out, uint64_t n) {
    const uint64_t base = (uint64_t)blockIdx.x * 256 * IT + threadIdx.x;
    uint32_t s[IT];
#pragma unroll
    for (int k = 0; k < IT; ++k) s[k] = __ldcs(idx + base + k * 256);
    V v[IT];
#pragma unroll
    for (int k = 0; k < IT; ++k) v[k] = __ldcg(in + s[k]);
#pragma unroll
    for (int k = 0; k < IT; ++k) __stcs(out + base + k * 256, v[k]);
}


// The library's k_resid_codes_sr phase 1 as written (U loads in flight,
// predicated, NT threads, MINB CTAs per SM), phase 2 reduced to the codes.
template <int NT, int MINB, int U>
__global__ void __launch_bounds__(NT, MINB) p1lib(const int16_t* __restrict__ Kp, const uint32_t* __restrict__ rPt,
                                                  const uint16_t* __restrict__ rLt, const uint32_t* __restrict__ dst,
                                                  uint16_t* __restrict__ out, uint64_t n) {
    extern __shared__ int16_t ks[];
    constexpr uint32_t T = 32768;
    const uint64_t t0 = (uint64_t)blockIdx.x * T;
    const uint32_t cnt = (uint32_t)min((uint64_t)T, n - t0);
    for (uint32_t k0 = threadIdx.x; k0 < cnt; k0 += NT * U) {
        uint32_t pp[U];
        uint32_t ll[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint32_t k = k0 + u * NT;
            pp[u] = k < cnt ? __ldcs(rPt + t0 + k) : 0u;
            ll[u] = k < cnt ? __ldcs(rLt + t0 + k) : 0u;
        }
        int16_t v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = k0 + u * NT < cnt ? __ldcg(Kp + pp[u]) : (int16_t)0;
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (k0 + u * NT < cnt) ks[ll[u]] = v[u];
    }
    __syncthreads();
    const int32_t prev0 = t0 ? (int32_t)__ldg(Kp + __ldg(dst + t0 - 1)) : 0;
    for (uint32_t i0 = threadIdx.x * 8; i0 < cnt; i0 += NT * 8) {
        int32_t prev = i0 ? (int32_t)ks[i0 - 1] : prev0;
        uint32_t w[4];
#pragma unroll
        for (int k = 0; k < 8; k += 2) {
            const int32_t a = ks[i0 + k], b = ks[i0 + k + 1];
            const int32_t q0 = a - prev, q1 = b - a;
            prev = b;
            w[k / 2] = ((uint32_t)((q0 << 1) ^ (q0 >> 31)) & 0xffffu) | ((uint32_t)((q1 << 1) ^ (q1 >> 31)) << 16);
        }
        *reinterpret_cast<uint4*>(out + t0 + i0) = make_uint4(w[0], w[1], w[2], w[3]);
    }
}

int main() {
    const uint64_t n = 134217728ull, EP = 1ull << 22;
    const uint32_t NB = (uint32_t)(n / 4096);
    std::mt19937_64 rng(7);
    // layout E
    std::vector<uint32_t> bucket(n), srcE(n), dstE(n);
    for (uint64_t i = 0; i < n; ++i) bucket[i] = (uint32_t)(rng() % NB);
    {
        std::vector<uint32_t> cnt(NB + 1);
        for (uint64_t e0 = 0; e0 < n; e0 += EP) {
            std::fill(cnt.begin(), cnt.end(), 0);
            for (uint64_t i = e0; i < e0 + EP; ++i) cnt[bucket[i] + 1]++;
            for (uint32_t b = 0; b < NB; ++b) cnt[b + 1] += cnt[b];
            for (uint64_t i = e0; i < e0 + EP; ++i) {
                const uint64_t p = e0 + cnt[bucket[i]]++;
                srcE[p] = (uint32_t)i;
                dstE[i] = (uint32_t)p;
            }
        }
    }
    double *dx, *dxe;
    uint32_t *dsrc, *ddst, *dPt;
    int16_t* dK;
    uint16_t *dcodes, *dLt;
    CK(cudaMalloc(&dx, n * 8)); CK(cudaMalloc(&dxe, n * 8));
    CK(cudaMalloc(&dsrc, n * 4)); CK(cudaMalloc(&ddst, n * 4)); CK(cudaMalloc(&dPt, n * 4));
    CK(cudaMalloc(&dK, n * 2)); CK(cudaMalloc(&dcodes, n * 2)); CK(cudaMalloc(&dLt, n * 2));
    {
        std::vector<double> hx(n);
        for (uint64_t i = 0; i < n; ++i) hx[i] = (double)(i % 1000) * 0.5;
        CK(cudaMemcpy(dx, hx.data(), n * 8, cudaMemcpyHostToDevice));
        std::vector<int16_t> hk(n);
        for (uint64_t i = 0; i < n; ++i) hk[i] = (int16_t)(rng() % 2001) - 1000;
        CK(cudaMemcpy(dK, hk.data(), n * 2, cudaMemcpyHostToDevice));
    }
    CK(cudaMemcpy(dsrc, srcE.data(), n * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(ddst, dstE.data(), n * 4, cudaMemcpyHostToDevice));
    cudaTextureObject_t tx, tk;
    {
        cudaResourceDesc rd{};
        rd.resType = cudaResourceTypeLinear;
        rd.res.linear.devPtr = dx;
        rd.res.linear.desc = cudaCreateChannelDesc<int2>();
        rd.res.linear.sizeInBytes = n * 8;
        cudaTextureDesc td{};
        td.readMode = cudaReadModeElementType;
        CK(cudaCreateTextureObject(&tx, &rd, &td, nullptr));
        rd.res.linear.devPtr = dK;
        rd.res.linear.desc = cudaCreateChannelDesc<short>();
        rd.res.linear.sizeInBytes = n * 2;
        CK(cudaCreateTextureObject(&tk, &rd, &td, nullptr));
    }
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    // L2 flush buffer
    char* fl; CK(cudaMalloc(&fl, 256ull << 20));
    auto timeit = [&](auto launch, const char* name) {
        launch();
        CK(cudaDeviceSynchronize());
        std::vector<float> v;
        for (int r = 0; r < 7; ++r) {
            cudaMemsetAsync(fl, r, 256ull << 20);
            cudaEventRecord(a); launch(); cudaEventRecord(b); cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b); v.push_back(ms);
        }
        std::sort(v.begin(), v.end());
        CK(cudaGetLastError());
        printf("%-60s median %.4f ms  min %.4f ms\n", name, v[3], v[0]);
        return 0;
    };
    const unsigned G8 = (unsigned)(n / (256 * IT));
    timeit([&] { g8<0><<<G8, 256>>>(dx, tx, dsrc, dxe, n); }, "g8 LDG.cg  (k_gather_fwd pattern)");
    timeit([&] { g8<1><<<G8, 256>>>(dx, tx, dsrc, dxe, n); }, "g8 tex1Dfetch");
    timeit([&] { g8<2><<<G8, 256>>>(dx, tx, dsrc, dxe, n); }, "g8 half LDG / half tex");
    timeit([&] { g2<0><<<G8, 256>>>(dK, tk, ddst, dcodes, n); }, "g2 LDG.cg  (k_resid_codes pattern)");
    timeit([&] { g2<1><<<G8, 256>>>(dK, tk, ddst, dcodes, n); }, "g2 tex1Dfetch");
    timeit([&] { g2<2><<<G8, 256>>>(dK, tk, ddst, dcodes, n); }, "g2 half LDG / half tex");
    std::vector<uint16_t> ref(n), got(n);
    CK(cudaMemcpy(ref.data(), dcodes, n * 2, cudaMemcpyDeviceToHost));
    // sorted-run tables for several tile sizes
    auto run_sorted = [&](auto kern, uint32_t T, int NT, const char* name) {
        std::vector<uint32_t> Pt(n);
        std::vector<uint16_t> Lt(n);
        std::vector<std::pair<uint32_t, uint16_t>> tmp(T);
        uint64_t runs = 0;
        for (uint64_t t0 = 0; t0 < n; t0 += T) {
            for (uint32_t k = 0; k < T; ++k) tmp[k] = {dstE[t0 + k], (uint16_t)k};
            std::sort(tmp.begin(), tmp.end());
            for (uint32_t k = 0; k < T; ++k) {
                Pt[t0 + k] = tmp[k].first;
                Lt[t0 + k] = tmp[k].second;
                runs += (k == 0 || tmp[k].first != tmp[k - 1].first + 1);
            }
        }
        if (cudaMemcpy(dPt, Pt.data(), n * 4, cudaMemcpyHostToDevice) != cudaSuccess) return 1;
        if (cudaMemcpy(dLt, Lt.data(), n * 2, cudaMemcpyHostToDevice) != cudaSuccess) return 1;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(T * 2));
        cudaMemset(dcodes, 0, n * 2);
        char nm[160];
        snprintf(nm, sizeof nm, "%s T=%u (mean run %.2f)", name, T, (double)n / runs);
        timeit([&] { kern<<<(unsigned)(n / T), NT, T * 2>>>(dK, dPt, dLt, ddst, dcodes, n); }, nm);
        cudaMemcpy(got.data(), dcodes, n * 2, cudaMemcpyDeviceToHost);
        printf("   matches LDG codes: %s\n", got == ref ? "yes" : "NO");
        return 0;
    };
    run_sorted(g2sorted<32768, 1024>, 32768, 1024, "g2 sorted-run");
    // the library kernel's phase 1 on the same tables (T = 32768 built last)
    {
        auto lib = [&](auto kern, int NT, const char* name) {
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
            cudaMemset(dcodes, 0, n * 2);
            timeit([&] { kern<<<(unsigned)(n / 32768), NT, 65536>>>(dK, dPt, dLt, ddst, dcodes, n); }, name);
            cudaMemcpy(got.data(), dcodes, n * 2, cudaMemcpyDeviceToHost);
            printf("   matches LDG codes: %s\n", got == ref ? "yes" : "NO");
        };
        lib(p1lib<256, 3, 8>, 256, "p1lib NT=256 MINB=3 U=8");
        lib(p1lib<256, 3, 4>, 256, "p1lib NT=256 MINB=3 U=4");
        lib(p1lib<1024, 1, 4>, 1024, "p1lib NT=1024 MINB=1 U=4");
        lib(p1lib<512, 2, 4>, 512, "p1lib NT=512 MINB=2 U=4");
        lib(p1lib<512, 1, 4>, 512, "p1lib NT=512 MINB=1 U=4");
        lib(p1lib<1024, 1, 2>, 1024, "p1lib NT=1024 MINB=1 U=2");
        lib(p1lib<1024, 1, 8>, 1024, "p1lib NT=1024 MINB=1 U=8");
        lib(p1lib<1024, 2, 4>, 1024, "p1lib NT=1024 MINB=2 U=4");
        lib(p1lib<256, 1, 4>, 256, "p1lib NT=256 MINB=1 U=4");
        {
            // carve-out: force the max shared-memory carveout for the 1024 variant
            cudaFuncSetAttribute(p1lib<1024, 1, 4>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
            lib(p1lib<1024, 1, 4>, 1024, "p1lib NT=1024 MINB=1 U=4 carveout100");
            cudaFuncSetAttribute(p1lib<256, 3, 8>, cudaFuncAttributePreferredSharedMemoryCarveout, 30);
            lib(p1lib<256, 3, 8>, 256, "p1lib NT=256 MINB=3 U=8 carveout30");
        }
    }
    // run-length curve: window-local (4M-element windows), runs of R
    {
        std::vector<uint32_t> idx(n);
        for (int R : {1, 2, 4, 8, 16}) {
            for (uint64_t w0 = 0; w0 < n; w0 += EP) {
                const uint64_t nr = EP / R;
                std::vector<uint32_t> starts(nr);
                for (uint64_t r = 0; r < nr; ++r) starts[r] = (uint32_t)(r * R);
                std::shuffle(starts.begin(), starts.end(), rng);
                for (uint64_t r = 0; r < nr; ++r)
                    for (int u = 0; u < R; ++u) idx[w0 + r * R + u] = (uint32_t)(w0 + starts[r] + u);
            }
            CK(cudaMemcpy(dsrc, idx.data(), n * 4, cudaMemcpyHostToDevice));
            char nm[96];
            snprintf(nm, sizeof nm, "grun f64 R=%d", R);
            timeit([&] { grun<double><<<G8, 256>>>(dx, dsrc, dxe, n); }, nm);
            snprintf(nm, sizeof nm, "grun i16 R=%d", R);
            timeit([&] { grun<int16_t><<<G8, 256>>>(dK, dsrc, (int16_t*)dcodes, n); }, nm);
        }
    }
    return 0;
}
