// mapping_digest (serialize.hpp:255-267, 300-303) on the device: FNV-1a-64 of
// the serialize_mapping bytes, computed in parallel.
//
// FNV-1a is a serial chain h <- (h ^ b) * P, and the reference pays it on
// every compress and decompress (pipeline.hpp:135, 188; 3.3 s at 134M
// vertices). The plan computes it once, but a byte-serial host loop over the
// 1.07 GB of u64 assignments still took ~1.2 s of a 1.4 s plan build. The
// chain parallelizes because the XOR touches only the low byte:
//
//   h ^ b = h + d,  d = ((l ^ b) - l),  l = h mod 256
//   l'    = ((l ^ b) * (P mod 256)) mod 256        (a 256-state automaton)
//
// so over any byte range, given the low byte s of the hash entering it, the
// hash leaving it is h_out = A * h_in + B_s (mod 2^64) with A = P^len and
// B_s accumulated by B <- (B + d) * P along the low-byte trajectory from s.
// k_fnv_chunks evaluates B_s of every chunk for all 256 entry states (thread
// s of the CTA), k_fnv_combine then chains the chunks with one table lookup
// each. A run of k zero bytes (the five high bytes of every u64 record
// holding a 24-bit slot) is one multiplication by P^k.
#include "common.cuh"
#include "plan.h"

namespace umcg {
namespace {

constexpr uint64_t kFnvP = 0x100000001b3ull;
constexpr uint32_t kFnvR = 16384;  // records per chunk
constexpr uint32_t kFnvStage = 1024;  // records staged per round

constexpr uint64_t fnv_pow(uint64_t e) {
    uint64_t r = 1, b = kFnvP;
    while (e) {
        if (e & 1) r *= b;
        b *= b;
        e >>= 1;
    }
    return r;
}

constexpr uint32_t fnv_lpow(uint32_t e) {
    uint32_t r = 1;
    for (uint32_t k = 0; k < e; ++k) r = (r * 0xb3u) & 0xffu;
    return r;
}
// P^k and (P mod 256)^k mod 256 for zero runs of k = 0..8 bytes
__constant__ uint64_t c_fnv_ppow[9] = {fnv_pow(0), fnv_pow(1), fnv_pow(2), fnv_pow(3), fnv_pow(4),
                                       fnv_pow(5), fnv_pow(6), fnv_pow(7), fnv_pow(8)};
__constant__ uint32_t c_fnv_lpow[9] = {fnv_lpow(0), fnv_lpow(1), fnv_lpow(2), fnv_lpow(3), fnv_lpow(4),
                                       fnv_lpow(5), fnv_lpow(6), fnv_lpow(7), fnv_lpow(8)};

// B_s and the low byte after `count` records of `T` (widened to u64, little
// endian: ByteWriter::u64, serialize.hpp:261), for the entry low byte s =
// threadIdx.x.
template <class T>
__global__ void __launch_bounds__(256) k_fnv_chunks(const T* __restrict__ rec, uint64_t n, uint64_t* __restrict__ tabB) {
    __shared__ T sr[kFnvStage];
    const uint64_t first = (uint64_t)blockIdx.x * kFnvR;
    const uint32_t cnt = (uint32_t)min((uint64_t)kFnvR, n - first);
    uint32_t l = threadIdx.x;
    uint64_t B = 0;
    for (uint32_t base = 0; base < cnt; base += kFnvStage) {
        const uint32_t m = min(kFnvStage, cnt - base);
        __syncthreads();
        for (uint32_t i = threadIdx.x; i < m; i += 256) sr[i] = rec[first + base + i];
        __syncthreads();
        for (uint32_t i = 0; i < m; ++i) {
            const uint64_t v = (uint64_t)sr[i];  // the same record for every thread
            const int hb = v ? (71 - __clzll((long long)v)) >> 3 : 0;  // significant bytes
            for (int k = 0; k < hb; ++k) {
                const uint32_t b = (uint32_t)(v >> (8 * k)) & 0xffu;
                const uint32_t t = l ^ b;
                B = (B + (uint64_t)(int64_t)((int)t - (int)l)) * kFnvP;
                l = (t * 0xb3u) & 0xffu;
            }
            // the record's high zero bytes: 8 - hb multiplications in one
            const uint64_t pz = c_fnv_ppow[8 - hb];
            const uint32_t lz = c_fnv_lpow[8 - hb];
            B *= pz;
            l = (l * lz) & 0xffu;
        }
    }
    tabB[(uint64_t)blockIdx.x * 256 + threadIdx.x] = B;
}

// h <- A_c * h + B_c[h mod 256] over the chunks in order (one thread: a
// dependent lookup per chunk, ~n / 16384 of them).
__global__ void k_fnv_combine(const uint64_t* __restrict__ tabB, uint64_t chunks, uint64_t a_full, uint64_t a_last,
                              uint64_t h, uint64_t* __restrict__ out) {
    for (uint64_t c = 0; c < chunks; ++c) {
        const uint64_t a = c + 1 == chunks ? a_last : a_full;
        h = a * h + tabB[c * 256 + (h & 0xffu)];
    }
    *out = h;
}

template <class T>
uint64_t fnv_records(uint64_t h, const T* d_rec, uint64_t n, DevBuf& scratch, cudaStream_t st) {
    if (!n) return h;
    const uint64_t chunks = cdiv(n, (uint64_t)kFnvR);
    uint64_t* tab = scratch.as<uint64_t>(chunks * 256 + 1);
    k_fnv_chunks<T><<<(unsigned)chunks, 256, 0, st>>>(d_rec, n, tab);
    UMCG_LAUNCHED();
    const uint64_t last = n - (chunks - 1) * kFnvR;
    k_fnv_combine<<<1, 1, 0, st>>>(tab, chunks, fnv_pow(8ull * kFnvR), fnv_pow(8ull * last), h, tab + chunks * 256);
    UMCG_LAUNCHED();
    uint64_t out = 0;
    UMCG_CUDA(cudaMemcpyAsync(&out, tab + chunks * 256, 8, cudaMemcpyDeviceToHost, st));
    UMCG_CUDA(cudaStreamSynchronize(st));
    return out;
}

struct FnvHost {
    uint64_t h = 0xcbf29ce484222325ull;
    void byte(uint8_t b) { h ^= b; h *= kFnvP; }
    void le(uint64_t v, int k) { for (int i = 0; i < k; ++i) byte((uint8_t)(v >> (8 * i))); }
};

}  // namespace

// serialize_mapping: "UMCP", u16 version 1, u8 mode, u64 n, n x u64
// assignment, and in seed mode u64 n_visited, n_visited x u64 node.
uint64_t mapping_digest_device(int mode, uint64_t n, const uint32_t* d_assign, uint64_t n_visited,
                               const uint64_t* d_visited, DevBuf& scratch, cudaStream_t st) {
    if (n >= (1ull << 40)) fail(UMCG_INVALID_ARGUMENT, "mapping too long for the device digest");
    FnvHost f;
    f.byte('U'); f.byte('M'); f.byte('C'); f.byte('P');
    f.le(1, 2);
    f.byte((uint8_t)mode);
    f.le(n, 8);
    f.h = fnv_records(f.h, d_assign, n, scratch, st);
    if (mode == 1) {
        f.le(n_visited, 8);
        f.h = fnv_records(f.h, d_visited, n_visited, scratch, st);
    }
    return f.h;
}

}  // namespace umcg
