// Device helpers shared by the stream encoder and the fused code kernels.
#pragma once

#include "kernels.h"

namespace umcg {

struct RleComposeOp {
    __device__ __forceinline__ RleSum operator()(const RleSum& a, const RleSum& b) const {
        return rle_compose(a, b);
    }
};

// Bytes one code occupies in the stream before RLE: varint(code) for the
// quantizer's codes (common.hpp:60-66); one raw byte for uint8_t "codes"
// (the verbatim codec and umcg_rle_compress feed raw bytes, lossless.hpp:24).
template <class T>
__device__ __forceinline__ uint32_t clen(T v) {
    if (sizeof(T) == 1) return 1u;
    if (sizeof(T) == 2) return 1u + (v >= 0x80) + (v >= 0x4000);
    return v == 0 ? 1u : vlen64((uint64_t)v);
}

template <class T>
__device__ __forceinline__ void write_varint(uint8_t* out, uint64_t pos, uint64_t base, uint64_t cap, T v) {
    uint64_t u = (uint64_t)v;
    uint64_t p = pos - base;
    while (u >= 0x80) {
        if (p < cap) out[p] = (uint8_t)u | 0x80;
        ++p;
        u >>= 7;
    }
    if (p < cap) out[p] = (uint8_t)u;
}

template <class T>
__device__ __forceinline__ int load_items(const T* codes, uint64_t n, uint64_t first, T (&v)[ENC_ITEMS]) {
    int cnt = 0;
    if (first + ENC_ITEMS <= n && sizeof(T) == 2 && (first % 8) == 0) {
        const uint4 a = __ldg(reinterpret_cast<const uint4*>(codes + first));
        const uint32_t w[4] = {a.x, a.y, a.z, a.w};
#pragma unroll
        for (int k = 0; k < ENC_ITEMS; ++k) v[k] = (T)(w[k >> 1] >> (16 * (k & 1)));
        return ENC_ITEMS;
    }
    if (first + ENC_ITEMS <= n && sizeof(T) == 4 && (first % 4) == 0) {
        const uint4* p = reinterpret_cast<const uint4*>(codes + first);
        const uint4 a = __ldg(p), b = __ldg(p + 1);
        const uint32_t w[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
        for (int k = 0; k < ENC_ITEMS; ++k) v[k] = (T)w[k];
        return ENC_ITEMS;
    }
#pragma unroll
    for (int k = 0; k < ENC_ITEMS; ++k) {
        const uint64_t i = first + k;
        if (i < n) { v[k] = codes[i]; cnt = k + 1; } else { v[k] = 0; }
    }
    return cnt;
}

template <class T>
__device__ __forceinline__ RleSum thread_summary(const T (&v)[ENC_ITEMS], int cnt, uint32_t origin) {
    // <= 8 codes cannot hold a zero run >= 8 strictly between two nonzeros,
    // so a thread summary never has interior runs.
    static_assert(ENC_ITEMS <= 9, "fast thread summary assumes <= 9 items");
    uint32_t zm = 0;
#pragma unroll
    for (int k = 0; k < ENC_ITEMS; ++k) zm |= (k < cnt && v[k] == 0) ? (1u << k) : 0u;
    const uint32_t valid = cnt >= 32 ? ~0u : ((1u << cnt) - 1u);
    const uint32_t nz = ~zm & valid;
    RleSum s;
    s.tz = s.lb = s.mid = 0;
    if (nz == 0) {
        s.lz = (uint64_t)cnt; s.fb = 0; s.origin = kNoOrigin; s.flags = 1u;
        return s;
    }
    const int lo = __ffs(nz) - 1, hi = 31 - __clz(nz);
    uint64_t fb = 0;
#pragma unroll
    for (int k = 0; k < ENC_ITEMS; ++k)
        if (k >= lo && k <= hi) fb += clen(v[k]);
    s.lz = (uint64_t)lo;
    s.tz = (uint64_t)(cnt - 1 - hi);
    s.fb = fb;
    s.origin = origin;
    s.flags = 0u;
    return s;
}

}  // namespace umcg
