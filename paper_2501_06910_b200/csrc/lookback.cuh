// Single-pass decoupled look-back scan across CTAs (prefix of tile
// aggregates under an associative op). Tiles take ids from a global ticket
// so every predecessor is already resident when a tile starts looking back.
#pragma once

#include "common.cuh"

namespace umcg {

enum : uint32_t { LB_NONE = 0, LB_AGG = 1, LB_INCL = 2 };

template <class T>
struct alignas(16) TileStatus {
    T agg;
    T incl;
    uint32_t flag;
};

// Ticket for dynamic tile ordering; `ctr` must be zero at launch.
__device__ __forceinline__ uint32_t lb_ticket(uint32_t* ctr) {
    __shared__ uint32_t s;
    if (threadIdx.x == 0) s = atomicAdd(ctr, 1u);
    __syncthreads();
    return s;
}

template <class T>
__device__ __forceinline__ void lb_store(T* dst, const T& v) {
    volatile uint32_t* d = reinterpret_cast<volatile uint32_t*>(dst);
    const uint32_t* s = reinterpret_cast<const uint32_t*>(&v);
#pragma unroll
    for (int k = 0; k < (int)(sizeof(T) / 4); ++k) d[k] = s[k];
}

template <class T>
__device__ __forceinline__ T lb_load(const T* src) {
    T v;
    const volatile uint32_t* s = reinterpret_cast<const volatile uint32_t*>(src);
    uint32_t* d = reinterpret_cast<uint32_t*>(&v);
#pragma unroll
    for (int k = 0; k < (int)(sizeof(T) / 4); ++k) d[k] = s[k];
    return v;
}

// Called by ONE thread of the tile. Publishes the tile aggregate, walks back
// over predecessors and returns the exclusive prefix (identity for tile 0).
// op(a, b) = a followed by b.
template <class T, class Op>
__device__ T lb_exclusive(TileStatus<T>* st, uint32_t tile, const T& agg, Op op, const T& identity) {
    static_assert(sizeof(T) % 4 == 0, "TileStatus payload must be 4-byte granular");
    if (tile == 0) {
        lb_store(&st[0].incl, agg);
        __threadfence();
        atomicExch(&st[0].flag, LB_INCL);
        return identity;
    }
    lb_store(&st[tile].agg, agg);
    __threadfence();
    atomicExch(&st[tile].flag, LB_AGG);
    T acc = identity;
    int64_t j = (int64_t)tile - 1;
    while (true) {
        uint32_t f;
        do {
            f = *reinterpret_cast<volatile uint32_t*>(&st[j].flag);
        } while (f == LB_NONE);
        __threadfence();
        if (f == LB_INCL) {
            acc = op(lb_load(&st[j].incl), acc);
            break;
        }
        acc = op(lb_load(&st[j].agg), acc);
        --j;
    }
    lb_store(&st[tile].incl, op(acc, agg));
    __threadfence();
    atomicExch(&st[tile].flag, LB_INCL);
    return acc;
}

template <class T>
__device__ __forceinline__ T shfl_down_t(const T& v, int off) {
    T r;
    const uint32_t* s = reinterpret_cast<const uint32_t*>(&v);
    uint32_t* d = reinterpret_cast<uint32_t*>(&r);
#pragma unroll
    for (int k = 0; k < (int)(sizeof(T) / 4); ++k) d[k] = __shfl_down_sync(0xffffffffu, s[k], off);
    return r;
}

template <class T>
__device__ __forceinline__ T shfl_idx_t(const T& v, int src) {
    T r;
    const uint32_t* s = reinterpret_cast<const uint32_t*>(&v);
    uint32_t* d = reinterpret_cast<uint32_t*>(&r);
#pragma unroll
    for (int k = 0; k < (int)(sizeof(T) / 4); ++k) d[k] = __shfl_sync(0xffffffffu, s[k], src);
    return r;
}

// Warp-wide look-back (all 32 lanes of one warp): each step inspects the 32
// closest unresolved predecessors at once and composes them in order, so a
// tile never waits on its immediate predecessor's inclusive prefix alone.
// Returns the exclusive prefix on every lane.
template <class T, class Op>
__device__ T lb_exclusive_warp(TileStatus<T>* st, uint32_t tile, const T& agg, Op op, const T& identity) {
    static_assert(sizeof(T) % 4 == 0, "TileStatus payload must be 4-byte granular");
    const int lane = threadIdx.x & 31;
    if (lane == 0) {
        if (tile == 0) {
            lb_store(&st[0].incl, agg);
            __threadfence();
            atomicExch(&st[0].flag, LB_INCL);
        } else {
            lb_store(&st[tile].agg, agg);
            __threadfence();
            atomicExch(&st[tile].flag, LB_AGG);
        }
    }
    if (tile == 0) return identity;
    T acc = identity;
    int64_t wend = (int64_t)tile - 1;
    while (true) {
        const int64_t j = wend - lane;
        uint32_t f = LB_INCL;
        T v = identity;
        if (j >= 0) {
            do {
                f = *reinterpret_cast<volatile uint32_t*>(&st[j].flag);
            } while (f == LB_NONE);
            __threadfence();
            v = f == LB_INCL ? lb_load(&st[j].incl) : lb_load(&st[j].agg);
        }
        const uint32_t m = __ballot_sync(0xffffffffu, f == LB_INCL);
        const int first = m ? __ffs(m) - 1 : 32;
        if (lane > first) v = identity;
        // ordered reduction: lane L ends with v_{L+..} o ... o v_L (older first)
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const T o = shfl_down_t(v, off);
            if (lane + off < 32) v = op(o, v);
        }
        const T w = shfl_idx_t(v, 0);
        acc = op(w, acc);
        if (m) break;
        wend -= 32;
    }
    if (lane == 0) {
        lb_store(&st[tile].incl, op(acc, agg));
        __threadfence();
        atomicExch(&st[tile].flag, LB_INCL);
    }
    return acc;
}

}  // namespace umcg
