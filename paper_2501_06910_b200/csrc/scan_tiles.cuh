// Exclusive prefix of per-tile (64-bit, 64-bit) sums, without a serial
// single-CTA scan: CTA b of k_scan_tiles owns tiles [1024 b, 1024 b + 1024),
// reduces every tile before its range itself (coalesced, at most a few
// dozen loads per thread for the tile counts of this code base) and
// block-scans its own range. T <= ~1M tiles.
#pragma once

#include <cstdint>

#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>

namespace umcg {

__device__ __forceinline__ ulonglong2 u2_add(ulonglong2 a, ulonglong2 b) {
    return make_ulonglong2(a.x + b.x, a.y + b.y);
}

struct u2_add_op {
    __device__ __forceinline__ ulonglong2 operator()(const ulonglong2& a, const ulonglong2& b) const {
        return u2_add(a, b);
    }
};

constexpr int SCAN_TILES_THREADS = 1024;

// out[t] = sum of in[0, t) for t < T; total -> *total (when non-null) and,
// when cnt_out is non-null, total.x -> *cnt_out. in and out must not alias.
static __global__ void __launch_bounds__(SCAN_TILES_THREADS) k_scan_tiles(const ulonglong2* __restrict__ in,
                                                                  ulonglong2* __restrict__ out, uint64_t T,
                                                                  ulonglong2* __restrict__ total,
                                                                  uint64_t* __restrict__ cnt_out) {
    using BR = cub::BlockReduce<ulonglong2, SCAN_TILES_THREADS>;
    using BS = cub::BlockScan<ulonglong2, SCAN_TILES_THREADS>;
    __shared__ union {
        typename BR::TempStorage r;
        typename BS::TempStorage s;
    } tmp;
    __shared__ ulonglong2 base;
    const uint64_t b0 = (uint64_t)blockIdx.x * SCAN_TILES_THREADS;
    ulonglong2 acc = make_ulonglong2(0, 0);
    uint64_t i = threadIdx.x;
    for (; i + 3 * SCAN_TILES_THREADS < b0; i += 4 * SCAN_TILES_THREADS) {
        const ulonglong2 a = in[i], b = in[i + SCAN_TILES_THREADS], c = in[i + 2 * SCAN_TILES_THREADS],
                         d = in[i + 3 * SCAN_TILES_THREADS];
        acc = u2_add(acc, u2_add(u2_add(a, b), u2_add(c, d)));
    }
    for (; i < b0; i += SCAN_TILES_THREADS) acc = u2_add(acc, in[i]);
    const ulonglong2 pre = BR(tmp.r).Reduce(acc, u2_add_op{});
    if (threadIdx.x == 0) base = pre;
    __syncthreads();
    const uint64_t t = b0 + threadIdx.x;
    const ulonglong2 v = t < T ? in[t] : make_ulonglong2(0, 0);
    ulonglong2 ex, agg;
    BS(tmp.s).ExclusiveScan(v, ex, make_ulonglong2(0, 0), u2_add_op{}, agg);
    const ulonglong2 bb = base;
    if (t < T) out[t] = u2_add(bb, ex);
    if (b0 + SCAN_TILES_THREADS >= T && threadIdx.x == 0) {
        const ulonglong2 tot = u2_add(bb, agg);
        if (total) *total = tot;
        if (cnt_out) *cnt_out = tot.x;
    }
}

inline unsigned scan_tiles_grid(uint64_t T) {
    return (unsigned)((T + SCAN_TILES_THREADS - 1) / SCAN_TILES_THREADS);
}

}  // namespace umcg
