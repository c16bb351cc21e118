// K0's sorts ("stable radix sort by node -> perm, seg_off"): a
// least-significant-digit radix sort of (u32 key, u32 value) pairs, 8 bits per
// pass, stable, and the exclusive scan it needs. Plan-time only (not in the
// timed path); hand-written so that the plan's vertex orders do not depend on
// a library's sort.
//
// One pass over digit d = (key >> shift) & mask, tiles of 4096 pairs:
//   k_rs_hist     per-tile digit counts            -> hist[d * T + tile]
//   exclusive_scan_u32 over (digit-major, tile-minor) -> first output position
//                                                     of each (digit, tile)
//   k_rs_scatter  every pair's stable rank inside its tile: warp w owns the
//                 tile's w-th run of 512 pairs and walks it 32 at a time;
//                 __match_any_sync groups the lanes of equal digit, a pair's
//                 rank is the warp's running count of its digit plus the
//                 number of lower lanes in its group; the running counts of
//                 the 8 warps are then prefixed per digit on top of the
//                 tile's scanned base.
#include "common.cuh"
#include "plan.h"

namespace umcg {
namespace {

constexpr int RS_T = 256;                  // threads
constexpr int RS_ITEMS = 16;               // pairs per thread
constexpr int RS_TILE = RS_T * RS_ITEMS;   // 4096 pairs per tile
constexpr int RS_W = RS_T / 32;            // warps
constexpr int RS_RUN = RS_TILE / RS_W;     // 512 consecutive pairs per warp

template <class K>
__global__ void __launch_bounds__(RS_T) k_rs_hist(const K* __restrict__ keys, uint64_t n, int shift,
                                                  uint32_t mask, uint64_t T, uint32_t* __restrict__ hist) {
    __shared__ uint32_t h[256];
    h[threadIdx.x] = 0;
    __syncthreads();
    const uint64_t base = (uint64_t)blockIdx.x * RS_TILE;
    const uint32_t lt = (1u << (threadIdx.x & 31)) - 1u;
#pragma unroll
    for (int j = 0; j < RS_ITEMS; ++j) {
        const uint64_t i = base + (uint64_t)j * RS_T + threadIdx.x;
        // one atomic per group of equal digits in the warp (clustered keys
        // would otherwise serialize on one counter)
        const uint32_t d = i < n ? (uint32_t)(keys[i] >> shift) & mask : 0x100u + (threadIdx.x & 31);
        const uint32_t peers = __match_any_sync(0xffffffffu, d);
        if (i < n && (peers & lt) == 0) atomicAdd(&h[d], (uint32_t)__popc(peers));
    }
    __syncthreads();
    hist[(uint64_t)threadIdx.x * T + blockIdx.x] = h[threadIdx.x];
}

// vals_out == nullptr: keys only; vals == nullptr: the values are the indices
template <class K>
__global__ void __launch_bounds__(RS_T) k_rs_scatter(const K* __restrict__ keys,
                                                     const uint32_t* __restrict__ vals, uint64_t n, int shift,
                                                     uint32_t mask, uint64_t T, const uint32_t* __restrict__ offs,
                                                     K* __restrict__ keys_out,
                                                     uint32_t* __restrict__ vals_out) {
    __shared__ uint32_t wc[RS_W][256];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int k = 0; k < RS_W; ++k) wc[k][threadIdx.x] = 0;
    __syncthreads();
    const uint64_t first = (uint64_t)blockIdx.x * RS_TILE + (uint64_t)w * RS_RUN;
    K key[RS_ITEMS];
    uint32_t val[RS_ITEMS], rank[RS_ITEMS];
#pragma unroll
    for (int j = 0; j < RS_ITEMS; ++j) {
        const uint64_t i = first + (uint64_t)j * 32 + lane;
        const bool ok = i < n;
        key[j] = ok ? keys[i] : (K)0;
        val[j] = ok && vals_out ? (vals ? vals[i] : (uint32_t)i) : 0u;
    }
    const uint32_t lt = (1u << lane) - 1u;
#pragma unroll
    for (int j = 0; j < RS_ITEMS; ++j) {
        const bool ok = first + (uint64_t)j * 32 + lane < n;
        // lanes past the end form groups of their own and count nothing
        const uint32_t d = ok ? (uint32_t)(key[j] >> shift) & mask : 0x100u + (uint32_t)lane;
        const uint32_t peers = __match_any_sync(0xffffffffu, d);
        const uint32_t before = ok ? wc[w][d] : 0u;
        rank[j] = before + __popc(peers & lt);
        __syncwarp();
        if (ok && (peers & lt) == 0) wc[w][d] = before + __popc(peers);
        __syncwarp();
    }
    __syncthreads();
    {   // digit threadIdx.x: the warps' counts -> their first output positions
        uint32_t run = offs[(uint64_t)threadIdx.x * T + blockIdx.x];
#pragma unroll
        for (int k = 0; k < RS_W; ++k) {
            const uint32_t c = wc[k][threadIdx.x];
            wc[k][threadIdx.x] = run;
            run += c;
        }
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < RS_ITEMS; ++j) {
        if (first + (uint64_t)j * 32 + lane >= n) continue;
        const uint32_t o = wc[w][(uint32_t)(key[j] >> shift) & mask] + rank[j];
        keys_out[o] = key[j];
        if (vals_out) vals_out[o] = val[j];
    }
}

// ---- exclusive scan of u32 (in place), 4096 entries per CTA -------------------
constexpr int SC_T = 256, SC_ITEMS = 16, SC_TILE = SC_T * SC_ITEMS;

__device__ __forceinline__ uint32_t block_exclusive(uint32_t v, uint32_t* total) {
    __shared__ uint32_t ws[SC_T / 32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    uint32_t inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += t;
    }
    __syncthreads();  // ws may still be read by a previous call
    if (lane == 31) ws[w] = inc;
    __syncthreads();
    uint32_t base = 0, tot = 0;
#pragma unroll
    for (int k = 0; k < SC_T / 32; ++k) {
        if (k < w) base += ws[k];
        tot += ws[k];
    }
    *total = tot;
    return base + inc - v;
}

__global__ void __launch_bounds__(SC_T) k_sc_sums(const uint32_t* __restrict__ a, uint64_t n, uint32_t* __restrict__ sums) {
    const uint64_t base = (uint64_t)blockIdx.x * SC_TILE + (uint64_t)threadIdx.x * SC_ITEMS;
    uint32_t s = 0;
#pragma unroll
    for (int k = 0; k < SC_ITEMS; ++k) s += base + k < n ? a[base + k] : 0u;
    uint32_t tot;
    block_exclusive(s, &tot);
    if (threadIdx.x == 0) sums[blockIdx.x] = tot;
}

// one CTA: exclusive scan of the tile sums, SC_TILE at a time with a carry
__global__ void __launch_bounds__(SC_T) k_sc_top(uint32_t* __restrict__ sums, uint64_t m) {
    uint32_t carry = 0;
    for (uint64_t o = 0; o < m; o += SC_TILE) {
        const uint64_t base = o + (uint64_t)threadIdx.x * SC_ITEMS;
        uint32_t v[SC_ITEMS], s = 0;
#pragma unroll
        for (int k = 0; k < SC_ITEMS; ++k) {
            v[k] = base + k < m ? sums[base + k] : 0u;
            s += v[k];
        }
        uint32_t tot;
        uint32_t run = carry + block_exclusive(s, &tot);
#pragma unroll
        for (int k = 0; k < SC_ITEMS; ++k) {
            if (base + k < m) sums[base + k] = run;
            run += v[k];
        }
        carry += tot;
    }
}

__global__ void __launch_bounds__(SC_T) k_sc_apply(uint32_t* __restrict__ a, uint64_t n, const uint32_t* __restrict__ sums) {
    const uint64_t base = (uint64_t)blockIdx.x * SC_TILE + (uint64_t)threadIdx.x * SC_ITEMS;
    uint32_t v[SC_ITEMS], s = 0;
#pragma unroll
    for (int k = 0; k < SC_ITEMS; ++k) {
        v[k] = base + k < n ? a[base + k] : 0u;
        s += v[k];
    }
    uint32_t tot;
    uint32_t run = sums[blockIdx.x] + block_exclusive(s, &tot);
#pragma unroll
    for (int k = 0; k < SC_ITEMS; ++k) {
        if (base + k < n) a[base + k] = run;
        run += v[k];
    }
}

}  // namespace

void exclusive_scan_u32(uint32_t* d_a, uint64_t n, DevBuf& scratch, cudaStream_t st) {
    if (!n) return;
    const uint64_t m = cdiv(n, (uint64_t)SC_TILE);
    uint32_t* sums = scratch.as<uint32_t>(m);
    k_sc_sums<<<(unsigned)m, SC_T, 0, st>>>(d_a, n, sums);
    UMCG_LAUNCHED();
    k_sc_top<<<1, SC_T, 0, st>>>(sums, m);
    UMCG_LAUNCHED();
    k_sc_apply<<<(unsigned)m, SC_T, 0, st>>>(d_a, n, sums);
    UMCG_LAUNCHED();
}

namespace {
template <class K>
void radix_sort_impl(const K* keys_in, K* keys_out, const uint32_t* vals_in, uint32_t* vals_out, uint64_t n,
                     int begin_bit, int end_bit, DevBuf& tmp_pairs, DevBuf& tmp_hist, DevBuf& tmp_scan,
                     cudaStream_t st) {
    if (!n) return;
    if (n >= (1ull << 32)) fail(UMCG_INVALID_ARGUMENT, "radix sort: more than 2^32-1 items");
    const int bits = end_bit - begin_bit;
    const int passes = bits <= 0 ? 1 : (bits + 7) / 8;
    const uint64_t T = cdiv(n, (uint64_t)RS_TILE);
    uint32_t* hist = tmp_hist.as<uint32_t>(256 * T);
    K* tk = nullptr;
    uint32_t* tv = nullptr;
    if (passes > 1) {
        auto* raw = tmp_pairs.as<uint8_t>(n * (sizeof(K) + 4) + 16);
        tk = reinterpret_cast<K*>(raw);
        tv = vals_out ? reinterpret_cast<uint32_t*>(raw + n * sizeof(K)) : nullptr;
    }
    const K* sk = keys_in;
    const uint32_t* sv = vals_in;  // nullptr: the values are 0..n-1
    for (int p = 0; p < passes; ++p) {
        // the last pass lands in the caller's arrays
        const bool to_out = ((passes - 1 - p) & 1) == 0;
        K* dk = to_out ? keys_out : tk;
        uint32_t* dv = to_out ? vals_out : tv;
        const int shift = begin_bit + 8 * p;
        const int nb = bits <= 0 ? 0 : std::min(8, end_bit - shift);
        const uint32_t mask = (1u << nb) - 1u;
        k_rs_hist<K><<<(unsigned)T, RS_T, 0, st>>>(sk, n, shift, mask, T, hist);
        UMCG_LAUNCHED();
        exclusive_scan_u32(hist, 256 * T, tmp_scan, st);
        k_rs_scatter<K><<<(unsigned)T, RS_T, 0, st>>>(sk, sv, n, shift, mask, T, hist, dk, dv);
        UMCG_LAUNCHED();
        sk = dk;
        sv = dv;
    }
}
}  // namespace

void radix_sort_pairs_u32(const uint32_t* keys_in, uint32_t* keys_out, const uint32_t* vals_in, uint32_t* vals_out,
                          uint64_t n, int begin_bit, int end_bit, DevBuf& tmp_pairs, DevBuf& tmp_hist,
                          DevBuf& tmp_scan, cudaStream_t st) {
    radix_sort_impl(keys_in, keys_out, vals_in, vals_out, n, begin_bit, end_bit, tmp_pairs, tmp_hist, tmp_scan, st);
}

void radix_sort_u64(const uint64_t* keys_in, uint64_t* keys_out, const uint32_t* vals_in, uint32_t* vals_out,
                    uint64_t n, int begin_bit, int end_bit, DevBuf& tmp_pairs, DevBuf& tmp_hist, DevBuf& tmp_scan,
                    cudaStream_t st) {
    radix_sort_impl(keys_in, keys_out, vals_in, vals_out, n, begin_bit, end_bit, tmp_pairs, tmp_hist, tmp_scan, st);
}

}  // namespace umcg
