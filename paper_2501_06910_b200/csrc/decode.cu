// Fused single-pass decode of a 1-D varint code stream on sm_100a:
//   unpacked varint bytes -> code boundaries (MSB-clear bytes) -> element
//   index and lattice index K = inclusive prefix of zigzag codes, both by one
//   decoupled look-back scan over 4 KiB byte tiles -> epilogue.
// Epilogues:
//   P64        K as int64 (grid component, further N-D scans follow)
//   VALUES     fl(K * bin)                       (codec.hpp:434 on the lattice)
//   RECOMPOSE  fl(fl(K1[node_i] * bin1) + fl(K * bin2))  (pipeline.hpp:206-208,
//              nearest g, grid component as int32 lattice indices: the decoded
//              grid value x1'[j] is exactly fl(K1[j] * bin1), so the gather
//              touches a 4-byte array that stays resident in L2)
#include <cub/block/block_scan.cuh>

#include "decode.h"
#include "scan_tiles.cuh"
#include <cub/block/block_reduce.cuh>

namespace umcg {

#ifndef UMCG_GATHER_LD
#define UMCG_GATHER_LD __ldcg  // load of the random K1 gathers: L2 only (A/B: __ldg 2 % slower)
#endif

namespace {


struct CS {
    uint64_t cnt;
    int64_t sum;
};
struct CSAdd {
    __device__ __forceinline__ CS operator()(const CS& a, const CS& b) const {
        return CS{a.cnt + b.cnt, a.sum + b.sum};
    }
};

// ---- three-phase (reduce, scan, apply) decode: every phase is fully
// parallel, no inter-CTA waiting. Tiles of 8 KiB of varint bytes.
constexpr int RT = 256;
constexpr int RB = 32;
constexpr uint64_t RTILE = (uint64_t)RT * RB;
constexpr int RHALO = 16;

// Stage tile bytes [base-16, base+RTILE) into 16-byte aligned shared memory:
// aligned 16-byte global loads (a 16-byte granule holding a valid byte lies
// inside the allocation) realigned with funnel shifts, then padding bytes:
// before the stream -> 0x00 (acts as a code end), past the end -> 0x80.
__device__ __forceinline__ void stage_tile(const uint8_t* __restrict__ U, uint64_t ulen, int64_t base,
                                           uint8_t* sb) {
    const int64_t lo = base - RHALO;
    const intptr_t A = (intptr_t)U + lo;  // address of smem byte 0 (may precede U)
    const intptr_t a0 = A & ~(intptr_t)15;
    const int sh = (int)(A - a0);
    const intptr_t g_lo = (intptr_t)U & ~(intptr_t)15;
    const intptr_t g_hi = ((intptr_t)U + (intptr_t)ulen + 15) & ~(intptr_t)15;
    constexpr int NCH = (RHALO + (int)RTILE) / 16;
    const uint64_t pol = l2_evict_first();
    uint4* dst = reinterpret_cast<uint4*>(sb);
    for (int j = threadIdx.x; j < NCH; j += RT) {
        const intptr_t c0 = a0 + 16 * (intptr_t)j, c1 = c0 + 16;
        uint4 x = make_uint4(0, 0, 0, 0), y = make_uint4(0, 0, 0, 0);
        if (c0 >= g_lo && c0 < g_hi) x = ld_v4_hint(reinterpret_cast<const void*>(c0), pol);
        if (sh && c1 >= g_lo && c1 < g_hi) y = ld_v4_hint(reinterpret_cast<const void*>(c1), pol);
        const uint32_t w[8] = {x.x, x.y, x.z, x.w, y.x, y.y, y.z, y.w};
        const int ws = sh >> 2, bs = 8 * (sh & 3);
        uint32_t o[4];
#pragma unroll
        for (int m = 0; m < 4; ++m) {
            uint32_t l = w[m], h = w[m + 1];
#pragma unroll
            for (int q = 1; q < 4; ++q)
                if (ws == q) { l = w[m + q]; h = w[m + q + 1]; }
            o[m] = __funnelshift_r(l, h, bs);
        }
        dst[j] = make_uint4(o[0], o[1], o[2], o[3]);
    }
    __syncthreads();
    if (lo < 0 || base + (int64_t)RTILE > (int64_t)ulen) {  // first / last tile only
        for (int k = threadIdx.x; k < RHALO + (int)RTILE; k += RT) {
            const int64_t off = lo + k;
            if (off < 0) sb[k] = 0x00;
            else if (off >= (int64_t)ulen) sb[k] = 0x80;
        }
    }
}

// Sequential varint walk over a thread's 32 bytes held in registers, seeded
// with the partial varint that straddles in from the 16 halo bytes. emit(v)
// is called for every code that ends inside the thread's bytes. Lossy PQ
// codes are zigzag(int32) < 2^32 (codec.hpp:305, 322), so values are
// accumulated in 32 bits; a longer varint sets *wide and the caller falls
// back to the general decoder.
// W: the thread's 48-byte window, 16 halo bytes then its 32 bytes, as words.
template <class F>
__device__ __forceinline__ void thread_walk(const uint32_t (&W)[12], int64_t gbase, uint64_t ulen, bool* bad,
                                            bool* wide, F&& emit) {
    const uint32_t hw[4] = {W[0], W[1], W[2], W[3]};
    const uint32_t w[8] = {W[4], W[5], W[6], W[7], W[8], W[9], W[10], W[11]};
    // continuation bytes immediately before my first byte
    int hlen = 0;
    bool run = true;
#pragma unroll
    for (int j = 15; j >= 6; --j) {
        const uint32_t hb = (hw[j >> 2] >> (8 * (j & 3))) & 0xffu;
        run = run && (hb & 0x80u);
        hlen += run ? 1 : 0;
    }
    uint32_t acc = 0;
    int shift = 0;
#pragma unroll
    for (int j = 11; j < 16; ++j) {
        const uint32_t hb = (hw[j >> 2] >> (8 * (j & 3))) & 0xffu;
        if (j >= 16 - hlen) {
            acc |= (hb & 0x7fu) << shift;
            shift += 7;
        }
    }
    int crun = hlen;
    bool wd = hlen > 4 && gbase < (int64_t)ulen;
#pragma unroll
    for (int k = 0; k < RB; ++k) {
        const uint32_t byte = (w[k >> 2] >> (8 * (k & 3))) & 0xffu;
        acc |= (byte & 0x7fu) << (shift & 31);
        wd |= (shift == 28) && (byte > 0x0fu) && (gbase + k < (int64_t)ulen);
        shift += 7;
        if (!(byte & 0x80u)) {
            emit(acc);
            acc = 0;
            shift = 0;
            crun = 0;
        } else {
            ++crun;
            if (crun >= 5 && gbase + k < (int64_t)ulen) {  // padding past the end is 0x80
                wd = true;
                if (crun >= 10) *bad = true;
            }
        }
    }
    *wide |= wd;
}

// 7-bit payloads of 4 varint bytes, concatenated (byte 0 lowest): 28 bits.
__device__ __forceinline__ uint32_t payload28(uint32_t x) {
    uint32_t y = x & 0x7f7f7f7fu;
    y = (y & 0x007f007fu) | ((y & 0x7f007f00u) >> 1);
    return (y & 0x00003fffu) | ((y & 0x3fff0000u) >> 2);
}
// Bit k set when byte k of x ends a varint (MSB clear).
__device__ __forceinline__ uint32_t ends4(uint32_t x) {
    return ((((~x) & 0x80808080u) >> 7) * 0x10204080u) >> 28;
}

// SWAR fast path of thread_walk for the common case: every code that ends
// in this thread's bytes is <= 4 bytes long (values < 2^28) and no run of 4
// continuation bytes touches them. Code ends come from a bit mask, values
// from a 64-bit window of concatenated 7-bit payloads, so the cost is per
// code rather than per byte. Returns false -- having emitted nothing -- when
// the general walk must run instead (long codes, end padding, corruption).
template <class F>
__device__ __forceinline__ bool thread_walk_fast(const uint32_t (&W)[12], F&& emit) {
    const uint32_t h3 = W[3];  // the 4 bytes before mine
    uint32_t w[RB / 4];
#pragma unroll
    for (int q = 0; q < RB / 4; ++q) w[q] = W[4 + q];
    uint64_t E = ends4(h3);  // bit i: byte i - 4 ends a code
#pragma unroll
    for (int q = 0; q < RB / 4; ++q) E |= (uint64_t)ends4(w[q]) << (4 + 4 * q);
    const uint64_t C = ~E & ((1ull << (4 + RB)) - 1);  // continuation bytes
    if (C & (C >> 1) & (C >> 2) & (C >> 3)) return false;
    // partial code entering from the halo: its trailing 0..3 continuation bytes
    const int hl = (C >> 3 & 1) ? ((C >> 2 & 1) ? ((C >> 1 & 1) ? 3 : 2) : 1) : 0;
    uint32_t acc = hl ? payload28(h3) >> (7 * (4 - hl)) : 0u;
    uint32_t shift = 7 * hl;
    // uniform byte loop without the long-code bookkeeping (ruled out above)
#pragma unroll
    for (int k = 0; k < RB; ++k) {
        const uint32_t byte = __byte_perm(w[k >> 2], 0, k & 3);
        acc |= (byte & 0x7fu) << shift;
        shift += 7;
        if (!(byte & 0x80u)) {
            emit(acc);
            acc = 0;
            shift = 0;
        }
    }
    return true;
}

__device__ __forceinline__ void smem_window(const uint8_t* sb, int my, uint32_t (&W)[12]) {
    const uint4* p = reinterpret_cast<const uint4*>(sb + my - 16);
#pragma unroll
    for (int q = 0; q < 3; ++q) {
        const uint4 a = p[q];
        W[4 * q] = a.x;
        W[4 * q + 1] = a.y;
        W[4 * q + 2] = a.z;
        W[4 * q + 3] = a.w;
    }
}

// The same window straight from global memory (no shared-memory staging: the
// L1 it leaves serves the random K1 gathers of k_dec_out): stream bytes
// [g - 16, g + 32) from 16-byte aligned loads realigned with funnel shifts,
// then the padding of stage_tile (before the stream 0x00, past its end 0x80).
__device__ __forceinline__ void global_window(const uint8_t* __restrict__ U, uint64_t ulen, int64_t g,
                                              uint64_t pol, uint32_t (&W)[12]) {
    const intptr_t A = (intptr_t)U + g - 16;
    const intptr_t a0 = A & ~(intptr_t)15;
    const int sh = (int)(A - a0);
    const intptr_t g_lo = (intptr_t)U & ~(intptr_t)15;
    const intptr_t g_hi = ((intptr_t)U + (intptr_t)ulen + 15) & ~(intptr_t)15;
    uint32_t r[16];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const intptr_t c = a0 + 16 * q;
        uint4 x = make_uint4(0, 0, 0, 0);
        if ((q < 3 || sh) && c >= g_lo && c < g_hi) x = ld_v4_hint(reinterpret_cast<const void*>(c), pol);
        r[4 * q] = x.x;
        r[4 * q + 1] = x.y;
        r[4 * q + 2] = x.z;
        r[4 * q + 3] = x.w;
    }
    const int ws = sh >> 2, bs = 8 * (sh & 3);
#pragma unroll
    for (int m = 0; m < 12; ++m) {
        uint32_t l = r[m], h = r[m + 1];
#pragma unroll
        for (int q = 1; q < 4; ++q)
            if (ws == q) { l = r[m + q]; h = r[m + q + 1]; }
        W[m] = __funnelshift_r(l, h, bs);
    }
    if (g - 16 < 0 || g + 32 > (int64_t)ulen) {  // first / last thread windows only
#pragma unroll
        for (int k = 0; k < 48; ++k) {
            const int64_t off = g - 16 + k;
            const uint32_t b = off < 0 ? 0x00u : 0x80u;
            if (off < 0 || off >= (int64_t)ulen)
                W[k >> 2] = (W[k >> 2] & ~(0xffu << (8 * (k & 3)))) | (b << (8 * (k & 3)));
        }
    }
}

__device__ __forceinline__ int64_t zz_dec32(uint32_t v) { return (int64_t)(v >> 1) ^ -(int64_t)(v & 1u); }

// Byte-parallel (count, sum of zigzag values) of the codes that end in the
// thread's 32 bytes, for the common case of codes of at most 2 bytes (the
// thread's window) -- no per-byte walk. With per-byte flag words (bit 7 of
// each byte): t = code ends here, s0 = code starts here (previous byte ends
// one), s1 = second byte of a code. A code c = p0 + 128 p1 (7-bit payloads)
// decodes to unzigzag(c) = +((p0 >> 1) + 64 p1) when p0 is even and
// -((p0 >> 1) + 64 p1) - 1 when odd, so the sum is four byte-masked dot
// products (dp4a against 0/1 byte masks) per word:
//   sum = A0 - 2 A0odd + 64 (A1 - 2 A1odd) - n_odd.
// Included bytes: the partial code entering from the halo (bytes of W[3]
// after its last end) and every byte of the thread up to its last end.
// Returns false (nothing computed) when a code of 3+ bytes touches the
// thread, or its first or last word has no code end: the walk then runs.
__device__ __forceinline__ bool thread_counts_swar(const uint32_t (&W)[12], uint32_t& cnt, int64_t& sum) {
    constexpr uint32_t M7 = 0x80808080u;
    const uint32_t t3 = ~W[3] & M7, t11 = ~W[11] & M7;
    if (!t3 || !t11) return false;
    const uint32_t keepH = (t3 & 0x80000000u) ? 0u : (0xffffffffu << (32 - __clz(t3)));
    const uint32_t keepL = (t11 & 0x80000000u) ? 0xffffffffu : (0xffffffffu >> __clz(t11));
    uint32_t tp = M7, s0p = 0, s1p = 0, wp = 0, more = 0;
    uint32_t a0 = 0, a0o = 0, a1 = 0, a1o = 0, no = 0, c = 0;
#pragma unroll
    for (int q = 3; q < 12; ++q) {
        const uint32_t w = W[q];
        const uint32_t t = ~w & M7;
        const uint32_t s0 = __funnelshift_l(tp, t, 8);
        const uint32_t s1 = __funnelshift_l(s0p, s0, 8) & ~s0;
        const uint32_t keep = q == 3 ? keepH : (q == 11 ? keepL : 0xffffffffu);
        more |= __funnelshift_l(s1p, s1, 8) & ~s0 & keep;  // third byte of a code
        const uint32_t sel0 = (s0 & keep) >> 7, sel1 = (s1 & keep) >> 7;
        const uint32_t odd0 = sel0 & w, odd1 = sel1 & __funnelshift_l(wp, w, 8);
        const uint32_t p0 = (w >> 1) & 0x3f3f3f3fu, p = w & 0x7f7f7f7fu;
        a0 = __dp4a(p0, sel0, a0);
        a0o = __dp4a(p0, odd0, a0o);
        a1 = __dp4a(p, sel1, a1);
        a1o = __dp4a(p, odd1, a1o);
        no = __dp4a(odd0, 0x01010101u, no);
        if (q >= 4) c += __popc(t);
        tp = t;
        s0p = s0;
        s1p = s1;
        wp = w;
    }
    if (more) return false;
    cnt = c;
    sum = (int64_t)a0 - 2 * (int64_t)a0o + 64 * ((int64_t)a1 - 2 * (int64_t)a1o) - (int64_t)no;
    return true;
}

__device__ __forceinline__ CS thread_counts(const uint8_t* sb, int my, bool* bad, bool* wide, int64_t base,
                                            uint64_t ulen) {
    uint32_t W[12];
    smem_window(sb, my, W);
    {
        uint32_t c2;
        int64_t s2;
        if (thread_counts_swar(W, c2, s2)) return CS{c2, s2};
    }
    uint32_t c = 0;
    // fast path: codes of <= 4 bytes ending in 32 bytes, so |sum| < 8 * 2^27
    // fits 32-bit accumulation (the emit runs predicated on every byte)
    int32_t s32 = 0;
    auto f32 = [&](uint32_t v) {
        ++c;
        s32 += (int32_t)(v >> 1) ^ -(int32_t)(v & 1u);
    };
    if (thread_walk_fast(W, f32)) return CS{c, (int64_t)s32};
    int64_t s = 0;
    auto f = [&](uint32_t v) {
        ++c;
        s += zz_dec32(v);
    };
    thread_walk(W, base + (my - RHALO), ulen, bad, wide, f);
    return CS{c, s};
}

// Per-thread prefix inside a tile, packed into one int64: sum * 2^16 + count
// (count <= 8192 codes per 8 KiB tile, |sum| < 2^44), so the block scan and
// the hand-off to k_dec_out move 8 bytes per thread instead of 16.
__device__ __forceinline__ int64_t cs_pack(const CS& a) { return (int64_t)((uint64_t)a.sum << 16) + (int64_t)a.cnt; }
__device__ __forceinline__ CS cs_unpack(int64_t v) { return CS{(uint64_t)(v & 0xffff), v >> 16}; }

// Tile aggregates (count, sum of zigzag values); tiles past the stream end
// (T is a host-side bound when the stream is resolved on the device) add 0.
// thr: every thread's exclusive (count, sum) inside its tile, so k_dec_out
// starts its walk without a counting walk + block scan of its own.
#ifndef UMCG_AGG_MINB
#define UMCG_AGG_MINB 6  // 6 CTAs per SM (A/B: 1 -> 0.178 ms, 6 or 8 -> 0.168 ms; 8 spills)
#endif
__global__ void __launch_bounds__(RT, UMCG_AGG_MINB) k_dec_agg(const DecSrc src, CS* __restrict__ aggs,
                                                               int64_t* __restrict__ thr, DevCtl* ctl) {
    const uint8_t* U;
    uint64_t ulen;
    resolve_src(src, U, ulen);
    if ((uint64_t)blockIdx.x * RTILE >= ulen) {
        if (threadIdx.x == 0) aggs[blockIdx.x] = CS{0, 0};
        return;
    }
    using BS = cub::BlockScan<int64_t, RT>;
    __shared__ typename BS::TempStorage tmp;
    __shared__ __align__(16) uint8_t sb[RHALO + RTILE + 16];
    const int64_t base = (int64_t)blockIdx.x * (int64_t)RTILE;
    stage_tile(U, ulen, base, sb);
    __syncthreads();
    bool bad = false, wide = false;
    const CS mine = thread_counts(sb, RHALO + threadIdx.x * RB, &bad, &wide, base, ulen);
    if (bad) set_err(ctl, DE_CORRUPT_VARINT);
    if (wide) ctl->aux[7] = 1;
    int64_t excl, t;
    BS(tmp).ExclusiveSum(cs_pack(mine), excl, t);
    if (threadIdx.x == 0) aggs[blockIdx.x] = cs_unpack(t);
    thr[blockIdx.x * (uint64_t)RT + threadIdx.x] = excl;
}

template <int MODE, class KT>
#ifndef UMCG_DEC_MINB
#define UMCG_DEC_MINB 6  // CTAs per SM (A/B with .cg gathers: 5 -> 0.739 ms, 6 -> 0.704 ms)
#endif
#ifndef UMCG_DEC_UN
#define UMCG_DEC_UN 8
#endif
__global__ void __launch_bounds__(RT, UMCG_DEC_MINB) k_dec_out(const DecSrc src, uint64_t n,
                                               const CS* __restrict__ pre, DevCtl* ctl,
                                               const uint32_t* __restrict__ node, const KT* __restrict__ K1,
                                               double bin1, double bin, double* __restrict__ out,
                                               int64_t* __restrict__ P64, const DevCtl* __restrict__ kctl,
                                               const int16_t* __restrict__ K16, const CS* __restrict__ raw,
                                               const int64_t* __restrict__ thr) {
    // lattice indices of the tile in element order, int16 (the decoded K of
    // a lossy residual stream fits; a tile that does not takes the direct
    // path below)
    constexpr bool PREFIX = MODE == DEC_P64 || MODE == DEC_Q32;
    __shared__ int16_t kb[PREFIX ? 1 : RTILE];
    // P64 mode: K - (tile prefix) as int32, written out coalesced afterwards;
    // Q32 mode: the zigzag-decoded code itself
    __shared__ int32_t kp[PREFIX ? RTILE : 1];
#ifdef UMCG_DEC_PAD  // (A/B: shared-memory footprint vs the L1 left for the K1 gathers)
    __shared__ volatile uint8_t pad_[PREFIX ? 1 : UMCG_DEC_PAD];
    if (threadIdx.x == 0) pad_[0] = 0;
#endif
    // int32 tables: switch to the int16 copy when the grid's max|K1| (known
    // on the device only) allows -- half the L2 footprint of the gather
    const bool use16 = sizeof(KT) == 4 && K16 && kctl && kctl->max_abs_k[0] < 32768;
    const uint8_t* U;
    uint64_t ulen;
    resolve_src(src, U, ulen);
    if ((uint64_t)blockIdx.x * RTILE >= ulen) return;
    const int64_t base = (int64_t)blockIdx.x * (int64_t)RTILE;
    const int my = RHALO + threadIdx.x * RB;
    uint32_t W[12];
    global_window(U, ulen, base + threadIdx.x * RB, l2_evict_first(), W);
    // the thread's prefix inside the tile and the tile's total (k_dec_agg)
    const CS excl = cs_unpack(thr[blockIdx.x * (uint64_t)RT + threadIdx.x]);
    const CS tot = raw[blockIdx.x];
    const CS tp = pre[blockIdx.x];
    const uint64_t e0 = tp.cnt;           // first element of the tile
    uint32_t li = (uint32_t)excl.cnt;     // local element index
    int64_t K = tp.sum + excl.sum;
    uint64_t kmax = 0;
    bool bad2 = false, wide2 = false;
    const uint32_t li0 = li;
    const int64_t K0 = K;
    bool ovf = false;  // P64: some K - tp.sum outside int32
    auto f = [&](uint32_t v) {
        K += zz_dec32(v);
        const uint64_t a = (uint64_t)(K < 0 ? -K : K);
        kmax = a > kmax ? a : kmax;
        if (MODE == DEC_Q32) {
            kp[li] = (int32_t)zz_dec32(v);  // exact: |q| <= 2^31 for a u32 code
        } else if (MODE == DEC_P64) {
            const int64_t d = K - tp.sum;
            ovf |= d != (int64_t)(int32_t)d;
            kp[li] = (int32_t)d;
        } else {
            kb[li] = (int16_t)K;  // exact when kmax < 2^15 (else the direct path)
        }
        ++li;
    };
    if (!thread_walk_fast(W, f)) thread_walk(W, base + (my - RHALO), ulen, &bad2, &wide2, f);
    for (int o = 16; o; o >>= 1) {
        const uint64_t b2 = __shfl_xor_sync(0xffffffffu, kmax, o);
        kmax = b2 > kmax ? b2 : kmax;
    }
    if ((threadIdx.x & 31) == 0 && kmax > ctl->max_abs_k[1]) atomicMax(&ctl->max_abs_k[1], (unsigned long long)kmax);
    if (MODE == DEC_Q32) {
        __syncthreads();
        int32_t* Q = reinterpret_cast<int32_t*>(P64);
        const uint32_t cnt = (uint32_t)tot.cnt;
        for (uint32_t e = threadIdx.x; e < cnt; e += RT) {
            const uint64_t i = e0 + e;
            if (i < n) Q[i] = kp[e];
        }
        return;
    }
    if (MODE == DEC_P64) {
        if (__syncthreads_or(ovf)) {  // rare: walk again, writing in the walk's order
            li = li0;
            K = K0;
            bool b3 = false, w3 = false;
            auto g = [&](uint32_t v) {
                K += zz_dec32(v);
                const uint64_t i = e0 + li;
                if (i < n) P64[i] = K;
                ++li;
            };
            if (!thread_walk_fast(W, g)) thread_walk(W, base + (my - RHALO), ulen, &b3, &w3, g);
            return;
        }
        const uint32_t cnt = (uint32_t)tot.cnt;
        for (uint32_t e = threadIdx.x; e < cnt; e += RT) {
            const uint64_t i = e0 + e;
            if (i < n) P64[i] = tp.sum + (int64_t)kp[e];
        }
        return;
    }
    const bool use16t = sizeof(KT) == 2 || use16;
    auto recompose = [&](uint64_t i, int64_t k) {
        const double r = __dmul_rn((double)k, bin);
        if (MODE == DEC_VALUES) {
            out[i] = r;
        } else if (MODE == DEC_RECOMPOSE_GE) {
            out[i] = __dadd_rn(reinterpret_cast<const double*>(K1)[node[i]], r);
        } else {
            const uint32_t nd = node[i];
            const int32_t g = use16t ? (int32_t)__ldg((sizeof(KT) == 2 ? reinterpret_cast<const int16_t*>(K1) : K16) + nd)
                                     : reinterpret_cast<const int32_t*>(K1)[nd];
            out[i] = __dadd_rn(__dmul_rn((double)g, bin1), r);
        }
    };
    if (__syncthreads_or(kmax >= 32768)) {
        // rare: some K of the tile does not fit int16 -- walk again and write
        // the outputs in the walk's order
        li = li0;
        K = K0;
        bool b3 = false, w3 = false;
        auto g = [&](uint32_t v) {
            K += zz_dec32(v);
            const uint64_t i = e0 + li;
            if (i < n) recompose(i, K);
            ++li;
        };
        if (!thread_walk_fast(W, g)) thread_walk(W, base + (my - RHALO), ulen, &b3, &w3, g);
        return;
    }
    const uint32_t cnt = (uint32_t)tot.cnt;
    constexpr int UN = UMCG_DEC_UN;  // independent gathers in flight per thread
    const uint64_t pf = l2_evict_first(), pl = l2_evict_last();
    for (uint32_t e0 = 0; e0 < cnt; e0 += RT * UN) {
        uint32_t nd[UN];
#pragma unroll
        for (int u = 0; u < UN; ++u) {
            const uint32_t e = e0 + u * RT + threadIdx.x;
            nd[u] = ((MODE == DEC_RECOMPOSE || MODE == DEC_RECOMPOSE_GE) && e < cnt && tp.cnt + e < n)
                        ? ld_u32_hint(&node[tp.cnt + e], pf)
                        : 0u;
        }
        int32_t g1[UN];
        double ge[UN];
#pragma unroll
        for (int u = 0; u < UN; ++u) {
            const uint32_t e = e0 + u * RT + threadIdx.x;
            ge[u] = (MODE == DEC_RECOMPOSE_GE && e < cnt && tp.cnt + e < n)
                        ? UMCG_GATHER_LD(reinterpret_cast<const double*>(K1) + nd[u])
                        : 0.0;
            if (MODE == DEC_RECOMPOSE && e < cnt && tp.cnt + e < n)
                g1[u] = sizeof(KT) == 2 || use16
                            ? (int32_t)UMCG_GATHER_LD((sizeof(KT) == 2 ? reinterpret_cast<const int16_t*>(K1) : K16) + nd[u])
                            : ld_s32_hint(reinterpret_cast<const int32_t*>(K1) + nd[u], pl);
            else
                g1[u] = 0;
        }
#pragma unroll
        for (int u = 0; u < UN; ++u) {
            const uint32_t e = e0 + u * RT + threadIdx.x;
            const uint64_t i = tp.cnt + e;
            if (e >= cnt || i >= n) continue;
            const double r = __dmul_rn((double)kb[e], bin);
            if (MODE == DEC_VALUES) st_f64_hint(&out[i], r, pf);
            else if (MODE == DEC_RECOMPOSE_GE) st_f64_hint(&out[i], __dadd_rn(ge[u], r), pf);  // approx + x2 (pipeline.hpp:208)
            else st_f64_hint(&out[i], __dadd_rn(__dmul_rn((double)g1[u], bin1), r), pf);
        }
    }
}

// Row differencing of a plain prefix P into per-row prefixes (scan along the
// fastest axis), i.e. the first axis of the N-D inclusive prefix sum.
__global__ void k_rows(const int64_t* __restrict__ P, uint64_t n, uint64_t R, int64_t* __restrict__ K) {
    const uint64_t i = blockIdx.x * 256ull + threadIdx.x;
    if (i >= n) return;
    const uint64_t r0 = i - i % R;
    K[i] = P[i] - (r0 ? P[r0 - 1] : 0);
}

// Inclusive scan along axis d (d < D-1): threads own consecutive positions
// of the fastest axis (coalesced), loop over the scanned axis.
__global__ void k_axis_cols(int64_t* __restrict__ K, uint64_t n, uint64_t len, uint64_t stride) {
    const uint64_t line = blockIdx.x * 256ull + threadIdx.x;
    const uint64_t n_lines = n / len;
    if (line >= n_lines) return;
    const uint64_t outer = line / stride, inner = line % stride;
    const uint64_t b = outer * len * stride + inner;
    int64_t acc = 0;
    for (uint64_t k = 0; k < len; ++k) {
        acc += K[b + k * stride];
        K[b + k * stride] = acc;
    }
}

// Fused N-D prefix for D = 2 / 3 from the plain row-major prefix P:
//   out[..., j, k] = sum_{j' <= j} (P[..., j', k] - P[row(..., j') - 1])
// i.e. the row scan (fastest axis) by differencing P, then the scan along
// the middle axis. Threads own (outer, k) lines, 8 loads in flight.
// For D == 2 the result is final (int32 + max|K|); for D == 3 an int64
// intermediate follows, finished by k_nd_outer.
// With few lines (2-D grids: one line per column) the middle axis is split
// into blockIdx.y chunks of rows: chunk sums (k_nd_mid_sums), their exclusive
// scan per line (k_nd_chunk_scan), then every chunk resumes from its offset.
__global__ void __launch_bounds__(256) k_nd_mid_sums(const int64_t* __restrict__ P, uint64_t d_out, uint64_t d_mid,
                                                    uint64_t d_fast, uint64_t rows, int64_t* __restrict__ csum) {
    const uint64_t lines = d_out * d_fast;
    const uint64_t line = blockIdx.x * 256ull + threadIdx.x;
    if (line >= lines) return;
    const uint64_t o = line / d_fast, k = line % d_fast;
    const uint64_t base = o * d_mid * d_fast;
    const uint64_t j0 = blockIdx.y * rows, j1 = min(d_mid, j0 + rows);
    int64_t acc = 0;
    for (uint64_t j = j0; j < j1; ++j) {
        const uint64_t r = base + j * d_fast;
        acc += __ldg(&P[r + k]) - (r ? __ldg(&P[r - 1]) : 0);
    }
    csum[blockIdx.y * lines + line] = acc;
}

__global__ void k_nd_chunk_scan(int64_t* __restrict__ csum, uint64_t lines, uint32_t nch) {
    const uint64_t line = blockIdx.x * 256ull + threadIdx.x;
    if (line >= lines) return;
    int64_t acc = 0;
    for (uint32_t c = 0; c < nch; ++c) {
        const int64_t v = csum[c * lines + line];
        csum[c * lines + line] = acc;
        acc += v;
    }
}

template <bool FINAL>
__global__ void __launch_bounds__(256) k_nd_mid(const int64_t* __restrict__ P, uint64_t d_out, uint64_t d_mid,
                                               uint64_t d_fast, int64_t* __restrict__ Kw, int32_t* __restrict__ K32,
                                               int16_t* __restrict__ K16, DevCtl* ctl,
                                               const int64_t* __restrict__ coff, uint64_t rows) {
    const uint64_t line = blockIdx.x * 256ull + threadIdx.x;  // over d_out * d_fast
    uint64_t amax = 0;
    if (line < d_out * d_fast) {
        const uint64_t o = line / d_fast, k = line % d_fast;
        const uint64_t base = o * d_mid * d_fast;
        int64_t acc = coff ? coff[blockIdx.y * d_out * d_fast + line] : 0;
        const uint64_t jb = blockIdx.y * rows, je = min(d_mid, jb + rows);
        for (uint64_t j0 = jb; j0 < je; j0 += 8) {
            int64_t v[8], rb[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const uint64_t j = j0 + u;
                if (j < je) {
                    const uint64_t r = base + j * d_fast;
                    v[u] = __ldcs(&P[r + k]);
                    rb[u] = r ? __ldg(&P[r - 1]) : 0;
                } else {
                    v[u] = 0;
                    rb[u] = 0;
                }
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const uint64_t j = j0 + u;
                if (j >= je) break;
                acc += v[u] - rb[u];
                const uint64_t idx = base + j * d_fast + k;
                if (FINAL) {
                    K32[idx] = (int32_t)acc;
                    if (K16) K16[idx] = (int16_t)acc;
                    const uint64_t a = (uint64_t)(acc < 0 ? -acc : acc);
                    amax = a > amax ? a : amax;
                } else {
                    Kw[idx] = acc;
                }
            }
        }
    }
    if (FINAL) {
        for (int o = 16; o; o >>= 1) {
            const uint64_t b = __shfl_xor_sync(0xffffffffu, amax, o);
            amax = b > amax ? b : amax;
        }
        if ((threadIdx.x & 31) == 0 && amax > ctl->max_abs_k[0]) atomicMax(&ctl->max_abs_k[0], (unsigned long long)amax);
    }
}

// Last scan for D == 3 along the outer axis (stride d1*d2), int32 out + max|K|.
__global__ void __launch_bounds__(256) k_nd_outer(const int64_t* __restrict__ Kw, uint64_t d0, uint64_t plane,
                                                 int32_t* __restrict__ K32, int16_t* __restrict__ K16, DevCtl* ctl) {
    const uint64_t c = blockIdx.x * 256ull + threadIdx.x;
    uint64_t amax = 0;
    if (c < plane) {
        int64_t acc = 0;
        for (uint64_t i0 = 0; i0 < d0; i0 += 8) {
            int64_t v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) v[u] = i0 + u < d0 ? __ldcs(&Kw[(i0 + u) * plane + c]) : 0;
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                if (i0 + u >= d0) break;
                acc += v[u];
                K32[(i0 + u) * plane + c] = (int32_t)acc;
                if (K16) K16[(i0 + u) * plane + c] = (int16_t)acc;
                const uint64_t a = (uint64_t)(acc < 0 ? -acc : acc);
                amax = a > amax ? a : amax;
            }
        }
    }
    for (int o = 16; o; o >>= 1) {
        const uint64_t b = __shfl_xor_sync(0xffffffffu, amax, o);
        amax = b > amax ? b : amax;
    }
    if ((threadIdx.x & 31) == 0 && amax > ctl->max_abs_k[0]) atomicMax(&ctl->max_abs_k[0], (unsigned long long)amax);
}

// 3-D inverse Lorenzo from the decoded codes q (int32, row-major d0 x d1 x d2,
// d2 <= 256), first stage: per plane i, the 2-D inclusive prefix over (j, k),
//   S[i, j, k] = sum_{j' <= j, k' <= k} q[i, j', k'] = K[i] - K[i - 1].
// One CTA per plane, thread = column k. The plane is walked in tiles of 32
// rows whose 32 loads per thread are all in flight (the next tile's loads are
// issued before the current tile is processed), so a plane costs d1 / 32
// memory round trips instead of one per row: column prefix in registers,
// row prefix by a shared-memory transpose (lane = 8 consecutive columns,
// in-lane prefix + one warp scan), S stored coalesced.
// Arithmetic is int32 modulo 2^32; it is exact when sum over the plane of |q|
// < 2^31 (then no partial sum leaves int32), which every plane checks -- a
// plane that does not fails the fast decompress's verdict (max|K| := ~0).
constexpr int ND3_T = 256;
constexpr int ND3_R = 32;
__global__ void __launch_bounds__(ND3_T) k_nd3_plane(const int32_t* __restrict__ Q, uint32_t d1, uint32_t d2,
                                                     int32_t* __restrict__ S, DevCtl* ctl) {
    __shared__ __align__(16) int32_t tile[ND3_R][ND3_T];
    const uint64_t plane = (uint64_t)d1 * d2;
    const int32_t* q = Q + (uint64_t)blockIdx.x * plane;
    int32_t* s = S + (uint64_t)blockIdx.x * plane;
    const uint32_t k = threadIdx.x;
    const bool col = k < d2;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    int32_t nx[ND3_R];
    auto load = [&](uint32_t j0) {
#pragma unroll
        for (int r = 0; r < ND3_R; ++r) nx[r] = (col && j0 + r < d1) ? __ldcs(&q[(uint64_t)(j0 + r) * d2 + k]) : 0;
    };
    load(0);
    uint64_t asum = 0;
    int32_t carry = 0;
    for (uint32_t j0 = 0; j0 < d1; j0 += ND3_R) {
        int32_t v[ND3_R];
#pragma unroll
        for (int r = 0; r < ND3_R; ++r) v[r] = nx[r];
        if (j0 + ND3_R < d1) load(j0 + ND3_R);
#pragma unroll
        for (int r = 0; r < ND3_R; ++r) {
            asum += (uint32_t)(v[r] < 0 ? -v[r] : v[r]);
            carry += v[r];  // column prefix (mod 2^32)
            tile[r][k] = carry;
        }
        __syncthreads();
        // row prefix of rows warp, warp + 8, ...: lane owns columns 8 lane .. 8 lane + 7
#pragma unroll
        for (int rr = 0; rr < ND3_R / (ND3_T / 32); ++rr) {
            const int r = warp + rr * (ND3_T / 32);
            const uint32_t j = j0 + r;
            const int4 a = *reinterpret_cast<const int4*>(&tile[r][8 * lane]);
            const int4 b = *reinterpret_cast<const int4*>(&tile[r][8 * lane + 4]);
            int32_t x[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
            for (int u = 1; u < 8; ++u) x[u] += x[u - 1];
            int32_t p = x[7];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int32_t y = __shfl_up_sync(0xffffffffu, p, o);
                if (lane >= o) p += y;
            }
            const int32_t off = p - x[7];  // exclusive prefix of the lane totals
            if (j < d1) {
                int32_t* row = s + (uint64_t)j * d2;
                const uint32_t kb = 8 * lane;
                if ((d2 & 7) == 0 && kb + 8 <= d2) {
                    int4 o0 = make_int4(x[0] + off, x[1] + off, x[2] + off, x[3] + off);
                    int4 o1 = make_int4(x[4] + off, x[5] + off, x[6] + off, x[7] + off);
                    if ((reinterpret_cast<uintptr_t>(row) & 15) == 0) {
                        *reinterpret_cast<int4*>(row + kb) = o0;
                        *reinterpret_cast<int4*>(row + kb + 4) = o1;
                    } else {
#pragma unroll
                        for (int u = 0; u < 8; ++u) row[kb + u] = x[u] + off;
                    }
                } else {
#pragma unroll
                    for (int u = 0; u < 8; ++u)
                        if (kb + u < d2) row[kb + u] = x[u] + off;
                }
            }
        }
        __syncthreads();
    }
    // exactness: with sum |q| < 2^31 over the plane no partial sum wrapped
    if (__syncthreads_or(asum >= 0x80000000ull) && threadIdx.x == 0) atomicMax(&ctl->max_abs_k[0], ~0ull);
}

// Second stage: K[i] = sum_{i' <= i} S[i'] along the outer axis (exact int64
// accumulation of the exact S), threads own (j, k) columns; planes in tiles
// of 32 with all loads of the next tile in flight. int32 + int16 tables and
// max|K|.
__global__ void __launch_bounds__(256) k_nd3_outer(const int32_t* __restrict__ S, uint32_t d0, uint64_t plane,
                                                  int32_t* __restrict__ K32, int16_t* __restrict__ K16,
                                                  DevCtl* ctl) {
    const uint64_t c = blockIdx.x * 256ull + threadIdx.x;
    uint64_t amax = 0;
    if (c < plane) {
        int32_t nx[ND3_R];
        auto load = [&](uint32_t i0) {
#pragma unroll
            for (int u = 0; u < ND3_R; ++u) nx[u] = i0 + u < d0 ? __ldcs(&S[(i0 + u) * plane + c]) : 0;
        };
        load(0);
        int64_t acc = 0;
        for (uint32_t i0 = 0; i0 < d0; i0 += ND3_R) {
            int32_t v[ND3_R];
#pragma unroll
            for (int u = 0; u < ND3_R; ++u) v[u] = nx[u];
            if (i0 + ND3_R < d0) load(i0 + ND3_R);
#pragma unroll
            for (int u = 0; u < ND3_R; ++u) {
                if (i0 + u >= d0) break;
                acc += v[u];
                K32[(i0 + u) * plane + c] = (int32_t)acc;
                if (K16) K16[(i0 + u) * plane + c] = (int16_t)acc;
                const uint64_t a = (uint64_t)(acc < 0 ? -acc : acc);
                amax = a > amax ? a : amax;
            }
        }
    }
    for (int o = 16; o; o >>= 1) {
        const uint64_t b = __shfl_xor_sync(0xffffffffu, amax, o);
        amax = b > amax ? b : amax;
    }
    if ((threadIdx.x & 31) == 0 && amax > ctl->max_abs_k[0]) atomicMax(&ctl->max_abs_k[0], (unsigned long long)amax);
}

__global__ void k_k32(const int64_t* __restrict__ K, uint64_t n, int32_t* __restrict__ K32,
                      int16_t* __restrict__ K16, DevCtl* ctl) {
    const uint64_t i = blockIdx.x * 256ull + threadIdx.x;
    uint64_t a = 0;
    if (i < n) {
        const int64_t v = K[i];
        K32[i] = (int32_t)v;
        if (K16) K16[i] = (int16_t)v;
        a = (uint64_t)(v < 0 ? -v : v);
    }
    for (int o = 16; o; o >>= 1) {
        const uint64_t b = __shfl_xor_sync(0xffffffffu, a, o);
        a = b > a ? b : a;
    }
    if ((threadIdx.x & 31) == 0 && a > ctl->max_abs_k[0]) atomicMax(&ctl->max_abs_k[0], (unsigned long long)a);
}

__global__ void k_k32_to_f64(const int32_t* __restrict__ K, uint64_t n, double bin, double* __restrict__ x) {
    const uint64_t i = blockIdx.x * 256ull + threadIdx.x;
    if (i < n) x[i] = __dmul_rn((double)K[i], bin);
}

}  // namespace

// status: exclusive tile prefixes CS[T + 1] | tile aggregates CS[T] |
// per-thread prefixes CS[T * RT]
size_t dec_status_bytes(uint64_t ulen) {
    const uint64_t T = cdiv(ulen, RTILE);
    return (2 * T + 1 + T * RT) * sizeof(CS);
}
uint64_t dec_tiles(uint64_t ulen_bound) { return cdiv(ulen_bound, RTILE); }

void dec_prepare(const DecSrc& src, uint64_t T, void* status, DevCtl* ctl, cudaStream_t st) {
    auto* aggs = static_cast<CS*>(status);
    if (!T) {
        UMCG_CUDA(cudaMemsetAsync(&ctl->count, 0, sizeof(ctl->count), st));
        return;
    }
    CS* raw = aggs + T + 1;
    auto* thr = reinterpret_cast<int64_t*>(raw + T);
    {
        ProfScope ps_a("k_dec_agg", st);
        k_dec_agg<<<(unsigned)T, RT, 0, st>>>(src, raw, thr, ctl);
        UMCG_LAUNCHED();
    }
    static_assert(sizeof(CS) == sizeof(ulonglong2), "CS scans as a pair of 64-bit sums");
    k_scan_tiles<<<scan_tiles_grid(T), SCAN_TILES_THREADS, 0, st>>>(reinterpret_cast<const ulonglong2*>(raw),
                                                                    reinterpret_cast<ulonglong2*>(aggs), T,
                                                                    nullptr, &ctl->count);
    UMCG_LAUNCHED();
}

void dec_fused(int mode, const DecSrc& src, uint64_t T, uint64_t n, void* status, DevCtl* ctl,
               const uint32_t* node, const int32_t* K1, double bin1, double bin, double* out, int64_t* P64,
               cudaStream_t st, const DevCtl* kctl, const int16_t* K16, bool prepared) {
    auto* aggs = static_cast<CS*>(status);
    if (!prepared) dec_prepare(src, T, status, ctl, st);
    if (!T) return;
    ProfScope ps_o(mode == DEC_P64 || mode == DEC_Q32 ? "k_dec_out_grid" : "k_dec_out", st);
    const CS* raw = aggs + T + 1;
    const auto* thr = reinterpret_cast<const int64_t*>(raw + T);
    if (mode == DEC_Q32)
        k_dec_out<DEC_Q32, int32_t><<<(unsigned)T, RT, 0, st>>>(src, n, aggs, ctl, node, K1, bin1, bin, out, P64,
                                                               nullptr, nullptr, raw, thr);
    else if (mode == DEC_P64)
        k_dec_out<DEC_P64, int32_t><<<(unsigned)T, RT, 0, st>>>(src, n, aggs, ctl, node, K1, bin1, bin, out, P64,
                                                               nullptr, nullptr, raw, thr);
    else if (mode == DEC_VALUES)
        k_dec_out<DEC_VALUES, int32_t><<<(unsigned)T, RT, 0, st>>>(src, n, aggs, ctl, node, K1, bin1, bin, out, P64,
                                                                  nullptr, nullptr, raw, thr);
    else if (mode == DEC_RECOMPOSE_GE)
        k_dec_out<DEC_RECOMPOSE_GE, int32_t><<<(unsigned)T, RT, 0, st>>>(src, n, aggs, ctl, node, K1, bin1, bin, out,
                                                                        P64, nullptr, nullptr, raw, thr);
    else if (mode == DEC_RECOMPOSE16)
        k_dec_out<DEC_RECOMPOSE, int16_t><<<(unsigned)T, RT, 0, st>>>(src, n, aggs, ctl, node,
                                                                     reinterpret_cast<const int16_t*>(K1), bin1, bin,
                                                                     out, P64, nullptr, nullptr, raw, thr);
    else
        k_dec_out<DEC_RECOMPOSE, int32_t><<<(unsigned)T, RT, 0, st>>>(src, n, aggs, ctl, node, K1, bin1, bin, out, P64,
                                                                     kctl, K16, raw, thr);
    UMCG_LAUNCHED();
}

void nd_from_prefix(const int64_t* P, uint64_t n, const NdShape& sh, int64_t* Kw, int32_t* K32, int16_t* K16,
                    DevCtl* ctl, cudaStream_t st) {
    const unsigned g = (unsigned)cdiv(n, 256);
    if (!n) return;
    const int64_t* src = P;
    if (sh.D == 2 || sh.D == 3) {
        const uint64_t d2 = sh.dims[sh.D - 1], d1 = sh.dims[sh.D - 2], d0 = sh.D == 3 ? sh.dims[0] : 1;
        const uint64_t lines = d0 * d2;
        const unsigned g1 = (unsigned)cdiv(lines, 256);
        // enough threads: split the middle axis into chunks when lines are few
        uint32_t nch = 1;
        while (nch < 64 && lines * nch < 65536 && d1 / (2 * nch) >= 16) nch *= 2;
        const uint64_t rows = cdiv(d1, (uint64_t)nch);
        int64_t* csum = nullptr;
        if (nch > 1) {
            // scratch: Kw is unused for D == 2; for D == 3 K32 is written only later
            csum = sh.D == 2 ? Kw : reinterpret_cast<int64_t*>(K32);
            k_nd_mid_sums<<<dim3(g1, nch), 256, 0, st>>>(P, d0, d1, d2, rows, csum);
            UMCG_LAUNCHED();
            k_nd_chunk_scan<<<g1, 256, 0, st>>>(csum, lines, nch);
            UMCG_LAUNCHED();
        }
        if (sh.D == 2) {
            k_nd_mid<true><<<dim3(g1, nch), 256, 0, st>>>(P, d0, d1, d2, nullptr, K32, K16, ctl, csum, rows);
            UMCG_LAUNCHED();
        } else {
            k_nd_mid<false><<<dim3(g1, nch), 256, 0, st>>>(P, d0, d1, d2, Kw, nullptr, nullptr, ctl, csum, rows);
            UMCG_LAUNCHED();
            k_nd_outer<<<(unsigned)cdiv(d1 * d2, 256), 256, 0, st>>>(Kw, d0, d1 * d2, K32, K16, ctl);
            UMCG_LAUNCHED();
        }
        return;
    }
    if (sh.D > 1) {
        k_rows<<<g, 256, 0, st>>>(P, n, sh.dims[sh.D - 1], Kw);
        UMCG_LAUNCHED();
        for (int d = sh.D - 2; d >= 0; --d) {
            const uint64_t lines = n / sh.dims[d];
            k_axis_cols<<<(unsigned)cdiv(lines, 256), 256, 0, st>>>(Kw, n, sh.dims[d], sh.strides[d]);
            UMCG_LAUNCHED();
        }
        src = Kw;
    }
    k_k32<<<g, 256, 0, st>>>(src, n, K32, K16, ctl);
    UMCG_LAUNCHED();
}

bool nd3_supported(const NdShape& sh) {
    return sh.D == 3 && sh.dims[2] >= 1 && sh.dims[2] <= (uint64_t)ND3_T && sh.dims[1] < (1ull << 31) &&
           sh.dims[0] < (1ull << 31);
}

void nd3_from_codes(const int32_t* Q, const NdShape& sh, int32_t* S, int32_t* K32, int16_t* K16, DevCtl* ctl,
                    cudaStream_t st) {
    const uint64_t d0 = sh.dims[0], d1 = sh.dims[1], d2 = sh.dims[2];
    if (!d0 || !d1 || !d2) return;
    k_nd3_plane<<<(unsigned)d0, ND3_T, 0, st>>>(Q, (uint32_t)d1, (uint32_t)d2, S, ctl);
    UMCG_LAUNCHED();
    k_nd3_outer<<<(unsigned)cdiv(d1 * d2, 256), 256, 0, st>>>(S, (uint32_t)d0, d1 * d2, K32, K16, ctl);
    UMCG_LAUNCHED();
}

void k32_to_f64(const int32_t* K, uint64_t n, double bin, double* x, cudaStream_t st) {
    if (!n) return;
    k_k32_to_f64<<<(unsigned)cdiv(n, 256), 256, 0, st>>>(K, n, bin, x);
    UMCG_LAUNCHED();
}

}  // namespace umcg
