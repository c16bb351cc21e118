// Partitioned compress path (nearest g): cluster means and residual lattice
// indices with coalesced HBM traffic only.
//
// The reference computes x1[j] = (sum of x_i over the vertices mapped to j,
// in ascending i) / count_j with a random scatter in vertex order
// (interp.hpp:58-64), then x2_i = x_i - x1[m_i] with a random gather
// (interp.hpp:145-147, 167-168). Vertex order carries no locality (the mesh
// is permuted), so on the GPU both would be random 8-byte accesses into
// 1 GB / 134 MB arrays. Instead, with the plan's static bucketing
// (plan.cu: contiguous slot ranges of <= 4096 vertices, vertices of a bucket
// in ascending vertex order):
//   k_partition   x -> xp (bucket order) + value range / finiteness
//                 (pipeline.hpp:31-41, mesh.hpp:58-64), one streaming pass;
//   k_bucket      per bucket, xp staged in shared memory: ordered segment
//                 sums (bit-exact: same additions in the same order as the
//                 reference), x1 written once, residual lattice index
//                 K2 = round((x - x1[m]) / bin2) per vertex (bucket order);
//   k_resid_codes back to vertex order through dst: q_i = K2_i - K2_{i-1},
//                 zigzag codes + the RLE tile summary in the same pass.
#include <cmath>
#include <cstdlib>
#include <type_traits>

#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>

#include "encode_dev.cuh"
#include "multilinear.cuh"
#include "plan.h"

namespace umcg {

#ifndef UMCG_GATHER_LD
#define UMCG_GATHER_LD __ldcg  // load of the random gathers: L2 only (A/B: __ldg 2-3 % slower)
#endif

namespace {

constexpr int PT = 256;

// Forward permutation into layout E: xE[p] = x[srcE[p]] (gather inside one
// epoch's window) + value range / finiteness over the same values.
constexpr int GI = 8;  // items per thread (strided by PT for coalescing)
template <class T>
__global__ void __launch_bounds__(PT) k_gather_fwd(const T* __restrict__ x, uint64_t n,
                                                  const uint32_t* __restrict__ srcE, double* __restrict__ xE,
                                                  DevCtl* ctl) {
    using BR = cub::BlockReduce<unsigned long long, PT>;
    __shared__ typename BR::TempStorage t1, t2;
    unsigned long long lo = ~0ull, hi = 0ull;
    int bad = 0;
    const uint64_t base = (uint64_t)blockIdx.x * PT * GI + threadIdx.x;
    uint32_t s[GI];
#pragma unroll
    for (int k = 0; k < GI; ++k) {
        const uint64_t p = base + (uint64_t)k * PT;
        s[k] = p < n ? __ldcs(srcE + p) : 0u;
    }
    double v[GI];
#pragma unroll
    for (int k = 0; k < GI; ++k) {
        const uint64_t p = base + (uint64_t)k * PT;
        v[k] = p < n ? (double)UMCG_GATHER_LD(x + s[k]) : 0.0;
    }
#pragma unroll
    for (int k = 0; k < GI; ++k) {
        const uint64_t p = base + (uint64_t)k * PT;
        if (p >= n) break;
        if (!isfinite(v[k])) { bad = 1; continue; }
        const unsigned long long key = dkey(v[k]);
        lo = key < lo ? key : lo;
        hi = key > hi ? key : hi;
        xE[p] = v[k];
    }
    const unsigned long long blo = BR(t1).Reduce(lo, cub::Min());
    const unsigned long long bhi = BR(t2).Reduce(hi, cub::Max());
    if (threadIdx.x == 0) {
        if (blo != ~0ull) atomicMin(&ctl->min_key, blo);
        if (bhi != 0ull) atomicMax(&ctl->max_key, bhi);
    }
    if (bad) ctl->nonfinite = 1;
}

constexpr int BT = 256;

__device__ __forceinline__ void flag_serial1(DevCtl* ctl) {
    if (ctl->need_serial[1] == 0) atomicExch(&ctl->need_serial[1], 1);
}

// lattice index with the escape / regime checks of codec.hpp:305-314
// (same as codes.cu lattice_k, 1-D limit 2^30). KT = int16_t is the narrow
// path: every |K| <= 16383 keeps each code zigzag(K_i - K_{i-1}) < 2^16. A
// larger |K| is not an escape, only too wide for int16 (e.g. multilinear g
// blending the 0.0 of unvisited nodes, interp.hpp:56, 78, 129, into a field
// far from zero): it flags need_wide and the host reruns the int32 path.
template <class KT>
__device__ __forceinline__ KT resid_k(double r, double bin, double inv, double tau, DevCtl* ctl) {
    double err;
    const double K = lattice_round(r, bin, inv, tau, &err);
    const bool bad = !(fabs(K) < 1073741824.0) || !(err <= tau);
    if (bad) flag_serial1(ctl);
    if (sizeof(KT) == 2 && !bad && !(fabs(K) <= 16383.0)) {
        if (ctl->need_wide == 0) atomicExch(&ctl->need_wide, 1);
        return 0;
    }
    return bad ? 0 : (KT)(int32_t)K;
}

// Grid lattice index of a cluster mean, fused into the bucket kernels for the
// dense N-D grid component (codes.cu lattice_k / k_lattice_nd, component 0).
struct GridK {
    int32_t* K1;  // nullptr: not fused
    double lim;   // 2^(31-D)
};
__device__ __forceinline__ void grid_k(const GridK& g, uint64_t j, double v, DevCtl* ctl) {
    if (!g.K1) return;
    double err;
    const double K = lattice_round(v, ctl->bin[0], ctl->inv_bin[0], ctl->tau_c[0], &err);
    if (!(fabs(K) < g.lim) || !(err <= ctl->tau_c[0])) {
        if (ctl->need_serial[0] == 0) atomicExch(&ctl->need_serial[0], 1);
    }
    g.K1[j] = (int32_t)K;
}

// Bucket b's elements, in bucket order l = 0..m-1, live in layout E as one
// chunk per epoch: pre[e] = first l of epoch e's chunk, cbase[e] = its
// layout-E position. Each warp moves whole chunks (coalesced).

template <class KT, uint32_t CAP, uint32_t NODES>
__global__ void __launch_bounds__(BT) k_bucket(const double* __restrict__ xE, const uint32_t* __restrict__ bk,
                                              uint64_t B, uint32_t E, const uint2* __restrict__ bct,
                                              const uint16_t* __restrict__ lnode,
                                              const uint16_t* __restrict__ lperm, const uint32_t* __restrict__ seg,
                                              DevCtl* ctl, double* __restrict__ x1, KT* __restrict__ KE,
                                              int heavy_only, GridK gk) {
    extern __shared__ __align__(128) unsigned char smem[];
    constexpr int PER = CAP / BT;  // elements per thread in a bucket
    double* xs = reinterpret_cast<double*>(smem);                      // [CAP]
    double* x1s = xs + CAP;                                            // [NODES]
    uint32_t* sg = reinterpret_cast<uint32_t*>(x1s + NODES);           // [NODES + 1]
    uint2* ch = reinterpret_cast<uint2*>(sg + NODES + 2);              // [E+1]
    uint16_t* lp = reinterpret_cast<uint16_t*>(ch + (E + 1));          // [CAP]
    uint16_t* ln = lp + CAP;                                           // [CAP]
    const uint32_t* bstart = bk;
    const uint32_t* bnode = bk + B + 1;
    const uint64_t b = blockIdx.x;
    const uint32_t s0 = bstart[b], s1 = bstart[b + 1], m = s1 - s0;
    const uint32_t j0 = bnode[b], j1 = bnode[b + 1], nj = j1 - j0;
    const double bin = ctl->bin[1], inv = ctl->inv_bin[1], tau = ctl->tau_c[1];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    constexpr int NW = BT / 32;
    // chunk table (one chunk per epoch, bucket-major) + segment offsets
    for (uint32_t e = threadIdx.x; e <= E; e += BT) ch[e] = __ldg(&bct[b * (uint64_t)(E + 1) + e]);
    const bool heavy = m > CAP;
    if (heavy_only && !heavy) return;
    if (!heavy)
        for (uint32_t j = threadIdx.x; j <= nj; j += BT) sg[j] = __ldg(&seg[j0 + j]) - s0;
    __syncthreads();
    if (heavy) {
        // one heavy slot: ordered sum straight from global memory
        if (threadIdx.x == 0) {
            double s = 0.0;
            for (uint32_t e = 0; e < E; ++e)
                for (uint32_t l = ch[e].x; l < ch[e + 1].x; ++l) s = __dadd_rn(s, xE[ch[e].y + (l - ch[e].x)]);
            x1s[0] = __ddiv_rn(s, (double)m);
            x1[j0] = x1s[0];
            grid_k(gk, j0, x1s[0], ctl);
        }
        __syncthreads();
        if (!KE) return;
        const double mean = x1s[0];
        for (uint32_t e = warp; e < E; e += NW)
            for (uint32_t l = ch[e].x + lane; l < ch[e + 1].x; l += 32) {
                const uint32_t q = ch[e].y + (l - ch[e].x);
                KE[q] = resid_k<KT>(__dsub_rn(xE[q], mean), bin, inv, tau, ctl);
            }
        return;
    }
    // each thread owns bucket elements l = t + k*BT; all loads issued up front
    uint32_t e_first = 0;
    {
        uint32_t lo = 0, hi = E;  // last chunk with first index <= threadIdx.x
        while (hi - lo > 1) {
            const uint32_t mid = (lo + hi) >> 1;
            if (ch[mid].x <= threadIdx.x) lo = mid; else hi = mid;
        }
        e_first = lo;
    }
    {
        double xv[PER];
        uint32_t e = e_first;
#pragma unroll
        for (int k = 0; k < PER; ++k) {
            const uint32_t l = threadIdx.x + k * BT;
            if (l < m) {
                while (l >= ch[e + 1].x) ++e;
                xv[k] = __ldcs(&xE[ch[e].y + (l - ch[e].x)]);
            }
        }
#pragma unroll
        for (int k = 0; k < PER; ++k) {
            const uint32_t l = threadIdx.x + k * BT;
            if (l < m) {
                lp[l] = __ldg(&lperm[s0 + l]);
                ln[l] = __ldg(&lnode[s0 + l]);
            }
        }
#pragma unroll
        for (int k = 0; k < PER; ++k) {
            const uint32_t l = threadIdx.x + k * BT;
            if (l < m) xs[l] = xv[k];
        }
    }
    __syncthreads();
    // interpolate_to_grid (interp.hpp:58-64): 0.0 + x_a + x_b + ... in ascending vertex order
    for (uint32_t j = threadIdx.x; j < nj; j += BT) {
        const uint32_t k0 = sg[j], k1 = sg[j + 1];
        double s = 0.0;
        for (uint32_t k = k0; k < k1; ++k) s = __dadd_rn(s, xs[lp[k]]);
        const double v = k1 > k0 ? __ddiv_rn(s, (double)(k1 - k0)) : 0.0;
        x1s[j] = v;
        x1[j0 + j] = v;
        grid_k(gk, j0 + j, v, ctl);
    }
    __syncthreads();
    if (!KE) return;
    // compute_residuals (interp.hpp:161-170) + lattice index (codec.hpp:307-314)
    {
        uint32_t e = e_first;
#pragma unroll 4
        for (int k = 0; k < PER; ++k) {
            const uint32_t l = threadIdx.x + k * BT;
            if (l < m) {
                while (l >= ch[e + 1].x) ++e;
                KE[ch[e].y + (l - ch[e].x)] = resid_k<KT>(__dsub_rn(xs[l], x1s[ln[l]]), bin, inv, tau, ctl);
            }
        }
    }
}


// ---- TMA variant ------------------------------------------------------------
// Persistent CTAs walk the regular (<= CAP vertices) buckets
// round-robin with two shared-memory stages: while bucket k is summed and
// quantized, bucket k+1 arrives through bulk asynchronous copies
// (cp.async.bulk, completion on an mbarrier): one copy
// per epoch chunk of xE, one each for the slot map, lnode and the segment
// offsets, issued by one warp. Chunk e is staged at slot base
// c0.x + 2e + phase_e (parity of the layout-E position, plan.cu k_lslot) so
// every copy is a 16-byte aligned superset of the chunk; the sums read xs
// through the plan's slot map instead of lperm.
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    uint32_t ok = 0;
    while (!ok) {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
            : "=r"(ok)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
    }
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

struct TmaStage {
    double* xs;     // [CAP + 2E + 4] slots
    uint16_t* ls;   // [CAP + 16]   slot map (node-sorted), phase s0 & 7
    uint16_t* ln;   // [CAP + 16]   lnode (bucket order),    phase s0 & 7
    uint2* ch;      // [E + 1]
};

// (segment offsets go straight to registers: two CTAs fit per SM)
template <uint32_t CAP>
__host__ __device__ __forceinline__ uint32_t tma_stage_bytes(uint32_t E) {
    const uint32_t b = (CAP + 2 * E + 4) * 8 + 2 * (CAP + 16) * 2 + (E + 1) * 8;
    return (b + 127) & ~127u;
}

template <uint32_t CAP>
__device__ __forceinline__ TmaStage make_tma_stage(unsigned char* p, uint32_t E) {
    TmaStage S;
    S.xs = reinterpret_cast<double*>(p);
    p += (CAP + 2 * E + 4) * 8;
    S.ls = reinterpret_cast<uint16_t*>(p);
    p += (CAP + 16) * 2;
    S.ln = reinterpret_cast<uint16_t*>(p);
    p += (CAP + 16) * 2;
    S.ch = reinterpret_cast<uint2*>(p);
    return S;
}

// Warp 0 issues the bulk copies of one bucket into S (its chunk table S.ch
// must already be in shared memory and visible to warp 0).
__device__ __forceinline__ void tma_issue(const TmaStage& S, uint64_t* bar, const double* __restrict__ xE,
                                          const uint16_t* __restrict__ lslot, const uint16_t* __restrict__ lnode,
                                          uint32_t s0, uint32_t m, uint32_t E) {
    const int lane = threadIdx.x & 31;
    // bytes of this lane's chunks
    uint32_t bytes = 0;
    for (uint32_t e = lane; e < E; e += 32) {
        const uint2 c0 = S.ch[e], c1 = S.ch[e + 1];
        const uint32_t cnt = c1.x - c0.x;
        if (!cnt) continue;
        const uint32_t glo = c0.y & ~1u, ghi = (c0.y + cnt + 1) & ~1u;
        bytes += 8 * (ghi - glo);
    }
    for (int o = 16; o; o >>= 1) bytes += __shfl_xor_sync(0xffffffffu, bytes, o);
    const uint32_t a0 = s0 & ~7u, a1 = (s0 + m + 7) & ~7u;  // u16 arrays
    const uint32_t small = (a1 - a0) * 2 * 2;
    // prior generic-proxy reads of this stage (ordered by __syncthreads) before
    // the async-proxy writes
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (lane == 0) {
        mbar_expect_tx(bar, bytes + small);
        if (a1 > a0) {
            bulk_g2s(S.ls, lslot + a0, (a1 - a0) * 2, bar);
            bulk_g2s(S.ln, lnode + a0, (a1 - a0) * 2, bar);
        }
    }
    __syncwarp();
    for (uint32_t e = lane; e < E; e += 32) {
        const uint2 c0 = S.ch[e], c1 = S.ch[e + 1];
        const uint32_t cnt = c1.x - c0.x;
        if (!cnt) continue;
        const uint32_t glo = c0.y & ~1u, ghi = (c0.y + cnt + 1) & ~1u;
        const uint32_t sbase = c0.x + 2 * e + ((c0.y - c0.x - 2 * e) & 1u);
        bulk_g2s(S.xs + (sbase - (c0.y & 1u)), xE + glo, 8 * (ghi - glo), bar);
    }
}


// The warp that issues the next bucket's bulk copies (~100 cycles per copy,
// E + 2 copies): the last warp, which owns slots only in buckets of more
// than 480 slots, so the issue overlaps the other warps' ordered sums.



// CAP vertices / NODES slots per bucket, BTP threads, MINB CTAs per SM.
template <class KT, uint32_t CAP, uint32_t NODES, int BTP, int MINB>
__global__ void __launch_bounds__(BTP, MINB) k_bucket_tma(const double* __restrict__ xE, const uint32_t* __restrict__ bk,
                                                  uint64_t B, uint32_t E, const uint2* __restrict__ bct,
                                                  const uint32_t* __restrict__ regular, uint32_t n_regular,
                                                  const uint16_t* __restrict__ lnode,
                                                  const uint16_t* __restrict__ lslot,
                                                  const uint32_t* __restrict__ seg, DevCtl* ctl,
                                                  double* __restrict__ x1, KT* __restrict__ KE, GridK gk) {
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ __align__(8) uint64_t bars[2];
    double* x1s = reinterpret_cast<double*>(smem);
    static_assert(NODES <= 2 * BTP, "k_bucket_tma keeps <= 2 slots per thread in registers");
    constexpr int BT_ISSUE_WARP = BTP / 32 - 1;
    const uint32_t stage_bytes = tma_stage_bytes<CAP>(E);
    auto stage = [&](int st) { return make_tma_stage<CAP>(smem + NODES * 8 + st * stage_bytes, E); };
    const uint32_t* bstart = bk;
    const uint32_t* bnode = bk + B + 1;
    const double bin = ctl->bin[1], inv = ctl->inv_bin[1], tau = ctl->tau_c[1];
    const uint32_t G = gridDim.x;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint32_t k = blockIdx.x;
    if (k >= n_regular) return;
    if (threadIdx.x == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    struct Info { uint32_t s0, m, j0, nj; };
    auto load_info = [&](uint32_t bb) {
        const uint32_t a0 = __ldg(&bstart[bb]), a1 = __ldg(&bstart[bb + 1]);
        const uint32_t c0 = __ldg(&bnode[bb]), c1 = __ldg(&bnode[bb + 1]);
        return Info{a0, a1 - a0, c0, c1 - c0};
    };
    uint32_t b = __ldg(&regular[k]);
    Info cur = load_info(b);
    if (threadIdx.x <= E) stage(0).ch[threadIdx.x] = __ldg(&bct[b * (uint64_t)(E + 1) + threadIdx.x]);
    __syncthreads();
    if (warp == BT_ISSUE_WARP) tma_issue(stage(0), &bars[0], xE, lslot, lnode, cur.s0, cur.m, E);
    uint2 chreg = make_uint2(0, 0);
    Info nxt{0, 0, 0, 0};
    uint32_t b2 = 0;
    if (k + G < n_regular) {
        const uint32_t bn = __ldg(&regular[k + G]);
        nxt = load_info(bn);
        if (threadIdx.x <= E) chreg = __ldg(&bct[bn * (uint64_t)(E + 1) + threadIdx.x]);
        if (k + 2 * G < n_regular) b2 = __ldg(&regular[k + 2 * G]);
    }
    // UMCG_BT_PROF: per-phase clock64 totals of thread 0 (printf, debug builds)
#ifdef UMCG_BT_PROF
    long long tp_issue = 0, tp_wait = 0, tp_sum = 0, tp_res = 0, tq = 0;
    uint32_t nb_prof = 0;
#define BT_T0() tq = clock64()
#define BT_ACC(v) do { const long long t_ = clock64(); v += t_ - tq; tq = t_; } while (0)
#else
#define BT_T0() do {} while (0)
#define BT_ACC(v) do {} while (0)
#endif
    for (uint32_t it = 0; k < n_regular; ++it, k += G) {
        const int st = it & 1;
        const bool has_next = k + G < n_regular;
        if (has_next && threadIdx.x <= E) stage(st ^ 1).ch[threadIdx.x] = chreg;
        __syncthreads();
        BT_T0();
        Info nn{0, 0, 0, 0};
        uint32_t b3 = 0;
        if (has_next) {
            if (warp == BT_ISSUE_WARP)
                tma_issue(stage(st ^ 1), &bars[st ^ 1], xE, lslot, lnode, nxt.s0, nxt.m, E);
            BT_ACC(tp_issue);
            if (k + 2 * G < n_regular) {
                nn = load_info(b2);
                if (threadIdx.x <= E) chreg = __ldg(&bct[b2 * (uint64_t)(E + 1) + threadIdx.x]);
                if (k + 3 * G < n_regular) b3 = __ldg(&regular[k + 3 * G]);
            }
        }
        const uint32_t s0 = cur.s0, j0 = cur.j0, nj = cur.nj;
        // segment offsets of this thread's slots (NODES <= 2 * BTP), in flight during the wait
        uint32_t sgr[2][2] = {{0, 0}, {0, 0}};
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const uint32_t j = threadIdx.x + h * BTP;
            if (j < nj) {
                sgr[h][0] = __ldg(&seg[j0 + j]);
                sgr[h][1] = __ldg(&seg[j0 + j + 1]);
            }
        }
        BT_T0();
        mbar_wait(&bars[st], (it >> 1) & 1u);
        BT_ACC(tp_wait);
        const TmaStage C = stage(st);
        const uint32_t lo8 = s0 & 7u;
        // interpolate_to_grid (interp.hpp:58-64): 0.0 + x_a + x_b + ... in ascending vertex order
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const uint32_t j = threadIdx.x + h * BTP;
            if (j >= nj) break;
            const uint32_t k0 = sgr[h][0] - s0, k1 = sgr[h][1] - s0;
            double sum = 0.0;
            for (uint32_t q = k0; q < k1; ++q) sum = __dadd_rn(sum, C.xs[C.ls[q + lo8]]);
            const double v = k1 > k0 ? __ddiv_rn(sum, (double)(k1 - k0)) : 0.0;
            x1s[j] = v;
            x1[j0 + j] = v;
            grid_k(gk, j0 + j, v, ctl);
        }
        __syncthreads();
        BT_ACC(tp_sum);
        // compute_residuals (interp.hpp:161-170) + lattice index (codec.hpp:307-314)
        for (uint32_t e = warp; KE && e < E; e += BTP / 32) {
            const uint2 c0 = C.ch[e], c1 = C.ch[e + 1];
            const uint32_t sbase = c0.x + 2 * e + ((c0.y - c0.x - 2 * e) & 1u);
            for (uint32_t l = c0.x + lane; l < c1.x; l += 32)
                KE[c0.y + (l - c0.x)] =
                    resid_k<KT>(__dsub_rn(C.xs[sbase + (l - c0.x)], x1s[C.ln[l + lo8]]), bin, inv, tau, ctl);
        }
        cur = nxt;
        nxt = nn;
        b2 = b3;
        __syncthreads();
        BT_ACC(tp_res);
#ifdef UMCG_BT_PROF
        ++nb_prof;
#endif
    }
#ifdef UMCG_BT_PROF
    if (threadIdx.x == 0 && (blockIdx.x == 0 || blockIdx.x == 150))
        printf("[bt prof] block %u buckets %u cycles: issue %lld wait %lld sum %lld res %lld\n", blockIdx.x, nb_prof,
               tp_issue, tp_wait, tp_sum, tp_res);
#endif
#undef BT_T0
#undef BT_ACC
}

// ---- multilinear g in bucket order -------------------------------------------
// A bucket is a contiguous range of grid slots, so the cells around its
// vertices -- and the 2^D corner values multilinear_at reads -- stay within a
// few grid rows: walking layout E bucket by bucket (one warp per epoch chunk)
// keeps the corner gathers in L1/L2, where vertex order would scatter them
// over the whole grid.
struct MlGrid {
    const double* axes;
    const uint64_t* axis_off;
    const double* inv_cell;
    double scale[3];
    uint64_t shape[3];
    int D;
};

// Corner staging: a bucket is a contiguous slot range [j0, j1), its vertices
// map to those slots (their nearest nodes), and a vertex's cell corners lie
// within one node of its slot per axis. So every corner lies in one of three
// bands of x1, a*s0 + [j0 - w, j1 + w) for a in {-1, 0, 1} (s0 the slowest
// axis' stride, w = s1 + 1 in 3-D, 1 in 2-D), staged once per bucket in
// shared memory at fixed offsets (a + 1) * Lb, Lb = j1 - j0 + 2w. A corner's
// band is the offset of its slowest-axis index from the vertex's slot, so
// its staged index is plain int32 arithmetic from the vertex's bucket-local
// slot -- no range search. The cell itself comes from the slot too (one
// comparison per axis, verified against the axis; a vertex whose slot is not
// its nearest node takes the search and global corner loads).
constexpr int ML_T = 256;

struct MlDims {
    uint32_t s1, s12;  // strides of axes 1 and 0 (3-D), s12 = axis-0 stride
    int32_t w, Lb;     // band half-width, band length (per bucket)
};

__device__ __forceinline__ void ml_stage_band(double* xs, const double* __restrict__ x1, int64_t lo, int64_t hi,
                                              int64_t n1) {
    // node v -> xs[v - lo]; nodes outside the grid are never a corner
    const int64_t a = lo < 0 ? 0 : lo, b = hi > n1 ? n1 : hi;
    for (int64_t v = a + threadIdx.x; v < b; v += ML_T) xs[v - lo] = __ldg(&x1[v]);
}

// The cell of a vertex whose slot m is its nearest node: along each axis
// the lower index is m_d - 1 or m_d (one comparison), verified against the
// axis like the clamped upper_bound; the fraction t_d is the certified
// quotient of multilinear_eval_c, the same operations. Returns false when the
// slot is not a valid hint (then the vertex takes the generic evaluation).
template <int D>
__device__ __forceinline__ bool ml_cell(const MlGrid& g, uint32_t m, const double* p, double* t, uint32_t& bits) {
    uint32_t hint[3] = {0, 0, 0};
    if (D == 3) {
        const uint32_t s12 = (uint32_t)(g.shape[1] * g.shape[2]), s1 = (uint32_t)g.shape[2];
        hint[0] = m / s12;
        const uint32_t r = m - hint[0] * s12;
        hint[1] = r / s1;
        hint[2] = r - hint[1] * s1;
    } else if (D == 2) {
        hint[0] = m / (uint32_t)g.shape[1];
        hint[1] = m - hint[0] * (uint32_t)g.shape[1];
    } else {
        hint[0] = m;
    }
    bits = 0;
#pragma unroll
    for (int d = D - 1; d >= 0; --d) {
        const uint32_t n = (uint32_t)g.shape[d];
        double td = 0.0;
        if (n > 1) {
            const double* axis = g.axes + g.axis_off[d];
            int32_t c = (p[d] >= axis[hint[d]]) ? (int32_t)hint[d] : (int32_t)hint[d] - 1;
            c = c < 0 ? 0 : c;
            c = c > (int32_t)n - 2 ? (int32_t)n - 2 : c;
            const bool found = (c == 0 || axis[c] <= p[d]) && (c == (int32_t)n - 2 || p[d] < axis[c + 1]);
            if (!found || (c != (int32_t)hint[d] && c != (int32_t)hint[d] - 1)) return false;
            const double num = __dsub_rn(p[d], axis[c]), den = __dsub_rn(axis[c + 1], axis[c]);
            const double y = g.inv_cell[g.axis_off[d] + c];
            const double q0 = __dmul_rn(num, y);
            double w = __fma_rn(__fma_rn(-q0, den, num), y, q0);
            if (!(fabs(num) > 0x1p-900) || !(fabs(num) < 0x1p900) || !quotient_certified(num, den, w))
                w = __ddiv_rn(num, den);
            td = (w < 0.0) ? 0.0 : ((1.0 < w) ? 1.0 : w);  // std::clamp
            if (c != (int32_t)hint[d]) bits |= 1u << d;
        }
        t[d] = td;
    }
    return true;
}

// Plan-time preparation (first multilinear call on a plan): t_d and the cell
// bits of every layout-E position, from the vertex's coordinates and slot.
template <int D>
__global__ void k_ml_prep(const double* __restrict__ coords, const uint32_t* __restrict__ srcE,
                          const uint32_t* __restrict__ node, uint64_t n, MlGrid g, double* __restrict__ tE,
                          uint8_t* __restrict__ bE) {
    const uint64_t q = blockIdx.x * 256ull + threadIdx.x;
    if (q >= n) return;
    const uint32_t v = srcE[q];
    double pc[3] = {0, 0, 0};
#pragma unroll
    for (int d = 0; d < D; ++d) pc[d] = coords[(uint64_t)v * D + d];
    double t[3] = {0, 0, 0};
    uint32_t bits = 0;
    const bool ok = ml_cell<D>(g, node[v], pc, t, bits);
#pragma unroll
    for (int d = 0; d < D; ++d) tE[d * n + q] = ok ? t[d] : 0.0;
    bE[q] = ok ? (uint8_t)bits : (uint8_t)0x80;
}

// multilinear_at (interp.hpp:97-132) from the prepared cell: weights
// ((1 * a_0) * a_1) * a_2 with a_d = t_d or 1 - t_d (corner bit d = axis d),
// corners skipped exactly when their weight is 0, accumulated from 0.0 in
// corner order -- the same operations as multilinear_eval_c. Corner values
// come from the staged bands: the corner (bits b_d) of a vertex with
// bucket-local slot ln sits at (1 - c_0 + b_0) Lb + w + ln + (b_1 - c_1) s1 +
// (b_2 - c_2) (3-D; c_d the cell bits), or at the global index m - sum c_d
// s_d + sum b_d s_d.
// Per-bucket constants of ml_eval_prepared (hoisted out of the element loop:
// the strides and band offsets would otherwise be reloaded from the kernel
// parameters for every element).
struct MlEvalC {
    int32_t so[3];   // corner offsets in the staged bands per axis
    uint64_t go[3];  // corner offsets in x1 per axis
    int32_t Lb, w;
    int32_t s1;      // axis-1 stride (3-D) / axis-0 cell step
    uint64_t st0, st1;
};
template <int D>
__device__ __forceinline__ MlEvalC ml_eval_const(const MlGrid& g, const MlDims& md) {
    MlEvalC c{};
    c.Lb = md.Lb;
    c.w = md.w;
    if (D == 3) {
        c.st1 = g.shape[2];
        c.st0 = g.shape[1] * g.shape[2];
        c.s1 = (int32_t)c.st1;
        c.so[0] = g.shape[0] > 1 ? md.Lb : 0;
        c.so[1] = g.shape[1] > 1 ? (int32_t)c.st1 : 0;
        c.so[2] = g.shape[2] > 1 ? 1 : 0;
        c.go[0] = g.shape[0] > 1 ? c.st0 : 0;
        c.go[1] = g.shape[1] > 1 ? c.st1 : 0;
        c.go[2] = g.shape[2] > 1 ? 1 : 0;
    } else if (D == 2) {
        c.st0 = g.shape[1];
        c.so[0] = g.shape[0] > 1 ? md.Lb : 0;
        c.so[1] = g.shape[1] > 1 ? 1 : 0;
        c.go[0] = g.shape[0] > 1 ? g.shape[1] : 0;
        c.go[1] = g.shape[1] > 1 ? 1 : 0;
    } else {
        c.so[0] = g.shape[0] > 1 ? 1 : 0;
        c.go[0] = (uint64_t)c.so[0];
    }
    return c;
}

template <int D, bool STAGED>
__device__ __forceinline__ double ml_eval_prepared(const MlEvalC& k, const double* __restrict__ x1, const double* xs,
                                                   uint32_t m, uint32_t ln, const double* t, uint32_t cb) {
    double om[3] = {1, 1, 1};
#pragma unroll
    for (int d = 0; d < D; ++d) om[d] = __dsub_rn(1.0, t[d]);
    int32_t ib;
    uint64_t lb;
    const int c0 = cb & 1, c1 = (cb >> 1) & 1, c2 = (cb >> 2) & 1;
    if (D == 3) {
        ib = (1 - c0) * k.Lb + k.w + (int32_t)ln - c1 * k.s1 - c2;
        lb = (uint64_t)m - c0 * k.st0 - c1 * k.st1 - c2;
    } else if (D == 2) {
        ib = (1 - c0) * k.Lb + k.w + (int32_t)ln - c1;
        lb = (uint64_t)m - c0 * k.st0 - c1;
    } else {
        ib = k.w + (int32_t)ln - c0;
        lb = (uint64_t)m - c0;
    }
    auto val = [&](unsigned corner) {
        if (STAGED) {
            int32_t si = ib;
#pragma unroll
            for (int d = 0; d < D; ++d)
                if ((corner >> d) & 1u) si += k.so[d];
            return xs[si];
        } else {
            uint64_t gi = lb;
#pragma unroll
            for (int d = 0; d < D; ++d)
                if ((corner >> d) & 1u) gi += k.go[d];
            return __ldg(&x1[gi]);
        }
    };
    double acc = 0.0;
    if (D == 1) {
        if (om[0] != 0.0) acc = __dadd_rn(acc, __dmul_rn(om[0], val(0)));
        if (t[0] != 0.0) acc = __dadd_rn(acc, __dmul_rn(t[0], val(1)));
        return acc;
    }
    if (D == 2) {
#pragma unroll
        for (unsigned corner = 0; corner < 4; ++corner) {
            const double w = __dmul_rn((corner & 1u) ? t[0] : om[0], (corner & 2u) ? t[1] : om[1]);
            if (w != 0.0) acc = __dadd_rn(acc, __dmul_rn(w, val(corner)));
        }
        return acc;
    }
    double p01[4];
#pragma unroll
    for (unsigned c = 0; c < 4; ++c) p01[c] = __dmul_rn((c & 1u) ? t[0] : om[0], (c & 2u) ? t[1] : om[1]);
    double v[8];
#pragma unroll
    for (unsigned corner = 0; corner < 8; ++corner) v[corner] = val(corner);
#pragma unroll
    for (unsigned corner = 0; corner < 8; ++corner) {
        const double w = __dmul_rn(p01[corner & 3u], (corner & 4u) ? t[2] : om[2]);
        if (w != 0.0) acc = __dadd_rn(acc, __dmul_rn(w, v[corner]));
    }
    return acc;
}

// The generic evaluation from the coordinates, for a vertex whose slot is not
// a cell hint (out of line: it would crowd the hot loop's registers).
template <int D>
__device__ __noinline__ double ml_eval_generic(const MlGrid& g, const double* __restrict__ x1,
                                               const double* __restrict__ coords, uint32_t v) {
    double pc[3] = {0, 0, 0};
    for (int d = 0; d < D; ++d) pc[d] = __ldg(&coords[(uint64_t)v * D + d]);
    return multilinear_eval_c<D>(g.axes, g.axis_off, g.shape, GlobalCorners{x1}, pc, g.inv_cell, g.scale);
}

// MODE 0: KE[p] = lattice(xE[p] - g(p)) (compute_residuals, interp.hpp:161-170)
// MODE 1: gE[p] = g(p) (back_interpolate for the recomposition, pipeline.hpp:206-208)
#ifndef UMCG_ML_MINB
#define UMCG_ML_MINB 4
#endif
#ifndef UMCG_ML_U
#define UMCG_ML_U 2
#endif
template <int MODE, int DD, class KT>
__global__ void __launch_bounds__(ML_T, UMCG_ML_MINB) k_ml_bucket(const double* __restrict__ xE, const double* __restrict__ tE,
                                                  const uint8_t* __restrict__ bE, const double* __restrict__ coords,
                                                  const uint32_t* __restrict__ srcE, uint64_t n,
                                                  const uint2* __restrict__ bct, uint32_t E, MlGrid g,
                                                  const double* __restrict__ x1, uint64_t n1,
                                                  const uint32_t* __restrict__ bk, uint64_t B,
                                                  const uint16_t* __restrict__ lnode, uint32_t band_cap, MlDims md,
                                                  DevCtl* ctl, KT* __restrict__ KE, double* __restrict__ gE) {
    extern __shared__ __align__(16) double dsm[];
    double* xs = dsm;  // [band_cap] x1 bands
    const uint64_t b = blockIdx.x;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint2* ch = bct + b * (uint64_t)(E + 1);
    double bin = 0, inv = 0, tau = 0;
    if (MODE == 0) { bin = ctl->bin[1]; inv = ctl->inv_bin[1]; tau = ctl->tau_c[1]; }
    const uint32_t s0 = __ldg(&bk[b]), j0 = __ldg(&bk[B + 1 + b]), j1 = __ldg(&bk[B + 2 + b]);
    MlDims mdb = md;
    mdb.Lb = (int32_t)(j1 - j0) + 2 * md.w;
    const int nbands = DD == 1 ? 1 : 3;
    const bool staged = (uint32_t)(nbands * mdb.Lb) <= band_cap;
    if (staged) {
        const int64_t st0 = DD == 1 ? 0 : (int64_t)md.s12;
        for (int a = (DD == 1 ? 0 : -1); a <= (DD == 1 ? 0 : 1); ++a)
            ml_stage_band(xs + (DD == 1 ? 0 : (a + 1) * mdb.Lb), x1, (int64_t)j0 + a * st0 - md.w,
                          (int64_t)j1 + a * st0 + md.w, (int64_t)n1);
    }
    __syncthreads();
    // U vertices per thread and pass, every load issued before any is
    // evaluated (the kernel is bound by the latency of these streams)
    constexpr int U = UMCG_ML_U;
    const MlEvalC kc = ml_eval_const<DD>(g, mdb);
    auto run = [&](auto staged_tag) {
        constexpr bool STAGED = decltype(staged_tag)::value;
        for (uint32_t e = warp; e < E; e += ML_T / 32) {
            const uint2 c0 = __ldg(&ch[e]), c1 = __ldg(&ch[e + 1]);
            for (uint32_t l0 = c0.x + lane; l0 < c1.x; l0 += 32 * U) {
                double t[U][3], xv[U];
                uint32_t ln[U], cb[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const uint32_t l = l0 + 32 * u;
                    const bool ok = l < c1.x;
                    const uint64_t p = c0.y + (l - c0.x);
#pragma unroll
                    for (int d = 0; d < 3; ++d) t[u][d] = (d < DD && ok) ? __ldcs(&tE[d * n + p]) : 0.0;
                    ln[u] = ok ? __ldg(&lnode[s0 + l]) : 0u;
                    cb[u] = ok ? __ldcs(&bE[p]) : 0u;
                    xv[u] = (MODE == 0 && ok) ? __ldcs(&xE[p]) : 0.0;
                }
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const uint32_t l = l0 + 32 * u;
                    if (l >= c1.x) break;
                    const uint64_t p = c0.y + (l - c0.x);
                    const double gv = (cb[u] & 0x80u)  // slot is not a cell hint: from the coordinates
                                          ? ml_eval_generic<DD>(g, x1, coords, __ldg(&srcE[p]))
                                          : ml_eval_prepared<DD, STAGED>(kc, x1, xs, j0 + ln[u], ln[u], t[u], cb[u]);
                    if (MODE == 0) KE[p] = resid_k<KT>(__dsub_rn(xv[u], gv), bin, inv, tau, ctl);
                    else gE[p] = gv;
                }
            }
        }
    };
    if (staged) run(std::true_type{});
    else run(std::false_type{});
}

// x'_i = approx_i + x2'_i (pipeline.hpp:206-208) with approx gathered from
// layout E (window-local gather through dstE).
__global__ void k_add_gathered(const double* __restrict__ gE, const uint32_t* __restrict__ dstE, uint64_t n,
                               double* __restrict__ io) {
    const uint64_t i = blockIdx.x * 256ull + threadIdx.x;
    if (i < n) io[i] = __dadd_rn(__ldg(&gE[dstE[i]]), io[i]);
}

// Vertex order: q_i = K_i - K_{i-1} through dstE (gather inside an epoch
// window), zigzag codes, RLE tile summary.
template <class KT, class CT>
__global__ void __launch_bounds__(ENC_THREADS) k_resid_codes(const uint32_t* __restrict__ dst,
                                                            const KT* __restrict__ Kp, uint64_t n,
                                                            CT* __restrict__ codes, RleSum* __restrict__ sums,
                                                            const DevCtl* ctl) {
    if (pass_skipped(ctl)) return;
    using BR = cub::BlockReduce<RleSum, ENC_THREADS>;
    __shared__ typename BR::TempStorage tmp;
    const uint64_t tile = blockIdx.x;
    const uint64_t first = tile * ENC_TILE + (uint64_t)threadIdx.x * ENC_ITEMS;
    CT v[ENC_ITEMS];
    int cnt = 0;
    if (first < n) {
        int64_t prev = first ? (int64_t)Kp[dst[first - 1]] : 0;
        uint32_t d[ENC_ITEMS];
        if (first + ENC_ITEMS <= n) {
            const uint4 a = __ldg(reinterpret_cast<const uint4*>(dst + first));
            const uint4 c = __ldg(reinterpret_cast<const uint4*>(dst + first) + 1);
            d[0] = a.x; d[1] = a.y; d[2] = a.z; d[3] = a.w; d[4] = c.x; d[5] = c.y; d[6] = c.z; d[7] = c.w;
        } else {
#pragma unroll
            for (int k = 0; k < ENC_ITEMS; ++k) d[k] = first + k < n ? dst[first + k] : 0;
        }
        int32_t K[ENC_ITEMS];
#pragma unroll
        for (int k = 0; k < ENC_ITEMS; ++k) K[k] = first + k < n ? (int32_t)UMCG_GATHER_LD(&Kp[d[k]]) : 0;
#pragma unroll
        for (int k = 0; k < ENC_ITEMS; ++k) {
            if (first + k < n) {
                v[k] = (CT)zz_enc((int64_t)K[k] - prev);
                prev = K[k];
                cnt = k + 1;
            } else {
                v[k] = 0;
            }
        }
        if (cnt == ENC_ITEMS) {
            if (sizeof(CT) == 4) {
                uint4* o = reinterpret_cast<uint4*>(codes + first);
                o[0] = make_uint4(v[0], v[1], v[2], v[3]);
                o[1] = make_uint4(v[4], v[5], v[6], v[7]);
            } else {
                *reinterpret_cast<uint4*>(codes + first) =
                    make_uint4((uint32_t)v[0] | ((uint32_t)v[1] << 16), (uint32_t)v[2] | ((uint32_t)v[3] << 16),
                               (uint32_t)v[4] | ((uint32_t)v[5] << 16), (uint32_t)v[6] | ((uint32_t)v[7] << 16));
            }
        } else {
            for (int k = 0; k < cnt; ++k) codes[first + k] = v[k];
        }
    } else {
#pragma unroll
        for (int k = 0; k < ENC_ITEMS; ++k) v[k] = 0;
    }
    const RleSum s = thread_summary(v, cnt, (uint32_t)tile);
    const RleSum tot = BR(tmp).Reduce(s, RleComposeOp());
    if (threadIdx.x == 0) sums[tile] = tot;
}

// Vertex tiles of kRTile vertices, one per CTA: the tile's lattice indices
// are gathered in ascending layout-E order (plan rPt: a tile meets each
// bucket chunk in a run of consecutive positions, so a warp's 32 loads share
// sectors), scattered into shared memory by tile-local vertex (rLt), and the
// codes q_i = K_i - K_{i-1} leave in vertex order, coalesced. The RLE tile
// summaries follow from the codes (k_rle_tiles_fast, stream_plan_u16).
// A/B (tools/microbench_paths.cu, config 3): 2-byte gathers through dstE
// 0.59 ms per 134M vertices, run-sorted 0.42 ms; one CTA of 1024 threads per
// SM -- the gathers in flight are bounded by the L1 left beside the shared-
// memory carve-out (3 x 256 threads with 192 KB of shared memory: 0.69 ms);
// 4 loads in flight per thread (8: 0.62 ms). With the RLE summaries fused
// into this kernel (no overlap of the two phases at one CTA per SM) 0.70 ms.
template <class KT, class CT, int NT>
__global__ void __launch_bounds__(NT, 1) k_resid_codes_sr(const uint32_t* __restrict__ rPt,
                                                          const uint16_t* __restrict__ rLt,
                                                          const uint32_t* __restrict__ dst,
                                                          const KT* __restrict__ Kp, uint64_t n,
                                                          CT* __restrict__ codes, const DevCtl* ctl) {
    if (pass_skipped(ctl)) return;
    extern __shared__ __align__(16) unsigned char smem[];
    KT* ks = reinterpret_cast<KT*>(smem);
    const uint64_t t0 = (uint64_t)blockIdx.x * kRTile;
    const uint32_t cnt = (uint32_t)min((uint64_t)kRTile, n - t0);
    constexpr int U = 4;
    for (uint32_t k0 = threadIdx.x; k0 < cnt; k0 += NT * U) {
        uint32_t pp[U];
        uint32_t ll[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint32_t k = k0 + u * NT;
            pp[u] = k < cnt ? __ldcs(rPt + t0 + k) : 0u;
            ll[u] = k < cnt ? __ldcs(rLt + t0 + k) : 0u;
        }
        KT v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = k0 + u * NT < cnt ? UMCG_GATHER_LD(Kp + pp[u]) : (KT)0;
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (k0 + u * NT < cnt) ks[ll[u]] = v[u];
    }
    const int32_t prev0 = t0 ? (int32_t)UMCG_GATHER_LD(Kp + __ldg(dst + t0 - 1)) : 0;
    __syncthreads();
    for (uint32_t i0 = threadIdx.x * ENC_ITEMS; i0 < cnt; i0 += NT * ENC_ITEMS) {
        const uint64_t first = t0 + i0;
        const int c = (int)min((uint32_t)ENC_ITEMS, cnt - i0);
        int32_t prev = i0 ? (int32_t)ks[i0 - 1] : prev0;
        CT v[ENC_ITEMS];
#pragma unroll
        for (int k = 0; k < ENC_ITEMS; ++k) {
            const int32_t K = k < c ? (int32_t)ks[i0 + k] : prev;
            v[k] = (CT)zz_enc((int64_t)K - prev);
            prev = K;
        }
        if (c == ENC_ITEMS) {
            if (sizeof(CT) == 4) {
                uint4* o = reinterpret_cast<uint4*>(codes + first);
                o[0] = make_uint4(v[0], v[1], v[2], v[3]);
                o[1] = make_uint4(v[4], v[5], v[6], v[7]);
            } else {
                *reinterpret_cast<uint4*>(codes + first) = make_uint4(
                    (uint32_t)v[0] | ((uint32_t)v[1] << 16), (uint32_t)v[2] | ((uint32_t)v[3] << 16),
                    (uint32_t)v[4] | ((uint32_t)v[5] << 16), (uint32_t)v[6] | ((uint32_t)v[7] << 16));
            }
        } else {
            for (int k = 0; k < c; ++k) codes[first + k] = v[k];
        }
    }
}

}  // namespace

void partition_values(const void* x, int x_f32, umcg_plan* p, double* xE, DevCtl* ctl, cudaStream_t st) {
    const uint64_t n = p->n;
    if (!n) return;
    const unsigned g = (unsigned)cdiv(n, (uint64_t)PT * GI);
    const uint32_t* srcE = p->d_srcE.as<uint32_t>(1);
    ProfScope ps_("k_gather_fwd", st);
    if (x_f32) k_gather_fwd<float><<<g, PT, 0, st>>>(static_cast<const float*>(x), n, srcE, xE, ctl);
    else k_gather_fwd<double><<<g, PT, 0, st>>>(static_cast<const double*>(x), n, srcE, xE, ctl);
    UMCG_LAUNCHED();
}

// Buckets of CAP vertices / NODES slots: persistent BTP-thread CTAs, MINB per SM.
template <uint32_t CAP, uint32_t NODES, int BTP, int MINB>
static void run_buckets(umcg_plan* p, const double* xE, DevCtl* ctl, double* x1, void* KE, bool narrow,
                        const GridK& gk, cudaStream_t st) {
    const uint32_t E = (uint32_t)p->n_epochs;
    static DeviceOnce configured;
    configured([] {
        constexpr int kMaxDyn = MINB == 1 ? 224 * 1024 : 112 * 1024;
        UMCG_CUDA(cudaFuncSetAttribute(k_bucket<int32_t, CAP, NODES>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       200 * 1024));
        UMCG_CUDA(cudaFuncSetAttribute(k_bucket<int16_t, CAP, NODES>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       200 * 1024));
        UMCG_CUDA(cudaFuncSetAttribute(k_bucket_tma<int32_t, CAP, NODES, BTP, MINB>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxDyn));
        UMCG_CUDA(cudaFuncSetAttribute(k_bucket_tma<int16_t, CAP, NODES, BTP, MINB>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxDyn));
    });
    const size_t tma_smem = NODES * 8 + 2 * (size_t)tma_stage_bytes<CAP>(E);
    // persistent two-stage bulk-copy kernel for the regular buckets; when its
    // staging does not fit (many epochs, ~700M vertices) every bucket takes
    // the one-bucket-per-CTA kernel below
    const bool pipe = E + 1 <= BTP && p->n_regular > 0 && tma_smem <= (MINB == 1 ? 224 : 112) * 1024;
    if (pipe) {
        int dev = 0, sms = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        const unsigned g = (unsigned)std::min<uint64_t>(p->n_regular, (uint64_t)sms * MINB);
        auto launch = [&](auto* ke) {
            using KT = std::remove_pointer_t<decltype(ke)>;
            k_bucket_tma<KT, CAP, NODES, BTP, MINB><<<g, BTP, tma_smem, st>>>(
                xE, p->d_bk.as<uint32_t>(1), p->n_buckets, E, p->d_bct.as<uint2>(1), p->d_regular.as<uint32_t>(1),
                (uint32_t)p->n_regular, p->d_lnode.as<uint16_t>(1), p->d_lslot.as<uint16_t>(1),
                p->d_seg.as<uint32_t>(1), ctl, x1, ke, gk);
        };
        if (narrow) launch(static_cast<int16_t*>(KE));
        else launch(static_cast<int32_t*>(KE));
        UMCG_LAUNCHED();
    }
    if (!pipe || p->n_regular < p->n_buckets) {
        // all buckets (no pipeline possible) or the heavy single-slot buckets
        const size_t smem = CAP * 8 + NODES * 8 + (NODES + 2) * 4 + ((size_t)E + 1) * 8 + CAP * 4 + 16;
        auto launch = [&](auto* ke) {
            using KT = std::remove_pointer_t<decltype(ke)>;
            k_bucket<KT, CAP, NODES><<<(unsigned)p->n_buckets, BT, smem, st>>>(
                xE, p->d_bk.as<uint32_t>(1), p->n_buckets, E, p->d_bct.as<uint2>(1), p->d_lnode.as<uint16_t>(1),
                p->d_lperm.as<uint16_t>(1), p->d_seg.as<uint32_t>(1), ctl, x1, ke, pipe ? 1 : 0, gk);
        };
        if (narrow) launch(static_cast<int16_t*>(KE));
        else launch(static_cast<int32_t*>(KE));
        UMCG_LAUNCHED();
    }
}

void bucket_means_residuals(umcg_plan* p, const double* xE, DevCtl* ctl, double* x1, void* KE, bool narrow,
                            int32_t* K1, int D1, cudaStream_t st) {
    const GridK gk{K1, std::ldexp(1.0, 31 - (D1 < 1 ? 1 : D1))};
    if (!p->n_buckets) return;
    ProfScope ps_("k_bucket", st);
    if (p->bucket_cap == kBucketCapL)
        run_buckets<kBucketCapL, kBucketNodesL, 1024, 1>(p, xE, ctl, x1, KE, narrow, gk, st);
    else
        run_buckets<kBucketCap, kBucketNodes, 512, 2>(p, xE, ctl, x1, KE, narrow, gk, st);
}
bool resid_codes_tiles(umcg_plan* p, const void* KE, void* codes, bool narrow, bool fine, const StreamEncScratch& s,
                       const DevCtl* ctl, cudaStream_t st) {
    const uint64_t T = cdiv(p->n, ENC_TILE);
    if (!T) return true;
    ProfScope ps_("k_resid_codes", st);
#ifndef UMCG_RSR_OFF  // (A/B: the dstE gather kernel below)
    // Narrow (int16) lattice indices of a fine bound only. With int32 indices the tile takes
    // 128 KB of shared memory and the dstE kernel below (summaries fused) is faster (A/B:
    // absolute-bound config 3, compress 2.69 -> 2.56 ms); with coarse bounds (token-dense
    // streams) the exact summaries are better hidden under the dstE kernel's gathers than
    // run as a pass of their own (config 5 256^3 tau 1e-2: 5.35 -> 4.95 ms).
    if (narrow && fine && p->d_rPt.capacity() >= p->n * 4 && p->d_rLt.capacity() >= p->n * 2) {
        constexpr int NT = 1024;
        static DeviceOnce configured;
        configured([] {
            UMCG_CUDA(cudaFuncSetAttribute(k_resid_codes_sr<int16_t, uint16_t, NT>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, kRTile * 2));
        });
        const unsigned g = (unsigned)cdiv(p->n, (uint64_t)kRTile);
        k_resid_codes_sr<int16_t, uint16_t, NT><<<g, NT, kRTile * 2, st>>>(
            p->d_rPt.as<uint32_t>(1), p->d_rLt.as<uint16_t>(1), p->d_dstE.as<uint32_t>(1),
            static_cast<const int16_t*>(KE), p->n, static_cast<uint16_t*>(codes), ctl);
        UMCG_LAUNCHED();
        return false;
    }
#endif
    if (narrow)
        k_resid_codes<int16_t, uint16_t><<<(unsigned)T, ENC_THREADS, 0, st>>>(
            p->d_dstE.as<uint32_t>(1), static_cast<const int16_t*>(KE), p->n, static_cast<uint16_t*>(codes), s.sums,
            ctl);
    else
        k_resid_codes<int32_t, uint32_t><<<(unsigned)T, ENC_THREADS, 0, st>>>(
            p->d_dstE.as<uint32_t>(1), static_cast<const int32_t*>(KE), p->n, static_cast<uint32_t*>(codes), s.sums,
            ctl);
    UMCG_LAUNCHED();
    return true;
}

static MlGrid ml_grid(umcg_plan* p) {
    MlGrid g{};
    g.axes = p->d_axes.as<double>(1);
    g.axis_off = p->d_axis_off.as<uint64_t>(1);
    g.inv_cell = p->d_inv_cell.as<double>(1);
    for (int d = 0; d < 3; ++d) {
        g.shape[d] = p->shape[d];
        g.scale[d] = p->axis_scale[d];
    }
    g.D = p->dim;
    return g;
}

// t_d and cell bits of every layout-E position (first multilinear use of a plan)
static void ml_prep(umcg_plan* p, cudaStream_t st) {
    if (p->has_mlprep) return;
    const MlGrid g = ml_grid(p);
    double* tE = p->d_mlT.as<double>(p->n * p->dim + 1);
    uint8_t* bE = p->d_mlB.as<uint8_t>(p->n + 16);
    const unsigned blocks = (unsigned)cdiv(p->n, 256);
    const double* c = p->d_coords.as<double>(1);
    const uint32_t* srcE = p->d_srcE.as<uint32_t>(1);
    const uint32_t* node = p->d_node.as<uint32_t>(1);
    if (p->n) {
        if (p->dim == 3) k_ml_prep<3><<<blocks, 256, 0, st>>>(c, srcE, node, p->n, g, tE, bE);
        else if (p->dim == 2) k_ml_prep<2><<<blocks, 256, 0, st>>>(c, srcE, node, p->n, g, tE, bE);
        else k_ml_prep<1><<<blocks, 256, 0, st>>>(c, srcE, node, p->n, g, tE, bE);
        UMCG_LAUNCHED();
    }
    p->has_mlprep = true;
}

template <int MODE, class KT>
static void launch_ml(umcg_plan* p, const double* xE, const double* x1, DevCtl* ctl, KT* KE, double* gE,
                      cudaStream_t st) {
    ml_prep(p, st);
    const MlGrid g = ml_grid(p);
    const uint32_t E = (uint32_t)p->n_epochs;
    // x1 bands: three ranges of (bucket slots + one row either side) per bucket
    MlDims md{};
    md.w = g.D == 3 ? (int32_t)g.shape[2] + 1 : 1;
    md.s1 = g.D == 3 ? (uint32_t)g.shape[2] : 1;
    md.s12 = g.D == 3 ? (uint32_t)(g.shape[1] * g.shape[2]) : g.D == 2 ? (uint32_t)g.shape[1] : 1;
    const uint32_t band_cap =
        p->n_slots < (1u << 30) ? (uint32_t)std::min<uint64_t>((g.D == 1 ? 1 : 3) * (p->bucket_nodes + 2 * (uint64_t)md.w), 12288)
                                : 0;
    const size_t smem = 8 * (size_t)band_cap;
    const double* tE = p->d_mlT.as<double>(1);
    const uint8_t* bE = p->d_mlB.as<uint8_t>(1);
    auto go = [&](auto kern) {
        UMCG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        kern<<<(unsigned)p->n_buckets, ML_T, smem, st>>>(xE, tE, bE, p->d_coords.as<double>(1),
                                                        p->d_srcE.as<uint32_t>(1), p->n, p->d_bct.as<uint2>(1), E, g,
                                                        x1, p->n_slots, p->d_bk.as<uint32_t>(1), p->n_buckets,
                                                        p->d_lnode.as<uint16_t>(1), band_cap, md, ctl, KE, gE);
    };
    if (g.D == 3) go(k_ml_bucket<MODE, 3, KT>);
    else if (g.D == 2) go(k_ml_bucket<MODE, 2, KT>);
    else go(k_ml_bucket<MODE, 1, KT>);
    UMCG_LAUNCHED();
}

void ml_residuals(umcg_plan* p, const double* xE, const double* x1, DevCtl* ctl, void* KE, bool narrow,
                  cudaStream_t st) {
    if (!p->n_buckets) return;
    ml_prep(p, st);  // outside the timed scope: plan-time work, once per plan handle
    ProfScope ps_("k_ml_resid", st);
    if (narrow) launch_ml<0>(p, xE, x1, ctl, static_cast<int16_t*>(KE), nullptr, st);
    else launch_ml<0>(p, xE, x1, ctl, static_cast<int32_t*>(KE), nullptr, st);
}

void ml_layout_g(umcg_plan* p, const double* x1, double* gE, cudaStream_t st) {
    ml_prep(p, st);
    ProfScope ps_("k_ml_recompose", st);
    if (p->n_buckets) launch_ml<1>(p, nullptr, x1, nullptr, static_cast<int32_t*>(nullptr), gE, st);
}

void ml_recompose(umcg_plan* p, const double* x1, double* gE, double* d_out, cudaStream_t st) {
    if (!p->n) return;
    ml_prep(p, st);
    ProfScope ps_("k_ml_recompose", st);
    if (p->n_buckets) launch_ml<1>(p, nullptr, x1, nullptr, static_cast<int32_t*>(nullptr), gE, st);
    k_add_gathered<<<(unsigned)cdiv(p->n, 256), 256, 0, st>>>(gE, p->d_dstE.as<uint32_t>(1), p->n, d_out);
    UMCG_LAUNCHED();
}

}  // namespace umcg
