// Zero-RLE varint stream encoder on sm_100a.
//
// Byte format: the reference's ByteWriter::varint stream of the codes
// (common.hpp:60-66) passed through rle_compress (lossless.hpp:24-51):
// maximal zero runs of >= 8 bytes become {0x00, varint(len)}, everything in
// between becomes {0x01, varint(len), bytes}. A 0x00 byte occurs iff a code
// is 0, so the token structure is decided on codes (RleSum, common.cuh).
//
// Kernels (every phase fully parallel; no inter-CTA waiting):
//   tiles/chunks/cscan/states: reduce-then-scan of per-2048-code RleSum tile
//            summaries -> each tile's entry state; the tile that sees a
//            literal close records that literal's total byte length.
//   write:   per tile, output range [P_t, P_t+1) from the entry states.
//            Fast path (no zero run >= 8 strictly inside the tile): one u32
//            block scan of byte lengths places every varint; the head
//            (pending zeros, Z token, literal header) is written by thread 0.
//            General path: exact per-thread walk of the state machine.
//            Bytes are staged in shared memory and leave in 4-byte stores.
#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>

#include "encode_dev.cuh"

namespace umcg {

namespace {

// Phase 1: tile summaries (independent tiles).
template <class T>
__global__ void __launch_bounds__(ENC_THREADS) k_rle_tiles(const T* __restrict__ codes, uint64_t n,
                                                           RleSum* __restrict__ sums, const DevCtl* ctl) {
    if (pass_skipped(ctl)) return;
    using BR = cub::BlockReduce<RleSum, ENC_THREADS>;
    __shared__ typename BR::TempStorage tmp;
    const uint64_t tile = blockIdx.x;
    const uint64_t first = tile * ENC_TILE + (uint64_t)threadIdx.x * ENC_ITEMS;
    T v[ENC_ITEMS];
    const int cnt = load_items(codes, n, first, v);
    const RleSum s = thread_summary(v, cnt, (uint32_t)tile);
    const RleSum tot = BR(tmp).Reduce(s, RleComposeOp());
    if (threadIdx.x == 0) sums[tile] = tot;
}

// Phase 1 with the fast tile summary: a tile with no zero run of >=
// kMinZeroRun codes strictly inside has the summary {lz, tz, fb = code bytes
// from its first to its last nonzero} (the composition of its thread
// summaries has no interior pieces, common.cuh rle_compose), which three warp
// reductions give. Such a run either fills one thread's ENC_ITEMS codes or
// ends at a thread's first nonzero after lz >= 1 zeros that continue >= 8 - lz
// codes into the previous thread; tiles with either (and the partial last
// tile) take the exact RleSum block reduction of k_rle_tiles.
constexpr int FT = 4;  // tiles per CTA of k_rle_tiles_fast: every code load in flight up front
template <class T>
__global__ void __launch_bounds__(ENC_THREADS) k_rle_tiles_fast(const T* __restrict__ codes, uint64_t n,
                                                                RleSum* __restrict__ sums,
                                                                uint32_t* __restrict__ redo,
                                                                uint32_t* __restrict__ n_redo, const DevCtl* ctl) {
    static_assert(ENC_ITEMS == 8, "8-bit zero masks");
    if (pass_skipped(ctl)) return;
    constexpr int NW = ENC_THREADS / 32;
    __shared__ uint32_t wpart[FT][NW][4];  // per warp: code bytes, first / last nonzero, any bad
    const uint64_t T_ = (n + ENC_TILE - 1) / ENC_TILE;
    const uint64_t tile0 = (uint64_t)blockIdx.x * FT;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    // u16 codes of a full thread stay packed: halfword compares give the zero
    // mask and the varint byte count (clen: 1 + (v >= 0x80) + (v >= 0x4000);
    // the __vcmp*2 SIMD intrinsics are emulated and cost ~3x more)
    constexpr bool P16 = sizeof(T) == 2;
    T v[FT][P16 ? 1 : ENC_ITEMS];
    uint4 pw[FT];
    int cnt[FT];
#pragma unroll
    for (int t = 0; t < FT; ++t) {
        cnt[t] = 0;
        const uint64_t first = (tile0 + t) * ENC_TILE + (uint64_t)threadIdx.x * ENC_ITEMS;
        if (tile0 + t >= T_) continue;
        if constexpr (P16) {
            if (first + ENC_ITEMS <= n) {
                pw[t] = __ldg(reinterpret_cast<const uint4*>(codes + first));
                cnt[t] = ENC_ITEMS;
            } else {
                uint32_t w[4] = {0, 0, 0, 0};
                for (int k = 0; k < ENC_ITEMS; ++k)
                    if (first + k < n) {
                        w[k >> 1] |= (uint32_t)codes[first + k] << (16 * (k & 1));
                        cnt[t] = k + 1;
                    }
                pw[t] = make_uint4(w[0], w[1], w[2], w[3]);
            }
        } else {
            cnt[t] = load_items(codes, n, first, v[t]);
        }
    }
#pragma unroll
    for (int t = 0; t < FT; ++t) {
        const uint64_t tile = tile0 + t;
        if (tile >= T_) break;
        uint32_t zm = 0, bytes = 0;
        if constexpr (P16) {
            const uint32_t w[4] = {pw[t].x, pw[t].y, pw[t].z, pw[t].w};
            uint32_t g = 0;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const uint32_t lo = w[i] & 0xffffu, hi = w[i] >> 16;
                zm |= ((uint32_t)(lo == 0) | ((uint32_t)(hi == 0) << 1)) << (2 * i);
                g += (lo >= 0x80u) + (lo >= 0x4000u) + (hi >= 0x80u) + (hi >= 0x4000u);
            }
            const uint32_t valid = (1u << cnt[t]) - 1u;
            zm &= valid;  // (padding halfwords of a partial thread are 0: excluded here, and bad below)
            bytes = (uint32_t)cnt[t] + g;
        } else {
#pragma unroll
            for (int k = 0; k < ENC_ITEMS; ++k) {
                zm |= (k < cnt[t] && v[t][k] == 0) ? 1u << k : 0u;
                bytes += k < cnt[t] ? clen(v[t][k]) : 0u;
            }
        }
        const uint32_t lz = zm == 0xffu ? 8u : (uint32_t)(__ffs(~zm) - 1);
        const uint32_t tzr = (zm & 0x80u) ? (uint32_t)__clz(~(zm << 24)) : 0u;
        uint32_t tz_prev = __shfl_up_sync(0xffffffffu, tzr, 1);
        if (lane == 0 && threadIdx.x > 0 && lz > 0 && lz < 8 && cnt[t] == ENC_ITEMS) {
            // the previous thread's codes (previous warp): trailing zeros
            const T* pc = codes + tile * ENC_TILE + (uint64_t)threadIdx.x * ENC_ITEMS - ENC_ITEMS;
            tz_prev = 0;
            for (int k = ENC_ITEMS - 1; k >= 0 && pc[k] == 0; --k) ++tz_prev;
        }
        const bool bad = cnt[t] < ENC_ITEMS || zm == 0xffu ||
                         (threadIdx.x > 0 && lz > 0 && tz_prev + lz >= kMinZeroRun) || tile == T_ - 1;
        const uint32_t fnz = zm != 0xffu ? threadIdx.x * ENC_ITEMS + lz : 0xffffffffu;
        const uint32_t lnz = zm != 0xffu ? threadIdx.x * ENC_ITEMS + 7u - tzr : 0u;
        const uint32_t wb = __reduce_add_sync(0xffffffffu, bytes);
        const uint32_t wf = __reduce_min_sync(0xffffffffu, fnz);
        const uint32_t wl = __reduce_max_sync(0xffffffffu, lnz);
        const uint32_t wx = __any_sync(0xffffffffu, bad);
        if (lane == 0) {
            wpart[t][warp][0] = wb;
            wpart[t][warp][1] = wf;
            wpart[t][warp][2] = wl;
            wpart[t][warp][3] = wx;
        }
    }
    __syncthreads();
    if (threadIdx.x < FT && tile0 + threadIdx.x < T_) {
        const int t = threadIdx.x;
        const uint64_t tile = tile0 + t;
        uint32_t tb = 0, f = 0xffffffffu, l = 0, bad = 0;
#pragma unroll
        for (int w = 0; w < NW; ++w) {
            tb += wpart[t][w][0];
            f = min(f, wpart[t][w][1]);
            l = max(l, wpart[t][w][2]);
            bad |= wpart[t][w][3];
        }
        if (bad) {
            redo[atomicAdd(n_redo, 1u)] = (uint32_t)tile;
        } else {
            RleSum S;
            S.lz = f;
            S.tz = (uint64_t)(ENC_TILE - 1 - l);
            S.fb = (uint64_t)(tb - f - (ENC_TILE - 1 - l));
            S.lb = S.mid = 0;
            S.origin = (uint32_t)tile;
            S.flags = 0u;
            sums[tile] = S;
        }
    }
}

// The exact summaries of the listed tiles (grid-stride: the count is on the device).
template <class T>
__global__ void __launch_bounds__(ENC_THREADS) k_rle_tiles_redo(const T* __restrict__ codes, uint64_t n,
                                                                RleSum* __restrict__ sums,
                                                                const uint32_t* __restrict__ redo,
                                                                const uint32_t* __restrict__ n_redo) {
    using BR = cub::BlockReduce<RleSum, ENC_THREADS>;
    __shared__ typename BR::TempStorage tmp;
    const uint32_t cnt = *n_redo;
    for (uint32_t i = blockIdx.x; i < cnt; i += gridDim.x) {
        const uint64_t tile = redo[i];
        const uint64_t first = tile * ENC_TILE + (uint64_t)threadIdx.x * ENC_ITEMS;
        T v[ENC_ITEMS];
        const int c = load_items(codes, n, first, v);
        const RleSum s = thread_summary(v, c, (uint32_t)tile);
        const RleSum tot = BR(tmp).Reduce(s, RleComposeOp());
        if (threadIdx.x == 0) sums[tile] = tot;
        __syncthreads();
    }
}

constexpr int CH = 256;  // tiles per chunk

// Phase 2: chunk aggregates of CH tile summaries.
__global__ void __launch_bounds__(CH) k_rle_chunks(const RleSum* __restrict__ sums, uint64_t T,
                                                   RleSum* __restrict__ csum) {
    using BR = cub::BlockReduce<RleSum, CH>;
    __shared__ typename BR::TempStorage tmp;
    const uint64_t t = blockIdx.x * (uint64_t)CH + threadIdx.x;
    const RleSum s = t < T ? sums[t] : rle_identity();
    const RleSum tot = BR(tmp).Reduce(s, RleComposeOp());
    if (threadIdx.x == 0) csum[blockIdx.x] = tot;
}

// Phase 3: exclusive scan of chunk aggregates (one CTA).
__global__ void __launch_bounds__(256) k_rle_cscan(RleSum* __restrict__ csum, uint64_t C) {
    using BS = cub::BlockScan<RleSum, 256>;
    __shared__ typename BS::TempStorage tmp;
    const uint64_t per = (C + 255) / 256;
    const uint64_t c0 = threadIdx.x * per, c1 = min(C, c0 + per);
    RleSum local = rle_identity();
    for (uint64_t c = c0; c < c1; ++c) local = rle_compose(local, csum[c]);
    RleSum excl;
    BS(tmp).ExclusiveScan(local, excl, rle_identity(), RleComposeOp());
    for (uint64_t c = c0; c < c1; ++c) {
        const RleSum v = csum[c];
        csum[c] = excl;
        excl = rle_compose(excl, v);
    }
}

// Phase 4: per-tile entry states, literal totals (keyed by the tile the
// literal opened in), final length, and the list of tiles that need the
// general writer.
__global__ void __launch_bounds__(CH) k_rle_states(const RleSum* __restrict__ sums, uint64_t T,
                                                   const RleSum* __restrict__ csum, RleState* __restrict__ states,
                                                   uint64_t* __restrict__ lit_total, uint32_t* __restrict__ glist,
                                                   DevCtl* ctl, int comp) {
    if (pass_skipped(ctl)) return;
    using BS = cub::BlockScan<RleSum, CH>;
    __shared__ typename BS::TempStorage tmp;
    const uint64_t t = blockIdx.x * (uint64_t)CH + threadIdx.x;
    const RleSum S = t < T ? sums[t] : rle_identity();
    RleSum excl;
    BS(tmp).ExclusiveScan(S, excl, rle_identity(), RleComposeOp());
    if (t >= T) return;
    bool cl;
    uint64_t tt;
    const RleState st = rle_apply(rle_state0(), rle_compose(csum[blockIdx.x], excl), &cl, &tt);
    states[t] = st;
    const RleState nx = rle_apply(st, S, &cl, &tt);
    if (cl) lit_total[st.origin] = tt;
    const bool last = t == T - 1;
    if (S.has_int() || (S.allzero() && last))
        glist[atomicAdd(reinterpret_cast<unsigned int*>(&ctl->aux[4 + comp]), 1u)] = (uint32_t)t;
    if (last) {
        states[T] = nx;
        bool closes;
        uint64_t tl = 0;
        const uint64_t len = rle_finish(nx, &closes, &tl);
        if (closes && nx.has) lit_total[nx.origin] = tl;
        ctl->stream_len[comp] = len;
    }
}

__device__ __forceinline__ uint64_t state_pos(const RleState& s, const uint64_t* lit_total) {
    return s.has ? s.C + 1 + vlen64(lit_total[s.origin]) + s.Lb : s.C;
}

// Stream position of every tile's first byte (pos[T] = stream length), so
// the writers start from one load instead of a chain of dependent ones.
__global__ void k_rle_pos(const RleState* __restrict__ states, const uint64_t* __restrict__ lit_total, uint64_t T,
                          const DevCtl* __restrict__ ctl, int comp, uint64_t* __restrict__ pos) {
    if (pass_skipped(ctl)) return;
    const uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (t < T) pos[t] = state_pos(states[t], lit_total);
    else if (t == T) pos[t] = ctl->stream_len[comp];
}

// Byte writer into the staging buffer (no bounds checks: the tile's output
// fits CAP by construction). Returns the varint length.
template <class T>
__device__ __forceinline__ uint32_t put_code(uint8_t* o, T v);

template <class T>
__device__ __forceinline__ uint32_t put_varint(uint8_t* o, T v) {
    uint64_t u = (uint64_t)v;
    uint32_t k = 0;
    while (u >= 0x80) {
        o[k++] = (uint8_t)u | 0x80;
        u >>= 7;
    }
    o[k++] = (uint8_t)u;
    return k;
}

// One code's stream bytes (see clen).
template <class T>
__device__ __forceinline__ uint32_t put_code(uint8_t* o, T v) {
    if (sizeof(T) == 1) {
        o[0] = (uint8_t)v;
        return 1u;
    }
    if (sizeof(T) == 2) {  // <= 3 bytes, no loop
        const uint32_t x = (uint32_t)v;
        const bool b2 = x >= 0x80, b3 = x >= 0x4000;
        o[0] = (uint8_t)(x | (b2 ? 0x80u : 0u));
        if (b2) o[1] = (uint8_t)((x >> 7) | (b3 ? 0x80u : 0u));
        if (b3) o[2] = (uint8_t)(x >> 14);
        return 1u + b2 + b3;
    }
    return put_varint(o, v);
}

// Staged bytes out[ao, ao+len) -> d[0, len) where ao = d & 15: 16-byte
// stores for the aligned middle, bytes at the two ends.
template <uint32_t NT = ENC_THREADS>
__device__ __forceinline__ void copy_out16(const uint8_t* out, uint32_t ao, uint32_t len, uint8_t* d) {
    uint8_t* g = d - ao;  // 16-byte aligned
    const uint32_t end = ao + len;
    const uint32_t w0 = (ao + 15) / 16, w1 = end / 16;  // full words [w0, w1)
    if (w0 >= w1) {
        for (uint32_t k = ao + threadIdx.x; k < end; k += NT) g[k] = out[k];
        return;
    }
    for (uint32_t k = ao + threadIdx.x; k < 16 * w0; k += NT) g[k] = out[k];
    for (uint32_t k = 16 * w1 + threadIdx.x; k < end; k += NT) g[k] = out[k];
    const uint4* s4 = reinterpret_cast<const uint4*>(out);
    uint4* g4 = reinterpret_cast<uint4*>(g);
    for (uint32_t w = w0 + threadIdx.x; w < w1; w += NT) g4[w] = s4[w];
}

// ITEMS consecutive codes of one thread (vector loads when whole and aligned).
template <class T, int ITEMS>
__device__ __forceinline__ int load_items_n(const T* codes, uint64_t n, uint64_t first, T (&v)[ITEMS]) {
    if (first + ITEMS <= n && sizeof(T) == 2 && (first % 8) == 0 && ITEMS % 8 == 0) {
#pragma unroll
        for (int h = 0; h < ITEMS / 8; ++h) {
            const uint4 a = __ldg(reinterpret_cast<const uint4*>(codes + first) + h);
            const uint32_t w[4] = {a.x, a.y, a.z, a.w};
#pragma unroll
            for (int k = 0; k < 8; ++k) v[8 * h + k] = (T)(w[k >> 1] >> (16 * (k & 1)));
        }
        return ITEMS;
    }
    if (first + ITEMS <= n && sizeof(T) == 4 && (first % 4) == 0 && ITEMS % 4 == 0) {
#pragma unroll
        for (int h = 0; h < ITEMS / 4; ++h) {
            const uint4 a = __ldg(reinterpret_cast<const uint4*>(codes + first) + h);
            v[4 * h] = (T)a.x, v[4 * h + 1] = (T)a.y, v[4 * h + 2] = (T)a.z, v[4 * h + 3] = (T)a.w;
        }
        return ITEMS;
    }
    int cnt = 0;
#pragma unroll
    for (int k = 0; k < ITEMS; ++k) {
        const uint64_t i = first + k;
        if (i < n) { v[k] = codes[i]; cnt = k + 1; } else { v[k] = 0; }
    }
    return cnt;
}

#ifndef UMCG_WF_MINB
#define UMCG_WF_MINB 8  // 8 CTAs per SM (A/B: 6 -> 0.333 ms, 8 -> 0.303 ms for both writers' fast path)
#endif
// ITEMS codes per thread, ENC_TILE / ITEMS threads: the per-thread costs (block
// scan, tile state, head arithmetic) are shared by ITEMS codes.
template <class T, int ITEMS, int MINB>
__global__ void __launch_bounds__(ENC_TILE / ITEMS, MINB) k_rle_write_fast(const T* __restrict__ codes, uint64_t n,
                                                               const RleState* __restrict__ states,
                                                               const RleSum* __restrict__ sums,
                                                               const uint64_t* __restrict__ lit_total,
                                                               const uint64_t* __restrict__ tpos,
                                                               const DevCtl* __restrict__ ctl, int comp,
                                                               uint8_t* __restrict__ dst, int off_from_ctl) {
    if (pass_skipped(ctl)) return;
    constexpr uint32_t CAP = ENC_TILE * (sizeof(T) == 8 ? 10 : sizeof(T) == 2 ? 3 : 5) + 96;  // u16: <= 3 bytes per code
    constexpr int NT = ENC_TILE / ITEMS;
    using BS32 = cub::BlockScan<uint32_t, NT>;
    __shared__ typename BS32::TempStorage tmp;
    __shared__ __align__(16) uint8_t out[CAP];

    const uint64_t tile = blockIdx.x;
    // every load up front (codes too: they do not depend on the tile's kind)
    const uint64_t first = tile * ENC_TILE + (uint64_t)threadIdx.x * ITEMS;
    T v[ITEMS];
    const int cnt = load_items_n<T, ITEMS>(codes, n, first, v);
    const RleSum S = sums[tile];
    const RleState entry = states[tile];
    const uint64_t P0 = tpos[tile], P1 = tpos[tile + 1];
    if (S.has_int() || S.allzero()) return;  // general writer (or nothing to write)
    const uint64_t T_ = (n + ENC_TILE - 1) / ENC_TILE;
    const bool last = tile == T_ - 1;
    const uint32_t len = (uint32_t)(P1 - P0);
    uint8_t* d = dst + (off_from_ctl ? ctl->stream_off[comp] : 0) + P0;
    const uint32_t ao = (uint32_t)((uintptr_t)d & 15);
    uint8_t* o = out + ao - 0;  // o[pos - P0] is the staged byte of stream position pos

    // the core [lz, tile_cnt - tz) is one literal segment
    const uint32_t tile_cnt = (uint32_t)min((uint64_t)ENC_TILE, n - tile * ENC_TILE);
    const uint32_t core_lo = (uint32_t)S.lz, core_hi = tile_cnt - (uint32_t)S.tz;
    const uint32_t r0 = threadIdx.x * ITEMS;
    // common case: all of the thread's items are in the core (no per-item checks)
    const bool inner = cnt == ITEMS && r0 >= core_lo && r0 + ITEMS <= core_hi;
    uint32_t w = 0;
    if (inner) {
#pragma unroll
        for (int k = 0; k < ITEMS; ++k) w += clen(v[k]);
    } else {
#pragma unroll
        for (int k = 0; k < ITEMS; ++k) {
            const uint32_t r = r0 + k;
            if (k < cnt && r >= core_lo && r < core_hi) w += clen(v[k]);
        }
    }
    uint32_t off, core_total;
    BS32(tmp).ExclusiveSum(w, off, core_total);
    // head: pending zeros from before + this tile's leading zeros
    const uint64_t J0 = entry.Zp + S.lz;
    uint64_t data_base, zero_pos = 0, zpos = 0, lpos = 0, totn = 0;
    bool ztok = false, hdr = false;
    if (J0 >= kMinZeroRun) {
        zpos = entry.C + (entry.has ? lit_size(entry.Lb) : 0);
        ztok = true;
        lpos = zpos + z_size(J0);
        hdr = true;
        totn = lit_total[tile];
        data_base = lpos + 1 + vlen64(totn);
    } else if (entry.has) {
        zero_pos = P0;  // == state_pos(entry): the open literal's bytes so far
        data_base = zero_pos + J0;
    } else {
        lpos = entry.C;
        hdr = true;
        totn = lit_total[tile];
        zero_pos = lpos + 1 + vlen64(totn);
        data_base = zero_pos + J0;
    }
    if (threadIdx.x == 0) {
        if (ztok) {
            o[zpos - P0] = 0x00;
            put_varint(o + (zpos + 1 - P0), J0);
        }
        if (hdr) {
            o[lpos - P0] = 0x01;
            put_varint(o + (lpos + 1 - P0), totn);
        }
        if (!ztok)
            for (uint32_t k = 0; k < (uint32_t)J0; ++k) o[zero_pos - P0 + k] = 0;
        if (last) {  // rle_finish: trailing zeros close the stream
            const uint32_t ce = (uint32_t)(data_base - P0) + core_total;
            if (S.tz >= kMinZeroRun) {
                o[ce] = 0x00;
                put_varint(o + ce + 1, S.tz);
            } else {
                for (uint32_t k = 0; k < (uint32_t)S.tz; ++k) o[ce + k] = 0;
            }
        }
    }
    uint32_t pos = (uint32_t)(data_base - P0) + off;
    if (inner) {
#pragma unroll
        for (int k = 0; k < ITEMS; ++k) pos += put_code(o + pos, v[k]);
    } else {
#pragma unroll
        for (int k = 0; k < ITEMS; ++k) {
            const uint32_t r = r0 + k;
            if (k < cnt && r >= core_lo && r < core_hi) pos += put_code(o + pos, v[k]);
        }
    }
    __syncthreads();
    copy_out16<NT>(out, ao, len, d);
}

// General writer: tiles with a zero run >= 8 strictly inside, and the last
// tile. Units = the tile's nonzero codes; unit j carries the zero run before
// it (J_j, the first one including the zeros pending on entry). A long run
// (J_j >= 8) emits a Z token and opens a literal at j; so does the first unit
// when no literal is open on entry. Four u32 block scans place everything:
//   1. last nonzero before each thread       -> J_j, long/open flags
//   2. prefix of literal data bytes d_j      -> literal totals T_j =
//   3. suffix "next long unit"                  D(next long unit) - D(j)
//   4. prefix of unit bytes U_j              -> output positions
// (literals still open at the tile end take T from lit_total[tile]).
template <class T>
__device__ __forceinline__ void general_tile(const uint64_t tile, const T* __restrict__ codes, uint64_t n,
                                             const RleState* __restrict__ states, const RleSum* __restrict__ sums,
                                             const uint64_t* __restrict__ lit_total, const DevCtl* __restrict__ ctl,
                                             int comp, const uint64_t* __restrict__ tpos, uint8_t* __restrict__ dst,
                                             int off_from_ctl) {
    constexpr uint32_t CAP = ENC_TILE * (sizeof(T) == 8 ? 10 : 5) + 96;
    constexpr int NONE = 0x7fffffff;
    using BSi = cub::BlockScan<int, ENC_THREADS>;
    using BSu = cub::BlockScan<uint32_t, ENC_THREADS>;
    __shared__ union {
        typename BSi::TempStorage i;
        typename BSu::TempStorage u;
    } tmp;
    __shared__ uint32_t dpre[ENC_TILE + 1];  // exclusive prefix of d at each item
    __shared__ int sfx[ENC_THREADS];
    __shared__ __align__(16) uint8_t out[CAP];

    const uint64_t T_ = (n + ENC_TILE - 1) / ENC_TILE;
    const bool last = tile == T_ - 1;
    const RleState E = states[tile];
    const uint64_t P0 = tpos[tile], P1 = tpos[tile + 1];
    const uint32_t len = (uint32_t)(P1 - P0);
    if (len == 0) return;  // all-zero tile: its zeros stay pending
    uint8_t* d = dst + (off_from_ctl ? ctl->stream_off[comp] : 0) + P0;
    const uint32_t ao = (uint32_t)((uintptr_t)d & 15);
    uint8_t* o = out + ao;

    const uint32_t tile_cnt = (uint32_t)min((uint64_t)ENC_TILE, n - tile * ENC_TILE);
    const int r0 = threadIdx.x * ENC_ITEMS;
    T v[ENC_ITEMS];
    const int cnt = load_items(codes, n, tile * ENC_TILE + (uint64_t)r0, v);
    // zero-filled staging: short zero runs inside literals are then skipped
    // (the first __syncthreads below orders this before every byte write)
    for (uint32_t w = threadIdx.x; w < CAP / 16; w += ENC_THREADS)
        reinterpret_cast<uint4*>(out)[w] = make_uint4(0, 0, 0, 0);
    uint32_t nzm = 0;
#pragma unroll
    for (int k = 0; k < ENC_ITEMS; ++k) nzm |= (k < cnt && v[k] != 0) ? (1u << k) : 0u;

    // 1. last nonzero item before this thread (-1: none in the tile)
    int prev_t;
    BSi(tmp.i).ExclusiveScan(nzm ? r0 + 31 - __clz(nzm) : -1, prev_t, -1, cub::Max());
    __syncthreads();
    // J_j per unit (int64: the entry's pending zeros can be many tiles long)
    auto run_before = [&](int r, int prev) -> uint64_t {
        return prev >= 0 ? (uint64_t)(r - prev - 1) : (uint64_t)r + E.Zp;
    };
    uint32_t lngm = 0, opnm = 0, dsum = 0;
    {
        int prev = prev_t;
#pragma unroll
        for (int k = 0; k < ENC_ITEMS; ++k) {
            if (!(nzm >> k & 1)) continue;
            const uint64_t J = run_before(r0 + k, prev);
            const bool lng = J >= kMinZeroRun;
            lngm |= (uint32_t)lng << k;
            opnm |= (uint32_t)(lng || (prev < 0 && !E.has)) << k;
            dsum += (lng ? 0u : (uint32_t)J) + clen(v[k]);
            prev = r0 + k;
        }
    }
    // 2. prefix of literal data bytes
    uint32_t dex, dtot;
    BSu(tmp.u).ExclusiveSum(dsum, dex, dtot);
    {
        int prev = prev_t;
        uint32_t acc = dex;
#pragma unroll
        for (int k = 0; k < ENC_ITEMS; ++k) {
            dpre[r0 + k] = acc;
            if (!(nzm >> k & 1)) continue;
            const uint64_t J = run_before(r0 + k, prev);
            acc += (lngm >> k & 1 ? 0u : (uint32_t)J) + clen(v[k]);
            prev = r0 + k;
        }
        if (threadIdx.x == ENC_THREADS - 1) dpre[ENC_TILE] = acc;
    }
    // 3. next long unit after this thread (suffix min via a reversed scan)
    sfx[threadIdx.x] = lngm ? r0 + __ffs(lngm) - 1 : NONE;
    __syncthreads();
    int nl_rev;
    BSi(tmp.i).ExclusiveScan(sfx[ENC_THREADS - 1 - threadIdx.x], nl_rev, NONE, cub::Min());
    __syncthreads();
    sfx[ENC_THREADS - 1 - threadIdx.x] = nl_rev;
    __syncthreads();
    const int next_long_after = sfx[threadIdx.x];
    const uint64_t tail_total = lit_total[tile];
    auto lit_T = [&](int k) -> uint64_t {
        const uint32_t later = lngm & ~((2u << k) - 1u);
        const int kl = later ? r0 + __ffs(later) - 1 : next_long_after;
        return kl != NONE ? (uint64_t)(dpre[kl] - dpre[r0 + k]) : tail_total;
    };
    // 4. unit bytes -> positions
    uint32_t usum = 0;
    {
        int prev = prev_t;
#pragma unroll
        for (int k = 0; k < ENC_ITEMS; ++k) {
            if (!(nzm >> k & 1)) continue;
            const uint64_t J = run_before(r0 + k, prev);
            const bool lng = lngm >> k & 1;
            usum += (lng ? 1u + vlen64(J) : (uint32_t)J) + clen(v[k]);
            if (opnm >> k & 1) usum += 1u + vlen64(lit_T(k));
            prev = r0 + k;
        }
    }
    uint32_t pos, utot;
    BSu(tmp.u).ExclusiveSum(usum, pos, utot);
    {
        int prev = prev_t;
#pragma unroll
        for (int k = 0; k < ENC_ITEMS; ++k) {
            if (!(nzm >> k & 1)) continue;
            const uint64_t J = run_before(r0 + k, prev);
            const bool lng = lngm >> k & 1;
            if (lng) {
                o[pos] = 0x00;
                pos += 1 + put_varint(o + pos + 1, J);
            }
            if (opnm >> k & 1) {
                o[pos] = 0x01;
                pos += 1 + put_varint(o + pos + 1, lit_T(k));
            }
            if (!lng) pos += (uint32_t)J;  // zero bytes (pre-filled)
            pos += put_code(o + pos, v[k]);
            prev = r0 + k;
        }
    }
    if (last && threadIdx.x == ENC_THREADS - 1) {  // rle_finish: trailing zeros
        const int lastnz = nzm ? r0 + 31 - __clz(nzm) : prev_t;
        const uint64_t t = lastnz >= 0 ? (uint64_t)(tile_cnt - 1 - lastnz) : E.Zp + tile_cnt;
        const bool open = lastnz >= 0 || E.has;
        uint32_t q = utot;
        if (t >= kMinZeroRun) {
            o[q] = 0x00;
            put_varint(o + q + 1, t);
        } else {
            if (!open) {
                o[q] = 0x01;
                q += 1 + put_varint(o + q + 1, t);
            }
            for (uint32_t z = 0; z < (uint32_t)t; ++z) o[q++] = 0;
        }
    }
    __syncthreads();
    copy_out16(out, ao, len, d);
}

// Grid-stride over the general tiles (their count is on the device): a
// launch per tile of the stream would start and retire a CTA for every
// fast tile as well (~36 us at config 3).
template <class T>
__global__ void __launch_bounds__(ENC_THREADS, 6) k_rle_write_general(const T* __restrict__ codes, uint64_t n,
                                                           const RleState* __restrict__ states,
                                                           const RleSum* __restrict__ sums,
                                                           const uint64_t* __restrict__ lit_total,
                                                           const DevCtl* __restrict__ ctl, int comp, const uint32_t* __restrict__ glist,
                                                           const uint64_t* __restrict__ tpos,
                                                           uint8_t* __restrict__ dst, int off_from_ctl) {
    if (pass_skipped(ctl)) return;
    const uint32_t cnt = (uint32_t)ctl->aux[4 + comp];
    for (uint32_t i = blockIdx.x; i < cnt; i += gridDim.x) {
        general_tile<T>(glist[i], codes, n, states, sums, lit_total, ctl, comp, tpos, dst, off_from_ctl);
        __syncthreads();
    }
}

}  // namespace

size_t stream_enc_scratch_bytes(uint64_t n) {
    const uint64_t T = cdiv(n, ENC_TILE) + 1;
    return T * (2 * sizeof(RleSum) + sizeof(RleState) + 2 * sizeof(uint64_t) + sizeof(uint32_t)) + 4096;
}

StreamEncScratch stream_enc_carve(void* base, uint64_t n) {
    const uint64_t T = cdiv(n, ENC_TILE) + 1;
    StreamEncScratch s;
    char* p = static_cast<char*>(base);
    s.csum = reinterpret_cast<RleSum*>(p);
    p += T * sizeof(RleSum);
    s.sums = reinterpret_cast<RleSum*>(p);
    p += T * sizeof(RleSum);
    s.states = reinterpret_cast<RleState*>(p);
    p += T * sizeof(RleState);
    s.lit_total = reinterpret_cast<uint64_t*>(p);
    p += T * sizeof(uint64_t);
    s.pos = reinterpret_cast<uint64_t*>(p);
    p += T * sizeof(uint64_t);
    s.glist = reinterpret_cast<uint32_t*>(p);
    p += T * sizeof(uint32_t);
    s.n_redo = reinterpret_cast<uint32_t*>(p);  // inside the scratch's 4096-byte slack
    return s;
}

template <class T>
static void plan_impl(const T* codes, uint64_t n, const StreamEncScratch& s, DevCtl* ctl, int comp, cudaStream_t st,
                      bool fast = false) {
    const uint64_t T_ = cdiv(n, ENC_TILE);
    if (!T_) {
        UMCG_CUDA(cudaMemsetAsync(&ctl->stream_len[comp], 0, 8, st));
        return;
    }
    const uint64_t C = cdiv(T_, CH);
    UMCG_CUDA(cudaMemsetAsync(&ctl->aux[4 + comp], 0, 8, st));
    if (fast) {
        // the tile list doubles as the redo list (k_rle_states fills it afterwards)
        UMCG_CUDA(cudaMemsetAsync(s.n_redo, 0, 4, st));
        k_rle_tiles_fast<T><<<(unsigned)cdiv(T_, (uint64_t)FT), ENC_THREADS, 0, st>>>(codes, n, s.sums, s.glist,
                                                                                    s.n_redo, ctl);
        UMCG_LAUNCHED();
        int dev = 0, sms = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        k_rle_tiles_redo<T><<<(unsigned)std::min<uint64_t>(T_, (uint64_t)sms * 8), ENC_THREADS, 0, st>>>(
            codes, n, s.sums, s.glist, s.n_redo);
    } else {
        k_rle_tiles<T><<<(unsigned)T_, ENC_THREADS, 0, st>>>(codes, n, s.sums, ctl);
    }
    UMCG_LAUNCHED();
    k_rle_chunks<<<(unsigned)C, CH, 0, st>>>(s.sums, T_, s.csum);
    UMCG_LAUNCHED();
    k_rle_cscan<<<1, 256, 0, st>>>(s.csum, C);
    UMCG_LAUNCHED();
    k_rle_states<<<(unsigned)C, CH, 0, st>>>(s.sums, T_, s.csum, s.states, s.lit_total, s.glist, ctl, comp);
    UMCG_LAUNCHED();
}

void stream_plan_from_sums(uint64_t n, const StreamEncScratch& s, DevCtl* ctl, int comp, cudaStream_t st) {
    const uint64_t T_ = cdiv(n, ENC_TILE);
    if (!T_) {
        UMCG_CUDA(cudaMemsetAsync(&ctl->stream_len[comp], 0, 8, st));
        return;
    }
    const uint64_t C = cdiv(T_, CH);
    UMCG_CUDA(cudaMemsetAsync(&ctl->aux[4 + comp], 0, 8, st));
    k_rle_chunks<<<(unsigned)C, CH, 0, st>>>(s.sums, T_, s.csum);
    UMCG_LAUNCHED();
    k_rle_cscan<<<1, 256, 0, st>>>(s.csum, C);
    UMCG_LAUNCHED();
    k_rle_states<<<(unsigned)C, CH, 0, st>>>(s.sums, T_, s.csum, s.states, s.lit_total, s.glist, ctl, comp);
    UMCG_LAUNCHED();
}

template <class T>
static void write_impl(const T* codes, uint64_t n, const StreamEncScratch& s, DevCtl* ctl, int comp, uint8_t* dst,
                       bool off_ctl, cudaStream_t st) {
    const uint64_t T_ = cdiv(n, ENC_TILE);
    if (!T_) return;
    ProfScope ps_("k_rle_write", st);
    k_rle_pos<<<(unsigned)cdiv(T_ + 1, 256), 256, 0, st>>>(s.states, s.lit_total, T_, ctl, comp, s.pos);
    UMCG_LAUNCHED();
#ifndef UMCG_WF_ITEMS16
#define UMCG_WF_ITEMS16 16  // codes per thread of the u16 fast writer (A/B config 3, k_rle_write scope:
#endif                      // 8 x 256 threads 0.278 ms; 16 x 128, 8 / 12 / 16 CTAs per SM 0.257 / 0.234 / 0.233;
#ifndef UMCG_WF_MINB16      // 32 x 64, 16 / 24 CTAs per SM 0.228 / 0.244)
#define UMCG_WF_MINB16 16
#endif
    if constexpr (sizeof(T) == 2)
        k_rle_write_fast<T, UMCG_WF_ITEMS16, UMCG_WF_MINB16><<<(unsigned)T_, ENC_TILE / UMCG_WF_ITEMS16, 0, st>>>(
            codes, n, s.states, s.sums, s.lit_total, s.pos, ctl, comp, dst, off_ctl ? 1 : 0);
    else
        k_rle_write_fast<T, ENC_ITEMS, UMCG_WF_MINB><<<(unsigned)T_, ENC_THREADS, 0, st>>>(
            codes, n, s.states, s.sums, s.lit_total, s.pos, ctl, comp, dst, off_ctl ? 1 : 0);
    UMCG_LAUNCHED();
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
#ifndef UMCG_GENERAL_PER_SM
#define UMCG_GENERAL_PER_SM 32  // (A/B config 5, tau 1e-2: 6 per SM 6.79 ms, 24 or one CTA per tile 6.06 ms)
#endif
    const unsigned gg = (unsigned)std::min<uint64_t>(T_, (uint64_t)sms * UMCG_GENERAL_PER_SM);
    k_rle_write_general<T><<<gg, ENC_THREADS, 0, st>>>(codes, n, s.states, s.sums, s.lit_total, ctl,
                                                                 comp, s.glist, s.pos, dst, off_ctl ? 1 : 0);
    UMCG_LAUNCHED();
}

void stream_plan_u32(const uint32_t* c, uint64_t n, const StreamEncScratch& s, DevCtl* ctl, int comp,
                     cudaStream_t st, bool fast) { plan_impl(c, n, s, ctl, comp, st, fast); }
void stream_plan_u64(const uint64_t* c, uint64_t n, const StreamEncScratch& s, DevCtl* ctl, int comp,
                     cudaStream_t st) { plan_impl(c, n, s, ctl, comp, st); }
void stream_plan_u16(const uint16_t* c, uint64_t n, const StreamEncScratch& s, DevCtl* ctl, int comp,
                     cudaStream_t st, bool fast) { plan_impl(c, n, s, ctl, comp, st, fast); }
void stream_write_u32(const uint32_t* c, uint64_t n, const StreamEncScratch& s, DevCtl* ctl, int comp,
                      uint8_t* dst, bool o, cudaStream_t st) { write_impl(c, n, s, ctl, comp, dst, o, st); }
void stream_write_u64(const uint64_t* c, uint64_t n, const StreamEncScratch& s, DevCtl* ctl, int comp,
                      uint8_t* dst, bool o, cudaStream_t st) { write_impl(c, n, s, ctl, comp, dst, o, st); }
void stream_write_u16(const uint16_t* c, uint64_t n, const StreamEncScratch& s, DevCtl* ctl, int comp,
                      uint8_t* dst, bool o, cudaStream_t st) { write_impl(c, n, s, ctl, comp, dst, o, st); }
void stream_plan_u8(const uint8_t* c, uint64_t n, const StreamEncScratch& s, DevCtl* ctl, int comp,
                    cudaStream_t st) { plan_impl(c, n, s, ctl, comp, st); }
void stream_write_u8(const uint8_t* c, uint64_t n, const StreamEncScratch& s, DevCtl* ctl, int comp,
                     uint8_t* dst, bool o, cudaStream_t st) { write_impl(c, n, s, ctl, comp, dst, o, st); }
void stream_encode_u32(const uint32_t* c, uint64_t n, const StreamEncScratch& s, DevCtl* ctl, int comp,
                       uint8_t* dst, bool o, cudaStream_t st) {
    plan_impl(c, n, s, ctl, comp, st);
    write_impl(c, n, s, ctl, comp, dst, o, st);
}
void stream_encode_u64(const uint64_t* c, uint64_t n, const StreamEncScratch& s, DevCtl* ctl, int comp,
                       uint8_t* dst, bool o, cudaStream_t st) {
    plan_impl(c, n, s, ctl, comp, st);
    write_impl(c, n, s, ctl, comp, dst, o, st);
}

}  // namespace umcg
