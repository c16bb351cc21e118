// Zero-RLE varint stream encode/decode on sm_100a.
//
// Byte format: the reference's ByteWriter::varint stream of the codes
// (common.hpp:60-66) passed through rle_compress (lossless.hpp:24-51):
// maximal zero runs of >= 8 bytes become {0x00, varint(len)}, everything in
// between becomes {0x01, varint(len), bytes}. Because a 0x00 byte occurs iff
// a code is 0, run detection happens on codes (RleSum in common.cuh).
//
// Encode = 3 kernels:
//   summary (per 2048-code tile, block-level RleSum reduction)
//   scan    (one CTA: tile prefix states, literal totals, tile output offsets)
//   write   (per tile: re-walk the codes with the exact state machine and
//            emit bytes to shared memory, then one coalesced copy-out; every
//            tile owns a contiguous output byte range)
// Decode = serial token walk (token headers only) + parallel expand +
//          parallel varint decode with a tile-count scan.
#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>

#include "kernels.h"

namespace umcg {

namespace {

struct RleComposeOp {
    __device__ __forceinline__ RleSum operator()(const RleSum& a, const RleSum& b) const {
        return rle_compose(a, b);
    }
};

template <class T>
__device__ __forceinline__ void write_varint(uint8_t* out, uint64_t pos, uint64_t base,
                                             uint64_t cap, T v) {
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
#pragma unroll
    for (int k = 0; k < ENC_ITEMS; ++k) {
        const uint64_t i = first + k;
        if (i < n) { v[k] = codes[i]; cnt = k + 1; } else { v[k] = 0; }
    }
    return cnt;
}

template <class T>
__device__ __forceinline__ RleSum thread_summary(const T (&v)[ENC_ITEMS], int cnt, uint32_t origin) {
    RleSum s = rle_identity();
#pragma unroll
    for (int k = 0; k < ENC_ITEMS; ++k)
        if (k < cnt) s = rle_compose(s, rle_leaf(vlen64((uint64_t)v[k]), v[k] == 0, origin));
    return s;
}

template <class T>
__global__ void __launch_bounds__(ENC_THREADS) k_rle_summary(const T* __restrict__ codes, uint64_t n,
                                                             RleSum* __restrict__ sums) {
    using BR = cub::BlockReduce<RleSum, ENC_THREADS>;
    __shared__ typename BR::TempStorage tmp;
    const uint64_t tile = blockIdx.x;
    const uint64_t first = tile * ENC_TILE + (uint64_t)threadIdx.x * ENC_ITEMS;
    T v[ENC_ITEMS];
    const int cnt = load_items(codes, n, first, v);
    RleSum s = thread_summary(v, cnt, (uint32_t)tile);
    RleSum tot = BR(tmp).Reduce(s, RleComposeOp());
    if (threadIdx.x == 0) sums[tile] = tot;
}

// One CTA. Tile prefix states, literal totals (keyed by the tile where the
// literal opened), per-tile output offsets P[t] and the stream length.
constexpr int SCAN_THREADS = 256;
__global__ void __launch_bounds__(SCAN_THREADS) k_rle_scan(const RleSum* __restrict__ sums, uint64_t T,
                                                           RleState* __restrict__ states,
                                                           uint64_t* __restrict__ P,
                                                           uint64_t* __restrict__ lit_total,
                                                           DevCtl* ctl, int comp) {
    using BS = cub::BlockScan<RleSum, SCAN_THREADS>;
    __shared__ typename BS::TempStorage tmp;
    const uint64_t per = (T + SCAN_THREADS - 1) / SCAN_THREADS;
    const uint64_t t0 = (uint64_t)threadIdx.x * per;
    const uint64_t t1 = min(T, t0 + per);
    RleSum local = rle_identity();
    for (uint64_t t = t0; t < t1; ++t) local = rle_compose(local, sums[t]);
    RleSum excl;
    BS(tmp).ExclusiveScan(local, excl, rle_identity(), RleComposeOp());
    bool cl;
    uint64_t tot;
    RleState st = rle_apply(rle_state0(), excl, &cl, &tot);
    for (uint64_t t = t0; t < t1; ++t) {
        states[t] = st;
        const RleState nx = rle_apply(st, sums[t], &cl, &tot);
        if (cl) lit_total[st.origin] = tot;
        st = nx;
    }
    if (t0 < T && t1 == T) {  // owner of the last tile closes the stream
        states[T] = st;
        bool closes;
        uint64_t tl = 0;
        const uint64_t len = rle_finish(st, &closes, &tl);
        if (closes && st.has) lit_total[st.origin] = tl;
        P[T] = len;
        ctl->stream_len[comp] = len;
    }
    if (T == 0 && threadIdx.x == 0) ctl->stream_len[comp] = 0;
    __syncthreads();
    for (uint64_t t = t0; t < t1; ++t) {
        const RleState s = states[t];
        P[t] = s.has ? s.C + 1 + vlen64(lit_total[s.origin]) + s.Lb : s.C;
    }
}

constexpr uint32_t kEntry = ENC_THREADS;  // slot of the literal open on tile entry
constexpr uint64_t kUnknown = ~0ull;

// Per-thread exact walk of the RLE state machine over its codes.
// WRITE=false: record literal closes; WRITE=true: emit bytes.
template <bool WRITE, class T>
__device__ __forceinline__ void walk(RleState st, const T (&v)[ENC_ITEMS], int cnt, bool finalize,
                                     uint64_t* closeTot, uint8_t* out, uint64_t base, uint64_t cap) {
    const uint32_t me = threadIdx.x;
    auto slot = [](uint32_t o) { return o == kEntry ? kEntry : o; };
    auto data_pos = [&](const RleState& s) {
        return s.C + 1 + vlen64(closeTot[slot(s.origin)]) + s.Lb;
    };
    auto open_lit = [&](RleState& s) {
        s.origin = me;
        s.Lb = 0;
        s.has = 1;
        if (WRITE) {
            const uint64_t p = s.C - base;
            if (p < cap) out[p] = 0x01;
            write_varint(out, s.C + 1, base, cap, closeTot[me]);
        }
    };
    auto put_zeros = [&](RleState& s, uint64_t J) {
        if (WRITE) {
            const uint64_t p0 = data_pos(s) - base;
            for (uint64_t k = 0; k < J; ++k)
                if (p0 + k < cap) out[p0 + k] = 0;
        }
        s.Lb += J;
    };
    auto put_z = [&](RleState& s, uint64_t J) {
        if (WRITE) {
            const uint64_t p = s.C - base;
            if (p < cap) out[p] = 0x00;
            write_varint(out, s.C + 1, base, cap, J);
        }
        s.C += z_size(J);
    };
    auto close_lit = [&](RleState& s) {
        if (!WRITE) closeTot[slot(s.origin)] = s.Lb;
        s.C += lit_size(s.Lb);
        s.has = 0;
    };
#pragma unroll
    for (int k = 0; k < ENC_ITEMS; ++k) {
        if (k >= cnt) break;
        const T c = v[k];
        if (c == 0) { st.Zp += 1; continue; }
        const uint64_t J = st.Zp;
        if (J >= kMinZeroRun) {
            if (st.has) close_lit(st);
            put_z(st, J);
            open_lit(st);
        } else {
            if (!st.has) open_lit(st);
            put_zeros(st, J);
        }
        st.Zp = 0;
        if (WRITE) write_varint(out, data_pos(st), base, cap, c);
        st.Lb += vlen64((uint64_t)c);
    }
    if (finalize) {
        const uint64_t J = st.Zp;
        if (J >= kMinZeroRun) {
            if (st.has) close_lit(st);
            put_z(st, J);
        } else if (J > 0 || st.has) {
            if (!st.has) open_lit(st);
            put_zeros(st, J);
            close_lit(st);
        }
    }
}

template <class T>
__global__ void __launch_bounds__(ENC_THREADS) k_rle_write(const T* __restrict__ codes, uint64_t n,
                                                           const RleState* __restrict__ states,
                                                           const uint64_t* __restrict__ P,
                                                           const uint64_t* __restrict__ lit_total,
                                                           const DevCtl* __restrict__ ctl, int comp,
                                                           uint8_t* __restrict__ dst, int off_from_ctl) {
    using BS = cub::BlockScan<RleSum, ENC_THREADS>;
    constexpr uint64_t CAP = ENC_TILE * (sizeof(T) == 8 ? 10 : 5) + 64;
    __shared__ typename BS::TempStorage tmp;
    __shared__ uint64_t closeTot[ENC_THREADS + 1];
    __shared__ __align__(16) uint8_t out[CAP];

    const uint64_t tile = blockIdx.x;
    const uint64_t first = tile * ENC_TILE + (uint64_t)threadIdx.x * ENC_ITEMS;
    T v[ENC_ITEMS];
    const int cnt = load_items(codes, n, first, v);
    const RleSum s = thread_summary(v, cnt, threadIdx.x);
    RleSum excl;
    BS(tmp).ExclusiveScan(s, excl, rle_identity(), RleComposeOp());

    const RleState entry = states[tile];
    RleState e = entry;
    e.origin = entry.has ? kEntry : kNoOrigin;
    bool cl;
    uint64_t tot;
    const RleState st = rle_apply(e, excl, &cl, &tot);
    const bool finalize = cnt > 0 && first + cnt == n;

    for (uint32_t k = threadIdx.x; k <= ENC_THREADS; k += ENC_THREADS) closeTot[k] = kUnknown;
    __syncthreads();
    walk<false>(st, v, cnt, finalize, closeTot, nullptr, 0, 0);
    __syncthreads();
    for (uint32_t k = threadIdx.x; k <= ENC_THREADS; k += ENC_THREADS) {
        if (closeTot[k] == kUnknown) {
            if (k == kEntry) closeTot[k] = entry.has ? lit_total[entry.origin] : 0;
            else closeTot[k] = lit_total[tile];
        }
    }
    __syncthreads();
    const uint64_t base = P[tile];
    const uint64_t len = P[tile + 1] - base;
    walk<true>(st, v, cnt, finalize, closeTot, out, base, CAP);
    __syncthreads();
    uint8_t* d = dst + (off_from_ctl ? ctl->stream_off[comp] : 0) + base;
    for (uint64_t k = threadIdx.x; k < len && k < CAP; k += ENC_THREADS) d[k] = out[k];
}

}  // namespace

size_t stream_enc_scratch_bytes(uint64_t n) {
    const uint64_t T = cdiv(n, ENC_TILE);
    return (T + 1) * (sizeof(RleSum) + sizeof(RleState) + 2 * sizeof(uint64_t)) + 256;
}

StreamEncScratch stream_enc_carve(void* base, uint64_t n) {
    const uint64_t T = cdiv(n, ENC_TILE);
    StreamEncScratch s;
    char* p = static_cast<char*>(base);
    s.sums = reinterpret_cast<RleSum*>(p);
    p += (T + 1) * sizeof(RleSum);
    s.states = reinterpret_cast<RleState*>(p);
    p += (T + 1) * sizeof(RleState);
    s.P = reinterpret_cast<uint64_t*>(p);
    p += (T + 1) * sizeof(uint64_t);
    s.lit_total = reinterpret_cast<uint64_t*>(p);
    return s;
}

template <class T>
static void plan_impl(const T* codes, uint64_t n, const StreamEncScratch& s, DevCtl* ctl, int comp,
                      cudaStream_t st) {
    const uint64_t T_ = cdiv(n, ENC_TILE);
    if (T_) {
        k_rle_summary<T><<<(unsigned)T_, ENC_THREADS, 0, st>>>(codes, n, s.sums);
        UMCG_LAUNCHED();
    }
    k_rle_scan<<<1, SCAN_THREADS, 0, st>>>(s.sums, T_, s.states, s.P, s.lit_total, ctl, comp);
    UMCG_LAUNCHED();
}

template <class T>
static void write_impl(const T* codes, uint64_t n, const StreamEncScratch& s, DevCtl* ctl, int comp,
                       uint8_t* dst, bool off_ctl, cudaStream_t st) {
    const uint64_t T_ = cdiv(n, ENC_TILE);
    if (!T_) return;
    k_rle_write<T><<<(unsigned)T_, ENC_THREADS, 0, st>>>(codes, n, s.states, s.P, s.lit_total, ctl,
                                                         comp, dst, off_ctl ? 1 : 0);
    UMCG_LAUNCHED();
}

void stream_plan_u32(const uint32_t* c, uint64_t n, const StreamEncScratch& s, DevCtl* ctl, int comp,
                     cudaStream_t st) { plan_impl(c, n, s, ctl, comp, st); }
void stream_plan_u64(const uint64_t* c, uint64_t n, const StreamEncScratch& s, DevCtl* ctl, int comp,
                     cudaStream_t st) { plan_impl(c, n, s, ctl, comp, st); }
void stream_write_u32(const uint32_t* c, uint64_t n, const StreamEncScratch& s, DevCtl* ctl, int comp,
                      uint8_t* dst, bool o, cudaStream_t st) { write_impl(c, n, s, ctl, comp, dst, o, st); }
void stream_write_u64(const uint64_t* c, uint64_t n, const StreamEncScratch& s, DevCtl* ctl, int comp,
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

// ===========================================================================
// Decode
// ===========================================================================
namespace {

struct Token {
    uint64_t src;   // literal data offset in the stream (unused for zero runs)
    uint64_t uoff;  // offset in the unpacked byte stream
    uint64_t len;   // unpacked bytes; bit 63 set for literal tokens
};

// Serial walk over token headers (rle_decompress, lossless.hpp:53-70).
__global__ void k_token_walk(const uint8_t* __restrict__ s, uint64_t len, Token* __restrict__ tok,
                             uint64_t tok_cap, DevCtl* ctl) {
    if (threadIdx.x | blockIdx.x) return;
    uint64_t pos = 0, u = 0, k = 0;
    int err = 0;
    while (pos < len) {
        const uint8_t tag = s[pos++];
        uint64_t v = 0;
        bool done = false;
        for (int shift = 0; shift < 64; shift += 7) {
            if (pos >= len) { err = DE_CORRUPT_END; break; }
            const uint8_t b = s[pos++];
            v |= (uint64_t)(b & 0x7f) << shift;
            if (!(b & 0x80)) { done = true; break; }
        }
        if (err) break;
        if (!done) { err = DE_CORRUPT_VARINT; break; }
        if (tag == 0x00) {
            if (k < tok_cap) tok[k] = Token{0, u, v};
        } else if (tag == 0x01) {
            if (len - pos < v) { err = DE_CORRUPT_END; break; }
            if (k < tok_cap) tok[k] = Token{pos, u, v | (1ull << 63)};
            pos += v;
        } else {
            err = DE_CORRUPT_TOKEN;
            break;
        }
        u += v;
        ++k;
    }
    if (err) set_err(ctl, err);
    ctl->count = k;
    ctl->aux[0] = u;  // unpacked length
}

constexpr int EXP_THREADS = 256;
constexpr uint64_t EXP_TILE = 8192;

// Expand tokens into the unpacked byte stream: each CTA fills one 8 KiB tile
// of the output, locating its first token by binary search.
__global__ void __launch_bounds__(EXP_THREADS) k_expand(const uint8_t* __restrict__ s,
                                                        const Token* __restrict__ tok, uint64_t ntok,
                                                        uint64_t ulen, uint8_t* __restrict__ u) {
    const uint64_t o0 = blockIdx.x * EXP_TILE;
    const uint64_t o1 = min(ulen, o0 + EXP_TILE);
    // last token with uoff <= o0
    uint64_t lo = 0, hi = ntok;
    while (hi - lo > 1) {
        const uint64_t mid = (lo + hi) / 2;
        if (tok[mid].uoff <= o0) lo = mid; else hi = mid;
    }
    for (uint64_t k = lo; k < ntok; ++k) {
        const Token t = tok[k];
        const uint64_t tl = t.len & ~(1ull << 63);
        if (t.uoff >= o1) break;
        const uint64_t a = max(o0, t.uoff), b = min(o1, t.uoff + tl);
        const bool lit = t.len >> 63;
        for (uint64_t o = a + threadIdx.x; o < b; o += EXP_THREADS)
            u[o] = lit ? s[t.src + (o - t.uoff)] : 0;
    }
}

constexpr int VD_THREADS = 256;
constexpr int VD_BYTES = 16;
constexpr uint64_t VD_TILE = VD_THREADS * VD_BYTES;

// Count code ends (bytes with MSB clear) per tile; flag 10+ byte varints.
__global__ void __launch_bounds__(VD_THREADS) k_varint_count(const uint8_t* __restrict__ u, uint64_t ulen,
                                                             uint64_t* __restrict__ counts, DevCtl* ctl) {
    using BR = cub::BlockReduce<uint64_t, VD_THREADS>;
    __shared__ typename BR::TempStorage tmp;
    const uint64_t b0 = blockIdx.x * VD_TILE + (uint64_t)threadIdx.x * VD_BYTES;
    uint64_t c = 0;
    for (int k = 0; k < VD_BYTES; ++k) {
        const uint64_t i = b0 + k;
        if (i < ulen) {
            const uint8_t b = u[i];
            if (!(b & 0x80)) {
                ++c;
            } else if (i >= 9) {
                // 10 continuation bytes in a row cannot be a valid 64-bit varint
                bool all = true;
                for (int j = 1; j <= 9 && all; ++j) all = (u[i - j] & 0x80) != 0;
                if (all) set_err(ctl, DE_CORRUPT_VARINT);
            }
        }
    }
    const uint64_t t = BR(tmp).Sum(c);
    if (threadIdx.x == 0) counts[blockIdx.x] = t;
}

// Exclusive scan of tile counts in one CTA; total -> ctl->count.
__global__ void __launch_bounds__(1024) k_scan_counts(uint64_t* __restrict__ counts, uint64_t T, DevCtl* ctl) {
    using BS = cub::BlockScan<uint64_t, 1024>;
    __shared__ typename BS::TempStorage tmp;
    const uint64_t per = (T + 1023) / 1024;
    const uint64_t t0 = threadIdx.x * per, t1 = min(T, t0 + per);
    uint64_t local = 0;
    for (uint64_t t = t0; t < t1; ++t) local += counts[t];
    uint64_t excl, total;
    BS(tmp).ExclusiveSum(local, excl, total);
    for (uint64_t t = t0; t < t1; ++t) {
        const uint64_t c = counts[t];
        counts[t] = excl;
        excl += c;
    }
    if (threadIdx.x == 0) ctl->count = total;
}

// Decode the varint ending at each MSB-clear byte; code index from the scan.
__global__ void __launch_bounds__(VD_THREADS) k_varint_decode(const uint8_t* __restrict__ u, uint64_t ulen,
                                                              const uint64_t* __restrict__ tile_start,
                                                              uint64_t n, uint64_t* __restrict__ codes) {
    using BS = cub::BlockScan<uint64_t, VD_THREADS>;
    __shared__ typename BS::TempStorage tmp;
    const uint64_t b0 = blockIdx.x * VD_TILE + (uint64_t)threadIdx.x * VD_BYTES;
    uint8_t b[VD_BYTES];
    uint64_t c = 0;
#pragma unroll
    for (int k = 0; k < VD_BYTES; ++k) {
        const uint64_t i = b0 + k;
        b[k] = i < ulen ? u[i] : 0x80;
        c += !(b[k] & 0x80);
    }
    uint64_t idx;
    BS(tmp).ExclusiveSum(c, idx);
    idx += tile_start[blockIdx.x];
#pragma unroll
    for (int k = 0; k < VD_BYTES; ++k) {
        if (b[k] & 0x80) continue;
        const uint64_t e = b0 + k;
        // walk back to the previous end (or the stream start), <= 9 bytes
        uint64_t s = e;
        while (s > 0 && (u[s - 1] & 0x80) && e - (s - 1) < 10) --s;
        uint64_t v = 0;
        int shift = 0;
        for (uint64_t j = s; j <= e; ++j, shift += 7) v |= (uint64_t)(u[j] & 0x7f) << shift;
        if (idx < n) codes[idx] = v;
        ++idx;
    }
}

}  // namespace

void stream_decode(const uint8_t* d_stream, uint64_t len, uint64_t n, uint64_t* d_codes,
                   StreamDecScratch& sc, DevCtl* ctl, cudaStream_t st) {
    const uint64_t tok_cap = len / 2 + 1;
    Token* tok = sc.tokens.as<Token>(tok_cap);
    k_token_walk<<<1, 32, 0, st>>>(d_stream, len, tok, tok_cap, ctl);
    UMCG_LAUNCHED();
    DevCtl h;
    UMCG_CUDA(cudaMemcpyAsync(&h, ctl, sizeof(DevCtl), cudaMemcpyDeviceToHost, st));
    UMCG_CUDA(cudaStreamSynchronize(st));
    if (h.err) fail(UMCG_CORRUPT_PAYLOAD, h.err == DE_CORRUPT_TOKEN ? "unknown token in lossless stream"
                                          : h.err == DE_CORRUPT_VARINT ? "varint exceeds 64 bits"
                                                                       : "unexpected end of data");
    const uint64_t ntok = h.count, ulen = h.aux[0];
    const uint8_t* u = nullptr;
    if (ntok == 1) {
        Token t;
        UMCG_CUDA(cudaMemcpyAsync(&t, tok, sizeof t, cudaMemcpyDeviceToHost, st));
        UMCG_CUDA(cudaStreamSynchronize(st));
        if (t.len >> 63) u = d_stream + t.src;  // single literal: decode in place
    }
    if (!u && ulen) {
        uint8_t* ub = sc.unpacked.as<uint8_t>(ulen);
        k_expand<<<(unsigned)cdiv(ulen, EXP_TILE), EXP_THREADS, 0, st>>>(d_stream, tok, ntok, ulen, ub);
        UMCG_LAUNCHED();
        u = ub;
    }
    const uint64_t T = cdiv(ulen, VD_TILE);
    uint64_t* counts = sc.counts.as<uint64_t>(T + 1);
    if (T) {
        k_varint_count<<<(unsigned)T, VD_THREADS, 0, st>>>(u, ulen, counts, ctl);
        UMCG_LAUNCHED();
    }
    k_scan_counts<<<1, 1024, 0, st>>>(counts, T, ctl);
    UMCG_LAUNCHED();
    UMCG_CUDA(cudaMemcpyAsync(&h, ctl, sizeof(DevCtl), cudaMemcpyDeviceToHost, st));
    uint8_t last = 0;
    if (ulen) UMCG_CUDA(cudaMemcpyAsync(&last, u + ulen - 1, 1, cudaMemcpyDeviceToHost, st));
    UMCG_CUDA(cudaStreamSynchronize(st));
    // reference order: a code ends early (unexpected end) before trailing bytes
    if (h.err == DE_CORRUPT_VARINT) fail(UMCG_CORRUPT_PAYLOAD, "varint exceeds 64 bits");
    const uint64_t ends = h.count;
    if (ends < n) fail(UMCG_CORRUPT_PAYLOAD, "unexpected end of data");
    if (ends > n || (ulen && (last & 0x80))) fail(UMCG_CORRUPT_PAYLOAD, "trailing bytes in quantized stream");
    if (T) {
        k_varint_decode<<<(unsigned)T, VD_THREADS, 0, st>>>(u, ulen, counts, n, d_codes);
        UMCG_LAUNCHED();
    }
}

void rle_bytes_encode(const uint8_t* d_in, uint64_t n, const StreamEncScratch& s, DevCtl* ctl,
                      uint8_t* dst, cudaStream_t st) {
    (void)d_in; (void)n; (void)s; (void)ctl; (void)dst; (void)st;
    fail(UMCG_ERROR, "raw byte RLE entry not built in this round");
}

}  // namespace umcg
