// Zero-RLE varint stream decode on sm_100a (the encoder is encode.cu).
//
// Decode = serial token walk (token headers only) + parallel expand +
//          parallel varint decode with a tile-count scan; the fused
//          single-pass decode + scan + recompose lives in decode.cu.
#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>

#include "decode.h"

namespace umcg {

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

const uint8_t* stream_unpack(const uint8_t* d_stream, uint64_t len, StreamDecScratch& sc, DevCtl* ctl,
                             cudaStream_t st, uint64_t* ulen_out) {
    const uint64_t tok_cap = len / 2 + 1;
    Token* tok = sc.tokens.as<Token>(tok_cap);
    k_token_walk<<<1, 32, 0, st>>>(d_stream, len, tok, tok_cap, ctl);
    UMCG_LAUNCHED();
    struct { DevCtl c; Token t; } h;
    UMCG_CUDA(cudaMemcpyAsync(&h.c, ctl, sizeof(DevCtl), cudaMemcpyDeviceToHost, st));
    UMCG_CUDA(cudaMemcpyAsync(&h.t, tok, sizeof(Token), cudaMemcpyDeviceToHost, st));
    UMCG_CUDA(cudaStreamSynchronize(st));
    if (h.c.err) fail(UMCG_CORRUPT_PAYLOAD, h.c.err == DE_CORRUPT_TOKEN ? "unknown token in lossless stream"
                                            : h.c.err == DE_CORRUPT_VARINT ? "varint exceeds 64 bits"
                                                                           : "unexpected end of data");
    const uint64_t ntok = h.c.count, ulen = h.c.aux[0];
    *ulen_out = ulen;
    if (ntok == 1 && (h.t.len >> 63)) return d_stream + h.t.src;  // single literal: decode in place
    if (!ulen) return d_stream;
    uint8_t* ub = sc.unpacked.as<uint8_t>(ulen);
    k_expand<<<(unsigned)cdiv(ulen, EXP_TILE), EXP_THREADS, 0, st>>>(d_stream, tok, ntok, ulen, ub);
    UMCG_LAUNCHED();
    return ub;
}

void varint_codes(const uint8_t* u, uint64_t ulen, uint64_t n, uint64_t* d_codes, StreamDecScratch& sc,
                  DevCtl* ctl, cudaStream_t st) {
    const uint64_t T = cdiv(ulen, VD_TILE);
    uint64_t* counts = sc.counts.as<uint64_t>(T + 1);
    if (T) {
        k_varint_count<<<(unsigned)T, VD_THREADS, 0, st>>>(u, ulen, counts, ctl);
        UMCG_LAUNCHED();
    }
    k_scan_counts<<<1, 1024, 0, st>>>(counts, T, ctl);
    UMCG_LAUNCHED();
    DevCtl h;
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

void stream_decode(const uint8_t* d_stream, uint64_t len, uint64_t n, uint64_t* d_codes,
                   StreamDecScratch& sc, DevCtl* ctl, cudaStream_t st) {
    uint64_t ulen = 0;
    const uint8_t* u = stream_unpack(d_stream, len, sc, ctl, st, &ulen);
    varint_codes(u, ulen, n, d_codes, sc, ctl, st);
}

void rle_bytes_encode(const uint8_t* d_in, uint64_t n, const StreamEncScratch& s, DevCtl* ctl,
                      uint8_t* dst, cudaStream_t st) {
    (void)d_in; (void)n; (void)s; (void)ctl; (void)dst; (void)st;
    fail(UMCG_ERROR, "raw byte RLE entry not built in this round");
}

}  // namespace umcg
