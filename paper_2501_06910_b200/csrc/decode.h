// Fused stream decode (decode.cu) + N-D lattice reconstruction helpers.
#pragma once

#include "kernels.h"

namespace umcg {

// DEC_RECOMPOSE_GE: x'_i = g_i + fl(K * bin) with g prepared in layout E
// (multilinear g, partition.cu): node = dstE, K1 = the fp64 gE array.
enum DecMode : int { DEC_P64 = 0, DEC_VALUES = 1, DEC_RECOMPOSE = 2, DEC_RECOMPOSE16 = 3, DEC_RECOMPOSE_GE = 4,
                     DEC_Q32 = 5 };  // Q32: the zigzag-decoded codes as int32 (P64 points to them)

// One RLE token (stream.cu): literal data offset, unpacked offset, length
// (bit 63 set for literal tokens).
struct Token {
    uint64_t src;
    uint64_t uoff;
    uint64_t len;
};

// Where a fused decode reads its unpacked varint bytes: known on the host
// (U, ulen), or resolved on the device from the token walk (base + tok[0]
// when the stream is exactly one literal; otherwise ulen = 0 and the caller's
// verdict fails), so no host synchronization sits between the two.
struct DecSrc {
    const uint8_t* U;
    uint64_t ulen;
    const uint8_t* base;
    const Token* tok;
    const DevCtl* tctl;
};
inline DecSrc host_src(const uint8_t* U, uint64_t ulen) { return DecSrc{U, ulen, nullptr, nullptr, nullptr}; }
#ifdef __CUDACC__
__device__ __forceinline__ void resolve_src(const DecSrc& s, const uint8_t*& U, uint64_t& ulen) {
    if (!s.tok) {
        U = s.U;
        ulen = s.ulen;
        return;
    }
    const Token t = s.tok[0];
    const bool one = s.tctl->count == 1 && (t.len >> 63) && s.tctl->err == 0 && s.tctl->aux[1] == 0;
    U = s.base + (one ? t.src : 0);
    ulen = one ? (t.len & ~(1ull << 63)) : 0;
}
#endif

size_t dec_status_bytes(uint64_t ulen);
// One pass over the unpacked varint bytes U[0..ulen): see decode.cu. Writes
// ctl->count (number of complete varints), ctl->max_abs_k[1], flags
// DE_CORRUPT_VARINT, and ctl->aux[7] = 1 when a varint longer than a lossy
// PQ code (> 5 bytes / >= 2^32) was seen (caller must use the general path).
// With DEC_RECOMPOSE16, K1 points to an int16 table.
// t_tiles: tiles launched (>= cdiv(ulen, 8 KiB); extra CTAs exit).
uint64_t dec_tiles(uint64_t ulen_bound);
// DEC_RECOMPOSE with kctl/K16: gathers from K16 (int16 copy of K1) when
// kctl->max_abs_k[0] < 2^15 on the device.
// prepared: dec_prepare (tile aggregates + their scan) already ran for this
// source/status/ctl, possibly on another stream ordered before st.
void dec_fused(int mode, const DecSrc& src, uint64_t t_tiles, uint64_t n, void* status, DevCtl* ctl,
               const uint32_t* node, const int32_t* K1, double bin1, double bin, double* out, int64_t* P64,
               cudaStream_t st, const DevCtl* kctl = nullptr, const int16_t* K16 = nullptr, bool prepared = false);
void dec_prepare(const DecSrc& src, uint64_t t_tiles, void* status, DevCtl* ctl, cudaStream_t st);
// N-D inclusive prefix from the plain 1-D prefix P of row-major codes:
// row differencing (fastest axis) + scans along the other axes -> int32 K,
// max|K| -> ctl->max_abs_k[0]. Kw is int64 scratch [n] (unused when D == 1).
void nd_from_prefix(const int64_t* P, uint64_t n, const NdShape& sh, int64_t* Kw, int32_t* K32, int16_t* K16,
                    DevCtl* ctl,
                    cudaStream_t st);
// 3-D grids with d2 <= 1024: N-D inclusive prefix straight from the decoded
// codes Q (DEC_Q32), int32 plane prefixes S [n] as scratch.
bool nd3_supported(const NdShape& sh);
void nd3_from_codes(const int32_t* Q, const NdShape& sh, int32_t* S, int32_t* K32, int16_t* K16, DevCtl* ctl,
                    cudaStream_t st);
void k32_to_f64(const int32_t* K, uint64_t n, double bin, double* x, cudaStream_t st);

// Launch the serial token probe (<= 64 tokens) without synchronizing;
// returns the device token table (tok[0] valid when it is one literal).
const Token* stream_probe(const uint8_t* d_stream, uint64_t len, StreamDecScratch& s, DevCtl* tctl,
                          cudaStream_t st);

// RLE token stream -> unpacked varint bytes (in place for a single literal
// token). Synchronizes; throws corrupt_payload on malformed token streams.
const uint8_t* stream_unpack(const uint8_t* d_stream, uint64_t len, StreamDecScratch& s, DevCtl* ctl,
                             cudaStream_t st, uint64_t* ulen);
// varint bytes -> codes[n] (u64); validates counts (corrupt_payload).
void varint_codes(const uint8_t* U, uint64_t ulen, uint64_t n, uint64_t* d_codes, StreamDecScratch& s,
                  DevCtl* ctl, cudaStream_t st);

}  // namespace umcg
