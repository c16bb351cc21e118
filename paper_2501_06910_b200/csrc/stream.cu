// Zero-RLE varint stream decode on sm_100a (the encoder is encode.cu).
//
// Decode = serial token walk (token headers only) + parallel expand +
//          parallel varint decode with a tile-count scan; the fused
//          single-pass decode + scan + recompose lives in decode.cu.
#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>

#include "decode.h"
#include "scan_tiles.cuh"

namespace umcg {

// ===========================================================================
// Decode
// ===========================================================================
namespace {

// Serial walk over token headers (rle_decompress, lossless.hpp:53-70).
// Stops after max_tok tokens; aux[1] = 1 when the stream is not finished
// (the caller then switches to the parallel parse below).
__global__ void k_token_walk(const uint8_t* __restrict__ s, uint64_t len, Token* __restrict__ tok,
                             uint64_t tok_cap, uint64_t max_tok, DevCtl* ctl) {
    if (threadIdx.x | blockIdx.x) return;
    uint64_t pos = 0, u = 0, k = 0;
    int err = 0;
    while (pos < len && k < max_tok) {
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
    ctl->aux[1] = !err && pos < len;
    ctl->aux[2] = pos;  // bytes the probe covered (token density estimate)
}

// ---------------------------------------------------------------------------
// Parallel token parse for streams with many tokens.
//
// The token chain is a functional graph on stream offsets: next(p) = p + 1 +
// |varint| (+ literal length). Every offset is a potential token start.
//  1. k_tok_jump: per chunk of PJ_C offsets, the "exit" of EVERY offset (the
//     first chain offset at or past the chunk end) by pointer jumping in
//     shared memory, plus the chunk's set of distinct live exits (<= PJ_K;
//     garbage chains inside literal data converge to a handful of exits).
//  2. k_tok_groups: per group of PJ_G chunks, one lane per possible entry
//     (the distinct exits of the chunk before the group) follows its chain
//     through the group's exit tables; records each chunk's entry per lane
//     and the group's exit per lane.
//  3. k_tok_resolve: one warp chains the groups from offset 0 -- a shared
//     memory match per group -- and picks each group's true lane (groups with
//     too many possible entries are chained chunk by chunk instead).
//  4. k_tok_walk_chunks: every chunk re-walks its own tokens from its
//     resolved entry, verifying the chain (must land exactly on the next
//     chunk's entry, no malformed header) and counting, then emitting, the
//     token table.
// Any disagreement sends the caller to the serial walk, which reports the
// reference's exact error.
// ---------------------------------------------------------------------------
constexpr int PJ_THREADS = 1024;
constexpr uint64_t PJ_C = 8192;  // offsets per chunk
constexpr int PJ_HALO = 16;      // tag + 10-byte varint past the chunk end
constexpr int PJ_K = 32;         // distinct exits kept per chunk (one warp)
constexpr int PJ_HS = 128;       // hash slots for the distinct-exit set
constexpr uint64_t PJ_G = 64;    // chunks per group
constexpr int PJ_SB = 8;         // sub-chunks of 2^PJ_SB bytes for the token walks
constexpr uint64_t PJ_NS = PJ_C >> PJ_SB;  // sub-chunks per chunk
constexpr uint64_t PJ_DEAD = ~0ull;
constexpr uint32_t PJ_DEAD32 = 0xFFFFFFFFu;
constexpr uint32_t PJ_MANY = 0xFFFFFFFFu;
constexpr uint8_t PJ_SLOW = 0xFF;
constexpr size_t PJ_SMEM = PJ_C * 4 + PJ_C + PJ_HALO + 16;

// One token header at p (< len), the checks of k_token_walk: next token
// start, or PJ_DEAD when the header is malformed or the literal overruns.
template <class At>
__device__ __forceinline__ uint64_t tok_next(At at, uint64_t len, uint64_t p, uint64_t& v, uint32_t& tag) {
    tag = at(p++);
    v = 0;
    if (tag > 1) return PJ_DEAD;
    for (int shift = 0; shift < 64; shift += 7) {
        if (p >= len) return PJ_DEAD;
        const uint32_t b = at(p++);
        v |= (uint64_t)(b & 0x7f) << shift;
        if (!(b & 0x80)) {
            if (tag == 0) return p;
            return len - p < v ? PJ_DEAD : p + v;
        }
    }
    return PJ_DEAD;
}

__global__ void __launch_bounds__(PJ_THREADS) k_tok_jump(const uint8_t* __restrict__ s, uint64_t len,
                                                         uint32_t* __restrict__ ex, uint32_t* __restrict__ dcount,
                                                         uint64_t* __restrict__ dvals, uint32_t* __restrict__ subex) {
    extern __shared__ __align__(16) uint8_t pj_smem[];
    __shared__ unsigned long long hs[PJ_HS];
    __shared__ int hcount, hpos;
    // nx[i]: successor of offset P + i, relative to P (>= n: an exit; PJ_DEAD32: malformed)
    uint32_t* nx = reinterpret_cast<uint32_t*>(pj_smem);
    const uint64_t P = blockIdx.x * PJ_C;
    const uint64_t E = min(len, P + PJ_C);
    const uint32_t n = (uint32_t)(E - P);
    // Warp w owns sub-chunk w (2^PJ_SB offsets) up to the sub-chunk exits:
    // staging, successors and the first jumping rounds are warp-local.
    // Bytes come by aligned 16-byte loads from the 16-byte boundary at or
    // below s + P (the stream sits at any offset of the archive): sb[k] =
    // s[P + k] for the warp's [2^PJ_SB w, 2^PJ_SB (w + 1) + HALO).
    static_assert(PJ_NS * 32 == PJ_THREADS, "one warp per sub-chunk");
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t sh = (uint32_t)((uintptr_t)(s + P) & 15);
    uint8_t* raw = pj_smem + PJ_C * 4;
    uint8_t* sb = raw + sh;
    const uint32_t s0 = (uint32_t)warp << PJ_SB, s1 = min(n, s0 + (1u << PJ_SB));
    {
        const uint4* src = reinterpret_cast<const uint4*>(s + P - sh);
        const uint32_t want = (uint32_t)min((uint64_t)(PJ_C + PJ_HALO), len - P);
        const uint32_t nw = (sh + want + 15) / 16;
        const uint32_t w0 = (s0 + sh) / 16, w1 = min(nw, (s0 + (1u << PJ_SB) + PJ_HALO + sh + 15) / 16);
        for (uint32_t w = w0 + lane; w < w1; w += 32) reinterpret_cast<uint4*>(raw)[w] = __ldg(src + w);
    }
    for (int i = threadIdx.x; i < PJ_HS; i += PJ_THREADS) hs[i] = PJ_DEAD;
    if (threadIdx.x == 0) hcount = hpos = 0;
    __syncwarp();
    auto at = [&](uint64_t q) -> uint32_t { return sb[q - P]; };
    const uint64_t rem = len - P;  // bytes from the chunk start to the stream end
    for (uint32_t i = s0 + lane; i < s1; i += 32) {
        // common case first: a 1-byte varint (32-bit offsets, rem >= i + 2)
        const uint32_t tag = sb[i], b = sb[i + 1];
        uint32_t r;
        if (tag > 1) {
            r = PJ_DEAD32;
        } else if (b < 0x80 && i + 2 <= rem) {
            const uint64_t e = (uint64_t)i + 2 + (tag ? b : 0);
            r = e > rem ? PJ_DEAD32 : (uint32_t)e;
        } else {
            uint64_t v;
            uint32_t tg;
            const uint64_t q = tok_next(at, len, P + i, v, tg);
            r = q == PJ_DEAD ? PJ_DEAD32 : (uint32_t)(q - P);
        }
        nx[i] = r;
    }
    __syncwarp();
    // Pointer jumping. Updates are in place: a reader sees either the old or
    // the new successor, both on the same chain, so the fixed point is exact.
    // First, warp-local, to the end of each offset's own sub-chunk (v < s1
    // implies v lies in the same sub-chunk): the sub-chunk exits the token
    // walks start from; then, block-wide on those, to the end of the chunk
    // (<= log2(PJ_NS) more rounds).
    for (;;) {
        int moved = 0;
        for (uint32_t i = s0 + lane; i < s1; i += 32) {
            const uint32_t v = nx[i];
            if (v < s1) {
                const uint32_t w = nx[v];
                nx[i] = w;
                moved |= w < s1;
            }
        }
        __syncwarp();
        if (!__any_sync(0xffffffffu, moved)) break;
    }
    if (subex)
        for (uint32_t i = s0 + lane; i < s1; i += 32) subex[P + i] = nx[i];
    __syncthreads();
    for (;;) {
        int moved = 0;
        for (uint32_t i = threadIdx.x; i < n; i += PJ_THREADS) {
            const uint32_t v = nx[i];
            if (v < n) {
                const uint32_t w = nx[v];
                nx[i] = w;
                moved |= w < n;
            }
        }
        if (!__syncthreads_or(moved)) break;
    }
    // exit table + distinct live exits (warp-deduplicated hash insert)
    for (uint32_t base = 0; base < n; base += PJ_THREADS) {
        const uint32_t i = base + threadIdx.x;
        const uint32_t r = i < n ? nx[i] : PJ_DEAD32;
        if (i < n) ex[P + i] = r;
        const uint64_t v = r == PJ_DEAD32 ? PJ_DEAD : P + r;
        const unsigned m = __match_any_sync(0xffffffffu, v);
        if (v != PJ_DEAD && __ffs(m) - 1 == lane && *(volatile int*)&hcount <= PJ_K) {
            unsigned h = (unsigned)((v * 0x9E3779B97F4A7C15ull) >> 57);
            int k = 0;
            for (; k < PJ_HS; ++k, h = (h + 1) & (PJ_HS - 1)) {
                const unsigned long long old = atomicCAS(&hs[h], PJ_DEAD, v);
                if (old == PJ_DEAD) { atomicAdd(&hcount, 1); break; }
                if (old == v) break;
            }
            if (k == PJ_HS) atomicAdd(&hcount, PJ_K + 1);
        }
    }
    __syncthreads();
    const int hc = hcount;
    if (threadIdx.x < PJ_HS && hc <= PJ_K) {
        const uint64_t v = hs[threadIdx.x];
        if (v != PJ_DEAD) dvals[blockIdx.x * PJ_K + atomicAdd(&hpos, 1)] = v;
    }
    if (threadIdx.x == 0) dcount[blockIdx.x] = hc <= PJ_K ? (uint32_t)hc : PJ_MANY;
}

// Entry of every sub-chunk from its chunk's entry: 32 steps through the
// sub-exit table per chunk (one thread per chunk); must land on the next
// chunk's entry.
__device__ __forceinline__ uint64_t chunk_entry(uint64_t c, uint64_t nc, const uint8_t* glane,
                                                const uint64_t* gent, const uint64_t* eslow,
                                                const uint64_t* entry_end);
__global__ void __launch_bounds__(128) k_tok_sub_entries(uint64_t len, uint64_t nc, const uint8_t* __restrict__ glane,
                                                         const uint64_t* __restrict__ gent,
                                                         const uint64_t* __restrict__ eslow,
                                                         const uint64_t* __restrict__ entry_end,
                                                         const uint32_t* __restrict__ subex, int sb_shift,
                                                         uint64_t* __restrict__ sent, DevCtl* ctl) {
    const uint64_t c = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (c >= nc) return;
    const uint64_t P = c * PJ_C;
    uint64_t e = chunk_entry(c, nc, glane, gent, eslow, entry_end);
    if (!subex) {  // chunk-level walks
        sent[c] = e;
        return;
    }
    const uint64_t nsub = PJ_C >> sb_shift;
    for (uint64_t j = 0; j < nsub; ++j) {
        sent[c * nsub + j] = e;
        const uint64_t send = min(len, P + ((j + 1) << sb_shift));
        if (e < send) {
            const uint32_t r = subex[e];
            if (r == PJ_DEAD32) { ctl->aux[1] = 1; return; }
            e = P + r;
        }
    }
    if (e != chunk_entry(c + 1, nc, glane, gent, eslow, entry_end)) ctl->aux[1] = 1;
}

// One warp per group of PJ_G chunks; lane = one possible group entry.
__global__ void __launch_bounds__(32) k_tok_groups(const uint32_t* __restrict__ ex,
                                                   const uint32_t* __restrict__ dcount,
                                                   const uint64_t* __restrict__ dvals, uint64_t nc, uint64_t len,
                                                   uint64_t* __restrict__ gent, uint64_t* __restrict__ gin,
                                                   uint64_t* __restrict__ gout, uint32_t* __restrict__ gn) {
    const uint64_t g = blockIdx.x;
    const int lane = threadIdx.x;
    const uint64_t c0 = g * PJ_G, c1 = min(nc, c0 + PJ_G);
    uint32_t ne = 1;
    uint64_t s = lane == 0 ? 0 : PJ_DEAD;
    if (g) {
        ne = dcount[c0 - 1];
        if (ne == PJ_MANY) {
            if (lane == 0) gn[g] = PJ_MANY;
            return;
        }
        s = lane < (int)ne ? dvals[(c0 - 1) * PJ_K + lane] : PJ_DEAD;
    }
    gin[g * 32 + lane] = s;
    for (uint64_t c = c0; c < c1; ++c) {
        gent[c * 32 + lane] = s;
        const uint64_t P = c * PJ_C, E = min(len, P + PJ_C);
        if (s < E) {
            const uint32_t r = ex[s];
            s = r == 0xFFFFFFFFu ? PJ_DEAD : P + r;
        }
    }
    gout[g * 32 + lane] = s;
    if (lane == 0) gn[g] = ne;
}

// Chain the groups from offset 0: glane[g] = true lane of group g (PJ_SLOW:
// entries chained chunk by chunk into eslow -- too many possible entries, or
// an entry that a long literal carried past the chunk before the group). entry_end = chain end.
// aux[1] = 1 when the chain breaks.
__global__ void __launch_bounds__(1024) k_tok_resolve(const uint32_t* __restrict__ ex,
                                                      const uint64_t* __restrict__ gin,
                                                      const uint64_t* __restrict__ gout,
                                                      const uint32_t* __restrict__ gn, uint64_t nc, uint64_t len,
                                                      uint8_t* __restrict__ glane, uint64_t* __restrict__ eslow,
                                                      uint64_t* __restrict__ entry_end, DevCtl* ctl) {
    __shared__ uint64_t si[1024], so[1024];
    __shared__ uint32_t sn[32];
    const uint64_t ng = (nc + PJ_G - 1) / PJ_G;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint64_t s = 0;  // warp 0's chain position
    bool bad = false;
    for (uint64_t gb = 0; gb < ng; gb += 32) {
        const uint64_t g = gb + warp;
        __syncthreads();
        if (g < ng) {
            si[threadIdx.x] = gin[g * 32 + lane];
            so[threadIdx.x] = gout[g * 32 + lane];
            if (lane == 0) sn[warp] = gn[g];
        }
        __syncthreads();
        if (warp == 0) {
            const int m = (int)min((uint64_t)32, ng - gb);
            for (int k = 0; k < m; ++k) {
                const uint64_t gg = gb + k;
                uint8_t gl = PJ_SLOW;
                if (sn[k] != PJ_MANY) {
                    const unsigned hit = __ballot_sync(0xffffffffu, lane < (int)sn[k] && si[k * 32 + lane] == s);
                    if (hit) {
                        gl = (uint8_t)(__ffs(hit) - 1);
                        s = so[k * 32 + gl];
                    }
                    // no hit: the entry came from a literal that jumped over
                    // the chunk before the group -- chain this group slowly
                }
                if (gl == PJ_SLOW && !bad) {  // chunk-by-chunk through this group
                    const uint64_t c0 = gg * PJ_G, c1 = min(nc, c0 + PJ_G);
                    for (uint64_t c = c0; c < c1; ++c) {
                        if (lane == 0) eslow[c] = s;
                        const uint64_t P = c * PJ_C, E = min(len, P + PJ_C);
                        if (s < E) {
                            const uint32_t r = ex[s];
                            if (r == 0xFFFFFFFFu) { bad = true; break; }
                            s = P + r;
                        }
                    }
                }
                if (lane == 0) glane[gg] = gl;
                if (bad) break;
            }
        }
        if (__syncthreads_or(bad)) break;
    }
    if (threadIdx.x == 0) {
        *entry_end = s;
        if (bad || s != len) ctl->aux[1] = 1;
    }
}

__device__ __forceinline__ uint64_t chunk_entry(uint64_t c, uint64_t nc, const uint8_t* glane,
                                                const uint64_t* gent, const uint64_t* eslow,
                                                const uint64_t* entry_end) {
    if (c >= nc) return *entry_end;
    const uint8_t l = glane[c / PJ_G];
    return l == PJ_SLOW ? eslow[c] : gent[c * 32 + l];
}

// One thread per sub-chunk: walk its tokens from its entry. EMIT = false
// verifies (must land exactly on the next sub-chunk's entry, no malformed
// header) and counts (tokens, unpacked bytes); EMIT = true writes the token
// table at the scanned offsets.
// Count pass (EMIT false): per sub-chunk token count and unpacked bytes
// (cnt, ub) and their per-block sums (bsum); emit pass: block scan of (cnt,
// ub) + the block's prefix (bpre, k_scan_tiles of bsum) = the sub-chunk's
// first token index and unpacked offset.
template <bool EMIT>
__global__ void __launch_bounds__(128) k_tok_walk_subs(const uint8_t* __restrict__ s, uint64_t len, uint64_t ns,
                                                       int shift, const uint64_t* __restrict__ sent,
                                                       const uint64_t* __restrict__ entry_end,
                                                       uint64_t* __restrict__ cnt, uint64_t* __restrict__ ub,
                                                       ulonglong2* __restrict__ bsum,
                                                       const ulonglong2* __restrict__ bpre,
                                                       Token* __restrict__ tok, DevCtl* ctl) {
    using BS = cub::BlockScan<ulonglong2, 128>;
    using BR = cub::BlockReduce<ulonglong2, 128>;
    __shared__ union {
        typename BS::TempStorage s;
        typename BR::TempStorage r;
    } tmp;
    const uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    uint64_t k = 0, u = 0;
    if (EMIT) {
        const ulonglong2 mine = q < ns ? make_ulonglong2(cnt[q], ub[q]) : make_ulonglong2(0, 0);
        ulonglong2 ex;
        BS(tmp.s).ExclusiveScan(mine, ex, make_ulonglong2(0, 0), u2_add_op{});
        const ulonglong2 b = bpre[blockIdx.x];
        k = b.x + ex.x;
        u = b.y + ex.y;
    }
    if (q < ns) {
        const uint64_t E = min(len, (q + 1) << shift);
        uint64_t p = sent[q];
        auto at = [&](uint64_t x) -> uint32_t { return s[x]; };
        while (p < E) {
            uint64_t v;
            uint32_t tag;
            const uint64_t nq = tok_next(at, len, p, v, tag);
            if (nq == PJ_DEAD) { ctl->aux[1] = 1; break; }
            if (EMIT) tok[k] = tag ? Token{nq - v, u, v | (1ull << 63)} : Token{0, u, v};
            ++k;
            u += v;
            p = nq;
        }
        if (!EMIT) {
            if (p != (q + 1 < ns ? sent[q + 1] : *entry_end)) ctl->aux[1] = 1;
            cnt[q] = k;
            ub[q] = u;
        }
    }
    if (!EMIT) {
        const ulonglong2 t = BR(tmp.r).Reduce(make_ulonglong2(k, u), u2_add_op{});
        if (threadIdx.x == 0) bsum[blockIdx.x] = t;
    }
}

constexpr int EXP_THREADS = 256;
constexpr uint64_t EXP_TILE = EXP_THREADS * 16;  // 16 output bytes per thread
constexpr int EXP_TOK = 1024;                   // tokens staged per tile

// Expand tokens into the unpacked byte stream. Each CTA fills one 4 KiB
// tile: the tokens overlapping it are staged in shared memory, then every
// thread assembles 16 bytes (binary search for its first token) and writes
// one 16-byte store. Tiles overlapping more than EXP_TOK tokens (zero-length
// tokens) take the token-by-token loop.
__global__ void __launch_bounds__(EXP_THREADS) k_expand(const uint8_t* __restrict__ s,
                                                        const Token* __restrict__ tok, uint64_t ntok,
                                                        uint64_t ulen, uint8_t* __restrict__ u) {
    __shared__ uint64_t t_uoff[EXP_TOK], t_src[EXP_TOK], t_len[EXP_TOK];
    __shared__ uint64_t range[2];
    const uint64_t o0 = blockIdx.x * EXP_TILE;
    const uint64_t o1 = min(ulen, o0 + EXP_TILE);
    if (threadIdx.x < 2) {
        // last token with uoff <= target (tokens are sorted by uoff)
        const uint64_t target = threadIdx.x ? o1 - 1 : o0;
        uint64_t lo = 0, hi = ntok;
        while (hi - lo > 1) {
            const uint64_t mid = (lo + hi) / 2;
            if (tok[mid].uoff <= target) lo = mid; else hi = mid;
        }
        range[threadIdx.x] = lo;
    }
    __syncthreads();
    const uint64_t k0 = range[0], nt = range[1] - range[0] + 1;
    if (nt > (uint64_t)EXP_TOK) {
        for (uint64_t k = k0; k < ntok; ++k) {
            const Token t = tok[k];
            const uint64_t tl = t.len & ~(1ull << 63);
            if (t.uoff >= o1) break;
            const uint64_t a = max(o0, t.uoff), b = min(o1, t.uoff + tl);
            const bool lit = t.len >> 63;
            for (uint64_t o = a + threadIdx.x; o < b; o += EXP_THREADS) u[o] = lit ? s[t.src + (o - t.uoff)] : 0;
        }
        return;
    }
    for (uint32_t k = threadIdx.x; k < (uint32_t)nt; k += EXP_THREADS) {
        const Token t = tok[k0 + k];
        t_uoff[k] = t.uoff;
        t_src[k] = t.src;
        t_len[k] = t.len;
    }
    __syncthreads();
    const uint64_t o = o0 + threadIdx.x * 16ull;
    if (o >= o1) return;
    uint32_t lo = 0, hi = (uint32_t)nt;
    while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) / 2;
        if (t_uoff[mid] <= o) lo = mid; else hi = mid;
    }
    uint32_t w[4] = {0, 0, 0, 0};
    const int m = (int)min((uint64_t)16, o1 - o);
    uint32_t k = lo;
    uint64_t tu = t_uoff[k], tl = t_len[k] & ~(1ull << 63), ts = t_src[k];
    bool lit = t_len[k] >> 63;
    for (int j = 0; j < m; ++j) {
        const uint64_t q = o + j;
        while (q >= tu + tl) {  // next token (zero-length ones are skipped)
            ++k;
            tu = t_uoff[k];
            tl = t_len[k] & ~(1ull << 63);
            ts = t_src[k];
            lit = t_len[k] >> 63;
        }
        if (lit) w[j >> 2] |= (uint32_t)s[ts + (q - tu)] << (8 * (j & 3));
    }
    if (m == 16) {
        *reinterpret_cast<uint4*>(u + o) = make_uint4(w[0], w[1], w[2], w[3]);
    } else {
        for (int j = 0; j < m; ++j) u[o + j] = (uint8_t)(w[j >> 2] >> (8 * (j & 3)));
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

// Parallel parse; returns false when the chain is broken (corrupt stream).
// fine: token-dense stream (the probe saw > 1 token per KiB): token walks
// per 256-byte sub-chunk (exits from the same pointer jumping); otherwise per
// 8 KiB chunk, without the sub-exit table.
static bool parallel_tokens(const uint8_t* d_stream, uint64_t len, Token* tok, StreamDecScratch& sc, DevCtl* ctl,
                            cudaStream_t st, uint64_t* ntok, uint64_t* ulen, bool fine) {
    static DeviceOnce attr;
    attr([] { UMCG_CUDA(cudaFuncSetAttribute(k_tok_jump, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)PJ_SMEM)); });
    const int shift = fine ? PJ_SB : 13;  // 2^13 == PJ_C
    static_assert(PJ_C == (1ull << 13), "chunk-level walks use shift 13");
    const uint64_t nc = cdiv(len, PJ_C), ng = cdiv(nc, PJ_G), ns = nc * (PJ_C >> shift);
    // scratch: tot u64[2] | bsum, bpre u64[2][g] (16-byte aligned at the base) | ex, subex u32[len] |
    //          dcount u32[nc] | dvals u64[nc*K] | gent u64[nc*32] | gin, gout u64[ng*32] | gn u32[ng] |
    //          eslow u64[nc] | sent, cnt, ub u64[ns] | entry_end | glane u8[ng]
    const uint64_t g = cdiv(ns, 128);
    const uint64_t ex_b = (len * 4 + 7) & ~7ull, dc_b = (nc * 4 + 7) & ~7ull, gn_b = (ng * 4 + 7) & ~7ull;
    const uint64_t bytes = 2 * ex_b + dc_b + nc * PJ_K * 8 + nc * 32 * 8 + ng * 32 * 16 + gn_b + nc * 8 +
                           ns * 24 + 24 + ng + 8 + g * 32;
    uint8_t* q = sc.parse.as<uint8_t>(bytes);
    uint64_t* tot = reinterpret_cast<uint64_t*>(q); q += 16;
    ulonglong2* bsum = reinterpret_cast<ulonglong2*>(q); q += g * 16;
    ulonglong2* bpre = reinterpret_cast<ulonglong2*>(q); q += g * 16;
    uint32_t* ex = reinterpret_cast<uint32_t*>(q); q += ex_b;
    uint32_t* subex = reinterpret_cast<uint32_t*>(q); q += ex_b;
    uint32_t* dcount = reinterpret_cast<uint32_t*>(q); q += dc_b;
    uint64_t* dvals = reinterpret_cast<uint64_t*>(q); q += nc * PJ_K * 8;
    uint64_t* gent = reinterpret_cast<uint64_t*>(q); q += nc * 32 * 8;
    uint64_t* gin = reinterpret_cast<uint64_t*>(q); q += ng * 32 * 8;
    uint64_t* gout = reinterpret_cast<uint64_t*>(q); q += ng * 32 * 8;
    uint32_t* gn = reinterpret_cast<uint32_t*>(q); q += gn_b;
    uint64_t* eslow = reinterpret_cast<uint64_t*>(q); q += nc * 8;
    uint64_t* sent = reinterpret_cast<uint64_t*>(q); q += ns * 8;
    uint64_t* cnt = reinterpret_cast<uint64_t*>(q); q += ns * 8;
    uint64_t* ub = reinterpret_cast<uint64_t*>(q); q += ns * 8;
    uint64_t* entry_end = reinterpret_cast<uint64_t*>(q); q += 8;
    uint8_t* glane = q;
    UMCG_CUDA(cudaMemsetAsync(&ctl->aux[1], 0, 8, st));
    {
        ProfScope ps("k_tok_jump", st);
        k_tok_jump<<<(unsigned)nc, PJ_THREADS, PJ_SMEM, st>>>(d_stream, len, ex, dcount, dvals,
                                                              fine ? subex : nullptr);
        UMCG_LAUNCHED();
    }
    {
        ProfScope ps("k_tok_resolve", st);
        k_tok_groups<<<(unsigned)ng, 32, 0, st>>>(ex, dcount, dvals, nc, len, gent, gin, gout, gn);
        UMCG_LAUNCHED();
        k_tok_resolve<<<1, 1024, 0, st>>>(ex, gin, gout, gn, nc, len, glane, eslow, entry_end, ctl);
        UMCG_LAUNCHED();
        k_tok_sub_entries<<<(unsigned)cdiv(nc, 128), 128, 0, st>>>(len, nc, glane, gent, eslow, entry_end,
                                                                     fine ? subex : nullptr, shift, sent, ctl);
        UMCG_LAUNCHED();
    }
    {
        ProfScope ps("k_tok_count", st);
        k_tok_walk_subs<false><<<(unsigned)g, 128, 0, st>>>(d_stream, len, ns, shift, sent, entry_end, cnt, ub, bsum, bpre,
                                                  tok, ctl);
        UMCG_LAUNCHED();
    }
    k_scan_tiles<<<scan_tiles_grid(g), SCAN_TILES_THREADS, 0, st>>>(bsum, bpre, g,
                                                                    reinterpret_cast<ulonglong2*>(tot), nullptr);
    UMCG_LAUNCHED();
    {
        ProfScope ps("k_tok_emit", st);
        k_tok_walk_subs<true><<<(unsigned)g, 128, 0, st>>>(d_stream, len, ns, shift, sent, entry_end, cnt, ub, bsum, bpre,
                                                 tok, ctl);
        UMCG_LAUNCHED();
    }
    struct { uint64_t bad, t[2]; } h;
    UMCG_CUDA(cudaMemcpyAsync(&h.bad, &ctl->aux[1], 8, cudaMemcpyDeviceToHost, st));
    UMCG_CUDA(cudaMemcpyAsync(h.t, tot, 16, cudaMemcpyDeviceToHost, st));
    UMCG_CUDA(cudaStreamSynchronize(st));
    *ntok = h.t[0];
    *ulen = h.t[1];
    return !h.bad;
}

const Token* stream_probe(const uint8_t* d_stream, uint64_t len, StreamDecScratch& sc, DevCtl* tctl,
                          cudaStream_t st) {
    const uint64_t tok_cap = len / 2 + 1;
    Token* tok = sc.tokens.as<Token>(tok_cap);
    k_token_walk<<<1, 32, 0, st>>>(d_stream, len, tok, tok_cap, 64, tctl);
    UMCG_LAUNCHED();
    return tok;
}

const uint8_t* stream_unpack(const uint8_t* d_stream, uint64_t len, StreamDecScratch& sc, DevCtl* ctl,
                             cudaStream_t st, uint64_t* ulen_out) {
    const uint64_t tok_cap = len / 2 + 1;
    Token* tok = sc.tokens.as<Token>(tok_cap);
    // Short serial probe: a lossy stream is usually a handful of tokens.
    constexpr uint64_t kProbe = 64;
    const bool par_ok = len >= 2 * PJ_C && len < 0xFFFFFFF0ull;
    k_token_walk<<<1, 32, 0, st>>>(d_stream, len, tok, tok_cap, par_ok ? kProbe : ~0ull, ctl);
    UMCG_LAUNCHED();
    struct { DevCtl c; Token t; } h;
    UMCG_CUDA(cudaMemcpyAsync(&h.c, ctl, sizeof(DevCtl), cudaMemcpyDeviceToHost, st));
    UMCG_CUDA(cudaMemcpyAsync(&h.t, tok, sizeof(Token), cudaMemcpyDeviceToHost, st));
    UMCG_CUDA(cudaStreamSynchronize(st));
    uint64_t ntok = h.c.count, ulen = h.c.aux[0];
    if (!h.c.err && h.c.aux[1]) {
        const bool fine = h.c.aux[2] < 64 * 1024;  // the probe's 64 tokens spanned < 64 KiB
        if (!parallel_tokens(d_stream, len, tok, sc, ctl, st, &ntok, &ulen, fine)) {
            // broken chain: the serial walk reports the reference's error
            k_token_walk<<<1, 32, 0, st>>>(d_stream, len, tok, tok_cap, ~0ull, ctl);
            UMCG_LAUNCHED();
            UMCG_CUDA(cudaMemcpyAsync(&h.c, ctl, sizeof(DevCtl), cudaMemcpyDeviceToHost, st));
            UMCG_CUDA(cudaStreamSynchronize(st));
            if (!h.c.err) fail(UMCG_INTERNAL_INCONSISTENCY, "parallel token parse disagrees with the serial walk");
        }
    }
    if (h.c.err) fail(UMCG_CORRUPT_PAYLOAD, h.c.err == DE_CORRUPT_TOKEN ? "unknown token in lossless stream"
                                            : h.c.err == DE_CORRUPT_VARINT ? "varint exceeds 64 bits"
                                                                           : "unexpected end of data");
    *ulen_out = ulen;
    if (ntok == 1 && (h.t.len >> 63)) return d_stream + h.t.src;  // single literal: decode in place
    if (!ulen) return d_stream;
    uint8_t* ub = sc.unpacked.as<uint8_t>(ulen);
    ProfScope ps("k_expand", st);
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
