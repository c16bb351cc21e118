// Escapes in parallel (codec.hpp:300-326 encode, 408-437 decode).
//
// The reference quantizes serially against the reconstructed predecessor; an
// element escapes when its quantum leaves the int32 range or its
// reconstruction misses the bound in floating point. It is then stored
// verbatim (index, value), coded as 0, and the chain continues from the exact
// value: recon_e = v_e. For lorenzo_1d this splits the chain into segments
// that restart at each escape, so the lattice reformulation of codes.cu holds
// per segment with the escape's value as the offset:
//   S_i = round((v_i - v_e) / bin)   (S_e = 0),    q_i = S_i - S_{i-1},
//   recon_i = fl(v_e + fl(S_i * bin)),
// with v_e = 0 before the first escape (the plain lattice). The element right
// after an escape is bit-exact with the reference (p = v_e exactly); later
// ones differ only by the serial chain's rounding drift, as without escapes.
//
// Which elements escape depends on the segment bases, i.e. on earlier
// escapes. seg_encode_1d iterates to the fixed point: round r evaluates every
// element against the escape set of round r-1 (base = value of the last
// escape before it, found by a max-scan of flagged indices). Element i's
// verdict depends only on the set restricted to [0, i), so a fixed point is
// the serial answer by induction, and every round fixes at least the first
// differing element; in practice two or three rounds.
//
// Decode: recon_i = fl(v_e + fl((K_i - K_e) * bin)) with K the plain prefix
// sum of the codes and e the last escape <= i (binary search in the sorted
// escape list); the escaped element's own code is read but ignored, as in
// the reference.
//
// N-D Lorenzo grids with escapes use the exact hyperplane wavefront
// (codes.cu). Elements whose reconstruction leaves the lattice regime
// (|S| >= 2^30 or |recon| >= 2^30 bin: FP spacing near the bin, the serial
// chain's drift no longer bounded by the rounding window) still go to the
// one-thread replica; they are counted (umcg_serial_fallbacks). Exempt are
// the element right after an escape (its prediction is v_e exactly, so it is
// bit-exact with the reference at any magnitude) and every element whose
// reconstruction fl(v_e + fl(S * bin)) involves no rounding (then the
// reference's chain reaches the same value exactly, e.g. runs of equal
// outliers coding q = 0).
#include <cmath>

#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>

#include "kernels.h"

namespace umcg {

namespace {

constexpr int ET = 256;
constexpr int EI = 8;
constexpr uint64_t ETILE = (uint64_t)ET * EI;
constexpr double kQLimit = 2147483647.0;  // codec.hpp:305
constexpr double kRegime = 1073741824.0;  // 2^30

struct MaxOp {
    __device__ int64_t operator()(int64_t a, int64_t b) const { return a > b ? a : b; }
};

// last flagged index per tile (-1: none)
__global__ void __launch_bounds__(ET) k_tile_last(const uint8_t* __restrict__ F, uint64_t n,
                                                 int64_t* __restrict__ tl) {
    using BR = cub::BlockReduce<int64_t, ET>;
    __shared__ typename BR::TempStorage tmp;
    const uint64_t b = blockIdx.x * ETILE + (uint64_t)threadIdx.x * EI;
    int64_t m = -1;
#pragma unroll
    for (int k = 0; k < EI; ++k)
        if (b + k < n && F[b + k]) m = (int64_t)(b + k);
    const int64_t t = BR(tmp).Reduce(m, MaxOp());
    if (threadIdx.x == 0) tl[blockIdx.x] = t;
}

// exclusive max-scan over tiles, one CTA (T = n / 2048 tiles)
__global__ void __launch_bounds__(1024) k_scan_last(int64_t* __restrict__ tl, uint64_t T) {
    using BS = cub::BlockScan<int64_t, 1024>;
    __shared__ typename BS::TempStorage tmp;
    const uint64_t per = (T + 1023) / 1024;
    const uint64_t t0 = threadIdx.x * per, t1 = min(T, t0 + per);
    int64_t local = -1;
    for (uint64_t t = t0; t < t1; ++t) local = tl[t] > local ? tl[t] : local;
    int64_t excl;
    BS(tmp).ExclusiveScan(local, excl, (int64_t)-1, MaxOp());
    for (uint64_t t = t0; t < t1; ++t) {
        const int64_t c = tl[t];
        tl[t] = excl;
        excl = c > excl ? c : excl;
    }
}

// base + S * bin with no rounding at all (exact product: fma residual 0;
// exact sum: TwoSum error 0). A segment whose reconstructions are all exact
// is the reference's chain bit for bit, at any magnitude (e.g. runs of equal
// huge values coding q = 0 after an escape).
__device__ __forceinline__ bool seg_exact(double base, double S, double bin) {
    const double pr = __dmul_rn(S, bin);
    if (__fma_rn(S, bin, -pr) != 0.0) return false;
    const double r = __dadd_rn(base, pr);
    const double bb = __dsub_rn(r, base);
    const double e = __dadd_rn(__dsub_rn(base, __dsub_rn(r, bb)), __dsub_rn(pr, bb));
    return e == 0.0;
}

__device__ __forceinline__ void flag_regime(DevCtl* ctl) {  // ctl->aux[6]: left the lattice regime
    if (ctl->aux[6] == 0) atomicExch(reinterpret_cast<unsigned long long*>(&ctl->aux[6]), 1ull);
}

// One fixed-point round: every element against the escape set Fin.
// Writes Fout, the codes (0 for escapes), counts changed verdicts
// (ctl->count) and flags the non-lattice regime (ctl->aux[6]).
__global__ void __launch_bounds__(ET) k_seg_eval(const double* __restrict__ v, uint64_t n,
                                                const uint8_t* __restrict__ Fin, const int64_t* __restrict__ carry,
                                                double bin, double inv, double tau, uint8_t* __restrict__ Fout,
                                                uint64_t* __restrict__ codes, DevCtl* ctl) {
    using BS = cub::BlockScan<int64_t, ET>;
    using BR = cub::BlockReduce<int, ET>;
    __shared__ typename BS::TempStorage ts;
    __shared__ typename BR::TempStorage tr;
    const uint64_t b = blockIdx.x * ETILE + (uint64_t)threadIdx.x * EI;
    uint8_t f[EI];
    int64_t mine = -1;
#pragma unroll
    for (int k = 0; k < EI; ++k) {
        f[k] = b + k < n ? Fin[b + k] : 0;
        if (f[k]) mine = (int64_t)(b + k);
    }
    int64_t excl;
    BS(ts).ExclusiveScan(mine, excl, (int64_t)-1, MaxOp());
    const int64_t c = carry[blockIdx.x];
    int64_t e = excl > c ? excl : c;  // last escape before this thread's first element
    int changed = 0, regime = 0;
    // predecessor of the first element: flag and value
    bool fprev = false;
    double vprev = 0.0;
    if (b < n && b > 0) {
        fprev = Fin[b - 1] != 0;
        vprev = v[b - 1];
    }
#pragma unroll
    for (int k = 0; k < EI; ++k) {
        const uint64_t i = b + k;
        if (i >= n) break;
        const double vi = v[i];
        const double base = e >= 0 ? v[e] : 0.0;
        // S_{i-1} relative to the same base (0 after an escape or at i = 0)
        double Sp = 0.0;
        if (i > 0 && !fprev) Sp = round_div(e >= 0 ? __dsub_rn(vprev, base) : vprev, bin, inv);
        const double r = e >= 0 ? __dsub_rn(vi, base) : vi;
        const double S = round_div(r, bin, inv);
        const double q = __dsub_rn(S, Sp);
        bool esc = !(fabs(q) <= kQLimit);
        double rec = 0.0;
        if (!esc) {
            rec = __dadd_rn(base, __dmul_rn(S, bin));
            esc = !(fabs(__dsub_rn(vi, rec)) <= tau);
        }
        if (esc) {
            codes[i] = 0;
        } else {
            // right after an escape the element is exact (p = v_e, no chain
            // drift yet), whatever its magnitude
            if (!(i > 0 && fprev) && (!(fabs(S) < kRegime) || !(fabs(rec) < __dmul_rn(kRegime, bin))) &&
                !seg_exact(base, S, bin))
                regime = 1;
            codes[i] = zz_enc((int64_t)q);
        }
        Fout[i] = esc ? 1 : 0;
        changed += (esc ? 1 : 0) != (f[k] ? 1 : 0);
        if (f[k]) e = (int64_t)i;
        fprev = f[k] != 0;
        vprev = vi;
    }
    const int tot = BR(tr).Sum(changed);
    if (threadIdx.x == 0 && tot) atomicAdd(reinterpret_cast<unsigned long long*>(&ctl->count), (unsigned long long)tot);
    if (regime) flag_regime(ctl);
}

// ---- stable compaction of flagged elements: (index, value) ---------------
__global__ void __launch_bounds__(ET) k_flag_count(const uint8_t* __restrict__ F, uint64_t n,
                                                  uint64_t* __restrict__ cnt) {
    using BR = cub::BlockReduce<int, ET>;
    __shared__ typename BR::TempStorage tmp;
    const uint64_t b = blockIdx.x * ETILE + (uint64_t)threadIdx.x * EI;
    int c = 0;
#pragma unroll
    for (int k = 0; k < EI; ++k) c += (b + k < n && F[b + k]) ? 1 : 0;
    const int t = BR(tmp).Sum(c);
    if (threadIdx.x == 0) cnt[blockIdx.x] = (uint64_t)t;
}

__global__ void __launch_bounds__(1024) k_scan_count(uint64_t* __restrict__ cnt, uint64_t T, uint64_t* total) {
    using BS = cub::BlockScan<uint64_t, 1024>;
    __shared__ typename BS::TempStorage tmp;
    const uint64_t per = (T + 1023) / 1024;
    const uint64_t t0 = threadIdx.x * per, t1 = min(T, t0 + per);
    uint64_t local = 0;
    for (uint64_t t = t0; t < t1; ++t) local += cnt[t];
    uint64_t excl, agg;
    BS(tmp).ExclusiveSum(local, excl, agg);
    for (uint64_t t = t0; t < t1; ++t) {
        const uint64_t c = cnt[t];
        cnt[t] = excl;
        excl += c;
    }
    if (threadIdx.x == 0) *total = agg;
}

// Each thread owns 8 consecutive elements: its flags form one byte mask, its
// rank inside the tile is a block scan (warp shuffles) of the masks' popc,
// so the records come out in ascending index order (codec.hpp:408-416).
__global__ void __launch_bounds__(ET) k_flag_write(const uint8_t* __restrict__ F, const double* __restrict__ v,
                                                  uint64_t n, const uint64_t* __restrict__ off,
                                                  uint64_t* __restrict__ idx, double* __restrict__ val) {
    using BS = cub::BlockScan<int, ET>;
    __shared__ typename BS::TempStorage tmp;
    const uint64_t b = blockIdx.x * ETILE + (uint64_t)threadIdx.x * EI;
    uint32_t bits = 0;
#pragma unroll
    for (int k = 0; k < EI; ++k)
        if (b + k < n && F[b + k]) bits |= 1u << k;
    int excl;
    BS(tmp).ExclusiveSum(__popc(bits), excl);
    uint64_t o = off[blockIdx.x] + (uint64_t)excl;
#pragma unroll
    for (int k = 0; k < EI; ++k)
        if (bits & (1u << k)) {
            idx[o] = b + k;
            val[o] = v[b + k];
            ++o;
        }
}

// ---- decode -----------------------------------------------------------------
// K_i = inclusive prefix of zz_dec(codes) (tile carries from k_tile_sums /
// k_scan_sums of codes.cu, recomputed here to keep the file self-contained)
__global__ void __launch_bounds__(ET) k_code_tile_sums(const uint64_t* __restrict__ codes, uint64_t n,
                                                      int64_t* __restrict__ sums) {
    using BR = cub::BlockReduce<int64_t, ET>;
    __shared__ typename BR::TempStorage tmp;
    const uint64_t b = blockIdx.x * ETILE + (uint64_t)threadIdx.x * EI;
    int64_t s = 0;
#pragma unroll
    for (int k = 0; k < EI; ++k)
        if (b + k < n) s += zz_dec(codes[b + k]);
    const int64_t t = BR(tmp).Sum(s);
    if (threadIdx.x == 0) sums[blockIdx.x] = t;
}

__global__ void __launch_bounds__(1024) k_scan_sums64(int64_t* __restrict__ sums, uint64_t T) {
    using BS = cub::BlockScan<int64_t, 1024>;
    __shared__ typename BS::TempStorage tmp;
    const uint64_t per = (T + 1023) / 1024;
    const uint64_t t0 = threadIdx.x * per, t1 = min(T, t0 + per);
    int64_t local = 0;
    for (uint64_t t = t0; t < t1; ++t) local += sums[t];
    int64_t excl;
    BS(tmp).ExclusiveSum(local, excl);
    for (uint64_t t = t0; t < t1; ++t) {
        const int64_t c = sums[t];
        sums[t] = excl;
        excl += c;
    }
}

__global__ void __launch_bounds__(ET) k_prefix_k(const uint64_t* __restrict__ codes, uint64_t n,
                                                const int64_t* __restrict__ carry, int64_t* __restrict__ K) {
    using BS = cub::BlockScan<int64_t, ET>;
    __shared__ typename BS::TempStorage tmp;
    const uint64_t b = blockIdx.x * ETILE + (uint64_t)threadIdx.x * EI;
    int64_t q[EI];
    int64_t s = 0;
#pragma unroll
    for (int k = 0; k < EI; ++k) {
        q[k] = b + k < n ? zz_dec(codes[b + k]) : 0;
        s += q[k];
    }
    int64_t excl;
    BS(tmp).ExclusiveSum(s, excl);
    int64_t acc = excl + carry[blockIdx.x];
#pragma unroll
    for (int k = 0; k < EI; ++k) {
        if (b + k >= n) break;
        acc += q[k];
        K[b + k] = acc;
    }
}

__global__ void k_gather_ke(const int64_t* __restrict__ K, const uint64_t* __restrict__ eidx, uint64_t ne,
                            int64_t* __restrict__ Ke) {
    const uint64_t e = blockIdx.x * 256ull + threadIdx.x;
    if (e < ne) Ke[e] = K[eidx[e]];
}

// recon_i from K_i, the last escape e <= i (binary search) and K_e; flags the
// non-lattice regime in ctl->aux[6].
__global__ void __launch_bounds__(ET) k_recon_seg(const int64_t* __restrict__ K, uint64_t n, double bin,
                                                 const uint64_t* __restrict__ eidx, const double* __restrict__ eval,
                                                 const int64_t* __restrict__ Ke, uint64_t ne,
                                                 double* __restrict__ out, DevCtl* ctl) {
    const uint64_t i = blockIdx.x * (uint64_t)ET + threadIdx.x;
    if (i >= n) return;
    // last e with eidx[e] <= i
    uint64_t lo = 0, hi = ne;  // answer in [lo, hi): count of eidx <= i
    while (lo < hi) {
        const uint64_t mid = (lo + hi) >> 1;
        if (eidx[mid] <= i) lo = mid + 1; else hi = mid;
    }
    double r;
    int64_t S;
    double base = 0.0;
    if (lo > 0) {
        const uint64_t e = lo - 1;
        if (eidx[e] == i) {
            out[i] = eval[e];
            return;
        }
        base = eval[e];
        S = K[i] - Ke[e];
        r = __dadd_rn(base, __dmul_rn((double)S, bin));
        if (eidx[e] + 1 == i) {  // first element after an escape: exact (p = v_e)
            out[i] = r;
            return;
        }
    } else {
        S = K[i];
        r = __dmul_rn((double)S, bin);
    }
    const double a = (double)(S < 0 ? -S : S);
    if ((!(a < kRegime) || !(fabs(r) < __dmul_rn(kRegime, bin))) && !seg_exact(base, (double)S, bin))
        flag_regime(ctl);
    out[i] = r;
}

inline unsigned tiles(uint64_t n) { return (unsigned)cdiv(n, ETILE); }

}  // namespace

size_t esc_scratch_bytes(uint64_t n) {
    const uint64_t T = cdiv(n ? n : 1, ETILE);
    return 2 * ((n + 255) & ~255ull) + (T + 1) * 8 * 2 + 256;
}

uint64_t compact_flags(const uint8_t* F, const double* v, uint64_t n, uint64_t* idx, double* val, uint64_t* tile_off,
                       uint64_t* d_total, uint64_t* h_total, cudaStream_t st) {
    if (!n) return 0;
    const unsigned T = tiles(n);
    k_flag_count<<<T, ET, 0, st>>>(F, n, tile_off);
    UMCG_LAUNCHED();
    k_scan_count<<<1, 1024, 0, st>>>(tile_off, T, d_total);
    UMCG_LAUNCHED();
    k_flag_write<<<T, ET, 0, st>>>(F, v, n, tile_off, idx, val);
    UMCG_LAUNCHED();
    UMCG_CUDA(cudaMemcpyAsync(h_total, d_total, 8, cudaMemcpyDeviceToHost, st));
    UMCG_CUDA(cudaStreamSynchronize(st));
    return *h_total;
}

// Returns false when the component must take the serial replica (the
// non-lattice regime, or no fixed point within the round limit).
bool seg_encode_1d(const double* v, uint64_t n, double tau, uint64_t* codes, uint64_t* esc_idx, double* esc_val,
                   void* scratch, DevCtl* ectl, DevCtl* hctl, uint64_t* n_esc, cudaStream_t st) {
    *n_esc = 0;
    if (!n) return true;
    const double bin = 2.0 * tau;
    if (!(tau > 0.0) || !std::isfinite(bin)) return false;
    const double inv = 1.0 / bin;
    const unsigned T = tiles(n);
    auto* base = static_cast<uint8_t*>(scratch);
    uint8_t* F[2] = {base, base + ((n + 255) & ~255ull)};
    auto* tl = reinterpret_cast<int64_t*>(base + 2 * ((n + 255) & ~255ull));
    auto* toff = reinterpret_cast<uint64_t*>(tl + T + 1);
    UMCG_CUDA(cudaMemsetAsync(F[0], 0, n, st));
    int cur = 0;
    constexpr int kRounds = 12;
    for (int r = 0; r < kRounds; ++r) {
        UMCG_CUDA(cudaMemsetAsync(ectl, 0, sizeof(DevCtl), st));
        k_tile_last<<<T, ET, 0, st>>>(F[cur], n, tl);
        UMCG_LAUNCHED();
        k_scan_last<<<1, 1024, 0, st>>>(tl, T);
        UMCG_LAUNCHED();
        k_seg_eval<<<T, ET, 0, st>>>(v, n, F[cur], tl, bin, inv, tau, F[cur ^ 1], codes, ectl);
        UMCG_LAUNCHED();
        UMCG_CUDA(cudaMemcpyAsync(hctl, ectl, sizeof(DevCtl), cudaMemcpyDeviceToHost, st));
        UMCG_CUDA(cudaStreamSynchronize(st));
        const bool converged = hctl->count == 0;
        const bool regime = hctl->aux[6] != 0;
        cur ^= 1;
        if (converged) {
            if (regime) return false;
            // F[cur] == F[cur ^ 1]: the codes written this round are the final ones
            *n_esc = compact_flags(F[cur], v, n, esc_idx, esc_val, toff, &ectl->aux[0], &hctl->aux[0], st);
            return true;
        }
    }
    return false;
}

// Decode of a 1-D (lorenzo_1d) component with escapes. Returns false when the
// reconstruction leaves the lattice regime (the caller replays serially).
bool seg_decode_1d(const uint64_t* codes, uint64_t n, double tau, const uint64_t* esc_idx, const double* esc_val,
                   uint64_t n_esc, int64_t* K, int64_t* scratch, double* out, DevCtl* ectl, DevCtl* hctl,
                   cudaStream_t st) {
    if (!n) return true;
    const double bin = 2.0 * tau;
    if (!(tau > 0.0) || !std::isfinite(bin)) return false;
    const unsigned T = tiles(n);
    int64_t* sums = scratch;           // [T]
    int64_t* Ke = scratch + T + 1;     // [n_esc]
    UMCG_CUDA(cudaMemsetAsync(ectl, 0, sizeof(DevCtl), st));
    k_code_tile_sums<<<T, ET, 0, st>>>(codes, n, sums);
    UMCG_LAUNCHED();
    k_scan_sums64<<<1, 1024, 0, st>>>(sums, T);
    UMCG_LAUNCHED();
    k_prefix_k<<<T, ET, 0, st>>>(codes, n, sums, K);
    UMCG_LAUNCHED();
    if (n_esc) {
        k_gather_ke<<<(unsigned)cdiv(n_esc, 256), 256, 0, st>>>(K, esc_idx, n_esc, Ke);
        UMCG_LAUNCHED();
    }
    k_recon_seg<<<(unsigned)cdiv(n, ET), ET, 0, st>>>(K, n, bin, esc_idx, esc_val, Ke, n_esc, out, ectl);
    UMCG_LAUNCHED();
    UMCG_CUDA(cudaMemcpyAsync(hctl, ectl, sizeof(DevCtl), cudaMemcpyDeviceToHost, st));
    UMCG_CUDA(cudaStreamSynchronize(st));
    return hctl->aux[6] == 0;
}

}  // namespace umcg
