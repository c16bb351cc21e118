// Quantization codes and reconstruction on sm_100a.
//
// Fast path = lattice reformulation of the reference predictor-quantizer
// (codec.hpp:300-326). With bin = 2*tau', the serial reference produces
// recon_i ~= bin*K_i with K_i = round(v_i / bin); its code is then
// q_i = K_i - sum(+-K_nbr) over the same Lorenzo stencil
// (codec.hpp:61-80). Every element is independent, so codes are computed in
// parallel; decode is an exact integer (N-D) prefix sum and recon =
// fl(K * bin). Codes equal the reference's except where a value sits within
// the serial chain's rounding drift of a bin boundary.
//
// Whenever the lattice could disagree with the reference beyond that window
// (an escape would be needed, |K| large enough that FP spacing approaches the
// bin, non-finite bins) the component is flagged and re-encoded by
// serial_encode: a one-thread exact replica of the reference loop. That path
// is correct by construction and only exists for pathological inputs.
//
// All files compile with --fmad=false: no contraction, IEEE division and
// round-half-away-from-zero, exactly like the reference build
// (-ffp-contract=off, proj/CMakeLists.txt:16-17).
#include <cstdlib>

#include <cooperative_groups.h>
#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>

#include "kernels.h"
#include "multilinear.cuh"

namespace umcg {

NdShape make_shape(int D, const uint64_t* dims) {
    NdShape s;
    s.D = D;
    for (int d = 0; d < 8; ++d) { s.dims[d] = d < D ? dims[d] : 1; s.strides[d] = 1; }
    for (int d = D - 1; d >= 1; --d) s.strides[d - 1] = s.strides[d] * s.dims[d];  // codec.hpp:87-92
    return s;
}

namespace {

constexpr int THREADS = 256;
constexpr double kQLimit = 2147483647.0;  // codec.hpp:305

// |K| bound under which the lattice codes cannot overflow the int32 code
// range for a stencil of 2^D terms (|q| <= 2^D * max|K| < 2^31 - 1).
__host__ __device__ inline double k_limit(int pred, int D) {
    if (pred == 0) return kQLimit;
    if (pred == 1) return 1073741824.0;          // 2^30
    return ldexp(1.0, 31 - (D < 1 ? 1 : D));     // 2^(31-D)
}

__device__ __forceinline__ void flag_serial(DevCtl* ctl, int comp) {
    if (ctl->need_serial[comp] == 0) atomicExch(&ctl->need_serial[comp], 1);
}

// Lattice index of v with the escape / regime checks of codec.hpp:305-314.
__device__ __forceinline__ double lattice_k(double v, double bin, double tau, double lim,
                                            DevCtl* ctl, int comp) {
    double err;
    const double K = lattice_round(v, bin, ctl->inv_bin[comp], tau, &err);
    const bool bad = !(fabs(K) < lim) || !(err <= tau);
    if (bad) flag_serial(ctl, comp);
    return K;
}

__device__ __forceinline__ void multi_index(uint64_t lin, const NdShape& sh, uint64_t* idx) {
    for (int d = sh.D - 1; d >= 0; --d) {
        idx[d] = lin % sh.dims[d];
        lin /= sh.dims[d];
    }
}

// ---- lossy: none / 1-D over an array ---------------------------------------
__global__ void __launch_bounds__(THREADS) k_codes_1d(const double* __restrict__ v, uint64_t n, int pred,
                                                     DevCtl* ctl, int comp, uint32_t* __restrict__ codes) {
    const uint64_t i = blockIdx.x * (uint64_t)THREADS + threadIdx.x;
    if (i >= n) return;
    const double bin = ctl->bin[comp], tau = ctl->tau_c[comp];
    const double lim = k_limit(pred, 1);
    const double K = lattice_k(v[i], bin, tau, lim, ctl, comp);
    double Kp = 0.0;
    if (pred == 1 && i > 0) Kp = round_div(v[i - 1], bin, ctl->inv_bin[comp]);
    const int64_t q = (int64_t)K - (int64_t)Kp;
    codes[i] = (uint32_t)zz_enc(q);
}

// ---- lossy N-D: K grid, then the integer Lorenzo stencil --------------------
__global__ void __launch_bounds__(THREADS) k_lattice_nd(const double* __restrict__ v, uint64_t n, int D,
                                                       DevCtl* ctl, int comp, int32_t* __restrict__ K) {
    const uint64_t i = blockIdx.x * (uint64_t)THREADS + threadIdx.x;
    if (i >= n) return;
    const double bin = ctl->bin[comp], tau = ctl->tau_c[comp];
    K[i] = (int32_t)lattice_k(v[i], bin, tau, k_limit(2, D), ctl, comp);
}

__global__ void __launch_bounds__(THREADS) k_stencil_nd(const int32_t* __restrict__ K, uint64_t n,
                                                       NdShape sh, uint32_t* __restrict__ codes) {
    const uint64_t i = blockIdx.x * (uint64_t)THREADS + threadIdx.x;
    if (i >= n) return;
    uint64_t idx[8];
    multi_index(i, sh, idx);
    int64_t pred = 0;
    for (unsigned mask = 1; mask < (1u << sh.D); ++mask) {  // lorenzo_predict, codec.hpp:66-78
        uint64_t off = 0;
        bool ok = true;
        for (int d = 0; d < sh.D; ++d)
            if ((mask >> d) & 1u) {
                if (idx[d] == 0) { ok = false; break; }
                off += sh.strides[d];
            }
        if (!ok) continue;
        const int64_t term = K[i - off];
        pred += (__popc(mask) & 1) ? term : -term;
    }
    codes[i] = (uint32_t)zz_enc((int64_t)K[i] - pred);
}

// Integer Lorenzo stencil for D = 2 / 3 with the grid laid out by axis:
// blockIdx.x spans the fastest axis, blockIdx.y / z the others (no 64-bit
// division per element). Missing neighbours (index -1) contribute 0, which
// is exactly the reference's skipped masks (codec.hpp:70-75).
__global__ void __launch_bounds__(THREADS) k_stencil_3d(const int32_t* __restrict__ K, uint64_t d0, uint64_t d1,
                                                       uint64_t d2, uint32_t* __restrict__ codes, const DevCtl* ctl) {
    if (pass_skipped(ctl)) return;
    const uint64_t k = blockIdx.x * (uint64_t)THREADS + threadIdx.x;
    if (k >= d2) return;
    const uint64_t j = blockIdx.y, i = blockIdx.z;
    const uint64_t s1 = d2, s0 = d1 * d2;
    const uint64_t c = i * s0 + j * s1 + k;
    auto at = [&](bool ok, uint64_t off) -> int64_t { return ok ? (int64_t)K[c - off] : 0; };
    const bool ai = i > 0, aj = j > 0, ak = k > 0;
    const int64_t pred = at(ak, 1) + at(aj, s1) + at(ai, s0) - at(aj && ak, s1 + 1) - at(ai && ak, s0 + 1) -
                         at(ai && aj, s0 + s1) + at(ai && aj && ak, s0 + s1 + 1);
    codes[c] = (uint32_t)zz_enc((int64_t)K[c] - pred);
    (void)d0;
}

// ---- lossless XOR codes (codec.hpp:276-294) --------------------------------
__device__ __forceinline__ double lorenzo_fp(const double* __restrict__ v, uint64_t i, const NdShape& sh) {
    uint64_t idx[8];
    multi_index(i, sh, idx);
    double pred = 0.0;
    for (unsigned mask = 1; mask < (1u << sh.D); ++mask) {
        uint64_t off = 0;
        bool ok = true;
        for (int d = 0; d < sh.D; ++d)
            if ((mask >> d) & 1u) {
                if (idx[d] == 0) { ok = false; break; }
                off += sh.strides[d];
            }
        if (!ok) continue;
        const double term = v[i - off];
        pred = (__popc(mask) & 1) ? __dadd_rn(pred, term) : __dsub_rn(pred, term);
    }
    return pred;
}

__global__ void __launch_bounds__(THREADS) k_lossless(const double* __restrict__ v, uint64_t n, int pred,
                                                     NdShape sh, uint64_t* __restrict__ codes) {
    const uint64_t i = blockIdx.x * (uint64_t)THREADS + threadIdx.x;
    if (i >= n) return;
    double p = 0.0;
    if (pred == 1) p = i ? v[i - 1] : 0.0;
    else if (pred == 2) p = lorenzo_fp(v, i, sh);
    codes[i] = (uint64_t)__double_as_longlong(v[i]) ^ (uint64_t)__double_as_longlong(p);
}

// ---- residual component -----------------------------------------------------
// detail::multilinear_at (interp.hpp:97-132), same operation order.
// multilinear_at / axis_upper_bound: multilinear.cuh
__device__ __forceinline__ double multilinear_at(const ResidualSrc& s, const double* __restrict__ p) {
    return multilinear_eval(s.axes, s.axis_off, s.shape, s.D, s.x1, p, s.inv_cell, s.scale);
}

__device__ __forceinline__ double load_x(const ResidualSrc& s, uint64_t i) {
    return s.x_f32 ? (double)static_cast<const float*>(s.x)[i] : static_cast<const double*>(s.x)[i];
}

__device__ __forceinline__ double g_at(const ResidualSrc& s, uint64_t i) {
    if (s.g_kind == 0) return s.x1[s.node[i]];
    return multilinear_at(s, s.coords + i * (uint64_t)s.D);
}

// compute_residuals (interp.hpp:161-170): one IEEE subtract.
__device__ __forceinline__ double residual_at(const ResidualSrc& s, uint64_t i) {
    return __dsub_rn(load_x(s, i), g_at(s, i));
}

constexpr int RES_ITEMS = 4;
__global__ void __launch_bounds__(THREADS) k_codes_residual(ResidualSrc s, uint64_t n, DevCtl* ctl,
                                                           uint32_t* __restrict__ codes) {
    const uint64_t i0 = (blockIdx.x * (uint64_t)THREADS + threadIdx.x) * RES_ITEMS;
    if (i0 >= n) return;
    const double bin = ctl->bin[1], tau = ctl->tau_c[1];
    const double lim = k_limit(1, 1);
    double Kp = i0 ? round_div(residual_at(s, i0 - 1), bin, ctl->inv_bin[1]) : 0.0;
#pragma unroll
    for (int k = 0; k < RES_ITEMS; ++k) {
        const uint64_t i = i0 + k;
        if (i >= n) break;
        const double K = lattice_k(residual_at(s, i), bin, tau, lim, ctl, 1);
        codes[i] = (uint32_t)zz_enc((int64_t)K - (int64_t)Kp);
        Kp = K;
    }
}

__global__ void __launch_bounds__(THREADS) k_lossless_residual(ResidualSrc s, uint64_t n,
                                                              uint64_t* __restrict__ codes) {
    const uint64_t i = blockIdx.x * (uint64_t)THREADS + threadIdx.x;
    if (i >= n) return;
    const double r = residual_at(s, i);
    const double p = i ? residual_at(s, i - 1) : 0.0;
    codes[i] = (uint64_t)__double_as_longlong(r) ^ (uint64_t)__double_as_longlong(p);
}

__global__ void __launch_bounds__(THREADS) k_materialize_residual(ResidualSrc s, uint64_t n,
                                                                 double* __restrict__ out) {
    const uint64_t i = blockIdx.x * (uint64_t)THREADS + threadIdx.x;
    if (i < n) out[i] = residual_at(s, i);
}

__global__ void __launch_bounds__(THREADS) k_recompose(ResidualSrc s, uint64_t n, double* __restrict__ io) {
    const uint64_t i = blockIdx.x * (uint64_t)THREADS + threadIdx.x;
    if (i < n) io[i] = __dadd_rn(g_at(s, i), io[i]);  // approx[i] + x2[i], pipeline.hpp:208
}

// ---- exact serial replicas (one thread) -------------------------------------
struct SerialPred {
    NdShape sh;
    int pred;
    uint64_t idx[8];
    __device__ void init(const NdShape& s, int p) {
        sh = s;
        pred = p;
        for (int d = 0; d < 8; ++d) idx[d] = 0;
    }
    __device__ double predict(const double* recon, uint64_t lin) const {  // codec.hpp:94-102
        if (pred == 0) return 0.0;
        if (pred == 1) return lin == 0 ? 0.0 : recon[lin - 1];
        double p = 0.0;
        for (unsigned mask = 1; mask < (1u << sh.D); ++mask) {
            uint64_t off = 0;
            bool ok = true;
            for (int d = 0; d < sh.D; ++d)
                if ((mask >> d) & 1u) {
                    if (idx[d] == 0) { ok = false; break; }
                    off += sh.strides[d];
                }
            if (!ok) continue;
            const double term = recon[lin - off];
            p = (__popc(mask) & 1) ? __dadd_rn(p, term) : __dsub_rn(p, term);
        }
        return p;
    }
    __device__ void advance() {  // codec.hpp:104-109
        for (int d = sh.D - 1; d >= 0; --d) {
            if (++idx[d] < sh.dims[d]) return;
            idx[d] = 0;
        }
    }
};

__global__ void k_serial_encode(const double* __restrict__ v, uint64_t n, int pred, NdShape sh,
                                double tau, uint64_t* __restrict__ codes, double* __restrict__ recon,
                                uint64_t* __restrict__ esc_idx, double* __restrict__ esc_val,
                                DevCtl* ctl, int comp) {
    if (threadIdx.x | blockIdx.x) return;
    SerialPred ps;
    ps.init(sh, pred);
    const double bin = __dmul_rn(2.0, tau);
    uint64_t ne = 0;
    for (uint64_t i = 0; i < n; ++i) {
        const double p = ps.predict(recon, i);
        if (tau == 0.0) {
            codes[i] = (uint64_t)__double_as_longlong(v[i]) ^ (uint64_t)__double_as_longlong(p);
            recon[i] = v[i];
        } else {
            const double qd = round(__ddiv_rn(__dsub_rn(v[i], p), bin));
            bool escape = !(fabs(qd) <= kQLimit);
            double r = 0.0;
            if (!escape) {
                r = __dadd_rn(p, __dmul_rn(qd, bin));
                escape = !(fabs(__dsub_rn(v[i], r)) <= tau);
            }
            if (escape) {
                esc_idx[ne] = i;
                esc_val[ne] = v[i];
                ++ne;
                codes[i] = 0;
                recon[i] = v[i];
            } else {
                codes[i] = zz_enc((int64_t)qd);
                recon[i] = r;
            }
        }
        ps.advance();
    }
    ctl->n_esc[comp] = ne;
}

__global__ void k_serial_decode(const uint64_t* __restrict__ codes, uint64_t n, int pred, NdShape sh,
                                double tau, const uint64_t* __restrict__ esc_idx,
                                const double* __restrict__ esc_val, uint64_t n_esc,
                                double* __restrict__ recon) {
    if (threadIdx.x | blockIdx.x) return;
    SerialPred ps;
    ps.init(sh, pred);
    const double bin = __dmul_rn(2.0, tau);
    uint64_t next = 0;
    for (uint64_t i = 0; i < n; ++i) {
        const double p = ps.predict(recon, i);
        const uint64_t z = codes[i];
        if (tau == 0.0) {
            recon[i] = __longlong_as_double((long long)(z ^ (uint64_t)__double_as_longlong(p)));
        } else if (next < n_esc && esc_idx[next] == i) {
            recon[i] = esc_val[next++];
        } else {
            recon[i] = __dadd_rn(p, __dmul_rn((double)zz_dec(z), bin));
        }
        ps.advance();
    }
}

// ---- decode: lattice reconstruction ----------------------------------------
// 1-D inclusive scan of zz_dec(codes) in three passes (tile sums, one-CTA
// scan of tile sums, tile scan + epilogue).
constexpr int SC_ITEMS = 8;
constexpr uint64_t SC_TILE = THREADS * SC_ITEMS;

__global__ void __launch_bounds__(THREADS) k_tile_sums(const uint64_t* __restrict__ codes, uint64_t n,
                                                      int64_t* __restrict__ sums) {
    using BR = cub::BlockReduce<int64_t, THREADS>;
    __shared__ typename BR::TempStorage tmp;
    const uint64_t b = blockIdx.x * SC_TILE + (uint64_t)threadIdx.x * SC_ITEMS;
    int64_t s = 0;
    for (int k = 0; k < SC_ITEMS; ++k)
        if (b + k < n) s += zz_dec(codes[b + k]);
    const int64_t t = BR(tmp).Sum(s);
    if (threadIdx.x == 0) sums[blockIdx.x] = t;
}

__global__ void __launch_bounds__(1024) k_scan_sums(int64_t* __restrict__ sums, uint64_t T) {
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

__device__ __forceinline__ void note_k(DevCtl* ctl, int64_t K) {
    const unsigned long long a = (unsigned long long)(K < 0 ? -K : K);
    if (a > ctl->max_abs_k[0]) atomicMax(&ctl->max_abs_k[0], a);
}

__global__ void __launch_bounds__(THREADS) k_tile_recon_1d(const uint64_t* __restrict__ codes, uint64_t n,
                                                          const int64_t* __restrict__ carry, double bin,
                                                          double* __restrict__ out, DevCtl* ctl) {
    using BS = cub::BlockScan<int64_t, THREADS>;
    __shared__ typename BS::TempStorage tmp;
    const uint64_t b = blockIdx.x * SC_TILE + (uint64_t)threadIdx.x * SC_ITEMS;
    int64_t q[SC_ITEMS];
    int64_t s = 0;
#pragma unroll
    for (int k = 0; k < SC_ITEMS; ++k) {
        q[k] = b + k < n ? zz_dec(codes[b + k]) : 0;
        s += q[k];
    }
    int64_t excl;
    BS(tmp).ExclusiveSum(s, excl);
    int64_t K = excl + carry[blockIdx.x];
    int64_t kmax = 0;
#pragma unroll
    for (int k = 0; k < SC_ITEMS; ++k) {
        if (b + k >= n) break;
        K += q[k];
        out[b + k] = __dmul_rn((double)K, bin);
        const int64_t a = K < 0 ? -K : K;
        kmax = a > kmax ? a : kmax;
    }
    note_k(ctl, kmax);
}

__global__ void __launch_bounds__(THREADS) k_recon_none(const uint64_t* __restrict__ codes, uint64_t n,
                                                       double bin, double* __restrict__ out) {
    const uint64_t i = blockIdx.x * (uint64_t)THREADS + threadIdx.x;
    if (i < n) out[i] = __dmul_rn((double)zz_dec(codes[i]), bin);
}

__global__ void __launch_bounds__(THREADS) k_zz_to_k(const uint64_t* __restrict__ codes, uint64_t n,
                                                    int64_t* __restrict__ K) {
    const uint64_t i = blockIdx.x * (uint64_t)THREADS + threadIdx.x;
    if (i < n) K[i] = zz_dec(codes[i]);
}

// Inclusive prefix sum along axis d of an N-D int64 array, one thread per
// line (lines along the last axis are handled the same way; adequate for the
// grid component, which is ~n/8 of the residual component).
__global__ void __launch_bounds__(THREADS) k_axis_scan(int64_t* __restrict__ K, NdShape sh, int d,
                                                      uint64_t n_lines) {
    const uint64_t line = blockIdx.x * (uint64_t)THREADS + threadIdx.x;
    if (line >= n_lines) return;
    const uint64_t stride = sh.strides[d], len = sh.dims[d];
    // line -> base offset: decompose over all axes except d
    const uint64_t inner = stride;             // product of dims after d
    const uint64_t outer_i = line / inner, inner_i = line % inner;
    const uint64_t base = outer_i * (len * stride) + inner_i;
    int64_t acc = 0;
    for (uint64_t k = 0; k < len; ++k) {
        acc += K[base + k * stride];
        K[base + k * stride] = acc;
    }
}

__global__ void __launch_bounds__(THREADS) k_k_to_recon(const int64_t* __restrict__ K, uint64_t n, double bin,
                                                       double* __restrict__ out, DevCtl* ctl) {
    const uint64_t i = blockIdx.x * (uint64_t)THREADS + threadIdx.x;
    int64_t a = 0;
    if (i < n) {
        out[i] = __dmul_rn((double)K[i], bin);
        a = K[i] < 0 ? -K[i] : K[i];
    }
    using BR = cub::BlockReduce<int64_t, THREADS>;
    __shared__ typename BR::TempStorage tmp;
    const int64_t m = BR(tmp).Reduce(a, cub::Max());
    if (threadIdx.x == 0) note_k(ctl, m);
}

// lossless 1-D: recon bits = XOR prefix of codes (codec.hpp:429-430 with
// pred = previous exact value).
__global__ void __launch_bounds__(THREADS) k_tile_xor(const uint64_t* __restrict__ codes, uint64_t n,
                                                     uint64_t* __restrict__ sums) {
    using BR = cub::BlockReduce<uint64_t, THREADS>;
    __shared__ typename BR::TempStorage tmp;
    const uint64_t b = blockIdx.x * SC_TILE + (uint64_t)threadIdx.x * SC_ITEMS;
    uint64_t s = 0;
    for (int k = 0; k < SC_ITEMS; ++k)
        if (b + k < n) s ^= codes[b + k];
    struct X { __device__ uint64_t operator()(uint64_t a, uint64_t b) const { return a ^ b; } };
    const uint64_t t = BR(tmp).Reduce(s, X());
    if (threadIdx.x == 0) sums[blockIdx.x] = t;
}

__global__ void __launch_bounds__(1024) k_scan_xor(uint64_t* __restrict__ sums, uint64_t T) {
    using BS = cub::BlockScan<uint64_t, 1024>;
    __shared__ typename BS::TempStorage tmp;
    struct X { __device__ uint64_t operator()(uint64_t a, uint64_t b) const { return a ^ b; } };
    const uint64_t per = (T + 1023) / 1024;
    const uint64_t t0 = threadIdx.x * per, t1 = min(T, t0 + per);
    uint64_t local = 0;
    for (uint64_t t = t0; t < t1; ++t) local ^= sums[t];
    uint64_t excl;
    BS(tmp).ExclusiveScan(local, excl, 0ull, X());
    for (uint64_t t = t0; t < t1; ++t) {
        const uint64_t c = sums[t];
        sums[t] = excl;
        excl ^= c;
    }
}

__global__ void __launch_bounds__(THREADS) k_tile_recon_xor(const uint64_t* __restrict__ codes, uint64_t n,
                                                           const uint64_t* __restrict__ carry,
                                                           double* __restrict__ out) {
    using BS = cub::BlockScan<uint64_t, THREADS>;
    __shared__ typename BS::TempStorage tmp;
    struct X { __device__ uint64_t operator()(uint64_t a, uint64_t b) const { return a ^ b; } };
    const uint64_t b = blockIdx.x * SC_TILE + (uint64_t)threadIdx.x * SC_ITEMS;
    uint64_t z[SC_ITEMS];
    uint64_t s = 0;
#pragma unroll
    for (int k = 0; k < SC_ITEMS; ++k) {
        z[k] = b + k < n ? codes[b + k] : 0;
        s ^= z[k];
    }
    uint64_t excl;
    BS(tmp).ExclusiveScan(s, excl, 0ull, X());
    uint64_t acc = excl ^ carry[blockIdx.x];
#pragma unroll
    for (int k = 0; k < SC_ITEMS; ++k) {
        if (b + k >= n) break;
        acc ^= z[k];
        out[b + k] = __longlong_as_double((long long)acc);
    }
}

__global__ void __launch_bounds__(THREADS) k_recon_lossless_none(const uint64_t* __restrict__ codes,
                                                                uint64_t n, double* __restrict__ out) {
    const uint64_t i = blockIdx.x * (uint64_t)THREADS + threadIdx.x;
    if (i < n) out[i] = __longlong_as_double((long long)codes[i]);
}

inline unsigned blocks(uint64_t n, uint64_t per = THREADS) { return (unsigned)cdiv(n, per); }

}  // namespace

void codes_lossy_values(const double* v, uint64_t n, int pred, const NdShape& sh, DevCtl* ctl, int comp,
                        uint32_t* codes, int32_t* kbuf, cudaStream_t st, bool k_ready) {
    if (!n) return;
    if (pred == 2 && sh.D > 1) {
        if (!k_ready) {  // else kbuf holds the lattice indices already (fused into the bucket kernels)
            k_lattice_nd<<<blocks(n), THREADS, 0, st>>>(v, n, sh.D, ctl, comp, kbuf);
            UMCG_LAUNCHED();
        }
        if ((sh.D == 2 || sh.D == 3) && sh.dims[0] < 65536 && (sh.D == 2 || sh.dims[1] < 65536)) {
            const uint64_t d0 = sh.D == 3 ? sh.dims[0] : 1, d1 = sh.D == 3 ? sh.dims[1] : sh.dims[0];
            const uint64_t d2 = sh.dims[sh.D - 1];
            dim3 g((unsigned)cdiv(d2, THREADS), (unsigned)d1, (unsigned)d0);
            k_stencil_3d<<<g, THREADS, 0, st>>>(kbuf, d0, d1, d2, codes, ctl);
        } else {
            k_stencil_nd<<<blocks(n), THREADS, 0, st>>>(kbuf, n, sh, codes);
        }
        UMCG_LAUNCHED();
    } else {
        // lorenzo_nd over a single axis is lorenzo_1d
        k_codes_1d<<<blocks(n), THREADS, 0, st>>>(v, n, pred == 0 ? 0 : 1, ctl, comp, codes);
        UMCG_LAUNCHED();
    }
}

void codes_lossless_values(const double* v, uint64_t n, int pred, const NdShape& sh, uint64_t* codes,
                           cudaStream_t st) {
    if (!n) return;
    k_lossless<<<blocks(n), THREADS, 0, st>>>(v, n, pred, sh, codes);
    UMCG_LAUNCHED();
}

void codes_lossy_residual(const ResidualSrc& src, uint64_t n, DevCtl* ctl, uint32_t* codes, cudaStream_t st) {
    if (!n) return;
    k_codes_residual<<<blocks(n, (uint64_t)THREADS * RES_ITEMS), THREADS, 0, st>>>(src, n, ctl, codes);
    UMCG_LAUNCHED();
}

void codes_lossless_residual(const ResidualSrc& src, uint64_t n, uint64_t* codes, cudaStream_t st) {
    if (!n) return;
    k_lossless_residual<<<blocks(n), THREADS, 0, st>>>(src, n, codes);
    UMCG_LAUNCHED();
}

void materialize_residual(const ResidualSrc& src, uint64_t n, double* out, cudaStream_t st) {
    if (!n) return;
    k_materialize_residual<<<blocks(n), THREADS, 0, st>>>(src, n, out);
    UMCG_LAUNCHED();
}

void recompose(const ResidualSrc& src, uint64_t n, double* inout, cudaStream_t st) {
    if (!n) return;
    k_recompose<<<blocks(n), THREADS, 0, st>>>(src, n, inout);
    UMCG_LAUNCHED();
}

void serial_encode(const double* v, uint64_t n, int pred, const NdShape& sh, double tau, uint64_t* codes,
                   double* recon_scratch, uint64_t* esc_idx, double* esc_val, DevCtl* ctl, int comp,
                   cudaStream_t st) {
    g_serial_fallbacks.fetch_add(1);
    k_serial_encode<<<1, 32, 0, st>>>(v, n, pred, sh, tau, codes, recon_scratch, esc_idx, esc_val, ctl, comp);
    UMCG_LAUNCHED();
}

// N-D lossless decode (codec.hpp:429-430 with lorenzo_nd): recon_i =
// bits^-1(code_i XOR bits(pred_i)) where pred_i is the floating-point Lorenzo
// prediction from already reconstructed neighbours, so the dependency is
// real. Every neighbour of (i, j[, k]) lies on an earlier hyperplane
// i + j [+ k] = s, so the hyperplanes are decoded in order, each fully in
// parallel with the reference's exact prediction (lorenzo_fp, same operation
// order). D = 2, 3; other ranks use the serial replica.
namespace {
__global__ void __launch_bounds__(THREADS) k_lossless_plane(const uint64_t* __restrict__ codes, NdShape sh,
                                                           uint64_t s, uint64_t i_lo, uint64_t cnt,
                                                           double* __restrict__ recon) {
    const uint64_t t = blockIdx.x * (uint64_t)THREADS + threadIdx.x;
    if (t >= cnt) return;
    uint64_t lin;
    if (sh.D == 2) {
        const uint64_t i = i_lo + t, j = s - i;
        lin = i * sh.dims[1] + j;
    } else {
        const uint64_t i = i_lo + t / sh.dims[1], j = t % sh.dims[1];
        if (i + j > s) return;
        const uint64_t k = s - i - j;
        if (k >= sh.dims[2]) return;
        lin = (i * sh.dims[1] + j) * sh.dims[2] + k;
    }
    const double p = lorenzo_fp(recon, lin, sh);
    recon[lin] = __longlong_as_double((long long)(codes[lin] ^ (uint64_t)__double_as_longlong(p)));
}

// Lossy N-D Lorenzo with escapes, exact: the reference loop (codec.hpp:300-326
// encode, 422-437 decode) per hyperplane, same operations in the same order.
__global__ void __launch_bounds__(THREADS) k_wave_enc(const double* __restrict__ v, NdShape sh, uint64_t s,
                                                     uint64_t i_lo, uint64_t cnt, double tau, double bin,
                                                     double* __restrict__ recon, uint64_t* __restrict__ codes,
                                                     uint8_t* __restrict__ F) {
    const uint64_t t = blockIdx.x * (uint64_t)THREADS + threadIdx.x;
    if (t >= cnt) return;
    uint64_t lin;
    if (sh.D == 2) {
        const uint64_t i = i_lo + t, j = s - i;
        lin = i * sh.dims[1] + j;
    } else {
        const uint64_t i = i_lo + t / sh.dims[1], j = t % sh.dims[1];
        if (i + j > s) return;
        const uint64_t k = s - i - j;
        if (k >= sh.dims[2]) return;
        lin = (i * sh.dims[1] + j) * sh.dims[2] + k;
    }
    const double p = lorenzo_fp(recon, lin, sh);
    const double x = v[lin];
    const double qd = round(__ddiv_rn(__dsub_rn(x, p), bin));
    bool escape = !(fabs(qd) <= kQLimit);
    double r = 0.0;
    if (!escape) {
        r = __dadd_rn(p, __dmul_rn(qd, bin));
        escape = !(fabs(__dsub_rn(x, r)) <= tau);
    }
    F[lin] = escape ? 1 : 0;
    codes[lin] = escape ? 0 : zz_enc((int64_t)qd);
    recon[lin] = escape ? x : r;
}

__global__ void __launch_bounds__(THREADS) k_wave_dec(const uint64_t* __restrict__ codes, NdShape sh, uint64_t s,
                                                     uint64_t i_lo, uint64_t cnt, double bin,
                                                     const int32_t* __restrict__ eslot,
                                                     const double* __restrict__ eval, double* __restrict__ recon) {
    const uint64_t t = blockIdx.x * (uint64_t)THREADS + threadIdx.x;
    if (t >= cnt) return;
    uint64_t lin;
    if (sh.D == 2) {
        const uint64_t i = i_lo + t, j = s - i;
        lin = i * sh.dims[1] + j;
    } else {
        const uint64_t i = i_lo + t / sh.dims[1], j = t % sh.dims[1];
        if (i + j > s) return;
        const uint64_t k = s - i - j;
        if (k >= sh.dims[2]) return;
        lin = (i * sh.dims[1] + j) * sh.dims[2] + k;
    }
    const double p = lorenzo_fp(recon, lin, sh);
    const int32_t e = eslot[lin];
    recon[lin] = e >= 0 ? eval[e] : __dadd_rn(p, __dmul_rn((double)zz_dec(codes[lin]), bin));
}

__global__ void k_esc_slots(const uint64_t* __restrict__ eidx, uint64_t ne, int32_t* __restrict__ eslot) {
    const uint64_t e = blockIdx.x * 256ull + threadIdx.x;
    if (e < ne) eslot[eidx[e]] = (int32_t)e;
}

// lorenzo_predict (codec.hpp:61-80) at node (i, j, k) of a 2-/3-D grid with
// the neighbours addressed directly: masks 1..2^D-1 in order, bit d = axis d
// (axis 0 slowest), a mask skipped when it steps off the grid, p accumulated
// from 0.0 with + for odd and - for even popcounts -- lorenzo_fp's operations
// without the index arithmetic.
__device__ __forceinline__ double lorenzo_direct(const double* __restrict__ r, uint64_t c, uint32_t D, bool ai,
                                                 bool aj, bool ak, uint64_t s0, uint64_t s1) {
    double p = 0.0;
    if (D == 2) {  // axes (i, j) = (0, 1); strides s0 = dims[1], 1
        if (ai) p = __dadd_rn(p, r[c - s0]);
        if (aj) p = __dadd_rn(p, r[c - 1]);
        if (ai && aj) p = __dsub_rn(p, r[c - s0 - 1]);
        return p;
    }
    if (ai) p = __dadd_rn(p, r[c - s0]);                       // mask 1
    if (aj) p = __dadd_rn(p, r[c - s1]);                       // mask 2
    if (ai && aj) p = __dsub_rn(p, r[c - s0 - s1]);            // mask 3
    if (ak) p = __dadd_rn(p, r[c - 1]);                        // mask 4
    if (ai && ak) p = __dsub_rn(p, r[c - s0 - 1]);             // mask 5
    if (aj && ak) p = __dsub_rn(p, r[c - s1 - 1]);             // mask 6
    if (ai && aj && ak) p = __dadd_rn(p, r[c - s0 - s1 - 1]);  // mask 7
    return p;
}

// One cooperative launch for the whole wavefront: the grid walks the planes
// in order with a grid-wide barrier between them (instead of one launch per
// plane: 766 for a 256^3 grid). Same per-node work as k_wave_enc / k_wave_dec.
// MODE 0: lossy encode with escapes, 1: lossy decode with escapes, 2: lossless
// decode (codec.hpp:429-430).
template <int MODE>
__global__ void __launch_bounds__(THREADS) k_wave_coop(const double* __restrict__ v, const uint64_t* __restrict__ cin,
                                                      NdShape sh, double tau, double bin, double* __restrict__ recon,
                                                      uint64_t* __restrict__ cout, uint8_t* __restrict__ F,
                                                      const int32_t* __restrict__ eslot,
                                                      const double* __restrict__ eval) {
    namespace cg = cooperative_groups;
    cg::grid_group grid = cg::this_grid();
    uint64_t smax = 0;
    for (int d = 0; d < sh.D; ++d) smax += sh.dims[d] - 1;
    const uint64_t d0 = sh.dims[0], rest = smax - (d0 - 1);
    const uint64_t tid = blockIdx.x * (uint64_t)THREADS + threadIdx.x, nth = (uint64_t)gridDim.x * THREADS;
    for (uint64_t s = 0; s <= smax; ++s) {
        const uint64_t i_lo = s > rest ? s - rest : 0, i_hi = d0 - 1 < s ? d0 - 1 : s;
        const uint64_t rows = i_hi - i_lo + 1;
        const uint64_t cnt = sh.D == 2 ? rows : rows * sh.dims[1];
        for (uint64_t t = tid; t < cnt; t += nth) {
            uint64_t lin;
            bool ai, aj, ak = false;
            uint64_t st0, st1 = 0;
            if (sh.D == 2) {
                const uint64_t i = i_lo + t, j = s - i;
                lin = i * sh.dims[1] + j;
                ai = i > 0;
                aj = j > 0;
                st0 = sh.dims[1];
            } else {
                const uint32_t d1 = (uint32_t)sh.dims[1];
                const uint32_t tq = (uint32_t)(t / d1);
                const uint64_t i = i_lo + tq, j = t - (uint64_t)tq * d1;
                if (i + j > s) continue;
                const uint64_t k = s - i - j;
                if (k >= sh.dims[2]) continue;
                lin = (i * sh.dims[1] + j) * sh.dims[2] + k;
                ai = i > 0;
                aj = j > 0;
                ak = k > 0;
                st1 = sh.dims[2];
                st0 = sh.dims[1] * sh.dims[2];
            }
            const double p = lorenzo_direct(recon, lin, (uint32_t)sh.D, ai, aj, ak, st0, st1);
            if (MODE == 2) {
                recon[lin] = __longlong_as_double((long long)(cin[lin] ^ (uint64_t)__double_as_longlong(p)));
            } else if (MODE == 0) {
                const double x = v[lin];
                const double qd = round(__ddiv_rn(__dsub_rn(x, p), bin));
                bool escape = !(fabs(qd) <= kQLimit);
                double r = 0.0;
                if (!escape) {
                    r = __dadd_rn(p, __dmul_rn(qd, bin));
                    escape = !(fabs(__dsub_rn(x, r)) <= tau);
                }
                F[lin] = escape ? 1 : 0;
                cout[lin] = escape ? 0 : zz_enc((int64_t)qd);
                recon[lin] = escape ? x : r;
            } else {
                const int32_t e = eslot[lin];
                recon[lin] = e >= 0 ? eval[e] : __dadd_rn(p, __dmul_rn((double)zz_dec(cin[lin]), bin));
            }
        }
        __threadfence();
        grid.sync();
    }
}

// Launches the cooperative wavefront; false when the device cannot (the
// caller then launches plane by plane).
// Tiled wavefront: the grid is cut into T^D tiles; tiles on one tile-plane
// (I + J [+ K] = S) are independent given the earlier tile-planes, so the
// grid barrier runs once per tile-plane (46 for 256^3 with T = 16, instead of
// 766). Each tile is reconstructed in shared memory with its one-node halo
// from the earlier tiles, plane by plane inside the tile (i + j [+ k] = s,
// __syncthreads between), with lorenzo_direct on the shared copy -- the
// reference's operations, in its order -- then written back.
template <int D>
struct WaveTile {
    static constexpr int T = D == 3 ? 16 : 64;
    static constexpr int P = T + 1;  // tile + one halo node per axis
    // shared strides padded off multiples of 128 bytes: the nodes of one
    // plane (stepping +1 / -1 along two axes) then fall into different banks
    static constexpr int Q1 = D == 3 ? P + 1 : 1;
    static constexpr int Q0 = D == 3 ? (P + 1) * Q1 : P + 1;
    static constexpr int SM = P * Q0;
};

template <int MODE, int D>
__global__ void __launch_bounds__(THREADS) k_wave_tiled(const double* __restrict__ v, const uint64_t* __restrict__ cin,
                                                       NdShape sh, double tau, double bin, double* __restrict__ recon,
                                                       uint64_t* __restrict__ cout, uint8_t* __restrict__ F,
                                                       const int32_t* __restrict__ eslot,
                                                       const double* __restrict__ eval) {
    namespace cg = cooperative_groups;
    cg::grid_group grid = cg::this_grid();
    constexpr int T = WaveTile<D>::T, P = WaveTile<D>::P;
    constexpr int TN = D == 3 ? T * T * T : T * T;  // nodes per tile
    extern __shared__ __align__(16) double wsm[];
    double* sr = wsm;                                              // [SM] reconstruction + halo
    uint64_t* sin = reinterpret_cast<uint64_t*>(wsm + WaveTile<D>::SM);  // [TN] the tile's values / codes
    int32_t* ses = reinterpret_cast<int32_t*>(sin + TN);              // [TN] escape slots (decode)
    const uint64_t n0 = sh.dims[0], n1 = sh.dims[1], n2 = D == 3 ? sh.dims[2] : 1;
    const uint32_t tI = (uint32_t)((n0 + T - 1) / T), tJ = (uint32_t)((n1 + T - 1) / T),
                   tK = D == 3 ? (uint32_t)((n2 + T - 1) / T) : 1;
    const uint32_t Smax = (tI - 1) + (tJ - 1) + (tK - 1);
    const uint64_t g0 = D == 3 ? n1 * n2 : n1, g1 = D == 3 ? n2 : 1;  // global strides of axes 0, 1
    constexpr uint64_t q0 = WaveTile<D>::Q0, q1 = WaveTile<D>::Q1;       // shared strides
    for (uint32_t S = 0; S <= Smax; ++S) {
        const uint32_t ntile = D == 3 ? tI * tJ : tI;
        for (uint32_t t = blockIdx.x; t < ntile; t += gridDim.x) {
            uint32_t I, J, K = 0;
            if (D == 3) {
                I = t / tJ;
                J = t - I * tJ;
                if (I + J > S || S - I - J >= tK) continue;
                K = S - I - J;
            } else {
                I = t;
                if (I > S || S - I >= tJ) continue;
                J = S - I;
            }
            const uint64_t i0 = (uint64_t)I * T, j0 = (uint64_t)J * T, k0 = (uint64_t)K * T;
            // halo (local index 0 on some axis) from the finished earlier tiles
            constexpr uint32_t HN = D == 3 ? P * P * P : P * P;
            for (uint32_t x = threadIdx.x; x < HN; x += THREADS) {
                const uint32_t a = D == 3 ? x / (P * P) : x / P;
                const uint32_t b = D == 3 ? (x / P) % P : x % P;
                const uint32_t c = D == 3 ? x % P : 1;
                if (a != 0 && b != 0 && (D == 2 || c != 0)) continue;
                const int64_t gi = (int64_t)i0 + a - 1, gj = (int64_t)j0 + b - 1, gk = D == 3 ? (int64_t)k0 + c - 1 : 0;
                double val = 0.0;
                if (gi >= 0 && gj >= 0 && gk >= 0 && (uint64_t)gi < n0 && (uint64_t)gj < n1 && (uint64_t)gk < n2)
                    val = recon[(uint64_t)gi * g0 + (uint64_t)gj * g1 + (uint64_t)gk];
                sr[a * q0 + (D == 3 ? b * q1 + c : b)] = val;
            }
            // the tile's inputs, once (the plane loop below touches shared memory only)
            for (uint32_t x = threadIdx.x; x < (uint32_t)TN; x += THREADS) {
                const uint32_t a = D == 3 ? x / (T * T) : x / T;
                const uint32_t b = D == 3 ? (x / T) % T : x % T;
                const uint32_t c = D == 3 ? x % T : 0;
                const uint64_t gi = i0 + a, gj = j0 + b, gk = k0 + c;
                if (gi >= n0 || gj >= n1 || gk >= n2) continue;
                const uint64_t lin = gi * g0 + gj * g1 + gk;
                sin[x] = MODE == 0 ? (uint64_t)__double_as_longlong(v[lin]) : cin[lin];
                if (MODE == 1) ses[x] = eslot[lin];
            }
            __syncthreads();
            const int nloc = D == 3 ? 3 * T - 2 : 2 * T - 1;
            for (int sl = 0; sl < nloc; ++sl) {
                // nodes (a, b[, c]) of the tile with a + b [+ c] = sl
                const uint32_t cand = D == 3 ? T * T : T;
                for (uint32_t x = threadIdx.x; x < cand; x += THREADS) {
                    uint32_t a, b, c = 0;
                    if (D == 3) {
                        a = x / T;
                        b = x % T;
                        if ((int)(a + b) > sl || sl - (int)(a + b) >= T) continue;
                        c = (uint32_t)sl - a - b;
                    } else {
                        a = x;
                        if ((int)a > sl || sl - (int)a >= T) continue;
                        b = (uint32_t)sl - a;
                    }
                    const uint64_t gi = i0 + a, gj = j0 + b, gk = k0 + c;
                    if (gi >= n0 || gj >= n1 || gk >= n2) continue;
                    const uint64_t lin = gi * g0 + gj * g1 + gk;
                    const uint32_t tx = D == 3 ? (a * T + b) * T + c : a * T + b;
                    const uint64_t pos = (uint64_t)(a + 1) * q0 + (uint64_t)(b + 1) * q1 + (D == 3 ? c + 1 : 0);
                    const double p = D == 3 ? lorenzo_direct(sr, pos, 3, gi > 0, gj > 0, gk > 0, q0, q1)
                                            : lorenzo_direct(sr, pos, 2, gi > 0, gj > 0, false, q0, 0);
                    double r;
                    if (MODE == 2) {
                        r = __longlong_as_double((long long)(sin[tx] ^ (uint64_t)__double_as_longlong(p)));
                    } else if (MODE == 0) {
                        const double xv = __longlong_as_double((long long)sin[tx]);
                        const double qd = round(__ddiv_rn(__dsub_rn(xv, p), bin));
                        bool escape = !(fabs(qd) <= kQLimit);
                        r = 0.0;
                        if (!escape) {
                            r = __dadd_rn(p, __dmul_rn(qd, bin));
                            escape = !(fabs(__dsub_rn(xv, r)) <= tau);
                        }
                        F[lin] = escape ? 1 : 0;
                        cout[lin] = escape ? 0 : zz_enc((int64_t)qd);
                        if (escape) r = xv;
                    } else {
                        const int32_t e = ses[tx];
                        r = e >= 0 ? eval[e] : __dadd_rn(p, __dmul_rn((double)zz_dec(sin[tx]), bin));
                    }
                    sr[pos] = r;
                }
                __syncthreads();
            }
            // the tile back to global memory
            for (uint32_t x = threadIdx.x; x < (uint32_t)(D == 3 ? T * T * T : T * T); x += THREADS) {
                const uint32_t a = D == 3 ? x / (T * T) : x / T;
                const uint32_t b = D == 3 ? (x / T) % T : x % T;
                const uint32_t c = D == 3 ? x % T : 0;
                const uint64_t gi = i0 + a, gj = j0 + b, gk = k0 + c;
                if (gi >= n0 || gj >= n1 || gk >= n2) continue;
                recon[gi * g0 + gj * g1 + gk] = sr[(uint64_t)(a + 1) * q0 + (uint64_t)(b + 1) * q1 + (D == 3 ? c + 1 : 0)];
            }
            __syncthreads();
        }
        __threadfence();
        grid.sync();
    }
}

template <int MODE>
bool wave_tiled(const double* v, const uint64_t* cin, const NdShape& sh, double tau, double bin, double* recon,
                uint64_t* cout, uint8_t* F, const int32_t* eslot, const double* eval, cudaStream_t st) {
    if (std::getenv("UMCG_WAVE_LAUNCHES") || std::getenv("UMCG_WAVE_UNTILED")) return false;
    int dev = 0, sms = 0, coop = 0, per = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const void* fn = sh.D == 3 ? (const void*)k_wave_tiled<MODE, 3> : (const void*)k_wave_tiled<MODE, 2>;
    const int tn = sh.D == 3 ? WaveTile<3>::T * WaveTile<3>::T * WaveTile<3>::T : WaveTile<2>::T * WaveTile<2>::T;
    const size_t smem = 8 * (size_t)(sh.D == 3 ? WaveTile<3>::SM : WaveTile<2>::SM) + 12 * (size_t)tn;
    if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    cudaError_t oe = sh.D == 3 ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_wave_tiled<MODE, 3>, THREADS, smem)
                               : cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_wave_tiled<MODE, 2>, THREADS, smem);
    if (!coop || oe != cudaSuccess || per < 1) {
        cudaGetLastError();
        return false;
    }
    void* args[] = {(void*)&v, (void*)&cin, (void*)&sh, (void*)&tau, (void*)&bin, (void*)&recon, (void*)&cout,
                    (void*)&F, (void*)&eslot, (void*)&eval};
    const dim3 grid((unsigned)(sms * std::min(per, 2)));
    if (cudaLaunchCooperativeKernel(fn, grid, dim3(THREADS), args, smem, st) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    UMCG_LAUNCHED();
    return true;
}

#ifndef UMCG_WAVE_BPS_DEFAULT
#define UMCG_WAVE_BPS_DEFAULT 2
#endif
template <int MODE>
bool wave_coop(const double* v, const uint64_t* cin, const NdShape& sh, double tau, double bin, double* recon,
               uint64_t* cout, uint8_t* F, const int32_t* eslot, const double* eval, cudaStream_t st) {
    if (std::getenv("UMCG_WAVE_LAUNCHES")) return false;
    int dev = 0, sms = 0, coop = 0, per = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (!coop || cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_wave_coop<MODE>, THREADS, 0) != cudaSuccess ||
        per < 1) {
        cudaGetLastError();
        return false;
    }
    void* args[] = {(void*)&v, (void*)&cin, (void*)&sh, (void*)&tau, (void*)&bin, (void*)&recon, (void*)&cout,
                    (void*)&F, (void*)&eslot, (void*)&eval};
    // blocks per SM: the grid barrier's cost grows with the block count (A/B: UMCG_WAVE_BPS)
    static const int bps = [] {
        const char* e = std::getenv("UMCG_WAVE_BPS");
        return e ? std::max(1, std::atoi(e)) : UMCG_WAVE_BPS_DEFAULT;
    }();
    const dim3 grid((unsigned)(sms * std::min(per, bps)));
    if (cudaLaunchCooperativeKernel((const void*)k_wave_coop<MODE>, grid, dim3(THREADS), args, 0, st) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    UMCG_LAUNCHED();
    return true;
}

template <class F>
void for_planes(const NdShape& sh, F&& f) {
    uint64_t smax = 0;
    for (int d = 0; d < sh.D; ++d) smax += sh.dims[d] - 1;
    const uint64_t d0 = sh.dims[0], rest = smax - (d0 - 1);
    for (uint64_t s = 0; s <= smax; ++s) {
        const uint64_t i_lo = s > rest ? s - rest : 0, i_hi = std::min<uint64_t>(d0 - 1, s);
        const uint64_t rows = i_hi - i_lo + 1;
        const uint64_t cnt = sh.D == 2 ? rows : rows * sh.dims[1];
        f(s, i_lo, cnt);
    }
}
}  // namespace

bool wave_encode_nd(const double* v, uint64_t n, const NdShape& sh, double tau, uint64_t* codes, double* recon,
                    uint8_t* F, cudaStream_t st) {
    if (sh.D != 2 && sh.D != 3) return false;
    if (!n) return true;
    const double bin = 2.0 * tau;
    if (wave_tiled<0>(v, nullptr, sh, tau, bin, recon, codes, F, nullptr, nullptr, st)) return true;
    if (wave_coop<0>(v, nullptr, sh, tau, bin, recon, codes, F, nullptr, nullptr, st)) return true;
    for_planes(sh, [&](uint64_t s, uint64_t i_lo, uint64_t cnt) {
        k_wave_enc<<<(unsigned)cdiv(cnt, THREADS), THREADS, 0, st>>>(v, sh, s, i_lo, cnt, tau, bin, recon, codes, F);
        UMCG_LAUNCHED();
    });
    return true;
}

bool wave_decode_nd(const uint64_t* codes, uint64_t n, const NdShape& sh, double tau, const uint64_t* esc_idx,
                    const double* esc_val, uint64_t n_esc, int32_t* eslot, double* out, cudaStream_t st) {
    if (sh.D != 2 && sh.D != 3) return false;
    if (!n) return true;
    const double bin = 2.0 * tau;
    UMCG_CUDA(cudaMemsetAsync(eslot, 0xff, n * sizeof(int32_t), st));
    if (n_esc) {
        k_esc_slots<<<(unsigned)cdiv(n_esc, 256), 256, 0, st>>>(esc_idx, n_esc, eslot);
        UMCG_LAUNCHED();
    }
    if (wave_tiled<1>(nullptr, codes, sh, tau, bin, out, nullptr, nullptr, eslot, esc_val, st)) return true;
    if (wave_coop<1>(nullptr, codes, sh, tau, bin, out, nullptr, nullptr, eslot, esc_val, st)) return true;
    for_planes(sh, [&](uint64_t s, uint64_t i_lo, uint64_t cnt) {
        k_wave_dec<<<(unsigned)cdiv(cnt, THREADS), THREADS, 0, st>>>(codes, sh, s, i_lo, cnt, bin, eslot, esc_val, out);
        UMCG_LAUNCHED();
    });
    return true;
}

bool lossless_nd_wavefront(const uint64_t* codes, uint64_t n, const NdShape& sh, double* out, cudaStream_t st) {
    if (sh.D != 2 && sh.D != 3) return false;
    if (!n) return true;
    if (wave_tiled<2>(nullptr, codes, sh, 0.0, 0.0, out, nullptr, nullptr, nullptr, nullptr, st)) return true;
    if (wave_coop<2>(nullptr, codes, sh, 0.0, 0.0, out, nullptr, nullptr, nullptr, nullptr, st)) return true;
    uint64_t smax = 0;
    for (int d = 0; d < sh.D; ++d) smax += sh.dims[d] - 1;
    const uint64_t d0 = sh.dims[0], rest = smax - (d0 - 1);  // max of the other coordinates' sum
    for (uint64_t s = 0; s <= smax; ++s) {
        const uint64_t i_lo = s > rest ? s - rest : 0, i_hi = std::min<uint64_t>(d0 - 1, s);
        const uint64_t rows = i_hi - i_lo + 1;
        const uint64_t cnt = sh.D == 2 ? rows : rows * sh.dims[1];
        k_lossless_plane<<<(unsigned)cdiv(cnt, THREADS), THREADS, 0, st>>>(codes, sh, s, i_lo, cnt, out);
        UMCG_LAUNCHED();
    }
    return true;
}

void serial_decode(const uint64_t* codes, uint64_t n, int pred, const NdShape& sh, double tau,
                   const uint64_t* esc_idx, const double* esc_val, uint64_t n_esc, double* out,
                   cudaStream_t st) {
    g_serial_fallbacks.fetch_add(1);
    k_serial_decode<<<1, 32, 0, st>>>(codes, n, pred, sh, tau, esc_idx, esc_val, n_esc, out);
    UMCG_LAUNCHED();
}

void recon_lossy(const uint64_t* codes, uint64_t n, int pred, const NdShape& sh, double bin, int64_t* kbuf,
                 double* out, DevCtl* ctl, cudaStream_t st) {
    if (!n) return;
    if (pred == 0) {
        k_recon_none<<<blocks(n), THREADS, 0, st>>>(codes, n, bin, out);
        UMCG_LAUNCHED();
        return;
    }
    if (pred == 1 || sh.D <= 1) {
        const uint64_t T = cdiv(n, SC_TILE);
        k_tile_sums<<<(unsigned)T, THREADS, 0, st>>>(codes, n, kbuf);
        UMCG_LAUNCHED();
        k_scan_sums<<<1, 1024, 0, st>>>(kbuf, T);
        UMCG_LAUNCHED();
        k_tile_recon_1d<<<(unsigned)T, THREADS, 0, st>>>(codes, n, kbuf, bin, out, ctl);
        UMCG_LAUNCHED();
        return;
    }
    k_zz_to_k<<<blocks(n), THREADS, 0, st>>>(codes, n, kbuf);
    UMCG_LAUNCHED();
    for (int d = sh.D - 1; d >= 0; --d) {
        const uint64_t lines = n / sh.dims[d];
        k_axis_scan<<<blocks(lines), THREADS, 0, st>>>(kbuf, sh, d, lines);
        UMCG_LAUNCHED();
    }
    k_k_to_recon<<<blocks(n), THREADS, 0, st>>>(kbuf, n, bin, out, ctl);
    UMCG_LAUNCHED();
}

void recon_lossless(const uint64_t* codes, uint64_t n, int pred, double* out, uint64_t* scratch,
                    cudaStream_t st) {
    if (!n) return;
    if (pred == 0) {
        k_recon_lossless_none<<<blocks(n), THREADS, 0, st>>>(codes, n, out);
        UMCG_LAUNCHED();
        return;
    }
    // pred == 1 only (N-D lossless goes through serial_decode)
    const uint64_t T = cdiv(n, SC_TILE);
    uint64_t* sums = scratch;  // [cdiv(n, SC_TILE)]
    k_tile_xor<<<(unsigned)T, THREADS, 0, st>>>(codes, n, sums);
    UMCG_LAUNCHED();
    k_scan_xor<<<1, 1024, 0, st>>>(sums, T);
    UMCG_LAUNCHED();
    k_tile_recon_xor<<<(unsigned)T, THREADS, 0, st>>>(codes, n, sums, out);
    UMCG_LAUNCHED();
}

}  // namespace umcg
