// detail::multilinear_at (interp.hpp:97-132) on the device, same operation
// order as the reference (no contraction: --fmad=false), shared by the
// vertex-order kernels (codes.cu) and the bucket-order ones (partition.cu).
#pragma once

#include <cstdint>

namespace umcg {

// std::upper_bound(axis, axis + n, p): guessed from the end points (any
// guess is fine), then corrected against the actual axis values -- same
// result as the binary search, which remains the fallback (outside the axis
// range, NaN, or a strongly graded axis).
__device__ __forceinline__ uint64_t axis_upper_bound(const double* __restrict__ axis, uint64_t n, double p,
                                                    double scale) {
    const double a0 = axis[0], a1 = axis[n - 1];
    if (p >= a0 && p < a1) {
        const double f = (p - a0) * scale;  // (n - 1) / (a1 - a0): only a guess
        uint64_t g = (uint64_t)f + 1;
        if (g > n - 1) g = n - 1;
        int steps = 0;
        while (g > 0 && p < axis[g - 1] && steps < 4) { --g; ++steps; }
        while (g < n && !(p < axis[g]) && steps < 8) { ++g; ++steps; }
        // verify: first index with axis[g] > p
        if ((g == 0 || !(p < axis[g - 1])) && (g == n || p < axis[g])) return g;
    }
    uint64_t lo = 0, hi = n;
    while (lo < hi) {
        const uint64_t mid = lo + (hi - lo) / 2;
        if (!(p < axis[mid])) lo = mid + 1; else hi = mid;
    }
    return lo;
}

// Corner weights are w = ((1.0 * a_0) * a_1) * a_2 with a_d = t_d or 1 - t_d
// (interp.hpp:120-125, dimension 0 = lowest corner bit); 1.0 * a_0 == a_0, so
// the partial products a_0 * a_1 are shared between corners without changing
// any rounding. Corners whose weight is 0 are skipped exactly as in the
// reference.
//
// Certificate that w == RN(num / den): the remainder r = num - w * den is
// exact (one fma) whenever w is within an ulp of the quotient, and w is the
// correctly rounded quotient if the true quotient lies strictly inside w's
// rounding interval, i.e. |r| < |den| * u / 2 with u the smaller of the two
// ulps next to w (the lower one is half at a power of two). A w more than an
// ulp off fails the test (its remainder is at least |den| * u), so a passing
// w is exact, with no assumption on how it was computed. Zero, subnormal and
// extreme exponents are not certified (the caller divides).
__device__ __forceinline__ bool quotient_certified(double num, double den, double w) {
    const unsigned long long b = (unsigned long long)__double_as_longlong(w) & 0x7fffffffffffffffull;
    const int e = (int)(b >> 52);  // biased exponent of w
    const int eh = e - 53 - ((b & 0xfffffffffffffull) == 0 ? 1 : 0);  // biased exponent of u_min / 2
    if (e == 0 || e > 2000 || eh < 200) return false;
    const double half = __longlong_as_double((long long)((unsigned long long)eh << 52));
    const double r = fabs(__fma_rn(-w, den, num));
    return r < __dmul_rn(fabs(den), half);
}

// Corner values from the grid component: x1[lin] straight from global memory
// (the bucket kernel passes a loader over its shared-memory staging).
struct GlobalCorners {
    const double* __restrict__ x1;
    __device__ __forceinline__ double operator()(uint64_t lin) const { return x1[lin]; }
};

// The cell fraction (p - a_l) / (a_h - a_l) is the correctly rounded quotient
// RN(num / den): Markstein's iteration from inv = RN(1 / (a_h - a_l))
// (precomputed per cell) -- q0 = RN(num * inv), r = num - q0 * den (fma),
// q = RN(q0 + r * inv) -- accepted only with the certificate above; any
// uncertified quotient (and operands outside [2^-900, 2^900]) takes the IEEE
// divide, so the result is RN(num / den) in every case, as the reference's
// `/` (interp.hpp:118).
// D is a compile-time rank (1-3) so the per-axis state stays in registers.
// hint (optional): per axis, the index of the vertex's nearest node (its
// slot in a dense mapping). The vertex then lies in the cell below or above
// it, so the cell is one comparison away; it is verified against the axis
// (axis[l] <= p < axis[l + 1], open at the ends exactly like the clamped
// upper_bound) and any mapping that does not satisfy it takes the search.
template <int D, class Corners>
__device__ __forceinline__ double multilinear_eval_c(const double* __restrict__ axes,
                                                    const uint64_t* __restrict__ axis_off, const uint64_t* shape,
                                                    const Corners& x1, const double* __restrict__ p,
                                                    const double* __restrict__ inv_cell, const double* scale,
                                                    const uint32_t* hint = nullptr) {
    double t[3] = {0, 0, 0}, om[3] = {1, 1, 1};
    uint64_t base = 0, step[3] = {0, 0, 0};
    uint64_t stride = 1;
#pragma unroll
    for (int d = D - 1; d >= 0; --d) {
        const uint64_t n = shape[d];
        uint64_t l = 0;
        double td = 0.0;
        if (n > 1) {
            const double* axis = axes + axis_off[d];
            uint64_t h = 0;
            bool found = false;
            if (hint) {
                const int64_t md = hint[d];
                int64_t c = (p[d] >= axis[md]) ? md : md - 1;
                c = c < 0 ? 0 : c;
                c = c > (int64_t)n - 2 ? (int64_t)n - 2 : c;
                found = (c == 0 || axis[c] <= p[d]) && (c == (int64_t)n - 2 || p[d] < axis[c + 1]);
                h = (uint64_t)c + 1;
            }
            if (!found) h = axis_upper_bound(axis, n, p[d], scale[d]);
            h = h < 1 ? 1 : h;
            if (h > n - 1) h = n - 1;
            l = h - 1;
            const double num = __dsub_rn(p[d], axis[l]), den = __dsub_rn(axis[h], axis[l]);
            const double y = inv_cell[axis_off[d] + l];
            const double q0 = __dmul_rn(num, y);
            double w = __fma_rn(__fma_rn(-q0, den, num), y, q0);
            if (!(fabs(num) > 0x1p-900) || !(fabs(num) < 0x1p900) || !quotient_certified(num, den, w))
                w = __ddiv_rn(num, den);
            td = (w < 0.0) ? 0.0 : ((1.0 < w) ? 1.0 : w);  // std::clamp
            step[d] = stride;  // l + 1 <= n - 1 always here
        }
        t[d] = td;
        om[d] = __dsub_rn(1.0, td);
        base += l * stride;
        stride *= n;
    }
    double acc = 0.0;
    if (D == 1) {
        if (om[0] != 0.0) acc = __dadd_rn(acc, __dmul_rn(om[0], x1(base)));
        if (t[0] != 0.0) acc = __dadd_rn(acc, __dmul_rn(t[0], x1(base + step[0])));
        return acc;
    }
    if (D == 2) {
#pragma unroll
        for (unsigned corner = 0; corner < 4; ++corner) {
            const bool h0 = corner & 1u, h1 = corner & 2u;
            const double w = __dmul_rn(h0 ? t[0] : om[0], h1 ? t[1] : om[1]);
            const uint64_t lin = base + (h0 ? step[0] : 0) + (h1 ? step[1] : 0);
            if (w != 0.0) acc = __dadd_rn(acc, __dmul_rn(w, x1(lin)));
        }
        return acc;
    }
    double p01[4];
#pragma unroll
    for (unsigned c = 0; c < 4; ++c) p01[c] = __dmul_rn((c & 1u) ? t[0] : om[0], (c & 2u) ? t[1] : om[1]);
    double v[8];
#pragma unroll
    for (unsigned corner = 0; corner < 8; ++corner) {
        const uint64_t lin = base + ((corner & 1u) ? step[0] : 0) + ((corner & 2u) ? step[1] : 0) +
                             ((corner & 4u) ? step[2] : 0);
        v[corner] = x1(lin);
    }
#pragma unroll
    for (unsigned corner = 0; corner < 8; ++corner) {
        const double w = __dmul_rn(p01[corner & 3u], (corner & 4u) ? t[2] : om[2]);
        if (w != 0.0) acc = __dadd_rn(acc, __dmul_rn(w, v[corner]));
    }
    return acc;
}

__device__ __forceinline__ double multilinear_eval(const double* __restrict__ axes,
                                                  const uint64_t* __restrict__ axis_off, const uint64_t* shape,
                                                  int D, const double* __restrict__ x1,
                                                  const double* __restrict__ p, const double* __restrict__ inv_cell,
                                                  const double* scale) {
    const GlobalCorners c{x1};
    if (D == 3) return multilinear_eval_c<3>(axes, axis_off, shape, c, p, inv_cell, scale);
    if (D == 2) return multilinear_eval_c<2>(axes, axis_off, shape, c, p, inv_cell, scale);
    return multilinear_eval_c<1>(axes, axis_off, shape, c, p, inv_cell, scale);
}

}  // namespace umcg
