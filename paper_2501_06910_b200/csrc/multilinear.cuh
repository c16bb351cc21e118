// detail::multilinear_at (interp.hpp:97-132) on the device, same operation
// order as the reference (no contraction: --fmad=false), shared by the
// vertex-order kernels (codes.cu) and the bucket-order ones (partition.cu).
#pragma once

#include <cstdint>

namespace umcg {

// std::upper_bound(axis, axis + n, p): guessed from the end points (exact
// for uniform axes up to rounding), then corrected against the actual axis
// values -- same result as the binary search, which remains the fallback
// (outside the axis range, NaN, or a strongly graded axis).
__device__ __forceinline__ uint64_t axis_upper_bound(const double* __restrict__ axis, uint64_t n, double p) {
    const double a0 = axis[0], a1 = axis[n - 1];
    if (p >= a0 && p < a1) {
        const double f = (p - a0) / (a1 - a0) * (double)(n - 1);
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

__device__ __forceinline__ double multilinear_eval(const double* __restrict__ axes, const uint64_t* __restrict__ axis_off,
                                                  const uint64_t* shape, int D, const double* __restrict__ x1,
                                                  const double* __restrict__ p) {
    uint64_t lo_idx[3] = {0, 0, 0};
    double t[3] = {0, 0, 0};
    for (int d = 0; d < D; ++d) {
        const uint64_t n = shape[d];
        const double* axis = axes + axis_off[d];
        if (n == 1) { lo_idx[d] = 0; t[d] = 0.0; continue; }
        uint64_t h = axis_upper_bound(axis, n, p[d]);
        h = h < 1 ? 1 : h;
        if (h > n - 1) h = n - 1;
        const uint64_t l = h - 1;
        const double w = __ddiv_rn(__dsub_rn(p[d], axis[l]), __dsub_rn(axis[h], axis[l]));
        lo_idx[d] = l;
        t[d] = (w < 0.0) ? 0.0 : ((1.0 < w) ? 1.0 : w);  // std::clamp
    }
    double acc = 0.0;
    for (unsigned corner = 0; corner < (1u << D); ++corner) {
        double w = 1.0;
        uint64_t lin = 0;
        for (int d = 0; d < D; ++d) {
            const bool high = (corner >> d) & 1u;
            w = __dmul_rn(w, high ? t[d] : __dsub_rn(1.0, t[d]));
            const uint64_t n = shape[d];
            uint64_t idx = lo_idx[d] + (high ? 1 : 0);
            if (idx >= n) idx = n - 1;
            lin = lin * n + idx;
        }
        if (w != 0.0) acc = __dadd_rn(acc, __dmul_rn(w, x1[lin]));
    }
    return acc;
}


}  // namespace umcg
