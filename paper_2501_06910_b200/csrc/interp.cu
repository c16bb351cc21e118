// Value range, error budget, cluster means (mesh -> grid) on sm_100a.
#include <cub/block/block_reduce.cuh>

#include "kernels.h"

namespace umcg {

namespace {

constexpr int THREADS = 256;

// value_range + validate_field finiteness (pipeline.hpp:31-35, mesh.hpp:58-64).
// min/max are order-free, so a grid-stride reduction is exact.
template <class T>
__global__ void __launch_bounds__(THREADS) k_minmax(const T* __restrict__ x, uint64_t n, DevCtl* ctl) {
    using BR = cub::BlockReduce<unsigned long long, THREADS>;
    __shared__ typename BR::TempStorage t1, t2;
    unsigned long long lo = ~0ull, hi = 0ull;
    int bad = 0;
    const uint64_t stride = (uint64_t)gridDim.x * THREADS;
    for (uint64_t i = blockIdx.x * (uint64_t)THREADS + threadIdx.x; i < n; i += stride) {
        const double v = (double)x[i];
        if (!isfinite(v)) { bad = 1; continue; }
        const unsigned long long k = dkey(v);
        lo = k < lo ? k : lo;
        hi = k > hi ? k : hi;
    }
    const unsigned long long blo = BR(t1).Reduce(lo, cub::Min());
    const unsigned long long bhi = BR(t2).Reduce(hi, cub::Max());
    if (threadIdx.x == 0) {
        if (blo != ~0ull) atomicMin(&ctl->min_key, blo);
        if (bhi != 0ull) atomicMax(&ctl->max_key, bhi);
    }
    if (bad) ctl->nonfinite = 1;
}

// resolve_tau_abs + split_budget + shave (pipeline.hpp:37-57, 94), one thread,
// same operation order as the reference (no contraction).
__global__ void k_budget(BudgetArgs a, DevCtl* ctl) {
    if (threadIdx.x | blockIdx.x) return;
    double range = 0.0;
    if (a.n) range = __dsub_rn(dkey_inv(ctl->max_key), dkey_inv(ctl->min_key));
    const double tau_abs = a.bound_kind ? __dmul_rn(a.tau, range) : a.tau;
    double t1 = __ddiv_rn(__dmul_rn(a.rho, tau_abs), a.coeff_abs_sum);
    const double t2 = __dmul_rn(__dsub_rn(1.0, a.rho), tau_abs);
    while (__dadd_rn(__dmul_rn(a.coeff_abs_sum, t1), t2) > tau_abs) t1 = nextafter(t1, 0.0);
    ctl->tau_abs = tau_abs;
    ctl->tau1 = t1;
    ctl->tau2 = t2;
    const double shave = 1.0 - 1e-9;  // detail::shave
    ctl->tau_c[0] = __dmul_rn(t1, shave);
    ctl->tau_c[1] = __dmul_rn(t2, shave);
    ctl->bin[0] = __dmul_rn(2.0, ctl->tau_c[0]);
    ctl->bin[1] = __dmul_rn(2.0, ctl->tau_c[1]);
    ctl->inv_bin[0] = __ddiv_rn(1.0, ctl->bin[0]);
    ctl->inv_bin[1] = __ddiv_rn(1.0, ctl->bin[1]);
    ctl->lossless = (ctl->tau_c[0] == 0.0 ? 1 : 0) | (ctl->tau_c[1] == 0.0 ? 2 : 0);
}

// interpolate_to_grid (interp.hpp:46-64): x1[j] = (0.0 + x_{i1} + x_{i2} + ...)
// / count_j in ascending vertex order. perm is the plan's stable sort of
// vertices by slot, so one thread per slot reproduces the reference's
// summation order bit for bit without atomics.
template <class T>
__global__ void __launch_bounds__(THREADS) k_cluster_mean(const T* __restrict__ x, const uint32_t* __restrict__ perm,
                                                         const uint32_t* __restrict__ seg_off, uint64_t n_slots,
                                                         double* __restrict__ x1) {
    const uint64_t j = blockIdx.x * (uint64_t)THREADS + threadIdx.x;
    if (j >= n_slots) return;
    const uint32_t b = seg_off[j], e = seg_off[j + 1];
    double s = 0.0;
    for (uint32_t k = b; k < e; ++k) s = __dadd_rn(s, (double)x[perm[k]]);
    x1[j] = e > b ? __ddiv_rn(s, (double)(e - b)) : 0.0;
}

// FillPolicy::nearest_visited (interp.hpp:66-91): per row of the fastest
// axis, unvisited nodes copy the nearest visited node, ties to the lower
// index; all-unvisited rows keep zeros. One thread per row.
__global__ void __launch_bounds__(THREADS) k_fill(const uint32_t* __restrict__ seg_off, uint64_t n_rows,
                                                 uint64_t row, double* __restrict__ x1) {
    const uint64_t r = blockIdx.x * (uint64_t)THREADS + threadIdx.x;
    if (r >= n_rows) return;
    double* v = x1 + r * row;
    const uint32_t* so = seg_off + r * row;
    auto visited = [&](uint64_t t) { return so[t + 1] > so[t]; };
    int64_t prev = -1;
    int64_t next = -1;
    for (uint64_t t = 0; t < row; ++t) {
        if (visited(t)) { prev = (int64_t)t; continue; }
        if (next <= (int64_t)t) {
            next = -1;
            for (uint64_t u = t + 1; u < row; ++u)
                if (visited(u)) { next = (int64_t)u; break; }
        }
        if (prev < 0 && next < 0) return;  // whole row unvisited
        int64_t src;
        if (prev < 0) src = next;
        else if (next < 0) src = prev;
        else src = ((int64_t)t - prev <= next - (int64_t)t) ? prev : next;
        v[t] = v[src];
    }
}

}  // namespace

void minmax(const void* x, int x_f32, uint64_t n, DevCtl* ctl, cudaStream_t st) {
    if (!n) return;
    unsigned grid = (unsigned)std::min<uint64_t>(cdiv(n, THREADS), 148ull * 8);
    if (x_f32) k_minmax<float><<<grid, THREADS, 0, st>>>(static_cast<const float*>(x), n, ctl);
    else k_minmax<double><<<grid, THREADS, 0, st>>>(static_cast<const double*>(x), n, ctl);
    UMCG_LAUNCHED();
}

void budget(const BudgetArgs& a, DevCtl* ctl, cudaStream_t st) {
    k_budget<<<1, 32, 0, st>>>(a, ctl);
    UMCG_LAUNCHED();
}

void cluster_mean(const void* x, int x_f32, const uint32_t* perm, const uint32_t* seg_off, uint64_t n_slots,
                  double* x1, cudaStream_t st) {
    if (!n_slots) return;
    const unsigned g = (unsigned)cdiv(n_slots, THREADS);
    if (x_f32) k_cluster_mean<float><<<g, THREADS, 0, st>>>(static_cast<const float*>(x), perm, seg_off, n_slots, x1);
    else k_cluster_mean<double><<<g, THREADS, 0, st>>>(static_cast<const double*>(x), perm, seg_off, n_slots, x1);
    UMCG_LAUNCHED();
}

void fill_nearest_visited(const uint32_t* seg_off, uint64_t n_slots, uint64_t row, double* x1, cudaStream_t st) {
    const uint64_t n_rows = n_slots / row;
    if (!n_rows) return;
    k_fill<<<(unsigned)cdiv(n_rows, THREADS), THREADS, 0, st>>>(seg_off, n_rows, row, x1);
    UMCG_LAUNCHED();
}

}  // namespace umcg
