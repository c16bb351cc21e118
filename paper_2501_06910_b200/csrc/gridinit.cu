// umc::grid_init (grid_builder.hpp:201-282) on the device: per-axis edge
// deltas (cell edges, or each vertex's exact 1-nearest neighbour for point
// clouds), nearest-rank percentile by radix sort, then the reference's
// spacing loop and axis construction on the host.
//
//   traverse_mesh (:79-97)   k_cell_deltas: |c_u - c_v| per cell edge, per axis
//   knn_edge_stats (:100-196) bucket grid + exact 1-NN per vertex (ties toward
//                            the lower vertex index; dist2 accumulated in axis
//                            order without contraction, as the reference)
//   percentile (:201-214)    sort ascending, zeros excluded, element at
//                            ceil(k / 100 * N)
#include <algorithm>
#include <cmath>
#include <limits>
#include <vector>


#include "kernels.h"
#include "plan.h"

namespace umcg {

namespace {

constexpr int GT = 256;

// cell_edges (grid_builder.hpp:46-59): 3 tri, 4 quad, 8 hex
__constant__ int c_edges[12][2];

__global__ void k_cell_deltas(const double* __restrict__ xyz, int D, uint64_t n_v, const uint64_t* __restrict__ cells,
                              uint64_t n_c, int arity, int n_e, int d, double* __restrict__ out, DevCtl* ctl) {
    const uint64_t t = blockIdx.x * (uint64_t)GT + threadIdx.x;
    if (t >= n_c * n_e) return;
    const uint64_t j = t / n_e;
    const int e = (int)(t % n_e);
    const uint64_t u = cells[j * arity + c_edges[e][0]], v = cells[j * arity + c_edges[e][1]];
    if (u >= n_v || v >= n_v) {
        set_err(ctl, 1);
        out[t] = 0.0;
        return;
    }
    out[t] = fabs(__dsub_rn(xyz[u * D + d], xyz[v * D + d]));
}

__global__ void k_minmax_axis(const double* __restrict__ xyz, int D, uint64_t n_v, unsigned long long* mm) {
    const uint64_t v = blockIdx.x * (uint64_t)GT + threadIdx.x;
    if (v >= n_v) return;
    for (int d = 0; d < D; ++d) {
        const unsigned long long k = dkey(xyz[v * D + d]);
        atomicMin(&mm[2 * d], k);
        atomicMax(&mm[2 * d + 1], k);
    }
}

struct KnnGrid {
    double lo[3], span[3];
    uint64_t per_axis;
    int D;
    double min_sep;
};

__device__ __forceinline__ int64_t bucket_of(const KnnGrid& g, double c, int d) {
    const double t = __ddiv_rn(__dsub_rn(c, g.lo[d]), g.span[d]);
    int64_t b = (int64_t)__dmul_rn(t, (double)g.per_axis);
    if (b < 0) b = 0;
    if (b > (int64_t)g.per_axis - 1) b = (int64_t)g.per_axis - 1;
    return b;
}

__global__ void k_knn_keys(const double* __restrict__ xyz, uint64_t n_v, KnnGrid g, uint64_t* __restrict__ key,
                           uint32_t* __restrict__ idx, uint32_t* __restrict__ cnt) {
    const uint64_t v = blockIdx.x * (uint64_t)GT + threadIdx.x;
    if (v >= n_v) return;
    uint64_t lin = 0;
    for (int d = 0; d < g.D; ++d) lin = lin * g.per_axis + (uint64_t)bucket_of(g, xyz[v * g.D + d], d);
    key[v] = lin;
    idx[v] = (uint32_t)v;
    atomicAdd(&cnt[lin], 1u);
}

// Exact 1-NN of v over all other vertices by rings of buckets (the ring
// bound only prunes buckets that cannot hold a closer point), then the
// per-axis deltas to it.
__global__ void k_knn(const double* __restrict__ xyz, uint64_t n_v, KnnGrid g, const uint32_t* __restrict__ start,
                      const uint32_t* __restrict__ sorted, double* __restrict__ deltas) {
    const uint64_t v = blockIdx.x * (uint64_t)GT + threadIdx.x;
    if (v >= n_v) return;
    const int D = g.D;
    double pv[3] = {0, 0, 0};
    int64_t home[3] = {0, 0, 0};
    for (int d = 0; d < D; ++d) {
        pv[d] = xyz[v * D + d];
        home[d] = bucket_of(g, pv[d], d);
    }
    double best = INFINITY;
    uint64_t best_idx = n_v;
    const int64_t P = (int64_t)g.per_axis;
    for (int64_t ring = 0; ring < P; ++ring) {
        if (best_idx != n_v && ring > 1) {
            const double reach = __dmul_rn((double)(ring - 1), g.min_sep);
            if (__dmul_rn(reach, reach) > best) break;
        }
        const int64_t r = ring;
        int64_t b[3];
        const int64_t z0 = D == 3 ? home[2] - r : 0, z1 = D == 3 ? home[2] + r : 0;
        for (b[0] = home[0] - r; b[0] <= home[0] + r; ++b[0]) {
            if (b[0] < 0 || b[0] >= P) continue;
            for (b[1] = home[1] - r; b[1] <= home[1] + r; ++b[1]) {
                if (b[1] < 0 || b[1] >= P) continue;
                for (b[2] = z0; b[2] <= z1; ++b[2]) {
                    if (D == 3 && (b[2] < 0 || b[2] >= P)) continue;
                    const int64_t a0 = b[0] - home[0], a1 = b[1] - home[1], a2 = D == 3 ? b[2] - home[2] : 0;
                    int64_t cheb = a0 < 0 ? -a0 : a0;
                    cheb = (a1 < 0 ? -a1 : a1) > cheb ? (a1 < 0 ? -a1 : a1) : cheb;
                    cheb = (a2 < 0 ? -a2 : a2) > cheb ? (a2 < 0 ? -a2 : a2) : cheb;
                    if (cheb != r) continue;
                    uint64_t lin = (uint64_t)b[0] * P + (uint64_t)b[1];
                    if (D == 3) lin = lin * P + (uint64_t)b[2];
                    for (uint32_t q = start[lin]; q < start[lin + 1]; ++q) {
                        const uint64_t u = sorted[q];
                        if (u == v) continue;
                        double dist2 = 0.0;
                        for (int d = 0; d < D; ++d) {
                            const double dd = __dsub_rn(xyz[u * D + d], pv[d]);
                            dist2 = __dadd_rn(dist2, __dmul_rn(dd, dd));
                        }
                        if (dist2 < best || (dist2 == best && u < best_idx)) {
                            best = dist2;
                            best_idx = u;
                        }
                    }
                }
            }
        }
    }
    for (int d = 0; d < D; ++d)
        deltas[d * n_v + v] = best_idx < n_v ? fabs(__dsub_rn(xyz[best_idx * D + d], pv[d])) : 0.0;
}

// IEEE doubles as u64 keys of the same order (sign bit flipped for positive
// values, all bits for negative ones), and back in place.
__global__ void k_double_keys(const double* __restrict__ v, uint64_t n, uint64_t* __restrict__ k) {
    const uint64_t i = blockIdx.x * (uint64_t)GT + threadIdx.x;
    if (i >= n) return;
    const uint64_t u = (uint64_t)__double_as_longlong(v[i]);
    k[i] = (u >> 63) ? ~u : u | 0x8000000000000000ull;
}
__global__ void k_keys_double(uint64_t* __restrict__ k, uint64_t n) {
    const uint64_t i = blockIdx.x * (uint64_t)GT + threadIdx.x;
    if (i >= n) return;
    const uint64_t u = k[i];
    k[i] = (u >> 63) ? u & 0x7fffffffffffffffull : ~u;
}

__global__ void k_count_zero(const double* __restrict__ s, uint64_t n, unsigned long long* z) {
    const uint64_t i = blockIdx.x * (uint64_t)GT + threadIdx.x;
    if (i < n && s[i] == 0.0) atomicAdd(z, 1ull);
}

unsigned gblocks(uint64_t n) { return (unsigned)cdiv(n, GT); }

// Sorted nonzero samples of one axis on the device (zeros sort first).
struct SortedAxis {
    DevBuf keys;
    uint64_t zeros = 0, total = 0;
    double at(uint64_t i, cudaStream_t st) const {  // i-th nonzero (0-based)
        double v = 0;
        UMCG_CUDA(cudaMemcpyAsync(&v, static_cast<const double*>(keys.get()) + zeros + i, 8, cudaMemcpyDeviceToHost, st));
        UMCG_CUDA(cudaStreamSynchronize(st));
        return v;
    }
};

void sort_axis(double* in, uint64_t n, SortedAxis& out, cudaStream_t st) {
    out.total = n;
    double* o = out.keys.as<double>(n ? n : 1);
    if (n) {
        // ascending doubles = ascending order-preserving u64 keys (radix.cu)
        DevBuf kb, tmp, rs_hist, rs_scan;
        uint64_t* k = kb.as<uint64_t>(n);
        k_double_keys<<<gblocks(n), GT, 0, st>>>(in, n, k);
        UMCG_LAUNCHED();
        radix_sort_u64(k, reinterpret_cast<uint64_t*>(o), nullptr, nullptr, n, 0, 64, tmp, rs_hist, rs_scan, st);
        k_keys_double<<<gblocks(n), GT, 0, st>>>(reinterpret_cast<uint64_t*>(o), n);
        UMCG_LAUNCHED();
    }
    DevBuf zb;
    auto* z = zb.as<unsigned long long>(1);
    UMCG_CUDA(cudaMemsetAsync(z, 0, 8, st));
    if (n) {
        k_count_zero<<<gblocks(n), GT, 0, st>>>(o, n, z);
        UMCG_LAUNCHED();
    }
    unsigned long long hz = 0;
    UMCG_CUDA(cudaMemcpyAsync(&hz, z, 8, cudaMemcpyDeviceToHost, st));
    UMCG_CUDA(cudaStreamSynchronize(st));
    out.zeros = hz;
}

}  // namespace

void grid_init_gpu(int D, uint64_t n_v, const double* xyz, int arity, uint64_t n_c, const uint64_t* cells,
                   double pk, uint64_t g_max, double delta, double thr, std::vector<std::vector<double>>& axes,
                   cudaStream_t st) {
    // validate_config (grid_builder.hpp:25-33)
    if (!(pk > 0.0) || pk > 100.0) fail(UMCG_ERROR, "percentile must be in (0, 100]");
    if (g_max < 2) fail(UMCG_ERROR, "g_max must be >= 2");
    if (!(delta > 0.0)) fail(UMCG_ERROR, "delta must be positive");
    if (!(thr > 0.0) || thr > 1.0) fail(UMCG_ERROR, "seed-mode threshold must be in (0, 1]");
    if (D != 2 && D != 3) fail(UMCG_MALFORMED_FILE, "mesh dimension must be 2 or 3");
    if (!n_v) fail(UMCG_DEGENERATE_MESH, "mesh has no vertices");
    // collect_extrema (:61-74)
    DevBuf mmb;
    auto* mm = mmb.as<unsigned long long>(6);
    std::vector<unsigned long long> init = {~0ull, 0ull, ~0ull, 0ull, ~0ull, 0ull};
    UMCG_CUDA(cudaMemcpyAsync(mm, init.data(), 48, cudaMemcpyHostToDevice, st));
    k_minmax_axis<<<gblocks(n_v), GT, 0, st>>>(xyz, D, n_v, mm);
    UMCG_LAUNCHED();
    std::vector<unsigned long long> hm(6);
    UMCG_CUDA(cudaMemcpyAsync(hm.data(), mm, 48, cudaMemcpyDeviceToHost, st));
    UMCG_CUDA(cudaStreamSynchronize(st));
    double lo[3], hi[3];
    for (int d = 0; d < D; ++d) {
        lo[d] = dkey_inv(hm[2 * d]);
        hi[d] = dkey_inv(hm[2 * d + 1]);
    }
    // deltas per axis: cell edges (traverse_mesh) or 1-NN (knn_edge_stats)
    std::vector<SortedAxis> sorted(D);
    DevBuf dl;
    if (n_c > 0 && arity != 0) {
        int edges[12][2];
        int n_e = 0;
        if (arity == 3) { int e[3][2] = {{0, 1}, {1, 2}, {2, 0}}; n_e = 3; std::memcpy(edges, e, sizeof e); }
        else if (arity == 4) { int e[4][2] = {{0, 1}, {1, 2}, {2, 3}, {3, 0}}; n_e = 4; std::memcpy(edges, e, sizeof e); }
        else if (arity == 8) {
            int e[12][2] = {{0, 1}, {1, 2}, {2, 3}, {3, 0}, {4, 5}, {5, 6}, {6, 7}, {7, 4}, {0, 4}, {1, 5}, {2, 6}, {3, 7}};
            n_e = 12;
            std::memcpy(edges, e, sizeof e);
        } else {
            fail(UMCG_MALFORMED_FILE, "unsupported cell arity " + std::to_string(arity));
        }
        UMCG_CUDA(cudaMemcpyToSymbolAsync(c_edges, edges, sizeof edges, 0, cudaMemcpyHostToDevice, st));
        const uint64_t ne = n_c * (uint64_t)n_e;
        double* buf = dl.as<double>(ne);
        DevBuf cb;
        auto* ctl = cb.as<DevCtl>(1);
        UMCG_CUDA(cudaMemsetAsync(ctl, 0, sizeof(DevCtl), st));
        for (int d = 0; d < D; ++d) {
            k_cell_deltas<<<gblocks(ne), GT, 0, st>>>(xyz, D, n_v, cells, n_c, arity, n_e, d, buf, ctl);
            UMCG_LAUNCHED();
            sort_axis(buf, ne, sorted[d], st);
        }
        int err = 0;
        UMCG_CUDA(cudaMemcpyAsync(&err, &ctl->err, 4, cudaMemcpyDeviceToHost, st));
        UMCG_CUDA(cudaStreamSynchronize(st));
        if (err) fail(UMCG_INDEX_OUT_OF_RANGE, "cell references a vertex out of range");
    } else if (n_v >= 2) {
        KnnGrid g{};
        g.D = D;
        g.per_axis = std::max<uint64_t>(1, (uint64_t)std::floor(std::pow((double)n_v, 1.0 / D)));
        double min_sep = std::numeric_limits<double>::infinity();
        const double cell_w = 1.0 / (double)g.per_axis;
        for (int d = 0; d < D; ++d) {
            g.lo[d] = lo[d];
            const double s = hi[d] - lo[d];
            g.span[d] = s > 0 ? s : 1.0;
            min_sep = std::min(min_sep, g.span[d] * cell_w);
        }
        g.min_sep = min_sep;
        uint64_t nb = 1;
        for (int d = 0; d < D; ++d) nb *= g.per_axis;
        DevBuf kb, ib, cntb, stb, sk, si, tmp;
        auto* key = kb.as<uint64_t>(n_v);
        auto* idx = ib.as<uint32_t>(n_v);
        auto* cnt = cntb.as<uint32_t>(nb + 1);
        auto* start = stb.as<uint32_t>(nb + 1);
        UMCG_CUDA(cudaMemsetAsync(cnt, 0, (nb + 1) * 4, st));
        k_knn_keys<<<gblocks(n_v), GT, 0, st>>>(xyz, n_v, g, key, idx, cnt);
        UMCG_LAUNCHED();
        DevBuf rs_hist, rs_scan;
        UMCG_CUDA(cudaMemcpyAsync(start, cnt, (nb + 1) * 4, cudaMemcpyDeviceToDevice, st));
        exclusive_scan_u32(start, nb + 1, rs_scan, st);
        auto* ks = sk.as<uint64_t>(n_v);
        auto* is = si.as<uint32_t>(n_v);
        int end_bit = 1;
        while (end_bit < 64 && (1ull << end_bit) < nb) ++end_bit;
        radix_sort_u64(key, ks, idx, is, n_v, 0, end_bit, tmp, rs_hist, rs_scan, st);
        double* buf = dl.as<double>(n_v * D);
        k_knn<<<gblocks(n_v), GT, 0, st>>>(xyz, n_v, g, start, is, buf);
        UMCG_LAUNCHED();
        for (int d = 0; d < D; ++d) sort_axis(buf + d * n_v, n_v, sorted[d], st);
    }
    // spacing per axis (grid_init, :224-270)
    axes.assign(D, {});
    for (int d = 0; d < D; ++d) {
        auto& axis = axes[d];
        const double a = lo[d], b = hi[d];
        double gs = 0.0;
        bool degenerate = b <= a;
        const SortedAxis& S = sorted[d];
        const uint64_t kept = S.total - S.zeros;
        auto percentile = [&](double k) -> double {  // :201-214
            const double nk = (double)kept;
            uint64_t rank = (uint64_t)std::ceil(k / 100.0 * nk);
            rank = std::clamp<uint64_t>(rank, 1, kept);
            return S.at(rank - 1, st);
        };
        if (!degenerate) {
            if (kept == 0) {
                degenerate = true;  // empty_after_filtering
            } else {
                double k = pk;
                gs = percentile(k);
                double gn = (b - a) / gs;
                while (gn >= (double)g_max) {
                    if (k >= 100.0) {
                        gs = (b - a) / (double)(g_max - 1);
                        break;
                    }
                    k = std::min(100.0, k + delta);
                    gs = percentile(k);
                    gn = (b - a) / gs;
                }
            }
        }
        if (degenerate) {
            axis = {a};
        } else {
            const double gn = (b - a) / gs;
            const auto steps = (uint64_t)std::floor(gn);
            axis.reserve(steps + 2);
            for (uint64_t t = 0; t <= steps; ++t) axis.push_back(a + (double)t * gs);
            if (b - axis.back() > gs / 2.0) axis.push_back(b);
        }
    }
    // validate_grid (grid.hpp:34-47)
    for (int d = 0; d < D; ++d)
        for (size_t i = 1; i < axes[d].size(); ++i)
            if (!(axes[d][i] > axes[d][i - 1])) fail(UMCG_MALFORMED_FILE, "grid axis not strictly increasing");
}

}  // namespace umcg
