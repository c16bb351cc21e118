// Drop-in GPU replacement for umc::compress / umc::decompress
// (reference proj/include/umc/pipeline.hpp:117-148, 180-210).
//
// Include this header next to the reference's own headers and call
// umc::b200::compress / umc::b200::decompress with exactly the arguments of
// the reference functions. Archives are byte-identical to the reference's
// (up to rounding-window code flips) and every
// failure is rethrown as the reference's exception type (common.hpp:19-38).
// Link with libumcg.so (paper_2501_06910_b200/libumcg.so) and the CUDA
// runtime. There is no CPU fallback: without a usable GPU the calls throw.
//
// Plans: the device plan (mapping upload, slot sort, bucketed layout,
// mapping digest) is built once per distinct MappingTable object and cached
// by address + content size; mutate a MappingTable only through a new
// object (the reference treats mappings as immutable) or
// call umc::b200::clear_plan_cache().
#ifndef UMC_B200_PIPELINE_GPU_HPP
#define UMC_B200_PIPELINE_GPU_HPP

#include <cstdint>
#include <cstring>
#include <map>
#include <memory>
#include <atomic>
#include <mutex>
#include <string>
#include <tuple>
#include <vector>

#include <cuda_runtime_api.h>

#include "umc/grid_builder.hpp"
#include "umc/pipeline.hpp"
#include "../umcg.h"

namespace umc {
namespace b200 {

namespace detail {

[[noreturn]] inline void rethrow(umcg_status s) {
    const std::string msg = umcg_last_error();
    switch (s) {
        case UMCG_MALFORMED_FILE: throw malformed_file(msg);
        case UMCG_INDEX_OUT_OF_RANGE: throw index_out_of_range(msg);
        case UMCG_NON_FINITE_VALUE: throw non_finite_value(msg);
        case UMCG_IO_FAILURE: throw io_failure(msg);
        case UMCG_DEGENERATE_MESH: throw degenerate_mesh(msg);
        case UMCG_EMPTY_AFTER_FILTERING: throw empty_after_filtering(msg);
        case UMCG_INTERNAL_INCONSISTENCY: throw internal_inconsistency(msg);
        case UMCG_SEED_MODE_UNSUPPORTED: throw seed_mode_unsupported(msg);
        case UMCG_UNKNOWN_CODEC: throw unknown_codec(msg);
        case UMCG_CORRUPT_PAYLOAD: throw corrupt_payload(msg);
        case UMCG_EXTERNAL_CODEC_VIOLATION: throw external_codec_violation(msg);
        case UMCG_SUBPROCESS_FAILURE: throw subprocess_failure(msg);
        case UMCG_BUDGET_INADMISSIBLE: throw budget_inadmissible(msg);
        case UMCG_MAPPING_MISMATCH: throw mapping_mismatch(msg);
        case UMCG_ZERO_NORM_REFERENCE: throw zero_norm_reference(msg);
        case UMCG_MISMATCHED_RUNS: throw mismatched_runs(msg);
        default: throw error(msg);
    }
}

inline void check(umcg_status s) {
    if (s != UMCG_OK) rethrow(s);
}

struct PlanDeleter {
    void operator()(umcg_plan* p) const { umcg_plan_destroy(p); }
};
using PlanPtr = std::unique_ptr<umcg_plan, PlanDeleter>;

struct PlanKey {
    const MappingTable* map;
    const void* assign_data;
    std::size_t n;
    std::size_t n_visited;
    std::uint64_t grid_nodes;
    bool coords;
    bool operator<(const PlanKey& o) const {
        return std::tie(map, assign_data, n, n_visited, grid_nodes, coords) <
               std::tie(o.map, o.assign_data, o.n, o.n_visited, o.grid_nodes, o.coords);
    }
};

inline std::mutex& cache_mutex() {
    static std::mutex m;
    return m;
}
inline std::map<PlanKey, PlanPtr>& cache() {
    static std::map<PlanKey, PlanPtr> c;
    return c;
}
inline std::atomic<std::uint64_t>& cache_generation() {
    static std::atomic<std::uint64_t> g{0};
    return g;
}

// Each host thread works on its own clone of a cached plan (umcg_plan_clone:
// own workspace, shared mapping arrays), so concurrent calls on one
// MappingTable run concurrently, as the reference allows.
inline umcg_plan* thread_handle(umcg_plan* origin) {
    thread_local std::uint64_t gen = 0;
    thread_local std::map<umcg_plan*, PlanPtr> clones;
    const std::uint64_t g = cache_generation().load();
    if (gen != g) {
        clones.clear();
        gen = g;
    }
    auto it = clones.find(origin);
    if (it != clones.end()) return it->second.get();
    umcg_plan* c = nullptr;
    check(umcg_plan_clone(origin, &c));
    clones.emplace(origin, PlanPtr(c));
    return c;
}

// Device plan for (map, grid, mesh); coordinates are uploaded only when the
// caller needs multilinear g.
inline umcg_plan* plan_for(const MappingTable& map, const RectGrid& grid, const Mesh& mesh, bool coords) {
    const PlanKey key{&map, map.assignments.data(), map.assignments.size(), map.visited_nodes.size(),
                      grid.node_count(), coords};
    std::lock_guard<std::mutex> lock(cache_mutex());
    auto it = cache().find(key);
    if (it != cache().end()) return thread_handle(it->second.get());
    std::vector<std::uint64_t> sizes;
    std::vector<double> axes;
    for (const auto& a : grid.axes) {
        sizes.push_back(a.size());
        axes.insert(axes.end(), a.begin(), a.end());
    }
    umcg_grid_desc g{grid.dim, sizes.data(), axes.data()};
    umcg_mapping_desc m{map.mode == MappingMode::seed ? 1 : 0, map.assignments.size(), map.assignments.data(),
                        map.visited_nodes.size(), map.visited_nodes.data()};
    umcg_plan* p = nullptr;
    check(umcg_plan_create(&g, &m, mesh.dim, coords ? mesh.vertices.data() : nullptr, &p));
    cache().emplace(key, PlanPtr(p));
    return thread_handle(p);
}

}  // namespace detail

inline void clear_plan_cache() {
    std::lock_guard<std::mutex> lock(detail::cache_mutex());
    detail::cache().clear();  // threads drop their clones on their next call
    detail::cache_generation().fetch_add(1);
}

/// umc::compress (pipeline.hpp:117-148) on the GPU. Same arguments, same
/// Archive, same exception types.
inline Archive compress(const Field& field, const MappingTable& map, const RectGrid& grid, const Mesh& mesh,
                        const ErrorBudget& budget, const CompressOptions& opt = {}) {
    validate_field(field, mesh);  // mesh.hpp:58-64, host-side like the reference
    if (field.values.size() != map.assignments.size())
        throw mapping_mismatch("mapping was built for a different vertex count");
    umcg_plan* plan = detail::plan_for(map, grid, mesh, opt.g.kind == BackInterpKind::multilinear);
    umcg_params prm{budget.tau,
                    budget.split_rho,
                    budget.bound_kind == BoundKind::relative_to_range ? 1 : 0,
                    opt.g.kind == BackInterpKind::multilinear ? 1 : 0,
                    opt.g.coeff_abs_sum,
                    opt.fill == FillPolicy::nearest_visited ? 1 : 0,
                    opt.codec_id,
                    opt.backend_id};
    std::uint64_t cap = 0;
    detail::check(umcg_compress_bound(plan, field.name.c_str(), &cap));
    std::vector<std::uint8_t> bytes(cap);
    std::uint64_t len = 0;
    detail::check(umcg_compress_host(plan, &prm, field.values.data(), field.name.c_str(), bytes.data(), cap, &len));
    bytes.resize(len);
    return deserialize_archive(bytes);  // pipeline.hpp:237 builds the reference's Archive
}

namespace detail {
inline void validate_config_host(const GridBuildConfig& cfg) { validate_config(cfg); }  // grid_builder.hpp:25-33

struct DeviceCoords {
    void* p = nullptr;
    ~DeviceCoords() { cudaFree(p); }
};
}  // namespace detail

/// umc::grid_init (grid_builder.hpp:224-282) on the GPU: same RectGrid.
inline RectGrid grid_init(const Mesh& mesh, const GridBuildConfig& cfg = {}) {
    detail::validate_config_host(cfg);
    const std::uint64_t n = mesh.vertex_count();
    const std::uint64_t nc = mesh.cell_count();
    detail::DeviceCoords dc, dl;
    if (cudaMalloc(&dc.p, mesh.vertices.size() * 8 + 8) != cudaSuccess ||
        cudaMalloc(&dl.p, mesh.cells.size() * 8 + 8) != cudaSuccess)
        throw error("cudaMalloc failed");
    cudaMemcpy(dc.p, mesh.vertices.data(), mesh.vertices.size() * 8, cudaMemcpyHostToDevice);
    if (nc) cudaMemcpy(dl.p, mesh.cells.data(), mesh.cells.size() * 8, cudaMemcpyHostToDevice);
    const umcg_grid_config c{cfg.percentile_k, cfg.g_max, cfg.delta, cfg.seed_mode_threshold};
    std::uint64_t sizes[3] = {0, 0, 0};
    const auto* cells = nc ? static_cast<const std::uint64_t*>(dl.p) : nullptr;
    detail::check(umcg_grid_init(mesh.dim, n, static_cast<const double*>(dc.p), mesh.cell_arity, nc, cells, &c, sizes,
                                 nullptr, 0, nullptr));
    std::uint64_t tot = 0;
    for (int d = 0; d < mesh.dim; ++d) tot += sizes[d];
    std::vector<double> cat(tot);
    detail::check(umcg_grid_init(mesh.dim, n, static_cast<const double*>(dc.p), mesh.cell_arity, nc, cells, &c, sizes,
                                 cat.data(), tot, nullptr));
    RectGrid grid;
    grid.dim = mesh.dim;
    grid.axes.resize(mesh.dim);
    std::uint64_t o = 0;
    for (int d = 0; d < mesh.dim; ++d) {
        grid.axes[d].assign(cat.begin() + o, cat.begin() + o + sizes[d]);
        o += sizes[d];
    }
    return grid;
}

/// umc::grid_coarsen (grid_builder.hpp:365-421) on the GPU: same mapping,
/// coarsened grid and mode (umcg_plan_build + umcg_plan_export).
inline CoarsenResult grid_coarsen(const Mesh& mesh, const RectGrid& grid, const GridBuildConfig& cfg) {
    detail::validate_config_host(cfg);
    const std::uint64_t n = mesh.vertex_count();
    std::vector<std::uint64_t> sizes;
    std::vector<double> axes;
    for (const auto& a : grid.axes) {
        sizes.push_back(a.size());
        axes.insert(axes.end(), a.begin(), a.end());
    }
    umcg_grid_desc g{grid.dim, sizes.data(), axes.data()};
    detail::DeviceCoords dc;
    if (cudaMalloc(&dc.p, mesh.vertices.size() * 8 + 8) != cudaSuccess) throw error("cudaMalloc failed");
    cudaMemcpy(dc.p, mesh.vertices.data(), mesh.vertices.size() * 8, cudaMemcpyHostToDevice);
    umcg_plan* p = nullptr;
    detail::check(umcg_plan_build(&g, n, static_cast<const double*>(dc.p), cfg.seed_mode_threshold, 0, &p));
    detail::PlanPtr holder(p);
    umcg_plan_info info{};
    detail::check(umcg_plan_get_info(p, &info));
    CoarsenResult res;
    res.mapping.mode = info.mode ? MappingMode::seed : MappingMode::dense;
    res.mapping.assignments.resize(n);
    std::vector<std::uint64_t> visited(info.n_visited);
    std::uint64_t tot = 0;
    for (int d = 0; d < info.dim; ++d) tot += info.shape[d];
    std::vector<double> cax(tot);
    detail::check(umcg_plan_export(p, res.mapping.assignments.data(), visited.data(), cax.data()));
    if (info.mode) res.mapping.visited_nodes = std::move(visited);
    res.mapping.visited_fraction = info.visited_fraction;
    res.grid.dim = info.dim;
    res.grid.axes.resize(info.dim);
    std::uint64_t o = 0;
    for (int d = 0; d < info.dim; ++d) {
        res.grid.axes[d].assign(cax.begin() + o, cax.begin() + o + info.shape[d]);
        o += info.shape[d];
    }
    return res;
}

/// umc::compress_baseline (pipeline.hpp:152-162) on the GPU: one 1-D
/// component at tau_abs (umcg_encode, codec 0 or 1).
inline EncodedComponent compress_baseline(const Field& field, double tau_abs,
                                          std::uint8_t codec_id = kCodecBuiltinPQ, std::uint8_t backend_id = 0) {
    const std::uint64_t n = field.values.size();
    void* d_v = nullptr;
    void* d_p = nullptr;
    const std::uint64_t cap = umcg_encode_bound(n, 1);
    if (cudaMalloc(&d_v, n * 8 + 8) != cudaSuccess || cudaMalloc(&d_p, cap) != cudaSuccess) {
        cudaFree(d_v);
        throw error("cudaMalloc failed");
    }
    if (n) cudaMemcpy(d_v, field.values.data(), n * 8, cudaMemcpyHostToDevice);
    const std::uint64_t dims[1] = {n};
    std::uint64_t len = 0;
    const umcg_status s = umcg_encode(static_cast<const double*>(d_v), n, 1, 1, dims, tau_abs, codec_id, backend_id,
                                      static_cast<std::uint8_t*>(d_p), cap, &len, nullptr);
    EncodedComponent comp;
    if (s == UMCG_OK) {
        comp.payload.resize(len);
        cudaMemcpy(comp.payload.data(), d_p, len, cudaMemcpyDeviceToHost);
    }
    cudaFree(d_v);
    cudaFree(d_p);
    detail::check(s);
    comp.spec.codec_id = codec_id;
    comp.spec.backend_id = backend_id;
    comp.spec.predictor = Predictor::lorenzo_1d;
    comp.spec.dims = {n};
    comp.spec.tau_abs = tau_abs;
    comp.n_elements = n;
    comp.original_bytes = n * 8;
    return comp;
}

/// umc::baseline_archive (pipeline.hpp:164-176) on the GPU.
inline Archive baseline_archive(const Field& field, const ErrorBudget& budget,
                                std::uint8_t codec_id = kCodecBuiltinPQ, std::uint8_t backend_id = 0) {
    Archive ar;
    ar.baseline = true;
    ar.bound_kind = budget.bound_kind;
    ar.field_name = field.name;
    ar.tau = budget.tau;
    ar.rho = budget.split_rho;
    ar.component1 = b200::compress_baseline(field, resolve_tau_abs(budget, field.values), codec_id, backend_id);
    return ar;
}

/// umc::decompress (pipeline.hpp:180-210) on the GPU.
inline Field decompress(const Archive& archive, const MappingTable& map, const RectGrid& grid, const Mesh& mesh) {
    const auto bytes = serialize_archive(archive);
    Field out;
    out.name = archive.field_name;
    if (archive.baseline) {  // pipeline.hpp:184-187: the single component, decoded on the device
        const auto& p = archive.component1.payload;
        const std::uint64_t n = archive.component1.n_elements;
        void* d_p = nullptr;
        void* d_v = nullptr;
        if (cudaMalloc(&d_p, p.size() + 1) != cudaSuccess || cudaMalloc(&d_v, n * 8 + 8) != cudaSuccess) {
            cudaFree(d_p);
            throw error("cudaMalloc failed");
        }
        cudaMemcpy(d_p, p.data(), p.size(), cudaMemcpyHostToDevice);
        std::uint64_t got = 0;
        const umcg_status s = umcg_decode(static_cast<const std::uint8_t*>(d_p), p.size(),
                                          static_cast<double*>(d_v), n, &got, nullptr);
        out.values.resize(got);
        if (s == UMCG_OK && got) cudaMemcpy(out.values.data(), d_v, got * 8, cudaMemcpyDeviceToHost);
        cudaFree(d_p);
        cudaFree(d_v);
        detail::check(s);
        return out;
    }
    umcg_plan* plan = detail::plan_for(map, grid, mesh, archive.g_kind == BackInterpKind::multilinear);
    out.values.resize(map.assignments.size());
    detail::check(umcg_decompress_host(plan, bytes.data(), bytes.size(), out.values.data()));
    return out;
}

}  // namespace b200
}  // namespace umc

#endif  // UMC_B200_PIPELINE_GPU_HPP
