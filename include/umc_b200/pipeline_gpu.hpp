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
// mapping digest) is cached by CONTENT: every call fingerprints the mapping
// (assignments, visited nodes, mode), the grid axes and, for multilinear g,
// the vertex coordinates (a multi-threaded 64-bit word hash, ~10 ms per GB)
// and reuses a plan only when all of it matches -- an in-place edit of a
// MappingTable, or a new one at a recycled address, gets a new plan, as the
// reference recomputes mapping_digest on every call (pipeline.hpp:135, 188).
// The cache keeps the UMCG_PLAN_CACHE (default 4) most recently used plans;
// umc::b200::clear_plan_cache() drops them all.
#ifndef UMC_B200_PIPELINE_GPU_HPP
#define UMC_B200_PIPELINE_GPU_HPP

#include <cstdint>
#include <cstring>
#include <map>
#include <memory>
#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <list>
#include <mutex>
#include <thread>
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

// 64-bit fingerprint of a byte range: a multiply-rotate hash per 8-byte word,
// per 64 MiB chunk on its own thread, chunk hashes combined in order.
inline std::uint64_t hash_words(const std::uint64_t* w, std::size_t n, std::uint64_t h) {
    for (std::size_t i = 0; i < n; ++i) {
        h ^= w[i] * 0x9e3779b97f4a7c15ull;
        h = ((h << 31) | (h >> 33)) * 0xbf58476d1ce4e5b9ull;
    }
    return h;
}
inline std::uint64_t fingerprint(const void* data, std::size_t bytes) {
    const auto* p = static_cast<const std::uint8_t*>(data);
    const std::size_t nw = bytes / 8;
    constexpr std::size_t kChunk = (64u << 20) / 8;
    const std::size_t nc = nw ? (nw + kChunk - 1) / kChunk : 0;
    std::vector<std::uint64_t> part(nc, 0);
    auto run = [&](std::size_t c) {
        const std::size_t a = c * kChunk, b = std::min(nw, a + kChunk);
        part[c] = hash_words(reinterpret_cast<const std::uint64_t*>(p) + a, b - a, 0x243f6a8885a308d3ull ^ c);
    };
    if (nc <= 1) {
        if (nc) run(0);
    } else {
        const unsigned hw = std::max(1u, std::min<unsigned>(std::thread::hardware_concurrency(), 32u));
        std::vector<std::thread> th;
        std::atomic<std::size_t> next{0};
        for (unsigned t = 0; t < std::min<std::size_t>(hw, nc); ++t)
            th.emplace_back([&] {
                for (std::size_t c; (c = next.fetch_add(1)) < nc;) run(c);
            });
        for (auto& t : th) t.join();
    }
    std::uint64_t h = 0x13198a2e03707344ull ^ bytes;
    for (std::size_t c = 0; c < nc; ++c) h = hash_words(&part[c], 1, h);
    std::uint64_t tail = 0;
    std::memcpy(&tail, p + nw * 8, bytes - nw * 8);
    return hash_words(&tail, 1, h);
}

struct PlanKey {
    int mode, dim;
    std::size_t n, n_visited, grid_nodes;
    bool coords;
    std::uint64_t h_assign, h_visited, h_axes, h_coords;
    bool operator==(const PlanKey& o) const {
        return std::tie(mode, dim, n, n_visited, grid_nodes, coords, h_assign, h_visited, h_axes, h_coords) ==
               std::tie(o.mode, o.dim, o.n, o.n_visited, o.grid_nodes, o.coords, o.h_assign, o.h_visited,
                        o.h_axes, o.h_coords);
    }
};

inline PlanKey plan_key(const MappingTable& map, const RectGrid& grid, const Mesh& mesh, bool coords) {
    PlanKey k{};
    k.mode = map.mode == MappingMode::seed ? 1 : 0;
    k.dim = grid.dim;
    k.n = map.assignments.size();
    k.n_visited = map.visited_nodes.size();
    k.grid_nodes = grid.node_count();
    k.coords = coords;
    k.h_assign = fingerprint(map.assignments.data(), map.assignments.size() * 8);
    k.h_visited = fingerprint(map.visited_nodes.data(), map.visited_nodes.size() * 8);
    std::uint64_t h = 0;
    for (const auto& a : grid.axes) h = hash_words(&h, 1, fingerprint(a.data(), a.size() * 8) ^ a.size());
    k.h_axes = h;
    k.h_coords = coords ? fingerprint(mesh.vertices.data(), mesh.vertices.size() * 8) : 0;
    return k;
}

inline std::mutex& cache_mutex() {
    static std::mutex m;
    return m;
}
// most recently used first
inline std::list<std::pair<PlanKey, PlanPtr>>& cache() {
    static std::list<std::pair<PlanKey, PlanPtr>> c;
    return c;
}
inline std::size_t cache_capacity() {
    const char* e = std::getenv("UMCG_PLAN_CACHE");
    const long v = e ? std::strtol(e, nullptr, 10) : 4;
    return v > 0 ? static_cast<std::size_t>(v) : 1;
}
inline std::atomic<std::uint64_t>& cache_generation() {
    static std::atomic<std::uint64_t> g{0};
    return g;
}

// Each host thread works on its own clone of a cached plan (umcg_plan_clone:
// own workspace, shared mapping arrays; a clone keeps its origin's arrays
// alive), so concurrent calls on one MappingTable run concurrently, as the
// reference allows. Clones are dropped when the cache
// changes generation (eviction, clear_plan_cache).
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
    const PlanKey key = plan_key(map, grid, mesh, coords);  // outside the lock: the expensive part
    std::lock_guard<std::mutex> lock(cache_mutex());
    auto& c = cache();
    for (auto it = c.begin(); it != c.end(); ++it)
        if (it->first == key) {
            c.splice(c.begin(), c, it);  // most recently used
            return thread_handle(c.front().second.get());
        }
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
    c.emplace_front(key, PlanPtr(p));
    if (c.size() > cache_capacity()) {
        c.pop_back();  // least recently used; clones held by threads keep its arrays alive
        cache_generation().fetch_add(1);
    }
    return thread_handle(p);
}

// Per-thread pinned staging for archive bytes coming back from the device
// (D2H into pinned memory runs at the link rate; no zero-fill of a
// capacity-sized std::vector per call).
struct PinnedStage {
    void* p = nullptr;
    std::size_t cap = 0;
    ~PinnedStage() {
        if (p) cudaFreeHost(p);
    }
    std::uint8_t* get(std::size_t bytes) {
        if (bytes > cap) {
            if (p) cudaFreeHost(p);
            p = nullptr;
            cap = 0;
            if (cudaMallocHost(&p, bytes) != cudaSuccess) throw error("cudaMallocHost failed");
            cap = bytes;
        }
        return static_cast<std::uint8_t*>(p);
    }
};
inline PinnedStage& stage() {
    thread_local PinnedStage s;
    return s;
}

inline std::uint64_t rd_le(const std::uint8_t* b, int k) {
    std::uint64_t v = 0;
    for (int i = 0; i < k; ++i) v |= static_cast<std::uint64_t>(b[i]) << (8 * i);
    return v;
}
inline void put_le(std::vector<std::uint8_t>& w, std::uint64_t v, int k) {
    for (int i = 0; i < k; ++i) w.push_back(static_cast<std::uint8_t>(v >> (8 * i)));
}

// The UMCZ container header through component 1's length, and component 2's
// length (serialize_archive, pipeline.hpp:214-235), without the payloads.
inline void archive_frame(const Archive& ar, std::vector<std::uint8_t>& head, std::vector<std::uint8_t>& mid) {
    if (ar.field_name.size() > 0xffff) throw malformed_file("field name too long");
    head = {'U', 'M', 'C', 'Z'};
    put_le(head, kFormatVersion, 2);
    std::uint16_t flags = 0;
    if (ar.seed_mode) flags |= 1u;
    if (ar.g_kind == BackInterpKind::multilinear) flags |= 2u;
    if (ar.bound_kind == BoundKind::relative_to_range) flags |= 4u;
    if (ar.baseline) flags |= 8u;
    put_le(head, flags, 2);
    put_le(head, ar.field_name.size(), 2);
    head.insert(head.end(), ar.field_name.begin(), ar.field_name.end());
    put_le(head, ar.map_digest, 8);
    std::uint64_t u;
    std::memcpy(&u, &ar.tau, 8);
    put_le(head, u, 8);
    std::memcpy(&u, &ar.rho, 8);
    put_le(head, u, 8);
    put_le(head, ar.component1.payload.size(), 8);
    mid.clear();
    put_le(mid, ar.component2.payload.size(), 8);
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
    // validate_field (mesh.hpp:58-64): the length check here; finiteness is
    // checked on the device in the same pass that reads the field, and
    // reported before any budget error, in the reference's order
    if (field.values.size() != mesh.vertex_count())
        throw malformed_file("field length " + std::to_string(field.values.size()) +
                             " does not match vertex count " + std::to_string(mesh.vertex_count()));
    if (field.values.size() != map.assignments.size()) {
        validate_field(field, mesh);  // a non-finite value still wins, as in the reference
        throw mapping_mismatch("mapping was built for a different vertex count");
    }
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
    std::uint8_t* b = detail::stage().get(cap);
    std::uint64_t len = 0;
    detail::check(umcg_compress_host(plan, &prm, field.values.data(), field.name.c_str(), b, cap, &len));
    // the Archive of deserialize_archive (pipeline.hpp:237-267), built from the
    // staged bytes: header fields, then each payload copied once into its
    // component and parsed by the reference's parse_component
    Archive ar;
    const std::uint64_t flags = detail::rd_le(b + 6, 2), nl = detail::rd_le(b + 8, 2);
    ar.seed_mode = flags & 1u;
    ar.g_kind = (flags & 2u) ? BackInterpKind::multilinear : BackInterpKind::nearest;
    ar.bound_kind = (flags & 4u) ? BoundKind::relative_to_range : BoundKind::absolute;
    ar.baseline = flags & 8u;
    ar.field_name.assign(reinterpret_cast<const char*>(b + 10), nl);
    std::uint64_t o = 10 + nl;
    ar.map_digest = detail::rd_le(b + o, 8);
    std::uint64_t u = detail::rd_le(b + o + 8, 8);
    std::memcpy(&ar.tau, &u, 8);
    u = detail::rd_le(b + o + 16, 8);
    std::memcpy(&ar.rho, &u, 8);
    o += 24;
    const std::uint64_t l1 = detail::rd_le(b + o, 8);
    ar.component1 = parse_component(std::vector<std::uint8_t>(b + o + 8, b + o + 8 + l1));
    o += 8 + l1;
    const std::uint64_t l2 = detail::rd_le(b + o, 8);
    ar.component2 = parse_component(std::vector<std::uint8_t>(b + o + 8, b + o + 8 + l2));
    if (o + 8 + l2 != len) throw internal_inconsistency("archive length");
    return ar;
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
    // the archive's bytes (serialize_archive) uploaded piece by piece: the
    // header, payload 1, component 2's length, payload 2
    std::vector<std::uint8_t> head, mid;
    detail::archive_frame(archive, head, mid);
    const std::uint8_t* parts[4] = {head.data(), archive.component1.payload.data(), mid.data(),
                                    archive.component2.payload.data()};
    const std::uint64_t lens[4] = {head.size(), archive.component1.payload.size(), mid.size(),
                                   archive.component2.payload.size()};
    detail::check(umcg_decompress_host_parts(plan, parts, lens, 4, out.values.data()));
    return out;
}

}  // namespace b200
}  // namespace umc

#endif  // UMC_B200_PIPELINE_GPU_HPP
