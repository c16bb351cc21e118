// TEST INFRASTRUCTURE ONLY -- never linked into the product library.
//
// extern "C" shim over the UNMODIFIED reference library (header-only C++20,
// /root/reference/proj/include/umc). Built by oracle/Makefile into
// oracle/_ref/libumcref.so straight from the reference headers (nothing is
// copied). Used by the parity tests as the reference oracle, by the golden
// fixture generator, and by bench.py's cpu_baseline / --impl reference arm.
//
// Every entry point is a thin marshalling layer: host arrays in, host arrays
// out, exceptions mapped to the reference's error taxonomy
// (common.hpp:19-38) as small integers (see ERROR_KINDS in
// paper_2501_06910_b200/errors.py, same order as include/umcg.h).

#include <chrono>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "umc/codec.hpp"
#include "umc/datagen.hpp"
#include "umc/grid_builder.hpp"
#include "umc/interp.hpp"
#include "umc/lossless.hpp"
#include "umc/pipeline.hpp"
#include "umc/serialize.hpp"
#include "support/golden_recipe.hpp"  // proj/tests/support: the golden recipe itself

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const umc::mismatched_runs& e) { g_err = e.what(); return 17;
    } catch (const umc::zero_norm_reference& e) { g_err = e.what(); return 16;
    } catch (const umc::mapping_mismatch& e) { g_err = e.what(); return 15;
    } catch (const umc::budget_inadmissible& e) { g_err = e.what(); return 14;
    } catch (const umc::subprocess_failure& e) { g_err = e.what(); return 13;
    } catch (const umc::external_codec_violation& e) { g_err = e.what(); return 12;
    } catch (const umc::corrupt_payload& e) { g_err = e.what(); return 11;
    } catch (const umc::unknown_codec& e) { g_err = e.what(); return 10;
    } catch (const umc::seed_mode_unsupported& e) { g_err = e.what(); return 9;
    } catch (const umc::internal_inconsistency& e) { g_err = e.what(); return 8;
    } catch (const umc::empty_after_filtering& e) { g_err = e.what(); return 7;
    } catch (const umc::degenerate_mesh& e) { g_err = e.what(); return 6;
    } catch (const umc::io_failure& e) { g_err = e.what(); return 5;
    } catch (const umc::non_finite_value& e) { g_err = e.what(); return 4;
    } catch (const umc::index_out_of_range& e) { g_err = e.what(); return 3;
    } catch (const umc::malformed_file& e) { g_err = e.what(); return 2;
    } catch (const umc::error& e) { g_err = e.what(); return 1;
    } catch (const std::exception& e) { g_err = e.what(); return 99; }
}

umc::RectGrid make_grid(int dim, const std::uint64_t* axis_sizes, const double* axes_concat) {
    umc::RectGrid g;
    g.dim = dim;
    g.axes.resize(static_cast<std::size_t>(dim));
    std::size_t off = 0;
    for (int d = 0; d < dim; ++d) {
        g.axes[d].assign(axes_concat + off, axes_concat + off + axis_sizes[d]);
        off += axis_sizes[d];
    }
    return g;
}

umc::MappingTable make_map(int mode, std::uint64_t n_v, const std::uint64_t* assignments,
                           std::uint64_t n_visited, const std::uint64_t* visited) {
    umc::MappingTable m;
    m.mode = mode ? umc::MappingMode::seed : umc::MappingMode::dense;
    m.assignments.assign(assignments, assignments + n_v);
    if (mode) m.visited_nodes.assign(visited, visited + n_visited);
    return m;
}

umc::Mesh make_mesh(int dim, std::uint64_t n_v, const double* coords) {
    umc::Mesh mesh;
    mesh.dim = dim;
    mesh.cell_arity = dim == 2 ? 3 : 4;
    if (coords)
        mesh.vertices.assign(coords, coords + n_v * static_cast<std::uint64_t>(dim));
    else
        mesh.vertices.assign(n_v * static_cast<std::uint64_t>(dim), 0.0);  // nearest g never reads them
    return mesh;
}

std::uint8_t* dup_bytes(const std::vector<std::uint8_t>& v) {
    auto* p = static_cast<std::uint8_t*>(std::malloc(v.size() ? v.size() : 1));
    if (!v.empty()) std::memcpy(p, v.data(), v.size());
    return p;
}

struct Ctx {
    umc::RectGrid grid;
    umc::MappingTable map;
    umc::Mesh mesh;
};

}  // namespace

extern "C" {

const char* umcref_last_error(void) { return g_err.c_str(); }
void umcref_free(void* p) { std::free(p); }

// Persistent context (grid + mapping + mesh) so timing loops do not pay the
// marshalling copies; mirrors how a caller keeps these objects alive.
void* umcref_ctx_create(int dim, const std::uint64_t* axis_sizes, const double* axes_concat,
                        int mode, std::uint64_t n_v, const std::uint64_t* assignments,
                        std::uint64_t n_visited, const std::uint64_t* visited, int mesh_dim,
                        const double* coords) {
    auto* c = new Ctx;
    c->grid = make_grid(dim, axis_sizes, axes_concat);
    c->map = make_map(mode, n_v, assignments, n_visited, visited);
    c->mesh = make_mesh(mesh_dim, n_v, coords);
    return c;
}
void umcref_ctx_destroy(void* c) { delete static_cast<Ctx*>(c); }

// umc::compress (pipeline.hpp:117) + serialize_archive (pipeline.hpp:214).
int umcref_compress_ctx(void* ctx, const double* values, std::uint64_t n, const char* name,
                        double tau, double rho, int bound_kind, int g_kind, double coeff_abs_sum,
                        int fill, int codec_id, int backend_id, std::uint8_t** out,
                        std::uint64_t* out_len) {
    return guarded([&] {
        auto* c = static_cast<Ctx*>(ctx);
        umc::Field f;
        f.name = name ? name : "";
        f.values.assign(values, values + n);
        umc::ErrorBudget b;
        b.tau = tau;
        b.split_rho = rho;
        b.bound_kind = bound_kind ? umc::BoundKind::relative_to_range : umc::BoundKind::absolute;
        umc::CompressOptions opt;
        opt.g.kind = g_kind ? umc::BackInterpKind::multilinear : umc::BackInterpKind::nearest;
        opt.g.coeff_abs_sum = coeff_abs_sum;
        opt.fill = fill ? umc::FillPolicy::nearest_visited : umc::FillPolicy::zero;
        opt.codec_id = static_cast<std::uint8_t>(codec_id);
        opt.backend_id = static_cast<std::uint8_t>(backend_id);
        const auto ar = umc::compress(f, c->map, c->grid, c->mesh, b, opt);
        const auto bytes = umc::serialize_archive(ar);
        *out = dup_bytes(bytes);
        *out_len = bytes.size();
    });
}

// deserialize_archive (pipeline.hpp:237) + umc::decompress (pipeline.hpp:180).
int umcref_decompress_ctx(void* ctx, const std::uint8_t* ar, std::uint64_t len, double* out,
                          std::uint64_t n_cap, std::uint64_t* n_out) {
    return guarded([&] {
        auto* c = static_cast<Ctx*>(ctx);
        const std::vector<std::uint8_t> bytes(ar, ar + len);
        const auto archive = umc::deserialize_archive(bytes);
        const auto f = umc::decompress(archive, c->map, c->grid, c->mesh);
        *n_out = f.values.size();
        if (f.values.size() > n_cap) throw umc::error("output buffer too small");
        std::memcpy(out, f.values.data(), f.values.size() * 8);
    });
}

// Time compress+decompress repeatedly inside the library (steady_clock), so
// the CPU baseline is not polluted by Python overhead. Returns seconds.
int umcref_time_roundtrip(void* ctx, const double* values, std::uint64_t n, double tau,
                          double rho, int bound_kind, int reps, double* t_compress,
                          double* t_decompress, std::uint64_t* archive_bytes) {
    return guarded([&] {
        auto* c = static_cast<Ctx*>(ctx);
        umc::Field f;
        f.name = "x";
        f.values.assign(values, values + n);
        umc::ErrorBudget b;
        b.tau = tau;
        b.split_rho = rho;
        b.bound_kind = bound_kind ? umc::BoundKind::relative_to_range : umc::BoundKind::absolute;
        double tc = 0, td = 0;
        for (int r = 0; r < reps; ++r) {
            const auto t0 = std::chrono::steady_clock::now();
            const auto ar = umc::compress(f, c->map, c->grid, c->mesh, b);
            const auto bytes = umc::serialize_archive(ar);
            const auto t1 = std::chrono::steady_clock::now();
            const auto back = umc::deserialize_archive(bytes);
            const auto out = umc::decompress(back, c->map, c->grid, c->mesh);
            const auto t2 = std::chrono::steady_clock::now();
            tc += std::chrono::duration<double>(t1 - t0).count();
            td += std::chrono::duration<double>(t2 - t1).count();
            *archive_bytes = bytes.size();
            if (out.values.size() != n) throw umc::error("size");
        }
        *t_compress = tc / reps;
        *t_decompress = td / reps;
    });
}

// Single component codec: umc::encode (codec.hpp:220) / umc::decode (:364).
int umcref_encode(const double* v, std::uint64_t n, int predictor, int ndims,
                  const std::uint64_t* dims, double tau, int codec_id, int backend_id,
                  std::uint8_t** out, std::uint64_t* out_len) {
    return guarded([&] {
        umc::CodecSpec spec;
        spec.codec_id = static_cast<std::uint8_t>(codec_id);
        spec.backend_id = static_cast<std::uint8_t>(backend_id);
        spec.predictor = static_cast<umc::Predictor>(predictor);
        spec.dims.assign(dims, dims + ndims);
        spec.tau_abs = tau;
        const auto comp = umc::encode(v, n, spec);
        *out = dup_bytes(comp.payload);
        *out_len = comp.payload.size();
    });
}

// umc::baseline_archive (pipeline.hpp:164-176), serialized.
int umcref_baseline_archive(const double* values, std::uint64_t n, const char* name, double tau, double rho,
                            int bound_kind, int codec_id, std::uint8_t** out, std::uint64_t* out_len) {
    return guarded([&] {
        umc::Field f;
        f.name = name ? name : "";
        f.values.assign(values, values + n);
        umc::ErrorBudget b;
        b.tau = tau;
        b.split_rho = rho;
        b.bound_kind = bound_kind ? umc::BoundKind::relative_to_range : umc::BoundKind::absolute;
        const auto ar = umc::baseline_archive(f, b, static_cast<std::uint8_t>(codec_id));
        const auto bytes = umc::serialize_archive(ar);
        *out = dup_bytes(bytes);
        *out_len = bytes.size();
    });
}

int umcref_decode(const std::uint8_t* p, std::uint64_t len, double* out, std::uint64_t n_cap,
                  std::uint64_t* n_out) {
    return guarded([&] {
        umc::EncodedComponent comp;
        comp.payload.assign(p, p + len);
        const auto v = umc::decode(comp);
        *n_out = v.size();
        if (v.size() > n_cap) throw umc::error("output buffer too small");
        if (!v.empty()) std::memcpy(out, v.data(), v.size() * 8);
    });
}

// parse_component (codec.hpp:342): header fields only.
int umcref_parse_component(const std::uint8_t* p, std::uint64_t len, int* codec_id,
                           int* predictor, int* backend_id, double* tau,
                           std::uint64_t* n_elements, int* ndims, std::uint64_t* dims8) {
    return guarded([&] {
        const auto comp = umc::parse_component(std::vector<std::uint8_t>(p, p + len));
        *codec_id = comp.spec.codec_id;
        *predictor = static_cast<int>(comp.spec.predictor);
        *backend_id = comp.spec.backend_id;
        *tau = comp.spec.tau_abs;
        *n_elements = comp.n_elements;
        *ndims = static_cast<int>(comp.spec.dims.size());
        for (std::size_t d = 0; d < comp.spec.dims.size() && d < 8; ++d) dims8[d] = comp.spec.dims[d];
    });
}

// rle_compress / rle_decompress (lossless.hpp:24-70).
int umcref_rle_compress(const std::uint8_t* p, std::uint64_t n, std::uint8_t** out,
                        std::uint64_t* out_len) {
    return guarded([&] {
        const auto v = umc::rle_compress(p, n);
        *out = dup_bytes(v);
        *out_len = v.size();
    });
}
int umcref_rle_decompress(const std::uint8_t* p, std::uint64_t n, std::uint8_t** out,
                          std::uint64_t* out_len) {
    return guarded([&] {
        const auto v = umc::rle_decompress(p, n);
        *out = dup_bytes(v);
        *out_len = v.size();
    });
}

// split_budget (pipeline.hpp:43) and resolve_tau_abs (:37).
int umcref_split_budget(double tau_abs, double rho, double coeff_abs_sum, double* tau1,
                        double* tau2) {
    return guarded([&] {
        umc::BackInterpSpec g;
        g.coeff_abs_sum = coeff_abs_sum;
        const auto [a, b] = umc::split_budget(tau_abs, rho, g);
        *tau1 = a;
        *tau2 = b;
    });
}

// interpolate_to_grid (interp.hpp:46): the exact cluster-mean grid component.
int umcref_interpolate_to_grid(void* ctx, const double* values, std::uint64_t n, int fill,
                               double* out, std::uint64_t n_cap, std::uint64_t* n_out) {
    return guarded([&] {
        auto* c = static_cast<Ctx*>(ctx);
        umc::Field f;
        f.values.assign(values, values + n);
        const auto gf = umc::interpolate_to_grid(
            f, c->map, c->grid, fill ? umc::FillPolicy::nearest_visited : umc::FillPolicy::zero);
        *n_out = gf.values.size();
        if (gf.values.size() > n_cap) throw umc::error("output buffer too small");
        std::memcpy(out, gf.values.data(), gf.values.size() * 8);
    });
}

// mapping_digest (serialize.hpp:300).
int umcref_mapping_digest(void* ctx, std::uint64_t* digest) {
    return guarded([&] { *digest = umc::mapping_digest(static_cast<Ctx*>(ctx)->map); });
}

// grid_coarsen (grid_builder.hpp:365) for an explicit initial grid. Outputs are
// malloc'ed: coarse axes (concatenated), assignments, visited nodes.
int umcref_grid_coarsen(int dim, std::uint64_t n_v, const double* coords,
                        const std::uint64_t* axis_sizes, const double* axes_concat,
                        double seed_threshold, std::uint64_t* out_axis_sizes, double** out_axes,
                        int* out_mode, std::uint64_t** out_assign, std::uint64_t* out_n_visited,
                        std::uint64_t** out_visited, double* visited_fraction) {
    return guarded([&] {
        const auto mesh = make_mesh(dim, n_v, coords);
        const auto grid = make_grid(dim, axis_sizes, axes_concat);
        umc::GridBuildConfig cfg;
        cfg.seed_mode_threshold = seed_threshold;
        auto res = umc::grid_coarsen(mesh, grid, cfg);
        std::vector<double> axes;
        for (int d = 0; d < dim; ++d) {
            out_axis_sizes[d] = res.grid.axes[d].size();
            axes.insert(axes.end(), res.grid.axes[d].begin(), res.grid.axes[d].end());
        }
        *out_axes = static_cast<double*>(std::malloc(axes.size() * 8));
        std::memcpy(*out_axes, axes.data(), axes.size() * 8);
        *out_mode = res.mapping.mode == umc::MappingMode::seed ? 1 : 0;
        *out_assign = static_cast<std::uint64_t*>(std::malloc(n_v * 8 + 8));
        std::memcpy(*out_assign, res.mapping.assignments.data(), n_v * 8);
        *out_n_visited = res.mapping.visited_nodes.size();
        *out_visited = static_cast<std::uint64_t*>(std::malloc(*out_n_visited * 8 + 8));
        std::memcpy(*out_visited, res.mapping.visited_nodes.data(), *out_n_visited * 8);
        *visited_fraction = res.mapping.visited_fraction.value_or(-1.0);
    });
}

// umc::grid_init (grid_builder.hpp:224) on an explicit mesh (cells optional:
// n_cells == 0 takes the reference's 1-NN point-cloud path).
int umcref_grid_init(int dim, std::uint64_t n_v, const double* coords, int arity, std::uint64_t n_cells,
                     const std::uint64_t* cells, double pk, std::uint64_t g_max, double delta, double thr,
                     std::uint64_t* out_sizes, double** out_axes) {
    return guarded([&] {
        umc::Mesh mesh;
        mesh.dim = dim;
        mesh.cell_arity = n_cells ? arity : 0;
        mesh.vertices.assign(coords, coords + n_v * dim);
        if (n_cells) mesh.cells.assign(cells, cells + n_cells * arity);
        umc::GridBuildConfig cfg;
        cfg.percentile_k = pk;
        cfg.g_max = g_max;
        cfg.delta = delta;
        cfg.seed_mode_threshold = thr;
        const auto grid = umc::grid_init(mesh, cfg);
        std::vector<double> axes;
        for (int d = 0; d < dim; ++d) {
            out_sizes[d] = grid.axes[d].size();
            axes.insert(axes.end(), grid.axes[d].begin(), grid.axes[d].end());
        }
        *out_axes = static_cast<double*>(std::malloc(axes.size() * 8 + 8));
        std::memcpy(*out_axes, axes.data(), axes.size() * 8);
    });
}

// grid_init (grid_builder.hpp:224) on a synthetic mesh from gen_mesh.
// Synthetic mesh + field (datagen.hpp:116, 261); returns coords and values.
int umcref_gen_case(int dim, std::uint64_t n_target, int mesh_style, int field_kind,
                    std::uint64_t seed, std::uint64_t* n_v, double** coords, double** values) {
    return guarded([&] {
        umc::SynthSpec spec;
        spec.dim = dim;
        spec.n_target = n_target;
        spec.mesh_style = static_cast<umc::MeshStyle>(mesh_style);
        spec.field_kind = static_cast<umc::FieldKind>(field_kind);
        spec.rng_seed = seed;
        const auto mesh = umc::gen_mesh(spec);
        const auto field = umc::gen_field(mesh, spec);
        *n_v = mesh.vertex_count();
        *coords = static_cast<double*>(std::malloc(mesh.vertices.size() * 8));
        std::memcpy(*coords, mesh.vertices.data(), mesh.vertices.size() * 8);
        *values = static_cast<double*>(std::malloc(field.values.size() * 8));
        std::memcpy(*values, field.values.data(), field.values.size() * 8);
    });
}

// Full build of a synthetic case the way the reference tests do it:
// gen_mesh -> grid_init -> grid_coarsen. Outputs as umcref_grid_coarsen.
int umcref_build_case(int dim, std::uint64_t n_target, int mesh_style, int field_kind,
                      std::uint64_t seed, std::uint64_t* n_v, double** coords, double** values,
                      std::uint64_t* out_axis_sizes, double** out_axes, int* out_mode,
                      std::uint64_t** out_assign, std::uint64_t* out_n_visited,
                      std::uint64_t** out_visited) {
    return guarded([&] {
        umc::SynthSpec spec;
        spec.dim = dim;
        spec.n_target = n_target;
        spec.mesh_style = static_cast<umc::MeshStyle>(mesh_style);
        spec.field_kind = static_cast<umc::FieldKind>(field_kind);
        spec.rng_seed = seed;
        const auto mesh = umc::gen_mesh(spec);
        const auto field = umc::gen_field(mesh, spec);
        umc::GridBuildConfig cfg;
        const auto init = umc::grid_init(mesh, cfg);
        auto res = umc::grid_coarsen(mesh, init, cfg);
        *n_v = mesh.vertex_count();
        *coords = static_cast<double*>(std::malloc(mesh.vertices.size() * 8));
        std::memcpy(*coords, mesh.vertices.data(), mesh.vertices.size() * 8);
        *values = static_cast<double*>(std::malloc(field.values.size() * 8));
        std::memcpy(*values, field.values.data(), field.values.size() * 8);
        std::vector<double> axes;
        for (int d = 0; d < dim; ++d) {
            out_axis_sizes[d] = res.grid.axes[d].size();
            axes.insert(axes.end(), res.grid.axes[d].begin(), res.grid.axes[d].end());
        }
        *out_axes = static_cast<double*>(std::malloc(axes.size() * 8));
        std::memcpy(*out_axes, axes.data(), axes.size() * 8);
        *out_mode = res.mapping.mode == umc::MappingMode::seed ? 1 : 0;
        *out_assign = static_cast<std::uint64_t*>(std::malloc(*n_v * 8 + 8));
        std::memcpy(*out_assign, res.mapping.assignments.data(), *n_v * 8);
        *out_n_visited = res.mapping.visited_nodes.size();
        *out_visited = static_cast<std::uint64_t*>(std::malloc(*out_n_visited * 8 + 8));
        std::memcpy(*out_visited, res.mapping.visited_nodes.data(), *out_n_visited * 8);
    });
}

// serialize_grid / serialize_mapping (serialize.hpp:211, 255) for fixtures.
int umcref_serialize_grid(int dim, const std::uint64_t* axis_sizes, const double* axes_concat,
                          std::uint8_t** out, std::uint64_t* out_len) {
    return guarded([&] {
        const auto v = umc::serialize_grid(make_grid(dim, axis_sizes, axes_concat));
        *out = dup_bytes(v);
        *out_len = v.size();
    });
}
int umcref_serialize_mapping(void* ctx, std::uint8_t** out, std::uint64_t* out_len) {
    return guarded([&] {
        const auto v = umc::serialize_mapping(static_cast<Ctx*>(ctx)->map);
        *out = dup_bytes(v);
        *out_len = v.size();
    });
}

// The reference's own golden recipe (tests/support/golden_recipe.hpp:22-45):
// serialized grid, mapping and archive images.
int umcref_make_golden(std::uint64_t seed, std::uint8_t** grid, std::uint64_t* grid_len,
                       std::uint8_t** map, std::uint64_t* map_len, std::uint8_t** archive,
                       std::uint64_t* archive_len) {
    return guarded([&] {
        const auto g = umc_test::make_golden(seed);
        const auto gb = umc::serialize_grid(g.grid);
        const auto mb = umc::serialize_mapping(g.mapping);
        const auto ab = umc::serialize_archive(g.archive);
        *grid = dup_bytes(gb);
        *grid_len = gb.size();
        *map = dup_bytes(mb);
        *map_len = mb.size();
        *archive = dup_bytes(ab);
        *archive_len = ab.size();
    });
}

}  // extern "C"
