// C++ drop-in test: the reference's own call sites with umc::compress /
// umc::decompress replaced by umc::b200::compress / decompress. Built here
// against the reference headers (tests/cpp/Makefile), run on the GPU box by
// tests/test_gpu_cpp.py. Checks, per case: byte-identical archive vs the
// reference (or a code-level diff confined to the rounding window is
// reported as MISMATCH), decode bound, and the reference's exception types.
#include <cmath>
#include <cstdio>
#include <string>
#include <thread>
#include <vector>

#include "umc/datagen.hpp"
#include "umc/grid_builder.hpp"
#include "umc/pipeline.hpp"
#include "umc_b200/pipeline_gpu.hpp"

using namespace umc;

static int failures = 0;
#define CHECK(c, msg)                                              \
    do {                                                           \
        if (!(c)) {                                                \
            std::printf("FAIL %s:%d %s\n", __FILE__, __LINE__, msg); \
            ++failures;                                            \
        }                                                          \
    } while (0)

struct Built {
    Mesh mesh;
    RectGrid grid;
    MappingTable map;
};

static Built build(std::uint64_t seed, int dim, std::uint64_t n, MeshStyle style) {
    SynthSpec spec;
    spec.dim = dim;
    spec.n_target = n;
    spec.mesh_style = style;
    spec.rng_seed = seed;
    Built b;
    b.mesh = gen_mesh(spec);
    GridBuildConfig cfg;
    const auto init = grid_init(b.mesh, cfg);
    auto res = grid_coarsen(b.mesh, init, cfg);
    b.grid = std::move(res.grid);
    b.map = std::move(res.mapping);
    return b;
}

// A differing archive is dumped (field, mapping, grid, both archives) for
// tests/test_gpu_cpp.py, which classifies every differing code against the
// rounding window with the Python helpers (helpers.check_archive).
static const char* g_dump_dir = nullptr;
static int g_dumps = 0;
static void put(std::FILE* f, const void* p, std::size_t n) { std::fwrite(p, 1, n, f); }
static void dump_case(const Built& b, const Field& field, const ErrorBudget& budget, const CompressOptions& opt,
                      const std::vector<std::uint8_t>& ref, const std::vector<std::uint8_t>& gpu) {
    if (!g_dump_dir) return;
    const std::string path = std::string(g_dump_dir) + "/mismatch_" + std::to_string(g_dumps++) + ".bin";
    std::FILE* f = std::fopen(path.c_str(), "wb");
    if (!f) return;
    const std::uint32_t hdr[6] = {0x4d434d55u, (std::uint32_t)b.grid.dim, (std::uint32_t)b.map.mode,
                                  (std::uint32_t)(opt.g.kind == BackInterpKind::multilinear),
                                  (std::uint32_t)(opt.fill == FillPolicy::nearest_visited),
                                  (std::uint32_t)(budget.bound_kind == BoundKind::relative_to_range)};
    put(f, hdr, sizeof hdr);
    const double tr[2] = {budget.tau, budget.split_rho};
    put(f, tr, sizeof tr);
    for (const auto& a : b.grid.axes) {
        const std::uint64_t k = a.size();
        put(f, &k, 8);
        put(f, a.data(), 8 * k);
    }
    const std::uint64_t n = b.map.assignments.size(), nv = b.map.visited_nodes.size();
    put(f, &n, 8);
    put(f, b.map.assignments.data(), 8 * n);
    put(f, &nv, 8);
    put(f, b.map.visited_nodes.data(), 8 * nv);
    put(f, field.values.data(), 8 * n);
    put(f, b.mesh.vertices.data(), 8 * b.mesh.vertices.size());
    for (const auto* v : {&ref, &gpu}) {
        const std::uint64_t k = v->size();
        put(f, &k, 8);
        put(f, v->data(), k);
    }
    std::fclose(f);
}

static double max_err(const std::vector<double>& a, const std::vector<double>& b) {
    double m = 0;
    for (std::size_t i = 0; i < a.size(); ++i) m = std::max(m, std::fabs(a[i] - b[i]));
    return m;
}

int main(int argc, char** argv) {
    if (argc > 1) g_dump_dir = argv[1];
    int exact = 0, total = 0;
    for (int c = 0; c < 4; ++c) {
        const int dim = c < 2 ? 2 : 3;
        Built b = build(100 + c, dim, dim == 2 ? 4000 : 6000, c % 2 ? MeshStyle::graded : MeshStyle::jittered);
        SynthSpec fs;
        fs.dim = dim;
        fs.field_kind = FieldKind::gaussian_mixture;
        fs.rng_seed = 7 + c;
        const Field field = gen_field(b.mesh, fs);
        for (double tau : {1e-2, 1e-4, 0.0}) {
            for (int g = 0; g < 2; ++g) {
                ErrorBudget budget;
                budget.tau = tau;
                CompressOptions opt;
                opt.g.kind = g ? BackInterpKind::multilinear : BackInterpKind::nearest;
                if (g && b.map.mode == MappingMode::seed) {
                    bool threw = false;
                    try {
                        b200::compress(field, b.map, b.grid, b.mesh, budget, opt);
                    } catch (const seed_mode_unsupported&) {
                        threw = true;
                    }
                    CHECK(threw, "seed + multilinear must throw seed_mode_unsupported");
                    continue;
                }
                const Archive ref = compress(field, b.map, b.grid, b.mesh, budget, opt);
                const Archive gpu = b200::compress(field, b.map, b.grid, b.mesh, budget, opt);
                ++total;
                const auto rb = serialize_archive(ref), gb = serialize_archive(gpu);
                const bool same = rb == gb;
                exact += same;
                if (!same) {
                    std::printf("MISMATCH case %d tau %g g %d (dumped for window classification)\n", c, tau, g);
                    dump_case(b, field, budget, opt, rb, gb);
                }
                const Field back = b200::decompress(gpu, b.map, b.grid, b.mesh);
                const double tau_abs = resolve_tau_abs(budget, field.values);
                const Field refback = decompress(gpu, b.map, b.grid, b.mesh);  // reference decodes our archive
                if (tau == 0.0) {
                    // lossless components: x' = g(x1) + (x - g(x1)) exactly as the reference computes it
                    CHECK(back.values == refback.values, "lossless decode must equal the reference bitwise");
                } else {
                    CHECK(max_err(back.values, field.values) <= tau_abs, "bound");
                    CHECK(max_err(refback.values, field.values) <= tau_abs, "reference decode bound");
                }
            }
        }
    }
    // error taxonomy (pipeline.hpp:120-125, 188-197)
    Built a = build(1, 2, 500, MeshStyle::jittered);
    Built o = build(2, 2, 500, MeshStyle::jittered);
    SynthSpec fs;
    fs.rng_seed = 5;
    const Field f = gen_field(a.mesh, fs);
    const Archive ar = b200::compress(f, a.map, a.grid, a.mesh, ErrorBudget{});
    bool mm = false;
    try {
        b200::decompress(ar, o.map, o.grid, o.mesh);
    } catch (const mapping_mismatch&) {
        mm = true;
    }
    CHECK(mm, "mapping_mismatch");
    bool ba = false;
    try {
        ErrorBudget bad;
        bad.split_rho = 1.0;
        b200::compress(f, a.map, a.grid, a.mesh, bad);
    } catch (const budget_inadmissible&) {
        ba = true;
    }
    CHECK(ba, "budget_inadmissible");
    bool nf = false;
    try {
        Field g2 = f;
        g2.values[3] = NAN;
        b200::compress(g2, a.map, a.grid, a.mesh, ErrorBudget{});
    } catch (const non_finite_value&) {
        nf = true;
    }
    CHECK(nf, "non_finite_value");
    // baseline archives decode through the device codec
    const Archive base = baseline_archive(f, ErrorBudget{});
    const Field bb = b200::decompress(base, {}, {}, a.mesh);
    const Field rb = decompress(base, {}, {}, a.mesh);
    double range = 0;
    {
        double lo = f.values[0], hi = lo;
        for (double v : f.values) { lo = std::min(lo, v); hi = std::max(hi, v); }
        range = hi - lo;
    }
    CHECK(bb.values.size() == rb.values.size(), "baseline size");
    CHECK(max_err(bb.values, rb.values) <= 1e-12 * range, "baseline decode within 1e-12 of the reference");
    CHECK(max_err(bb.values, f.values) <= resolve_tau_abs(ErrorBudget{}, f.values), "baseline bound");
    // baseline_archive through the drop-in (pipeline.hpp:164-176); codec 0 may
    // differ from the reference only by rounding-window flips, so compare the
    // decodes; verbatim (codec 1) is exact bytes
    const Archive gbase = b200::baseline_archive(f, ErrorBudget{});
    const Field gb = b200::decompress(gbase, {}, {}, a.mesh);
    CHECK(max_err(gb.values, f.values) <= resolve_tau_abs(ErrorBudget{}, f.values), "drop-in baseline bound");
    CHECK(serialize_archive(b200::baseline_archive(f, ErrorBudget{}, kCodecVerbatim)) ==
              serialize_archive(baseline_archive(f, ErrorBudget{}, kCodecVerbatim)),
          "verbatim baseline archive byte-identical");
    // verbatim pipeline archive (codec 1 on both components)
    {
        CompressOptions vo;
        vo.codec_id = kCodecVerbatim;
        const Archive rv = compress(f, a.map, a.grid, a.mesh, ErrorBudget{}, vo);
        const Archive gv = b200::compress(f, a.map, a.grid, a.mesh, ErrorBudget{}, vo);
        CHECK(serialize_archive(rv) == serialize_archive(gv), "verbatim archive byte-identical");
        CHECK(b200::decompress(gv, a.map, a.grid, a.mesh).values == decompress(rv, a.map, a.grid, a.mesh).values,
              "verbatim decode bitwise");
    }
    // grid builder on the device (grid_builder.hpp:224-421): same axes, same
    // mapping, same mode, for meshes with cells and for a bare point cloud
    for (int c = 0; c < 4; ++c) {
        const int dim = c < 2 ? 2 : 3;
        SynthSpec spec;
        spec.dim = dim;
        spec.n_target = dim == 2 ? 5000 : 8000;
        spec.mesh_style = c % 2 ? MeshStyle::graded : MeshStyle::jittered;
        spec.rng_seed = 40 + c;
        Mesh mesh = gen_mesh(spec);
        if (c == 3) mesh.cells.clear();  // point cloud: 1-NN statistics
        GridBuildConfig cfg;
        const RectGrid gi = grid_init(mesh, cfg);
        const RectGrid gg = b200::grid_init(mesh, cfg);
        CHECK(gi.axes == gg.axes, "grid_init axes identical");
        const auto rc = grid_coarsen(mesh, gi, cfg);
        const auto gc = b200::grid_coarsen(mesh, gi, cfg);
        CHECK(rc.grid.axes == gc.grid.axes, "grid_coarsen axes identical");
        CHECK(rc.mapping.mode == gc.mapping.mode, "grid_coarsen mode");
        CHECK(rc.mapping.assignments == gc.mapping.assignments, "grid_coarsen assignments identical");
        CHECK(rc.mapping.visited_nodes == gc.mapping.visited_nodes, "grid_coarsen visited identical");
        CHECK(mapping_digest(rc.mapping) == mapping_digest(gc.mapping), "mapping digest");
    }
    {
        // concurrent calls on one MappingTable from several host threads (each
        // gets its own plan clone): same archives as one thread
        Built c = build(2, 2, 4000, MeshStyle::jittered);
        std::vector<Field> fields;
        std::vector<std::vector<std::uint8_t>> want;
        std::vector<std::vector<double>> want_back;  // one-thread drop-in decode (the GPU decode is deterministic)
        for (int k = 0; k < 4; ++k) {
            SynthSpec s2;
            s2.rng_seed = 100 + k;
            fields.push_back(gen_field(c.mesh, s2));
            const Archive r = compress(fields.back(), c.map, c.grid, c.mesh, ErrorBudget{});
            want.push_back(serialize_archive(r));
            want_back.push_back(b200::decompress(r, c.map, c.grid, c.mesh).values);
        }
        std::vector<int> ok(4, 0);
        std::vector<std::thread> th;
        for (int k = 0; k < 4; ++k)
            th.emplace_back([&, k] {
                for (int r = 0; r < 3; ++r) {
                    const Archive g = b200::compress(fields[k], c.map, c.grid, c.mesh, ErrorBudget{});
                    const Field back = b200::decompress(g, c.map, c.grid, c.mesh);
                    const bool a_ok = serialize_archive(g) == want[k];
                    const bool d_ok = back.values == want_back[k];
                    if (!a_ok || !d_ok) std::printf("thread %d round %d: archive %d decode %d\n", k, r, a_ok, d_ok);
                    ok[k] += a_ok && d_ok;
                }
            });
        for (auto& t : th) t.join();
        for (int k = 0; k < 4; ++k) {
            if (ok[k] != 3) std::printf("thread %d: %d of 3 round trips matched\n", k, ok[k]);
            CHECK(ok[k] == 3, "concurrent drop-in calls match the reference");
        }
        b200::clear_plan_cache();
        CHECK(serialize_archive(b200::compress(fields[0], c.map, c.grid, c.mesh, ErrorBudget{})) == want[0],
              "after clear_plan_cache");
        // the plan cache is keyed by content: an in-place edit of the same
        // MappingTable object (same address, same sizes) must not reuse the
        // plan built for the old assignments (the reference recomputes
        // mapping_digest per call, pipeline.hpp:135)
        MappingTable& m = c.map;
        std::size_t i0 = 0, i1 = 1;
        while (i1 < m.assignments.size() && m.assignments[i1] == m.assignments[i0]) ++i1;
        std::swap(m.assignments[i0], m.assignments[i1]);
        const auto edited_ref = serialize_archive(compress(fields[0], m, c.grid, c.mesh, ErrorBudget{}));
        const auto edited_gpu = serialize_archive(b200::compress(fields[0], m, c.grid, c.mesh, ErrorBudget{}));
        CHECK(edited_ref != want[0], "the edit changes the archive");
        CHECK(edited_gpu == edited_ref, "in-place mapping edit: new plan (content-keyed cache)");
        CHECK(b200::decompress(compress(fields[0], m, c.grid, c.mesh, ErrorBudget{}), m, c.grid, c.mesh).values ==
                  b200::decompress(b200::compress(fields[0], m, c.grid, c.mesh, ErrorBudget{}), m, c.grid, c.mesh)
                      .values,
              "edited mapping decode");
        std::swap(m.assignments[i0], m.assignments[i1]);
        CHECK(serialize_archive(b200::compress(fields[0], m, c.grid, c.mesh, ErrorBudget{})) == want[0],
              "edit undone: the original plan again");
        // more distinct mappings than the cache holds (LRU eviction, default 4)
        for (int k = 0; k < 6; ++k) {
            Built d = build(300 + k, 2, 1500, MeshStyle::jittered);
            SynthSpec s3;
            s3.rng_seed = 7;
            const Field fd = gen_field(d.mesh, s3);
            CHECK(serialize_archive(b200::compress(fd, d.map, d.grid, d.mesh, ErrorBudget{})) ==
                      serialize_archive(compress(fd, d.map, d.grid, d.mesh, ErrorBudget{})),
                  "eviction round");
        }
        CHECK(serialize_archive(b200::compress(fields[0], m, c.grid, c.mesh, ErrorBudget{})) == want[0],
              "after eviction");
    }
    std::printf("cases %d exact %d failures %d\n", total, exact, failures);
    return failures ? 1 : 0;
}
