// End-to-end throughput through the C++ drop-in API (the call a reference
// user makes): umc::b200::compress / umc::b200::decompress on std::vector
// fields, host buffers in and out, on BASELINE config 3 (512^3 jittered
// lattice, 256^3 grid, tau_rel 1e-4, rho 0.5, nearest g). Inputs come from
// the product's device generator (umcg_gen_config) and the mapping from the
// drop-in umc::b200::grid_coarsen; the plan is built by the first (warm-up)
// call. Prints one JSON line. Built here against the reference headers
// (tests/cpp/Makefile); run by bench.py (e2e.cpp_api).
#include <malloc.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "umc/pipeline.hpp"
#include "umc_b200/pipeline_gpu.hpp"

using namespace umc;
using clk = std::chrono::steady_clock;

int main(int argc, char** argv) {
    // A long-running caller: keep freed heap memory instead of returning every
    // 1 GB Field / 200 MB payload to the kernel (glibc would mmap/munmap them,
    // and each call would page-fault 1.3 GB back in -- the same cost the
    // reference API's value-semantics Field carries; not the compressor's).
    mallopt(M_MMAP_MAX, 0);       // large blocks from the heap (glibc caps M_MMAP_THRESHOLD at 32 MiB)
    mallopt(M_TRIM_THRESHOLD, -1);  // and never returned
    const int steps = argc > 1 ? std::atoi(argv[1]) : 5;
    const int warmup = argc > 2 ? std::atoi(argv[2]) : 2;
    const std::uint64_t lattice = argc > 3 ? std::strtoull(argv[3], nullptr, 10) : 512;
    const int g = argc > 4 ? std::atoi(argv[4]) : 256;
    const double tau = 1e-4;
    std::uint64_t n = 0;
    if (umcg_gen_config(3, lattice, 0x250106910ull + 3, nullptr, nullptr, &n, nullptr)) return 2;
    void *dc = nullptr, *dv = nullptr;
    if (cudaMalloc(&dc, n * 24) || cudaMalloc(&dv, n * 8)) return 3;
    if (umcg_gen_config(3, lattice, 0x250106910ull + 3, static_cast<double*>(dc), dv, &n, nullptr)) return 4;
    Mesh mesh;
    mesh.dim = 3;
    mesh.cell_arity = 4;
    mesh.vertices.resize(n * 3);
    Field field;
    field.name = "field";
    field.values.resize(n);
    cudaMemcpy(mesh.vertices.data(), dc, n * 24, cudaMemcpyDeviceToHost);
    cudaMemcpy(field.values.data(), dv, n * 8, cudaMemcpyDeviceToHost);
    cudaFree(dc);
    cudaFree(dv);
    RectGrid init;
    init.dim = 3;
    init.axes.resize(3);
    for (auto& a : init.axes) {
        a.resize(g);
        for (int k = 0; k < g; ++k) a[k] = (double)k / (double)(g - 1);
    }
    const CoarsenResult cr = b200::grid_coarsen(mesh, init, GridBuildConfig{});
    ErrorBudget budget;
    budget.tau = tau;
    double tc = 0, td = 0, tk = 0;
    std::uint64_t bytes = 0;
    double err = 0;
    for (int it = 0; it < warmup + steps; ++it) {
        const auto t0 = clk::now();
        const Archive ar = b200::compress(field, cr.mapping, cr.grid, mesh, budget);
        const auto t1 = clk::now();
        const Field back = b200::decompress(ar, cr.mapping, cr.grid, mesh);
        const auto t2 = clk::now();
        if (it >= warmup) {
            tc += std::chrono::duration<double>(t1 - t0).count();
            td += std::chrono::duration<double>(t2 - t1).count();
        }
        if (it == warmup + steps - 1) {
            bytes = ar.compressed_bytes();
            double lo = field.values[0], hi = lo;
            for (double v : field.values) { lo = v < lo ? v : lo; hi = v > hi ? v : hi; }
            for (std::uint64_t i = 0; i < n; ++i) {
                const double e = std::fabs(back.values[i] - field.values[i]);
                err = e > err ? e : err;
            }
            err /= tau * (hi - lo);
        }
    }
    {  // the per-call content fingerprint of the plan cache (mapping + axes)
        const auto t0 = clk::now();
        (void)b200::detail::plan_key(cr.mapping, cr.grid, mesh, false);
        tk = std::chrono::duration<double>(clk::now() - t0).count();
    }
    double t_alloc = 0;
    {  // what the value-semantics Field alone costs the caller: a 1 GB vector
        const auto t0 = clk::now();
        std::vector<double> v;
        v.resize(n);
        t_alloc = std::chrono::duration<double>(clk::now() - t0).count();
    }
    tc /= steps;
    td /= steps;
    const double gb = n * 8 / 1e9;
    std::printf("{\"path\": \"umc::b200::compress + umc::b200::decompress (C++ drop-in, std::vector fields)\", "
                "\"n\": %llu, \"steps\": %d, \"compress_ms\": %.3f, \"decompress_ms\": %.3f, \"ms_per_step\": %.3f, "
                "\"value\": %.4f, \"unit\": \"GB/s\", \"compress_gbs\": %.4f, \"decompress_gbs\": %.4f, "
                "\"plan_key_ms\": %.3f, \"field_vector_alloc_ms\": %.3f, \"archive_payload_bytes\": %llu, "
                "\"max_err_over_tau\": %.6f}\n",
                (unsigned long long)n, steps, tc * 1e3, td * 1e3, (tc + td) * 1e3, gb / (tc + td), gb / tc, gb / td,
                tk * 1e3, t_alloc * 1e3, (unsigned long long)bytes, err);
    return 0;
}
