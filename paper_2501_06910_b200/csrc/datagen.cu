// Synthetic BASELINE inputs generated on the device (BASELINE.json configs).
// The per-vertex recipe lives in datagen_core.h, shared with the host
// generator of the CPU reference arm (oracle/datagen_host.c): both produce
// the same bytes (IEEE-exact arithmetic only, no libm transcendental calls).
#include <cmath>
#include <vector>

#include "datagen_core.h"
#include "kernels.h"

namespace umcg {

namespace {

constexpr int THREADS = 256;

__constant__ DgModes c_md;

__global__ void k_gen_lattice(int config, uint64_t m, uint64_t n, uint64_t seed, DgFeistel perm,
                              double* __restrict__ xyz, void* __restrict__ f) {
    const uint64_t v = blockIdx.x * (uint64_t)THREADS + threadIdx.x;
    if (v >= n) return;
    const uint64_t L = dg_lattice_id(&perm, v);
    double p[3], fv;
    if (config == 3) {
        dg_gen3(m, seed, L, &c_md, p, f ? &fv : nullptr);
        if (xyz) { xyz[3 * v] = p[0]; xyz[3 * v + 1] = p[1]; xyz[3 * v + 2] = p[2]; }
        if (f) static_cast<double*>(f)[v] = fv;
    } else if (config == 1) {
        dg_gen1(m, seed, L, &c_md, p, f ? &fv : nullptr);
        if (xyz) { xyz[2 * v] = p[0]; xyz[2 * v + 1] = p[1]; }
        if (f) static_cast<double*>(f)[v] = fv;
    } else {
        float f5[5];
        dg_gen4(m, seed, L, v, &c_md, p, f ? f5 : nullptr);
        if (xyz) { xyz[2 * v] = p[0]; xyz[2 * v + 1] = p[1]; }
        if (f)
            for (int k = 0; k < 5; ++k) static_cast<float*>(f)[k * n + v] = f5[k];  // field-major
    }
}

__global__ void k_gen_iid(int config, uint64_t n, uint64_t seed, double* __restrict__ xyz, double* __restrict__ f) {
    const uint64_t v = blockIdx.x * (uint64_t)THREADS + threadIdx.x;
    if (v >= n) return;
    double p[3], fv;
    if (config == 2) {
        dg_gen2(seed, v, p, f ? &fv : nullptr);
        if (xyz) { xyz[2 * v] = p[0]; xyz[2 * v + 1] = p[1]; }
    } else {
        dg_gen5(seed, v, &c_md, p, f ? &fv : nullptr);
        if (xyz) { xyz[3 * v] = p[0]; xyz[3 * v + 1] = p[1]; xyz[3 * v + 2] = p[2]; }
    }
    if (f) f[v] = fv;
}

}  // namespace

void gen_config(int config, uint64_t m, uint64_t seed, double* d_coords, void* d_values, uint64_t* n_out,
                cudaStream_t st) {
    if (m < 2) fail(UMCG_INVALID_ARGUMENT, "lattice must have >= 2 points per axis");
    uint64_t n;
    if (config == 3) n = m * m * m;
    else if (config == 1 || config == 4) n = m * m;
    else if (config == 2 || config == 5) n = m;  // vertex count
    else fail(UMCG_INVALID_ARGUMENT, "config must be 1..5");
    if (n_out) *n_out = n;
    if (!d_coords && !d_values) return;
    DgModes md;
    dg_modes(seed, &md);
    UMCG_CUDA(cudaMemcpyToSymbolAsync(c_md, &md, sizeof md, 0, cudaMemcpyHostToDevice, st));
    UMCG_CUDA(cudaStreamSynchronize(st));
    const unsigned g = (unsigned)cdiv(n, THREADS);
    if (config == 2 || config == 5) {
        k_gen_iid<<<g, THREADS, 0, st>>>(config, n, seed, d_coords, static_cast<double*>(d_values));
    } else {
        k_gen_lattice<<<g, THREADS, 0, st>>>(config, m, n, seed, dg_make_feistel(n, seed), d_coords, d_values);
    }
    UMCG_LAUNCHED();
}

}  // namespace umcg

extern "C" umcg_status umcg_gen_config(int config, uint64_t lattice, uint64_t seed, double* d_coords,
                                       void* d_values, uint64_t* n_out, void* stream) {
    try {
        umcg::gen_config(config, lattice, seed, d_coords, d_values, n_out, static_cast<cudaStream_t>(stream));
        return UMCG_OK;
    } catch (const umcg::Error& e) {
        return e.status;
    }
}
