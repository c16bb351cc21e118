/* TEST INFRASTRUCTURE (CPU reference arm / parity tests): host generator of
 * the synthetic BASELINE inputs, byte-identical to the device generator
 * (paper_2501_06910_b200/csrc/datagen.cu). Both evaluate the shared per-vertex
 * recipe of datagen_core.h with IEEE-exact arithmetic only (this file is
 * built with -ffp-contract=off, the device side with --fmad=false), so the
 * reference arm of bench.py builds its inputs without loading the product
 * library. tests/test_datagen_host.py checks the identity on the GPU.
 *
 * OpenMP over vertices; the outputs do not depend on the thread count.
 */
#include <stdint.h>
#include <stdlib.h>

#include "datagen_core.h"

static uint64_t n_of(int config, uint64_t m) {
    if (config == 3) return m * m * m;
    if (config == 1 || config == 4) return m * m;
    return m;
}

/* The whole field (and coordinates) of one config, as umcg_gen_config. */
int dgh_gen(int config, uint64_t m, uint64_t seed, double* coords, void* values, uint64_t* n_out, int threads) {
    if (config < 1 || config > 5 || m < 2) return 1;
    const uint64_t n = n_of(config, m);
    if (n_out) *n_out = n;
    if (!coords && !values) return 0;
    DgModes md;
    dg_modes(seed, &md);
    const DgFeistel perm = dg_make_feistel(n, seed);
    const int dim = (config == 3 || config == 5) ? 3 : 2;
    if (threads < 1) threads = 1;
#pragma omp parallel for num_threads(threads) schedule(static, 65536)
    for (uint64_t v = 0; v < n; ++v) {
        double p[3], f = 0.0;
        float f5[5];
        if (config == 3) dg_gen3(m, seed, dg_lattice_id(&perm, v), &md, p, values ? &f : NULL);
        else if (config == 1) dg_gen1(m, seed, dg_lattice_id(&perm, v), &md, p, values ? &f : NULL);
        else if (config == 4) dg_gen4(m, seed, dg_lattice_id(&perm, v), v, &md, p, values ? f5 : NULL);
        else if (config == 2) dg_gen2(seed, v, p, values ? &f : NULL);
        else dg_gen5(seed, v, &md, p, values ? &f : NULL);
        if (coords)
            for (int d = 0; d < dim; ++d) coords[v * dim + d] = p[d];
        if (values) {
            if (config == 4)
                for (int k = 0; k < 5; ++k) ((float*)values)[k * n + v] = f5[k];
            else
                ((double*)values)[v] = f;
        }
    }
    return 0;
}

/* Config 3, restricted to the lattice points (i, j, k) in [lo, hi) per axis,
 * in the full mesh's permuted vertex order: the same coordinates and field
 * values the full-size run has at those vertices. Output count =
 * prod(hi - lo). */
int dgh_gen3_block(uint64_t m, uint64_t seed, const uint64_t* lo, const uint64_t* hi, double* coords,
                   double* values, uint64_t* n_out, int threads) {
    if (m < 2) return 1;
    for (int d = 0; d < 3; ++d)
        if (lo[d] >= hi[d] || hi[d] > m) return 1;
    const uint64_t n = m * m * m;
    const uint64_t cnt = (hi[0] - lo[0]) * (hi[1] - lo[1]) * (hi[2] - lo[2]);
    if (n_out) *n_out = cnt;
    if (!coords && !values) return 0;
    DgModes md;
    dg_modes(seed, &md);
    const DgFeistel perm = dg_make_feistel(n, seed);
    if (threads < 1) threads = 1;
    const uint64_t chunks = (uint64_t)threads * 16;
    uint64_t* off = (uint64_t*)calloc(chunks + 1, sizeof(uint64_t));
    if (!off) return 2;
#define DGH_IN(L) ((L) / (m * m) >= lo[0] && (L) / (m * m) < hi[0] && ((L) / m) % m >= lo[1] && \
                   ((L) / m) % m < hi[1] && (L) % m >= lo[2] && (L) % m < hi[2])
#pragma omp parallel for num_threads(threads) schedule(dynamic, 1)
    for (uint64_t c = 0; c < chunks; ++c) {
        const uint64_t a = n * c / chunks, b = n * (c + 1) / chunks;
        uint64_t k = 0;
        for (uint64_t v = a; v < b; ++v) {
            const uint64_t L = dg_lattice_id(&perm, v);
            k += DGH_IN(L);
        }
        off[c + 1] = k;
    }
    for (uint64_t c = 0; c < chunks; ++c) off[c + 1] += off[c];
    if (off[chunks] != cnt) { free(off); return 3; }
#pragma omp parallel for num_threads(threads) schedule(dynamic, 1)
    for (uint64_t c = 0; c < chunks; ++c) {
        const uint64_t a = n * c / chunks, b = n * (c + 1) / chunks;
        uint64_t o = off[c];
        for (uint64_t v = a; v < b; ++v) {
            const uint64_t L = dg_lattice_id(&perm, v);
            if (!DGH_IN(L)) continue;
            double p[3], f = 0.0;
            dg_gen3(m, seed, L, &md, p, values ? &f : NULL);
            if (coords) { coords[3 * o] = p[0]; coords[3 * o + 1] = p[1]; coords[3 * o + 2] = p[2]; }
            if (values) values[o] = f;
            ++o;
        }
    }
#undef DGH_IN
    free(off);
    return 0;
}
