// Synthetic BASELINE inputs generated on the device (BASELINE.json configs).
//
// Counter-based SplitMix64 (the reference's generator, common.hpp:150-173,
// applied to (seed, stream, index) so every element is independent), a
// Feistel bijection for the "vertex order randomly permuted" requirement
// (stand-in for the reference's Fisher-Yates shuffle, datagen.hpp:58-76),
// boundary lattice points left unjittered so the bounding box is exact.
#include <cmath>
#include <vector>

#include "kernels.h"

namespace umcg {

namespace {

constexpr int THREADS = 256;

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}
__host__ __device__ __forceinline__ uint64_t hash3(uint64_t seed, uint64_t stream, uint64_t i) {
    return mix64(seed + 0x9e3779b97f4a7c15ull * (stream * 0x100000001ull + i + 1));
}
__host__ __device__ __forceinline__ double u01(uint64_t h) { return (double)(h >> 11) * 0x1.0p-53; }

// 4-round Feistel permutation on [0, 2^(2b)), cycle-walked into [0, n).
struct Feistel {
    uint32_t b;
    uint64_t n, key;
    __host__ __device__ uint64_t round_fn(uint64_t r, int k) const {
        return mix64(r ^ (key + 0x632be59bd9b4e019ull * (uint64_t)(k + 1))) & ((1ull << b) - 1);
    }
    __host__ __device__ uint64_t once(uint64_t x) const {
        const uint64_t mask = (1ull << b) - 1;
        uint64_t L = x >> b, R = x & mask;
        for (int k = 0; k < 4; ++k) {
            const uint64_t t = L ^ round_fn(R, k);
            L = R;
            R = t;
        }
        return (L << b) | R;
    }
    __host__ __device__ uint64_t operator()(uint64_t x) const {
        do { x = once(x); } while (x >= n);
        return x;
    }
};

Feistel make_feistel(uint64_t n, uint64_t seed) {
    uint32_t b = 1;
    while ((1ull << (2 * b)) < n) ++b;
    return Feistel{b, n, mix64(seed ^ 0x5851f42d4c957f2dull)};
}

struct Modes3 {
    double k[64][3];
    double amp[64];
    double phase[64];
};
__constant__ Modes3 c_modes;
struct Bumps {
    double c[8][2];
};
__constant__ Bumps c_bumps;

__device__ __forceinline__ double jittered(uint64_t i, uint64_t m, double h, double jit, uint64_t seed,
                                           uint64_t stream, uint64_t lattice_id) {
    const double base = (double)i * h;
    if (i == 0 || i == m - 1) return base;
    return base + (u01(hash3(seed, stream, lattice_id)) - 0.5) * 2.0 * jit * h;
}

// Config 3: 3D jittered lattice (jitter +-0.25 h), 64 Fourier modes.
__global__ void k_gen3(uint64_t m, uint64_t seed, Feistel perm, double* __restrict__ xyz, double* __restrict__ f) {
    const uint64_t v = blockIdx.x * (uint64_t)THREADS + threadIdx.x;
    const uint64_t n = m * m * m;
    if (v >= n) return;
    const uint64_t L = perm(v);
    const uint64_t i = L / (m * m), j = (L / m) % m, k = L % m;
    const double h = 1.0 / (double)(m - 1);
    const double p[3] = {jittered(i, m, h, 0.25, seed, 1, L), jittered(j, m, h, 0.25, seed, 2, L),
                         jittered(k, m, h, 0.25, seed, 3, L)};
    if (xyz) { xyz[3 * v] = p[0]; xyz[3 * v + 1] = p[1]; xyz[3 * v + 2] = p[2]; }
    if (f) {
        double s = 0.0;
        for (int q = 0; q < 64; ++q) {
            const double arg = 2.0 * M_PI * (c_modes.k[q][0] * p[0] + c_modes.k[q][1] * p[1] + c_modes.k[q][2] * p[2]) +
                               c_modes.phase[q];
            s += c_modes.amp[q] * cos(arg);
        }
        f[v] = s;
    }
}

// Config 1: 2D jittered lattice (+-0.3 h), sin(4 pi x) cos(4 pi y) + 8 Gaussian bumps.
__global__ void k_gen1(uint64_t m, uint64_t seed, Feistel perm, double* __restrict__ xy, double* __restrict__ f) {
    const uint64_t v = blockIdx.x * (uint64_t)THREADS + threadIdx.x;
    const uint64_t n = m * m;
    if (v >= n) return;
    const uint64_t L = perm(v);
    const uint64_t i = L / m, j = L % m;
    const double h = 1.0 / (double)(m - 1);
    const double x = jittered(i, m, h, 0.3, seed, 1, L), y = jittered(j, m, h, 0.3, seed, 2, L);
    if (xy) { xy[2 * v] = x; xy[2 * v + 1] = y; }
    if (f) {
        double s = sin(4.0 * M_PI * x) * cos(4.0 * M_PI * y);
        for (int q = 0; q < 8; ++q) {
            const double dx = x - c_bumps.c[q][0], dy = y - c_bumps.c[q][1];
            s += 0.2 * exp(-(dx * dx + dy * dy) / 0.002);
        }
        f[v] = s;
    }
}

// Config 4: 2D jittered lattice, 5 fp32 variables (field-major).
__global__ void k_gen4(uint64_t m, uint64_t seed, Feistel perm, double* __restrict__ xy, float* __restrict__ f) {
    const uint64_t v = blockIdx.x * (uint64_t)THREADS + threadIdx.x;
    const uint64_t n = m * m;
    if (v >= n) return;
    const uint64_t L = perm(v);
    const uint64_t i = L / m, j = L % m;
    const double h = 1.0 / (double)(m - 1);
    const double x = jittered(i, m, h, 0.3, seed, 1, L), y = jittered(j, m, h, 0.3, seed, 2, L);
    if (xy) { xy[2 * v] = x; xy[2 * v + 1] = y; }
    if (!f) return;
    double b = 0.0;  // smooth Gaussian bumps
    for (int q = 0; q < 8; ++q) {
        const double dx = x - c_bumps.c[q][0], dy = y - c_bumps.c[q][1];
        b += exp(-(dx * dx + dy * dy) / 0.01);
    }
    double fm = 0.0;  // Fourier modes (2D projection of the config-3 modes)
    for (int q = 0; q < 16; ++q)
        fm += c_modes.amp[q] * cos(2.0 * M_PI * (c_modes.k[q][0] * x + c_modes.k[q][1] * y) + c_modes.phase[q]);
    const double step = (x > 0.5 + 0.1 * sin(2.0 * M_PI * y)) ? 1.0 : 0.0;  // discontinuity
    const double u1 = u01(hash3(seed, 11, v)), u2 = u01(hash3(seed, 12, v));
    const double g = sqrt(-2.0 * log(u1 > 0 ? u1 : 1e-300)) * cos(2.0 * M_PI * u2);
    const double sgn = (hash3(seed, 13, v) & 1) ? 1.0 : -1.0;
    const double logn = sgn * exp(2.0 * g);  // sign * lognormal(0, 2)
    const double uni = 2.0 * u01(hash3(seed, 14, v)) - 1.0;
    f[v] = (float)b;
    f[n + v] = (float)fm;
    f[2 * n + v] = (float)(step + 0.05 * x);
    f[3 * n + v] = (float)logn;
    f[4 * n + v] = (float)uni;
}

__device__ __forceinline__ double gauss(uint64_t seed, uint64_t stream, uint64_t i) {
    const double u1 = u01(hash3(seed, stream, i)), u2 = u01(hash3(seed, stream + 1, i));
    return sqrt(-2.0 * log(u1 > 0 ? u1 : 1e-300)) * cos(2.0 * M_PI * u2);
}

__device__ __forceinline__ double fourier3(const double* p) {
    double s = 0.0;
    for (int q = 0; q < 64; ++q) {
        const double arg = 2.0 * M_PI * (c_modes.k[q][0] * p[0] + c_modes.k[q][1] * p[1] + c_modes.k[q][2] * p[2]) +
                           c_modes.phase[q];
        s += c_modes.amp[q] * cos(arg);
    }
    return s;
}

// Config 2: graded 2D annulus around (0.5, 0.5), r in [0.3, 0.45]: 90 % of
// the vertices from the radial density exp(-((r - 0.4) / 0.02)^2) (a normal
// with sigma 0.02/sqrt(2), truncated to the annulus), 10 % uniform over the
// annulus area; theta ~ U[0, 2pi). Field tanh((r - 0.4) / 0.005) +
// 0.05 cos(12 theta) + N(0, 1e-4). Vertices are i.i.d., so their order is
// already random.
__global__ void k_gen2(uint64_t n, uint64_t seed, double* __restrict__ xy, double* __restrict__ f) {
    const uint64_t v = blockIdx.x * (uint64_t)THREADS + threadIdx.x;
    if (v >= n) return;
    double r;
    if (u01(hash3(seed, 1, v)) < 0.1) {
        const double a = u01(hash3(seed, 2, v));
        r = sqrt(0.09 + a * (0.2025 - 0.09));
    } else {
        r = 0.4;
        for (uint64_t t = 0; t < 64; ++t) {
            r = 0.4 + gauss(seed, 3 + 2 * t, v) * (0.02 / M_SQRT2);
            if (r >= 0.3 && r <= 0.45) break;
            r = 0.4;
        }
    }
    const double th = 2.0 * M_PI * u01(hash3(seed, 200, v));
    const double x = 0.5 + r * cos(th), y = 0.5 + r * sin(th);
    if (xy) { xy[2 * v] = x; xy[2 * v + 1] = y; }
    if (f) f[v] = tanh((r - 0.4) / 0.005) + 0.05 * cos(12.0 * th) + 1e-4 * gauss(seed, 201, v);
}

// Config 5: clustered 3D shell around the axis (0.5, 0.5, z): r = 0.2 +
// N(0, 0.01), theta ~ U[0, 2pi), z ~ U[0, 1]; field = the config-3 Fourier
// field x exp(-((r - 0.2) / 0.01)^2 / 2).
__global__ void k_gen5(uint64_t n, uint64_t seed, double* __restrict__ xyz, double* __restrict__ f) {
    const uint64_t v = blockIdx.x * (uint64_t)THREADS + threadIdx.x;
    if (v >= n) return;
    const double r = 0.2 + 0.01 * gauss(seed, 1, v);
    const double th = 2.0 * M_PI * u01(hash3(seed, 3, v));
    const double p[3] = {0.5 + r * cos(th), 0.5 + r * sin(th), u01(hash3(seed, 4, v))};
    if (xyz) { xyz[3 * v] = p[0]; xyz[3 * v + 1] = p[1]; xyz[3 * v + 2] = p[2]; }
    if (f) {
        const double d = (r - 0.2) / 0.01;
        f[v] = fourier3(p) * exp(-0.5 * d * d);
    }
}

void upload_modes(uint64_t seed) {
    Modes3 md;
    uint64_t s = seed ^ 0xa0761d6478bd642full;
    auto next = [&]() { s += 0x9e3779b97f4a7c15ull; return mix64(s); };
    for (int q = 0; q < 64; ++q) {
        const double km = 1.0 + 31.0 * u01(next());       // |k| ~ U[1, 32]
        const double cz = 2.0 * u01(next()) - 1.0;        // direction uniform on S^2
        const double az = 2.0 * M_PI * u01(next());
        const double r = std::sqrt(std::max(0.0, 1.0 - cz * cz));
        md.k[q][0] = km * r * std::cos(az);
        md.k[q][1] = km * r * std::sin(az);
        md.k[q][2] = km * cz;
        md.amp[q] = std::pow(km, -5.0 / 6.0);
        md.phase[q] = 2.0 * M_PI * u01(next());
    }
    UMCG_CUDA(cudaMemcpyToSymbol(c_modes, &md, sizeof md));
    Bumps bp;
    for (int q = 0; q < 8; ++q) { bp.c[q][0] = u01(next()); bp.c[q][1] = u01(next()); }
    UMCG_CUDA(cudaMemcpyToSymbol(c_bumps, &bp, sizeof bp));
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
    upload_modes(seed);
    const Feistel perm = make_feistel(n, seed);
    const unsigned g = (unsigned)cdiv(n, THREADS);
    if (config == 2) k_gen2<<<g, THREADS, 0, st>>>(n, seed, d_coords, static_cast<double*>(d_values));
    else if (config == 5) k_gen5<<<g, THREADS, 0, st>>>(n, seed, d_coords, static_cast<double*>(d_values));
    else if (config == 3) k_gen3<<<g, THREADS, 0, st>>>(m, seed, perm, d_coords, static_cast<double*>(d_values));
    else if (config == 1) k_gen1<<<g, THREADS, 0, st>>>(m, seed, perm, d_coords, static_cast<double*>(d_values));
    else k_gen4<<<g, THREADS, 0, st>>>(m, seed, perm, d_coords, static_cast<float*>(d_values));
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
