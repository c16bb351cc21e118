/* Synthetic BASELINE inputs (BASELINE.json configs 1-5): the per-vertex
 * generator shared by the device kernels (datagen.cu) and the host generator
 * the CPU reference arm uses (oracle/datagen_host.c), so both arms see the
 * same bytes without the reference process loading the product library.
 *
 * Bit-identity between nvcc device code and gcc host code holds because every
 * floating-point value is produced by IEEE-exact operations only (+ - * /
 * sqrt, no contraction: device --fmad=false, host -ffp-contract=off).
 * cos/sin/exp/log/tanh are therefore evaluated here with explicit
 * Cody-Waite range reduction and fixed Taylor polynomials instead of libm /
 * CUDA's math library (whose last-ulp results differ between the two).
 * Accuracy is ~1e-16 relative, far below anything the configs depend on.
 *
 * Randomness: counter-based SplitMix64 finalizer (the reference's generator,
 * common.hpp:150-173) on (seed, stream, index); the "vertex order randomly
 * permuted" requirement is a 4-round Feistel bijection cycle-walked into
 * [0, n) (stand-in for the reference's Fisher-Yates shuffle,
 * datagen.hpp:58-76); boundary lattice points are unjittered so the bounding
 * box is exact (datagen.hpp:131-134).
 */
#ifndef UMCG_DATAGEN_CORE_H
#define UMCG_DATAGEN_CORE_H

#include <stdint.h>
#include <string.h>
#include <math.h>

#ifdef __CUDACC__
#define DG_FN __host__ __device__ static inline
#else
#define DG_FN static inline
#endif

#define DG_PI 3.14159265358979311600e+00
#define DG_SQRT1_2 0.70710678118654757274

DG_FN uint64_t dg_bits(double x) { uint64_t u; memcpy(&u, &x, 8); return u; }
DG_FN double dg_from_bits(uint64_t u) { double x; memcpy(&x, &u, 8); return x; }

/* nearest integer (ties away from zero) of |x| < 2^52, as a double */
DG_FN double dg_nint(double x) {
    const double a = x < 0 ? -x : x;
    double k = (double)(int64_t)(a + 0.5);
    return x < 0 ? -k : k;
}

/* sin and cos of x (|x| < 2^20 * pi/2): Cody-Waite reduction by pi/2 with
 * the fdlibm three-part constant (33 significant bits each, so k * part is
 * exact), then Taylor polynomials on |r| <= pi/4. */
DG_FN void dg_sincos(double x, double* s_out, double* c_out) {
    const double k = dg_nint(x * 6.36619772367581382433e-01);
    double r = x - k * 1.57079632673412561417e+00;
    r = r - k * 6.07710050630396597660e-11;
    r = r - k * 2.02226624871116645580e-21;
    const double r2 = r * r;
    double ps = 1.0 / 355687428096000.0;          /* 1/17! */
    ps = ps * r2 - 1.0 / 1307674368000.0;         /* 1/15! */
    ps = ps * r2 + 1.0 / 6227020800.0;            /* 1/13! */
    ps = ps * r2 - 1.0 / 39916800.0;              /* 1/11! */
    ps = ps * r2 + 1.0 / 362880.0;                /* 1/9!  */
    ps = ps * r2 - 1.0 / 5040.0;                  /* 1/7!  */
    ps = ps * r2 + 1.0 / 120.0;                   /* 1/5!  */
    ps = ps * r2 - 1.0 / 6.0;                     /* 1/3!  */
    const double sn = r + r * (r2 * ps);
    double pc = 1.0 / 6402373705728000.0;         /* 1/18! */
    pc = pc * r2 - 1.0 / 20922789888000.0;        /* 1/16! */
    pc = pc * r2 + 1.0 / 87178291200.0;           /* 1/14! */
    pc = pc * r2 - 1.0 / 479001600.0;             /* 1/12! */
    pc = pc * r2 + 1.0 / 3628800.0;               /* 1/10! */
    pc = pc * r2 - 1.0 / 40320.0;                 /* 1/8!  */
    pc = pc * r2 + 1.0 / 720.0;                   /* 1/6!  */
    pc = pc * r2 - 1.0 / 24.0;                    /* 1/4!  */
    pc = pc * r2 + 0.5;
    const double cs = 1.0 - r2 * pc;
    const int q = (int)(((int64_t)k) & 3);
    if (q == 0) { *s_out = sn; *c_out = cs; }
    else if (q == 1) { *s_out = cs; *c_out = -sn; }
    else if (q == 2) { *s_out = -sn; *c_out = -cs; }
    else { *s_out = -cs; *c_out = sn; }
}
DG_FN double dg_cos(double x) { double s, c; dg_sincos(x, &s, &c); return c; }
DG_FN double dg_sin(double x) { double s, c; dg_sincos(x, &s, &c); return s; }

/* e^x: x = k ln2 + r (fdlibm ln2 split), Taylor to r^14 on |r| <= 0.35,
 * scaled by an exactly constructed 2^k. Results below e^-708 flush to 0. */
DG_FN double dg_exp(double x) {
    if (x < -708.0) return 0.0;
    if (x > 709.0) return dg_from_bits(0x7ff0000000000000ull);
    const double k = dg_nint(x * 1.44269504088896338700e+00);
    const double r = (x - k * 6.93147180369123816490e-01) - k * 1.90821492927058770002e-10;
    double p = 1.0 / 87178291200.0;   /* 1/14! */
    p = p * r + 1.0 / 6227020800.0;
    p = p * r + 1.0 / 479001600.0;
    p = p * r + 1.0 / 39916800.0;
    p = p * r + 1.0 / 3628800.0;
    p = p * r + 1.0 / 362880.0;
    p = p * r + 1.0 / 40320.0;
    p = p * r + 1.0 / 5040.0;
    p = p * r + 1.0 / 720.0;
    p = p * r + 1.0 / 120.0;
    p = p * r + 1.0 / 24.0;
    p = p * r + 1.0 / 6.0;
    p = p * r + 0.5;
    p = p * r + 1.0;
    p = p * r + 1.0;
    /* x >= -708 keeps k >= -1021: 2^k is a normal number, the product exact-rounded */
    return p * dg_from_bits((uint64_t)((int64_t)k + 1023) << 52);
}

/* ln(u), u > 0 normal: u = m 2^e with m in [sqrt(1/2), sqrt(2)),
 * ln m = 2 atanh(s), s = (m - 1) / (m + 1), series to s^25. */
DG_FN double dg_log(double u) {
    const uint64_t b = dg_bits(u);
    int64_t e = (int64_t)((b >> 52) & 0x7ff) - 1023;
    double m = dg_from_bits((b & 0x000fffffffffffffull) | 0x3ff0000000000000ull);
    if (m > 1.41421356237309514547) { m = m * 0.5; e = e + 1; }
    const double s = (m - 1.0) / (m + 1.0);
    const double s2 = s * s;
    double p = 1.0 / 25.0;
    p = p * s2 + 1.0 / 23.0;
    p = p * s2 + 1.0 / 21.0;
    p = p * s2 + 1.0 / 19.0;
    p = p * s2 + 1.0 / 17.0;
    p = p * s2 + 1.0 / 15.0;
    p = p * s2 + 1.0 / 13.0;
    p = p * s2 + 1.0 / 11.0;
    p = p * s2 + 1.0 / 9.0;
    p = p * s2 + 1.0 / 7.0;
    p = p * s2 + 1.0 / 5.0;
    p = p * s2 + 1.0 / 3.0;
    const double lm = 2.0 * s + 2.0 * s * (s2 * p);
    const double ed = (double)e;
    return ed * 6.93147180369123816490e-01 + (ed * 1.90821492927058770002e-10 + lm);
}

DG_FN double dg_tanh(double x) {
    if (x > 20.0) return 1.0;
    if (x < -20.0) return -1.0;
    const double e = dg_exp(2.0 * x);
    return (e - 1.0) / (e + 1.0);
}

/* ---- counter-based randomness ---- */
DG_FN uint64_t dg_mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}
DG_FN uint64_t dg_hash3(uint64_t seed, uint64_t stream, uint64_t i) {
    return dg_mix64(seed + 0x9e3779b97f4a7c15ull * (stream * 0x100000001ull + i + 1));
}
DG_FN double dg_u01(uint64_t h) { return (double)(h >> 11) * 0x1.0p-53; }

/* 4-round Feistel permutation on [0, 2^(2b)), cycle-walked into [0, n). */
typedef struct { uint32_t b; uint64_t n, key; } DgFeistel;
DG_FN DgFeistel dg_make_feistel(uint64_t n, uint64_t seed) {
    DgFeistel f;
    f.b = 1;
    while ((1ull << (2 * f.b)) < n) ++f.b;
    f.n = n;
    f.key = dg_mix64(seed ^ 0x5851f42d4c957f2dull);
    return f;
}
DG_FN uint64_t dg_feistel_once(const DgFeistel* f, uint64_t x) {
    const uint64_t mask = (1ull << f->b) - 1;
    uint64_t L = x >> f->b, R = x & mask;
    for (int k = 0; k < 4; ++k) {
        const uint64_t t = L ^ (dg_mix64(R ^ (f->key + 0x632be59bd9b4e019ull * (uint64_t)(k + 1))) & mask);
        L = R;
        R = t;
    }
    return (L << f->b) | R;
}
DG_FN uint64_t dg_feistel(const DgFeistel* f, uint64_t x) {
    do { x = dg_feistel_once(f, x); } while (x >= f->n);
    return x;
}

/* ---- per-seed tables ---- */
typedef struct {
    double k[64][3];   /* config-3 wave vectors: |k| ~ U[1, 32], direction uniform on S^2 */
    double amp[64];    /* |k|^(-5/6) */
    double phase[64];  /* U[0, 2 pi) */
    double bump[8][2]; /* Gaussian bump centres, U[0, 1]^2 */
} DgModes;

DG_FN void dg_modes(uint64_t seed, DgModes* md) {
    uint64_t s = seed ^ 0xa0761d6478bd642full;
#define DG_NEXT() (s += 0x9e3779b97f4a7c15ull, dg_mix64(s))
    for (int q = 0; q < 64; ++q) {
        const double km = 1.0 + 31.0 * dg_u01(DG_NEXT());
        const double cz = 2.0 * dg_u01(DG_NEXT()) - 1.0;
        const double az = 2.0 * DG_PI * dg_u01(DG_NEXT());
        double t = 1.0 - cz * cz;
        const double r = t > 0.0 ? sqrt(t) : 0.0;
        double sa, ca;
        dg_sincos(az, &sa, &ca);
        md->k[q][0] = km * r * ca;
        md->k[q][1] = km * r * sa;
        md->k[q][2] = km * cz;
        md->amp[q] = dg_exp((-5.0 / 6.0) * dg_log(km));
        md->phase[q] = 2.0 * DG_PI * dg_u01(DG_NEXT());
    }
    for (int q = 0; q < 8; ++q) {
        md->bump[q][0] = dg_u01(DG_NEXT());
        md->bump[q][1] = dg_u01(DG_NEXT());
    }
#undef DG_NEXT
}

DG_FN double dg_jittered(uint64_t i, uint64_t m, double h, double jit, uint64_t seed, uint64_t stream,
                         uint64_t lattice_id) {
    const double base = (double)i * h;
    if (i == 0 || i == m - 1) return base;
    return base + (dg_u01(dg_hash3(seed, stream, lattice_id)) - 0.5) * 2.0 * jit * h;
}

DG_FN double dg_gauss(uint64_t seed, uint64_t stream, uint64_t i) {
    const double u1 = dg_u01(dg_hash3(seed, stream, i)), u2 = dg_u01(dg_hash3(seed, stream + 1, i));
    return sqrt(-2.0 * dg_log(u1 > 0 ? u1 : 1e-300)) * dg_cos(2.0 * DG_PI * u2);
}

/* sum of the 64 Fourier modes at p (config 3's turbulence-like field) */
DG_FN double dg_fourier3(const DgModes* md, const double* p) {
    double s = 0.0;
    for (int q = 0; q < 64; ++q) {
        const double arg = 2.0 * DG_PI * (md->k[q][0] * p[0] + md->k[q][1] * p[1] + md->k[q][2] * p[2]) +
                           md->phase[q];
        s += md->amp[q] * dg_cos(arg);
    }
    return s;
}

/* Lattice id of vertex v for the permuted lattice configs (1, 3, 4). */
DG_FN uint64_t dg_lattice_id(const DgFeistel* perm, uint64_t v) { return dg_feistel(perm, v); }

/* Config 3: 3D jittered lattice (jitter +-0.25 h), 64 Fourier modes. */
DG_FN void dg_gen3(uint64_t m, uint64_t seed, uint64_t L, const DgModes* md, double* p, double* f) {
    const uint64_t i = L / (m * m), j = (L / m) % m, k = L % m;
    const double h = 1.0 / (double)(m - 1);
    p[0] = dg_jittered(i, m, h, 0.25, seed, 1, L);
    p[1] = dg_jittered(j, m, h, 0.25, seed, 2, L);
    p[2] = dg_jittered(k, m, h, 0.25, seed, 3, L);
    if (f) *f = dg_fourier3(md, p);
}

/* Config 1: 2D jittered lattice (+-0.3 h), sin(4 pi x) cos(4 pi y) + 8 Gaussian bumps. */
DG_FN void dg_gen1(uint64_t m, uint64_t seed, uint64_t L, const DgModes* md, double* p, double* f) {
    const uint64_t i = L / m, j = L % m;
    const double h = 1.0 / (double)(m - 1);
    const double x = dg_jittered(i, m, h, 0.3, seed, 1, L), y = dg_jittered(j, m, h, 0.3, seed, 2, L);
    p[0] = x;
    p[1] = y;
    if (!f) return;
    double s = dg_sin(4.0 * DG_PI * x) * dg_cos(4.0 * DG_PI * y);
    for (int q = 0; q < 8; ++q) {
        const double dx = x - md->bump[q][0], dy = y - md->bump[q][1];
        s += 0.2 * dg_exp(-(dx * dx + dy * dy) / 0.002);
    }
    *f = s;
}

/* Config 4: 2D jittered lattice, 5 fp32 variables: Gaussian bumps, Fourier
 * modes, a step discontinuity, sign * lognormal(0, 2), U(-1, 1) noise. */
DG_FN void dg_gen4(uint64_t m, uint64_t seed, uint64_t L, uint64_t v, const DgModes* md, double* p, float* f5) {
    const uint64_t i = L / m, j = L % m;
    const double h = 1.0 / (double)(m - 1);
    const double x = dg_jittered(i, m, h, 0.3, seed, 1, L), y = dg_jittered(j, m, h, 0.3, seed, 2, L);
    p[0] = x;
    p[1] = y;
    if (!f5) return;
    double b = 0.0;
    for (int q = 0; q < 8; ++q) {
        const double dx = x - md->bump[q][0], dy = y - md->bump[q][1];
        b += dg_exp(-(dx * dx + dy * dy) / 0.01);
    }
    double fm = 0.0;
    for (int q = 0; q < 16; ++q)
        fm += md->amp[q] * dg_cos(2.0 * DG_PI * (md->k[q][0] * x + md->k[q][1] * y) + md->phase[q]);
    const double step = (x > 0.5 + 0.1 * dg_sin(2.0 * DG_PI * y)) ? 1.0 : 0.0;
    const double u1 = dg_u01(dg_hash3(seed, 11, v)), u2 = dg_u01(dg_hash3(seed, 12, v));
    const double g = sqrt(-2.0 * dg_log(u1 > 0 ? u1 : 1e-300)) * dg_cos(2.0 * DG_PI * u2);
    const double sgn = (dg_hash3(seed, 13, v) & 1) ? 1.0 : -1.0;
    const double logn = sgn * dg_exp(2.0 * g);
    const double uni = 2.0 * dg_u01(dg_hash3(seed, 14, v)) - 1.0;
    f5[0] = (float)b;
    f5[1] = (float)fm;
    f5[2] = (float)(step + 0.05 * x);
    f5[3] = (float)logn;
    f5[4] = (float)uni;
}

/* Config 2: graded 2D annulus around (0.5, 0.5), r in [0.3, 0.45]: 90 % of
 * the vertices from the radial density exp(-((r - 0.4) / 0.02)^2) (a normal
 * with sigma 0.02/sqrt(2), truncated to the annulus), 10 % uniform over the
 * annulus area; theta ~ U[0, 2pi). Field tanh((r - 0.4) / 0.005) +
 * 0.05 cos(12 theta) + N(0, 1e-4). Vertices are i.i.d. (order already random). */
DG_FN void dg_gen2(uint64_t seed, uint64_t v, double* p, double* f) {
    double r;
    if (dg_u01(dg_hash3(seed, 1, v)) < 0.1) {
        const double a = dg_u01(dg_hash3(seed, 2, v));
        r = sqrt(0.09 + a * (0.2025 - 0.09));
    } else {
        r = 0.4;
        for (uint64_t t = 0; t < 64; ++t) {
            r = 0.4 + dg_gauss(seed, 3 + 2 * t, v) * (0.02 * DG_SQRT1_2);
            if (r >= 0.3 && r <= 0.45) break;
            r = 0.4;
        }
    }
    const double th = 2.0 * DG_PI * dg_u01(dg_hash3(seed, 200, v));
    double st, ct;
    dg_sincos(th, &st, &ct);
    p[0] = 0.5 + r * ct;
    p[1] = 0.5 + r * st;
    if (f) *f = dg_tanh((r - 0.4) / 0.005) + 0.05 * dg_cos(12.0 * th) + 1e-4 * dg_gauss(seed, 201, v);
}

/* Config 5: clustered 3D shell around the axis (0.5, 0.5, z): r = 0.2 +
 * N(0, 0.01), theta ~ U[0, 2pi), z ~ U[0, 1]; field = the config-3 Fourier
 * field x exp(-((r - 0.2) / 0.01)^2 / 2). */
DG_FN void dg_gen5(uint64_t seed, uint64_t v, const DgModes* md, double* p, double* f) {
    const double r = 0.2 + 0.01 * dg_gauss(seed, 1, v);
    const double th = 2.0 * DG_PI * dg_u01(dg_hash3(seed, 3, v));
    double st, ct;
    dg_sincos(th, &st, &ct);
    p[0] = 0.5 + r * ct;
    p[1] = 0.5 + r * st;
    p[2] = dg_u01(dg_hash3(seed, 4, v));
    if (f) {
        const double d = (r - 0.2) / 0.01;
        *f = dg_fourier3(md, p) * dg_exp(-0.5 * d * d);
    }
}

#endif /* UMCG_DATAGEN_CORE_H */
