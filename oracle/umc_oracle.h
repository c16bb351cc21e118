/* TEST INFRASTRUCTURE ONLY -- CPU oracle, never part of the product path.
 *
 * Plain-C restatement of the reference hot path (umc::compress /
 * umc::decompress with the built-in predictor-quantizer codec and the
 * zero-RLE byte stage). Each function cites the reference file:line it
 * restates (paths relative to /root/reference/proj/include/umc/).
 *
 * Pinned against: the reference's own golden images (regenerated from
 * tests/support/golden_recipe.hpp, sha256 recorded in SURVEY.md 8(c)) and
 * against oracle/_ref/libumcref.so (the unmodified reference compiled from
 * its headers) over the fixture set in tests/golden/.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load this library, and only as the checker.
 */
#ifndef UMC_ORACLE_H
#define UMC_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* error kinds: same numbering as include/umcg.h (umcg_status) */
const char* umco_last_error(void);
void umco_free(void* p);

uint64_t umco_fnv1a64(const uint8_t* p, uint64_t n, uint64_t seed);

int umco_rle_compress(const uint8_t* in, uint64_t n, uint8_t** out, uint64_t* out_len);
int umco_rle_decompress(const uint8_t* in, uint64_t n, uint8_t** out, uint64_t* out_len);

/* predictor: 0 none, 1 lorenzo_1d, 2 lorenzo_nd; codec 0 only */
int umco_encode(const double* v, uint64_t n, int predictor, int ndims, const uint64_t* dims,
                double tau, uint8_t** out, uint64_t* out_len);
int umco_decode(const uint8_t* p, uint64_t len, double** out, uint64_t* n_out);

int umco_split_budget(double tau_abs, double rho, double coeff_abs_sum, double* tau1,
                      double* tau2);

typedef struct {
    int dim;                       /* 2 or 3 */
    const uint64_t* axis_sizes;    /* dim entries */
    const double* axes;            /* concatenated axis coordinates */
    int mode;                      /* 0 dense, 1 seed */
    uint64_t n_v;
    const uint64_t* assignments;   /* n_v */
    uint64_t n_visited;
    const uint64_t* visited;       /* n_visited (seed mode) */
    const double* coords;          /* n_v * dim, or NULL (nearest g only) */
} umco_setup;

typedef struct {
    double tau, rho, coeff_abs_sum;
    int bound_kind; /* 0 absolute, 1 relative_to_range */
    int g_kind;     /* 0 nearest, 1 multilinear */
    int fill;       /* 0 zero, 1 nearest_visited */
} umco_params;

uint64_t umco_mapping_digest(const umco_setup* s);
int umco_interpolate_to_grid(const umco_setup* s, const double* x, int fill, double* x1);
int umco_residuals(const umco_setup* s, const double* x, int fill, int g_kind, double* x2);
int umco_compress(const umco_setup* s, const double* x, const char* name, const umco_params* p,
                  uint8_t** out, uint64_t* out_len);
int umco_decompress(const umco_setup* s, const uint8_t* ar, uint64_t len, double* out);

#ifdef __cplusplus
}
#endif
#endif
