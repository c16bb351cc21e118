/* TEST INFRASTRUCTURE ONLY -- CPU oracle restating the reference hot path.
 * See umc_oracle.h for scope and pinning. Reference paths are relative to
 * /root/reference/proj/include/umc/. Compiled with -ffp-contract=off like
 * the reference (proj/CMakeLists.txt:16-17) so every FP operation rounds
 * exactly as the reference's does.
 */
#include "umc_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static _Thread_local char g_err[256];

static int fail(int kind, const char* msg) {
    snprintf(g_err, sizeof g_err, "%s", msg);
    return kind;
}

const char* umco_last_error(void) { return g_err; }
void umco_free(void* p) { free(p); }

enum {
    E_ERROR = 1, E_MALFORMED = 2, E_INDEX = 3, E_NONFINITE = 4, E_SEED = 9, E_CODEC = 10,
    E_CORRUPT = 11, E_BUDGET = 14, E_MAPPING = 15
};

/* ---- byte buffer: ByteWriter (common.hpp:45-80) -------------------------- */
typedef struct { uint8_t* p; uint64_t n, cap; } buf_t;

static void bw_reserve(buf_t* b, uint64_t extra) {
    if (b->n + extra <= b->cap) return;
    uint64_t c = b->cap ? b->cap : 64;
    while (c < b->n + extra) c *= 2;
    b->p = (uint8_t*)realloc(b->p, c);
    b->cap = c;
}
static void bw_u8(buf_t* b, uint8_t v) { bw_reserve(b, 1); b->p[b->n++] = v; }
static void bw_le(buf_t* b, uint64_t v, int k) {           /* common.hpp:75-77 */
    bw_reserve(b, (uint64_t)k);
    for (int i = 0; i < k; ++i) b->p[b->n++] = (uint8_t)(v >> (8 * i));
}
static void bw_f64(buf_t* b, double v) { uint64_t u; memcpy(&u, &v, 8); bw_le(b, u, 8); }
static void bw_bytes(buf_t* b, const void* p, uint64_t n) {
    bw_reserve(b, n);
    if (n) memcpy(b->p + b->n, p, n);
    b->n += n;
}
static void bw_varint(buf_t* b, uint64_t v) {              /* common.hpp:60-66 */
    while (v >= 0x80) { bw_u8(b, (uint8_t)v | 0x80); v >>= 7; }
    bw_u8(b, (uint8_t)v);
}

/* ---- ByteReader (common.hpp:83-127); errors are corrupt_payload ----------- */
typedef struct { const uint8_t* p; uint64_t n, pos; int err; } rd_t;

static int rd_need(rd_t* r, uint64_t k) {
    if (r->err) return 0;
    if (r->n - r->pos < k) { r->err = 1; return 0; }
    return 1;
}
static uint8_t rd_u8(rd_t* r) { return rd_need(r, 1) ? r->p[r->pos++] : 0; }
static uint64_t rd_le(rd_t* r, int k) {
    if (!rd_need(r, (uint64_t)k)) return 0;
    uint64_t v = 0;
    for (int i = 0; i < k; ++i) v |= (uint64_t)r->p[r->pos + i] << (8 * i);
    r->pos += (uint64_t)k;
    return v;
}
static double rd_f64(rd_t* r) { uint64_t u = rd_le(r, 8); double v; memcpy(&v, &u, 8); return v; }
static uint64_t rd_varint(rd_t* r) {                       /* common.hpp:99-107 */
    uint64_t v = 0;
    for (int shift = 0; shift < 64; shift += 7) {
        uint8_t b = rd_u8(r);
        if (r->err) return 0;
        v |= (uint64_t)(b & 0x7f) << shift;
        if (!(b & 0x80)) return v;
    }
    r->err = 2; /* varint exceeds 64 bits */
    return 0;
}

static uint64_t zz_enc(int64_t v) { return ((uint64_t)v << 1) ^ (uint64_t)(v >> 63); } /* :129 */
static int64_t zz_dec(uint64_t v) { return (int64_t)(v >> 1) ^ -(int64_t)(v & 1); }       /* :133 */

uint64_t umco_fnv1a64(const uint8_t* p, uint64_t n, uint64_t seed) {   /* common.hpp:137-145 */
    uint64_t h = seed;
    for (uint64_t i = 0; i < n; ++i) { h ^= p[i]; h *= 0x100000001b3ull; }
    return h;
}

/* ---- zero-RLE byte stage (lossless.hpp:24-70) ----------------------------- */
static void rle_into(buf_t* w, const uint8_t* data, uint64_t n) {
    uint64_t i = 0, lit_start = 0;
    while (i < n) {
        if (data[i] == 0) {
            uint64_t j = i;
            while (j < n && data[j] == 0) ++j;
            if (j - i >= 8) {                                   /* kMinZeroRun */
                if (i > lit_start) {
                    bw_u8(w, 0x01); bw_varint(w, i - lit_start);
                    bw_bytes(w, data + lit_start, i - lit_start);
                }
                bw_u8(w, 0x00); bw_varint(w, j - i);
                lit_start = j;
            }
            i = j;
        } else {
            ++i;
        }
    }
    if (n > lit_start) {
        bw_u8(w, 0x01); bw_varint(w, n - lit_start);
        bw_bytes(w, data + lit_start, n - lit_start);
    }
}

int umco_rle_compress(const uint8_t* in, uint64_t n, uint8_t** out, uint64_t* out_len) {
    buf_t w = {0};
    rle_into(&w, in, n);
    *out = w.p ? w.p : (uint8_t*)malloc(1);
    *out_len = w.n;
    return 0;
}

static int rle_expand(const uint8_t* in, uint64_t n, buf_t* out) {
    rd_t r = {in, n, 0, 0};
    while (r.pos != r.n) {
        uint8_t tok = rd_u8(&r);
        uint64_t len = rd_varint(&r);
        if (r.err) return fail(E_CORRUPT, r.err == 2 ? "varint exceeds 64 bits" : "unexpected end of data");
        if (tok == 0x00) {
            bw_reserve(out, len);
            memset(out->p + out->n, 0, len);
            out->n += len;
        } else if (tok == 0x01) {
            if (!rd_need(&r, len)) return fail(E_CORRUPT, "unexpected end of data");
            bw_bytes(out, in + r.pos, len);
            r.pos += len;
        } else {
            return fail(E_CORRUPT, "unknown token in lossless stream");
        }
    }
    return 0;
}

int umco_rle_decompress(const uint8_t* in, uint64_t n, uint8_t** out, uint64_t* out_len) {
    buf_t w = {0};
    int e = rle_expand(in, n, &w);
    if (e) { free(w.p); return e; }
    *out = w.p ? w.p : (uint8_t*)malloc(1);
    *out_len = w.n;
    return 0;
}

/* ---- predictors (codec.hpp:61-110) ---------------------------------------- */
typedef struct {
    int predictor, D;
    uint64_t dims[8], strides[8], idx[8];
} pred_t;

static void pred_init(pred_t* s, int predictor, int D, const uint64_t* dims) {
    memset(s, 0, sizeof *s);
    s->predictor = predictor;
    s->D = D;
    for (int d = 0; d < D; ++d) { s->dims[d] = dims[d]; s->strides[d] = 1; }
    for (int d = D - 1; d >= 1; --d) s->strides[d - 1] = s->strides[d] * dims[d];   /* :87-92 */
}

static double pred_predict(const pred_t* s, const double* recon, uint64_t lin) {
    if (s->predictor == 0) return 0.0;
    if (s->predictor == 1) return lin == 0 ? 0.0 : recon[lin - 1];
    double pred = 0.0;                                            /* lorenzo_predict :61-80 */
    for (unsigned mask = 1; mask < (1u << s->D); ++mask) {
        uint64_t off = 0;
        int ok = 1;
        for (int d = 0; d < s->D; ++d) {
            if ((mask >> d) & 1u) {
                if (s->idx[d] == 0) { ok = 0; break; }
                off += s->strides[d];
            }
        }
        if (!ok) continue;
        const double term = recon[lin - off];
        pred += (__builtin_popcount(mask) & 1) ? term : -term;
    }
    return pred;
}

static void pred_advance(pred_t* s) {                             /* :104-109 */
    for (int d = s->D - 1; d >= 0; --d) {
        if (++s->idx[d] < s->dims[d]) return;
        s->idx[d] = 0;
    }
}

/* ---- builtin PQ encode (codec.hpp:220-334, codec_id 0, backend 0) --------- */
static int encode_into(buf_t* out, const double* values, uint64_t n, int predictor, int D,
                       const uint64_t* dims, double tau) {
    if (!(tau >= 0.0)) return fail(E_ERROR, "tau_abs must be >= 0");
    uint64_t prod = 1;
    for (int d = 0; d < D; ++d) prod *= dims[d];
    if (D == 0 || prod != n) return fail(E_ERROR, "codec dims product does not equal element count");
    if (D > 8) return fail(E_ERROR, "codec supports at most 8 dimensions");
    for (uint64_t i = 0; i < n; ++i)
        if (!isfinite(values[i])) return fail(E_NONFINITE, "non-finite input to encode");

    bw_u8(out, 0); bw_u8(out, (uint8_t)predictor); bw_u8(out, 0); bw_u8(out, 0);   /* :225-233 */
    bw_f64(out, tau);
    bw_le(out, n, 8);
    bw_u8(out, (uint8_t)D);
    for (int d = 0; d < D; ++d) bw_le(out, dims[d], 8);

    pred_t ps;
    pred_init(&ps, predictor, D, dims);
    double* recon = (double*)malloc((n ? n : 1) * sizeof(double));
    buf_t qs = {0}, esc = {0};
    uint64_t n_esc = 0;
    if (tau == 0.0) {                                              /* :276-294 */
        for (uint64_t i = 0; i < n; ++i) {
            const double p = pred_predict(&ps, recon, i);
            uint64_t a, b;
            memcpy(&a, &values[i], 8);
            memcpy(&b, &p, 8);
            bw_varint(&qs, a ^ b);
            recon[i] = values[i];
            pred_advance(&ps);
        }
    } else {                                                       /* :300-326 */
        const double bin = 2.0 * tau;
        const double kQLimit = 2147483647.0;
        for (uint64_t i = 0; i < n; ++i) {
            const double p = pred_predict(&ps, recon, i);
            const double qd = round((values[i] - p) / bin);
            int escape = !(fabs(qd) <= kQLimit);
            double r = 0.0;
            if (!escape) {
                r = p + qd * bin;
                escape = !(fabs(values[i] - r) <= tau);
            }
            if (escape) {
                bw_le(&esc, i, 8);
                bw_f64(&esc, values[i]);
                ++n_esc;
                bw_varint(&qs, 0);
                recon[i] = values[i];
            } else {
                bw_varint(&qs, zz_enc((int64_t)qd));
                recon[i] = r;
            }
            pred_advance(&ps);
        }
    }
    bw_le(out, n_esc, 8);                                          /* :329-331 */
    bw_bytes(out, esc.p, esc.n);
    rle_into(out, qs.p, qs.n);
    free(recon); free(qs.p); free(esc.p);
    return 0;
}

int umco_encode(const double* v, uint64_t n, int predictor, int ndims, const uint64_t* dims,
                double tau, uint8_t** out, uint64_t* out_len) {
    buf_t w = {0};
    int e = encode_into(&w, v, n, predictor, ndims, dims, tau);
    if (e) { free(w.p); return e; }
    *out = w.p;
    *out_len = w.n;
    return 0;
}

/* ---- decode (codec.hpp:364-441) ------------------------------------------- */
typedef struct { int codec, pred, backend, D; double tau; uint64_t n, dims[8]; } comp_hdr;

/* parse_component (codec.hpp:342-362) header; returns corrupt on truncation */
static int parse_hdr(rd_t* r, comp_hdr* h) {
    h->codec = rd_u8(r);
    h->pred = rd_u8(r);
    h->backend = rd_u8(r);
    (void)rd_u8(r);
    h->tau = rd_f64(r);
    h->n = rd_le(r, 8);
    h->D = rd_u8(r);
    if (r->err) return fail(E_CORRUPT, "unexpected end of data");
    if (h->pred > 2) return fail(E_CORRUPT, "bad predictor byte");
    uint64_t prod = 1;
    for (int d = 0; d < h->D; ++d) {
        uint64_t v = rd_le(r, 8);
        if (d < 8) h->dims[d] = v;
        prod *= v;
    }
    if (r->err) return fail(E_CORRUPT, "unexpected end of data");
    if (h->D == 0 || prod != h->n) return fail(E_CORRUPT, "dims product does not match element count");
    return 0;
}

static int decode_payload(const uint8_t* p, uint64_t len, double** out_v, uint64_t* n_out) {
    rd_t r = {p, len, 0, 0};
    comp_hdr h;
    int e = parse_hdr(&r, &h);
    if (e) return e;
    const uint64_t n_esc = rd_le(&r, 8);
    if (r.err) return fail(E_CORRUPT, "unexpected end of data");
    if (h.codec != 0) return fail(E_CODEC, "only the builtin PQ codec (id 0) is in scope");
    if (h.D > 8) return fail(E_CORRUPT, "too many dims");
    if (n_esc > h.n) return fail(E_CORRUPT, "escape count exceeds element count");
    uint64_t* esc_idx = (uint64_t*)malloc((n_esc ? n_esc : 1) * 8);
    double* esc_val = (double*)malloc((n_esc ? n_esc : 1) * 8);
    for (uint64_t k = 0; k < n_esc; ++k) {
        esc_idx[k] = rd_le(&r, 8);
        esc_val[k] = rd_f64(&r);
        if (r.err) { free(esc_idx); free(esc_val); return fail(E_CORRUPT, "unexpected end of data"); }
        if (esc_idx[k] >= h.n || (k > 0 && esc_idx[k] <= esc_idx[k - 1])) {
            free(esc_idx); free(esc_val);
            return fail(E_CORRUPT, "bad escape index sequence");
        }
    }
    if (h.backend != 0) { free(esc_idx); free(esc_val); return fail(E_CODEC, "lossless backend not registered"); }
    buf_t un = {0};
    e = rle_expand(p + r.pos, len - r.pos, &un);
    if (e) { free(esc_idx); free(esc_val); free(un.p); return e; }
    rd_t qs = {un.p, un.n, 0, 0};
    pred_t ps;
    pred_init(&ps, h.pred, h.D, h.dims);
    double* recon = (double*)malloc((h.n ? h.n : 1) * 8);
    const double bin = 2.0 * h.tau;
    uint64_t next_escape = 0;
    for (uint64_t i = 0; i < h.n; ++i) {
        const double pr = pred_predict(&ps, recon, i);
        const uint64_t z = rd_varint(&qs);
        if (qs.err) {
            free(esc_idx); free(esc_val); free(un.p); free(recon);
            return fail(E_CORRUPT, qs.err == 2 ? "varint exceeds 64 bits" : "unexpected end of data");
        }
        if (h.tau == 0.0) {
            uint64_t b;
            memcpy(&b, &pr, 8);
            b ^= z;
            memcpy(&recon[i], &b, 8);
        } else if (next_escape < n_esc && esc_idx[next_escape] == i) {
            recon[i] = esc_val[next_escape++];
        } else {
            recon[i] = pr + (double)zz_dec(z) * bin;
        }
        pred_advance(&ps);
    }
    const int trailing = qs.pos != qs.n;
    free(esc_idx); free(esc_val); free(un.p);
    if (trailing) { free(recon); return fail(E_CORRUPT, "trailing bytes in quantized stream"); }
    if (h.tau == 0.0 && n_esc != 0) { free(recon); return fail(E_CORRUPT, "lossless payload with escapes"); }
    *out_v = recon;
    *n_out = h.n;
    return 0;
}

int umco_decode(const uint8_t* p, uint64_t len, double** out, uint64_t* n_out) {
    return decode_payload(p, len, out, n_out);
}

/* ---- budget (pipeline.hpp:31-57, 94) --------------------------------------- */
int umco_split_budget(double tau_abs, double rho, double coeff_abs_sum, double* tau1, double* tau2) {
    if (!(rho > 0.0) || !(rho < 1.0)) return fail(E_BUDGET, "rho must lie strictly inside (0, 1)");
    if (!(tau_abs >= 0.0)) return fail(E_BUDGET, "tau must be >= 0");
    if (!(coeff_abs_sum > 0.0)) return fail(E_BUDGET, "coefficient sum must be positive");
    double t1 = rho * tau_abs / coeff_abs_sum;
    const double t2 = (1.0 - rho) * tau_abs;
    while (coeff_abs_sum * t1 + t2 > tau_abs) t1 = nextafter(t1, 0.0);
    *tau1 = t1;
    *tau2 = t2;
    return 0;
}

static double shave(double tau) { return tau * (1.0 - 1e-9); }

/* ---- mapping digest (serialize.hpp:255-267, 300-303) ----------------------- */
uint64_t umco_mapping_digest(const umco_setup* s) {
    uint8_t hdr[4 + 2 + 1 + 8];
    memcpy(hdr, "UMCP", 4);
    hdr[4] = 1; hdr[5] = 0;               /* u16 kFormatVersion */
    hdr[6] = (uint8_t)s->mode;
    for (int i = 0; i < 8; ++i) hdr[7 + i] = (uint8_t)(s->n_v >> (8 * i));
    uint64_t h = umco_fnv1a64(hdr, sizeof hdr, 0xcbf29ce484222325ull);
    uint8_t b[8];
    for (uint64_t i = 0; i < s->n_v; ++i) {
        for (int k = 0; k < 8; ++k) b[k] = (uint8_t)(s->assignments[i] >> (8 * k));
        h = umco_fnv1a64(b, 8, h);
    }
    if (s->mode == 1) {
        for (int k = 0; k < 8; ++k) b[k] = (uint8_t)(s->n_visited >> (8 * k));
        h = umco_fnv1a64(b, 8, h);
        for (uint64_t i = 0; i < s->n_visited; ++i) {
            for (int k = 0; k < 8; ++k) b[k] = (uint8_t)(s->visited[i] >> (8 * k));
            h = umco_fnv1a64(b, 8, h);
        }
    }
    return h;
}

static uint64_t node_count(const umco_setup* s) {
    uint64_t n = 1;
    for (int d = 0; d < s->dim; ++d) n *= s->axis_sizes[d];
    return n;
}

/* ---- f: cluster mean (interp.hpp:46-93) ------------------------------------ */
int umco_interpolate_to_grid(const umco_setup* s, const double* x, int fill, double* x1) {
    const uint64_t n_slots = s->mode == 1 ? s->n_visited : node_count(s);
    uint64_t* count = (uint64_t*)calloc(n_slots ? n_slots : 1, 8);
    for (uint64_t j = 0; j < n_slots; ++j) x1[j] = 0.0;
    for (uint64_t i = 0; i < s->n_v; ++i) {
        const uint64_t slot = s->assignments[i];
        if (slot >= n_slots) { free(count); return fail(E_INDEX, "assignment out of range"); }
        x1[slot] += x[i];
        count[slot] += 1;
    }
    for (uint64_t j = 0; j < n_slots; ++j)
        if (count[j]) x1[j] /= (double)count[j];
    if (s->mode == 0 && fill == 1) {                             /* :66-91 */
        const uint64_t row = s->axis_sizes[s->dim - 1];
        const uint64_t n_rows = n_slots / row;
        for (uint64_t r = 0; r < n_rows; ++r) {
            double* v = x1 + r * row;
            const uint64_t* c = count + r * row;
            int64_t prev = -1;
            for (uint64_t t = 0; t < row; ++t) {
                if (c[t]) { prev = (int64_t)t; continue; }
                int64_t next = -1;
                for (uint64_t u = t + 1; u < row; ++u) if (c[u]) { next = (int64_t)u; break; }
                if (prev < 0 && next < 0) break;           /* whole row unvisited */
                int64_t src;
                if (prev < 0) src = next;
                else if (next < 0) src = prev;
                else src = ((int64_t)t - prev <= next - (int64_t)t) ? prev : next;
                v[t] = v[src];
            }
        }
    }
    free(count);
    return 0;
}

/* ---- g: multilinear (interp.hpp:97-132) ------------------------------------ */
static double multilinear_at(const umco_setup* s, const double* node_values, const double* p) {
    const int D = s->dim;
    uint64_t lo_idx[3] = {0, 0, 0};
    double t[3] = {0, 0, 0};
    const double* axis = s->axes;
    for (int d = 0; d < D; ++d) {
        const uint64_t n = s->axis_sizes[d];
        if (n == 1) { lo_idx[d] = 0; t[d] = 0.0; axis += n; continue; }
        uint64_t lo = 0, hi = n;                      /* upper_bound */
        while (lo < hi) {
            uint64_t mid = lo + (hi - lo) / 2;
            if (!(p[d] < axis[mid])) lo = mid + 1; else hi = mid;
        }
        uint64_t h = lo;
        if (h < 1) h = 1;
        if (h > n - 1) h = n - 1;
        const uint64_t l = h - 1;
        const double w = (p[d] - axis[l]) / (axis[h] - axis[l]);
        lo_idx[d] = l;
        t[d] = w < 0.0 ? 0.0 : (w > 1.0 ? 1.0 : w);   /* std::clamp(w, 0, 1) */
        axis += n;
    }
    double acc = 0.0;
    for (unsigned corner = 0; corner < (1u << D); ++corner) {
        double w = 1.0;
        uint64_t lin = 0;
        for (int d = 0; d < D; ++d) {
            const int high = (corner >> d) & 1u;
            w *= high ? t[d] : 1.0 - t[d];
            const uint64_t n = s->axis_sizes[d];
            uint64_t idx = lo_idx[d] + (high ? 1 : 0);
            if (idx >= n) idx = n - 1;
            lin = lin * n + idx;
        }
        if (w != 0.0) acc += w * node_values[lin];
    }
    return acc;
}

/* back_interpolate (interp.hpp:140-158) */
static int back_interp(const umco_setup* s, const double* x1, int g_kind, int seed, double* out) {
    if (g_kind == 0) {
        for (uint64_t i = 0; i < s->n_v; ++i) out[i] = x1[s->assignments[i]];
        return 0;
    }
    if (seed) return fail(E_SEED, "multilinear back-interpolation needs a dense grid component");
    for (uint64_t i = 0; i < s->n_v; ++i)
        out[i] = multilinear_at(s, x1, s->coords + i * (uint64_t)s->dim);
    return 0;
}

/* compute_residuals (interp.hpp:161-170) against the exact grid component */
int umco_residuals(const umco_setup* s, const double* x, int fill, int g_kind, double* x2) {
    const int seed = s->mode == 1;
    const uint64_t n1 = seed ? s->n_visited : node_count(s);
    double* x1 = (double*)malloc((n1 ? n1 : 1) * 8);
    int e = umco_interpolate_to_grid(s, x, fill, x1);
    if (!e) e = back_interp(s, x1, g_kind, seed, x2);
    free(x1);
    if (e) return e;
    for (uint64_t i = 0; i < s->n_v; ++i) x2[i] = x[i] - x2[i];
    return 0;
}

/* ---- compress (pipeline.hpp:117-148) + serialize_archive (:214-235) -------- */
int umco_compress(const umco_setup* s, const double* x, const char* name, const umco_params* p,
                  uint8_t** out, uint64_t* out_len) {
    for (uint64_t i = 0; i < s->n_v; ++i)                         /* validate_field */
        if (!isfinite(x[i])) return fail(E_NONFINITE, "non-finite field value");
    if (!(p->tau >= 0.0)) return fail(E_BUDGET, "tau must be >= 0");
    double tau_abs = p->tau;
    if (p->bound_kind == 1) {                                     /* resolve_tau_abs */
        double lo = 0, hi = 0;
        if (s->n_v) {
            lo = hi = x[0];
            for (uint64_t i = 1; i < s->n_v; ++i) {
                if (x[i] < lo) lo = x[i];
                if (hi < x[i]) hi = x[i];
            }
        }
        tau_abs = p->tau * (hi - lo);
    }
    double tau1, tau2;
    int e = umco_split_budget(tau_abs, p->rho, p->coeff_abs_sum, &tau1, &tau2);
    if (e) return e;
    const int seed = s->mode == 1;
    const uint64_t n1 = seed ? s->n_visited : node_count(s);
    double* x1 = (double*)malloc((n1 ? n1 : 1) * 8);
    double* x2 = (double*)malloc((s->n_v ? s->n_v : 1) * 8);
    e = umco_interpolate_to_grid(s, x, p->fill, x1);
    if (!e) e = back_interp(s, x1, p->g_kind, seed, x2);
    if (e) { free(x1); free(x2); return e; }
    for (uint64_t i = 0; i < s->n_v; ++i) x2[i] = x[i] - x2[i];  /* compute_residuals */

    buf_t c1 = {0}, c2 = {0};
    uint64_t dims1[3];
    int D1;
    if (seed) { D1 = 1; dims1[0] = s->n_visited; }                /* grid_codec_spec :96-110 */
    else { D1 = s->dim; for (int d = 0; d < D1; ++d) dims1[d] = s->axis_sizes[d]; }
    e = encode_into(&c1, x1, n1, seed ? 1 : 2, D1, dims1, shave(tau1));
    uint64_t dn = s->n_v;
    if (!e) e = encode_into(&c2, x2, s->n_v, 1, 1, &dn, shave(tau2));
    free(x1); free(x2);
    if (e) { free(c1.p); free(c2.p); return e; }

    buf_t w = {0};
    bw_bytes(&w, "UMCZ", 4);
    bw_le(&w, 1, 2);
    uint16_t flags = 0;
    if (seed) flags |= 1u;
    if (p->g_kind == 1) flags |= 2u;
    if (p->bound_kind == 1) flags |= 4u;
    bw_le(&w, flags, 2);
    const uint64_t nl = name ? strlen(name) : 0;
    if (nl > 0xffff) { free(c1.p); free(c2.p); return fail(E_MALFORMED, "field name too long"); }
    bw_le(&w, nl, 2);
    bw_bytes(&w, name, nl);
    bw_le(&w, umco_mapping_digest(s), 8);
    bw_f64(&w, p->tau);
    bw_f64(&w, p->rho);
    bw_le(&w, c1.n, 8);
    bw_bytes(&w, c1.p, c1.n);
    bw_le(&w, c2.n, 8);
    bw_bytes(&w, c2.p, c2.n);
    free(c1.p); free(c2.p);
    *out = w.p;
    *out_len = w.n;
    return 0;
}

/* ---- deserialize_archive (pipeline.hpp:237-267) + decompress (:180-210) ---- */
int umco_decompress(const umco_setup* s, const uint8_t* ar, uint64_t len, double* out) {
    rd_t r = {ar, len, 0, 0};
    if (len < 4) return fail(E_MALFORMED, "file too short for archive header");
    if (memcmp(ar, "UMCZ", 4) != 0) return fail(E_MALFORMED, "bad magic for archive");
    r.pos = 4;
    const uint64_t ver = rd_le(&r, 2);
    if (r.err) return fail(E_MALFORMED, "truncated archive");
    if (ver != 1) return fail(E_MALFORMED, "unsupported archive format version");
    const uint64_t flags = rd_le(&r, 2);
    const uint64_t nl = rd_le(&r, 2);
    if (!rd_need(&r, nl)) return fail(E_MALFORMED, "truncated archive");
    r.pos += nl;
    const uint64_t digest = rd_le(&r, 8);
    (void)rd_f64(&r);
    (void)rd_f64(&r);
    const uint64_t l1 = rd_le(&r, 8);
    if (r.err || !rd_need(&r, l1)) return fail(E_MALFORMED, "truncated archive");
    const uint8_t* p1 = ar + r.pos;
    r.pos += l1;
    {
        rd_t h1 = {p1, l1, 0, 0};
        comp_hdr hh;
        if (parse_hdr(&h1, &hh)) return fail(E_MALFORMED, "truncated archive: bad component 1");
    }
    const uint64_t l2 = rd_le(&r, 8);
    if (r.err || !rd_need(&r, l2)) return fail(E_MALFORMED, "truncated archive");
    const uint8_t* p2 = ar + r.pos;
    r.pos += l2;
    const int baseline = (flags & 8u) != 0;
    comp_hdr h2 = {0};
    if (l2) {
        rd_t h2r = {p2, l2, 0, 0};
        if (parse_hdr(&h2r, &h2)) return fail(E_MALFORMED, "truncated archive: bad component 2");
    } else if (!baseline) {
        return fail(E_MALFORMED, "missing residual component");
    }
    if (r.pos != len) return fail(E_MALFORMED, "trailing bytes in archive");

    double* v1 = NULL;
    uint64_t n1 = 0;
    int e;
    if (baseline) {
        e = decode_payload(p1, l1, &v1, &n1);
        if (e) return e;
        memcpy(out, v1, n1 * 8);
        free(v1);
        return 0;
    }
    if (digest != umco_mapping_digest(s)) return fail(E_MAPPING, "archive was compressed with a different mapping");
    const int seed = s->mode == 1;
    if (seed != (int)(flags & 1u)) return fail(E_MAPPING, "mapping mode does not match archive");
    rd_t h1r = {p1, l1, 0, 0};
    comp_hdr h1;
    parse_hdr(&h1r, &h1);
    if (h1.n != (seed ? s->n_visited : node_count(s))) return fail(E_MAPPING, "grid size does not match archive component");
    if (h2.n != s->n_v) return fail(E_MAPPING, "vertex count does not match archive component");
    e = decode_payload(p1, l1, &v1, &n1);
    if (e) return e;
    double* v2 = NULL;
    uint64_t n2 = 0;
    e = decode_payload(p2, l2, &v2, &n2);
    if (e) { free(v1); return e; }
    e = back_interp(s, v1, (flags & 2u) ? 1 : 0, seed, out);
    if (!e)
        for (uint64_t i = 0; i < n2; ++i) out[i] = out[i] + v2[i];
    free(v1); free(v2);
    return e;
}
