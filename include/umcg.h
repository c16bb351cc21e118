/*
 * umcg -- B200 (sm_100a) implementation of the umc multi-component
 * compressor's data-parallel hot path, behind a plain C ABI.
 *
 * The reference exposes this path only as header-only C++ free functions:
 *   umc::compress   (reference proj/include/umc/pipeline.hpp:117-148)
 *   umc::decompress (pipeline.hpp:180-210)
 *   umc::encode / umc::decode / umc::parse_component (codec.hpp:220-441)
 *   umc::rle_compress / rle_decompress (lossless.hpp:24-70)
 *   umc::mapping_digest (serialize.hpp:300-303)
 *   umc::grid_coarsen (grid_builder.hpp:365-421)
 * Each entry point below names the reference function it replaces. Byte
 * formats (UMCZ archive, PQ component payload, zero-RLE stream) are the
 * reference's, bit for bit. The C++ drop-in wrapper that keeps the umc::
 * signatures is include/umc_b200/pipeline_gpu.hpp; the binding a maintainer
 * adds is shown in INTEGRATION.md.
 *
 * Conventions
 *  - Every function returns umcg_status; UMCG_OK == 0. The numeric values of
 *    the error statuses follow the order of the reference's exception types
 *    (common.hpp:19-38), so a C++ wrapper rethrows the identical type.
 *    umcg_last_error() returns a thread-local message for the last failure.
 *  - Device pointers are marked d_; they must be CUDA device memory on the
 *    plan's device. Host pointers are plain. Sizes are bytes or elements as
 *    named.
 *  - stream: a cudaStream_t passed as void* (NULL = legacy default stream).
 *    Compress/decompress wait for their device work before returning (they
 *    report lengths and data-dependent errors), so the call is complete on
 *    return: the last kernel of the call posts a completion ticket into
 *    pinned host memory after everything queued before it has finished, and
 *    the host waits for that ticket (UMCG_NO_MAILBOX=1: a plain
 *    cudaStreamSynchronize).
 *  - A plan is immutable after creation apart from its private workspace;
 *    calls on one plan are serialized by an internal mutex. For concurrency
 *    use one handle per thread: umcg_plan_clone gives a handle with its own
 *    workspace that shares the (read-only) mapping arrays of its origin.
 *  - Plans may live on different devices; every call runs on its plan's
 *    device (per-device kernel attributes, streams and buffers).
 *  - Unsupported inputs fail loudly: external codecs (>= 128) and lossless
 *    backends != 0 give UMCG_UNKNOWN_CODEC. There is no CPU fallback.
 */
#ifndef UMCG_H
#define UMCG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum umcg_status {
    UMCG_OK = 0,
    UMCG_ERROR = 1,                    /* umc::error */
    UMCG_MALFORMED_FILE = 2,           /* umc::malformed_file */
    UMCG_INDEX_OUT_OF_RANGE = 3,       /* umc::index_out_of_range */
    UMCG_NON_FINITE_VALUE = 4,         /* umc::non_finite_value */
    UMCG_IO_FAILURE = 5,               /* umc::io_failure */
    UMCG_DEGENERATE_MESH = 6,          /* umc::degenerate_mesh */
    UMCG_EMPTY_AFTER_FILTERING = 7,    /* umc::empty_after_filtering */
    UMCG_INTERNAL_INCONSISTENCY = 8,   /* umc::internal_inconsistency */
    UMCG_SEED_MODE_UNSUPPORTED = 9,    /* umc::seed_mode_unsupported */
    UMCG_UNKNOWN_CODEC = 10,           /* umc::unknown_codec */
    UMCG_CORRUPT_PAYLOAD = 11,         /* umc::corrupt_payload */
    UMCG_EXTERNAL_CODEC_VIOLATION = 12,/* umc::external_codec_violation */
    UMCG_SUBPROCESS_FAILURE = 13,      /* umc::subprocess_failure */
    UMCG_BUDGET_INADMISSIBLE = 14,     /* umc::budget_inadmissible */
    UMCG_MAPPING_MISMATCH = 15,        /* umc::mapping_mismatch */
    UMCG_ZERO_NORM_REFERENCE = 16,     /* umc::zero_norm_reference */
    UMCG_MISMATCHED_RUNS = 17,         /* umc::mismatched_runs */
    UMCG_CUDA_ERROR = 100,             /* CUDA runtime failure (no reference equivalent) */
    UMCG_INVALID_ARGUMENT = 101        /* NULL pointer / capacity too small */
} umcg_status;

/* umc::RectGrid (grid.hpp:16-32): dim axes, concatenated, strictly increasing. */
typedef struct umcg_grid_desc {
    int dim;                       /* 2 or 3 */
    const uint64_t* axis_sizes;    /* [dim], host */
    const double* axes;            /* [sum(axis_sizes)], host, axis 0 first */
} umcg_grid_desc;

/* umc::MappingTable (grid.hpp:79-92). */
typedef struct umcg_mapping_desc {
    int mode;                      /* 0 dense, 1 seed */
    uint64_t n_vertices;
    const uint64_t* assignments;   /* [n_vertices], host: node (dense) or visited position (seed) */
    uint64_t n_visited;
    const uint64_t* visited_nodes; /* [n_visited], host, seed mode only (strictly increasing) */
} umcg_mapping_desc;

/* umc::ErrorBudget (pipeline.hpp:25-29) + umc::CompressOptions (pipeline.hpp:81-86). */
typedef struct umcg_params {
    double tau;                    /* requested bound, in bound_kind units */
    double split_rho;              /* budget split, strictly inside (0,1) */
    int bound_kind;                /* 0 absolute, 1 relative_to_range */
    int g_kind;                    /* 0 nearest, 1 multilinear (BackInterpKind) */
    double coeff_abs_sum;          /* BackInterpSpec::coeff_abs_sum (1.0 for built-ins) */
    int fill;                      /* 0 zero, 1 nearest_visited (FillPolicy) */
    int codec_id;                  /* must be 0 (builtin PQ) */
    int backend_id;                /* must be 0 (builtin zero-RLE) */
} umcg_params;

typedef struct umcg_plan umcg_plan;

typedef struct umcg_plan_info {
    int dim;
    int mode;                      /* 0 dense, 1 seed */
    uint64_t n_vertices;
    uint64_t n_slots;              /* grid-component length: node count (dense) or visited count (seed) */
    uint64_t shape[3];             /* coarse grid axis sizes */
    uint64_t n_visited;            /* visited node count (both modes) */
    double visited_fraction;       /* n_visited / node count (grid_builder.hpp:409-410) */
    uint64_t digest;               /* mapping_digest (serialize.hpp:300-303), cached */
    int has_coords;                /* coordinates resident (multilinear g available) */
} umcg_plan_info;

/* Build the immutable device plan for a host mapping: uploads the grid and
 * mapping, stable-sorts vertices by slot (cluster-mean order), computes the
 * mapping digest once. coords (host, [n_vertices*mesh_dim]) may be NULL when
 * only nearest g is used. Replaces the per-call work of mapping_digest
 * (serialize.hpp:300) and the static inputs of interpolate_to_grid
 * (interp.hpp:46). */
umcg_status umcg_plan_create(const umcg_grid_desc* grid, const umcg_mapping_desc* mapping,
                             int mesh_dim, const double* coords, umcg_plan** out);

/* GPU grid_coarsen (grid_builder.hpp:365-421) from an initial grid and
 * device-resident vertex coordinates d_coords [n_vertices*dim]; builds the
 * plan directly (the mapping never leaves the GPU except for the digest).
 * keep_coords != 0 keeps a device copy of the coordinates for multilinear g. */
umcg_status umcg_plan_build(const umcg_grid_desc* init_grid, uint64_t n_vertices,
                            const double* d_coords, double seed_mode_threshold, int keep_coords,
                            umcg_plan** out);

umcg_status umcg_plan_destroy(umcg_plan* plan);
/* A second handle on the same plan with its own workspace (scratch buffers,
 * control block, streams): the static mapping arrays are shared, not copied.
 * Calls on different handles run concurrently (calls on one handle are
 * serialized). The origin's memory is released when it and every clone are
 * destroyed, in any order. */
umcg_status umcg_plan_clone(const umcg_plan* plan, umcg_plan** out);
umcg_status umcg_plan_get_info(const umcg_plan* plan, umcg_plan_info* info);

/* Copy the plan's mapping back to host arrays (tests / serialization):
 * assignments [n_vertices], visited [n_visited] (the visited node list in
 * both modes), axes [sum(shape)]. Any pointer may be NULL. */
umcg_status umcg_plan_export(const umcg_plan* plan, uint64_t* assignments, uint64_t* visited,
                             double* axes);

/* Upper bound of the archive size for a compress call on this plan. */
umcg_status umcg_compress_bound(const umcg_plan* plan, const char* name, uint64_t* bytes);

/* umc::compress + umc::serialize_archive (pipeline.hpp:117-148, 214-235) on
 * device memory: d_values [n_vertices] fp64 -> d_archive (UMCZ bytes). */
umcg_status umcg_compress(umcg_plan* plan, const umcg_params* params, const double* d_values,
                          const char* name, uint8_t* d_archive, uint64_t capacity,
                          uint64_t* archive_len, void* stream);

/* Batched entry: n_fields fp64 or fp32 fields of one mesh in one call
 * (BASELINE config 4). d_values is field-major [n_fields][n_vertices];
 * dtype 0 = fp64, 1 = fp32 (widened to fp64 in-kernel, as the oracle's
 * separate fp64 calls on (double)x). Archives are written back to back into
 * d_archive; archive_lens[f] receives each length. names may be NULL. */
umcg_status umcg_compress_batch(umcg_plan* plan, const umcg_params* params, const void* d_values,
                                int dtype, int n_fields, const char* const* names,
                                uint8_t* d_archive, uint64_t capacity, uint64_t* archive_lens,
                                void* stream);

/* Batched decompress (BASELINE config 4): n_fields archives packed back to
 * back in d_archives (archive_lens[f] each, as umcg_compress_batch writes
 * them) -> d_out field-major [n_fields][n_vertices]; dtype 0 = fp64 (the
 * reference's decode), 1 = fp32 (RN of the fp64 decode: the error bound holds
 * for the fp64 values; the narrowing adds at most half an fp32 ulp). */
umcg_status umcg_decompress_batch(umcg_plan* plan, const uint8_t* d_archives, const uint64_t* archive_lens,
                                  int n_fields, int dtype, void* d_out, void* stream);

/* umc::deserialize_archive + umc::decompress (pipeline.hpp:237-267, 180-210)
 * on device memory: d_archive [len] -> d_out [n_vertices] fp64. Baseline
 * archives (flag 8) decode the single component. */
umcg_status umcg_decompress(umcg_plan* plan, const uint8_t* d_archive, uint64_t len,
                            double* d_out, void* stream);

/* Host-buffer conveniences (the reference's value-semantics call shape):
 * H2D of the inputs, the device call, D2H of the outputs, all inside. */
umcg_status umcg_compress_host(umcg_plan* plan, const umcg_params* params, const double* values,
                               const char* name, uint8_t* archive, uint64_t capacity,
                               uint64_t* archive_len);
umcg_status umcg_decompress_host(umcg_plan* plan, const uint8_t* archive, uint64_t len,
                                 double* out);
/* umcg_decompress_host that calls uploaded(ctx) (on the calling thread) once
 * the next field's host->device copy can be queued without delaying this
 * archive's upload: after the upload when it uses a copy engine, right away
 * when the archive is pinned mapped memory (read by the SMs). Each host
 * thread's calls use their own CUDA stream. */
umcg_status umcg_decompress_host_notify(umcg_plan* plan, const uint8_t* archive, uint64_t len,
                                        double* out, void (*uploaded)(void* ctx), void* ctx);

/* umcg_decompress_host for an archive held in pieces (e.g. the container
 * header and the two component payloads of an umc::Archive, pipeline.hpp:
 * 214-235): the pieces are uploaded back to back, so the caller never
 * concatenates them on the host. */
umcg_status umcg_decompress_host_parts(umcg_plan* plan, const uint8_t* const* parts, const uint64_t* lens,
                                       int n_parts, double* out);

/* Single component codec: umc::encode (codec.hpp:220-334) with codec 0 /
 * backend 0, and umc::decode (codec.hpp:364-441). predictor: 0 none,
 * 1 lorenzo_1d, 2 lorenzo_nd; ndims <= 8. tau == 0 selects the lossless
 * XOR path (codec.hpp:276-294). */
uint64_t umcg_encode_bound(uint64_t n, int ndims);
umcg_status umcg_encode(const double* d_values, uint64_t n, int predictor, int ndims,
                        const uint64_t* dims, double tau, int codec_id, int backend_id,
                        uint8_t* d_out, uint64_t capacity, uint64_t* out_len, void* stream);
umcg_status umcg_decode(const uint8_t* d_payload, uint64_t len, double* d_out, uint64_t n_capacity,
                        uint64_t* n_out, void* stream);

/* umc::grid_init (grid_builder.hpp:201-282) on the device: the initial
 * rectilinear grid from the mesh's per-axis edge lengths -- cell edges
 * (arity 3 tri, 4 quad, 8 hex; traverse_mesh) or, with no cells, each
 * vertex's exact 1-nearest neighbour (knn_edge_stats) -- at the k-th
 * nearest-rank percentile, raised by delta while an axis would exceed g_max
 * nodes. d_coords [n_v*dim], d_cells [n_cells*arity] (u64 vertex ids).
 * Writes axis_sizes[dim] and, when axes != NULL, the concatenated axes
 * (axes_cap doubles). cfg NULL = the reference defaults (50, 4096, 5, 0.35).
 * The result feeds umcg_plan_build (grid_coarsen). */
typedef struct umcg_grid_config {
    double percentile_k;
    uint64_t g_max;
    double delta;
    double seed_mode_threshold;
} umcg_grid_config;
umcg_status umcg_grid_init(int dim, uint64_t n_vertices, const double* d_coords, int cell_arity,
                           uint64_t n_cells, const uint64_t* d_cells, const umcg_grid_config* cfg,
                           uint64_t* axis_sizes, double* axes, uint64_t axes_cap, void* stream);

/* Serialization baseline (pipeline.hpp:152-176, baseline_archive): the
 * field in file order as ONE lorenzo_1d component at the full budget,
 * tau_abs = resolve_tau_abs(budget, values); archive flag 8, digest 0, empty
 * residual component. Decoded by umcg_decode on component 1 (the drop-in
 * wrapper's decompress does this, pipeline.hpp:184-187). */
uint64_t umcg_baseline_bound(uint64_t n, uint64_t name_len);
umcg_status umcg_compress_baseline(const umcg_params* params, const double* d_values, uint64_t n,
                                   const char* name, uint8_t* d_archive, uint64_t capacity,
                                   uint64_t* out_len, void* stream);

/* Zero-RLE byte stage alone (lossless.hpp:24-70, rle_compress /
 * rle_decompress), device to device. umcg_rle_bound(n) bounds the output of
 * umcg_rle_compress; errors follow rle_decompress (corrupt_payload). */
uint64_t umcg_rle_bound(uint64_t n);
umcg_status umcg_rle_compress(const uint8_t* d_in, uint64_t n, uint8_t* d_out, uint64_t capacity,
                              uint64_t* out_len, void* stream);
umcg_status umcg_rle_decompress(const uint8_t* d_in, uint64_t n, uint8_t* d_out,
                                uint64_t capacity, uint64_t* out_len, void* stream);

/* Synthetic BASELINE inputs generated on the device (SplitMix64-seeded,
 * counter-based). config: 1 (2D jittered lattice),
 * 2 (2D graded annulus), 3 (3D jittered lattice), 4 (2D lattice, 5 fp32
 * variables), 5 (3D clustered cylinder shell). lattice = points per axis for
 * configs 1, 3, 4 and the vertex count for configs 2, 5. d_coords [n*dim]
 * fp64; d_values [n_fields*n] (fp64, or fp32 for config 4). Returns n via
 * *n_out when pointers are NULL. */
umcg_status umcg_gen_config(int config, uint64_t lattice, uint64_t seed, double* d_coords,
                            void* d_values, uint64_t* n_out, void* stream);

/* Instrumentation: number of kernels this library launched since load, and
 * how many times a component took the exact one-thread replica of the
 * reference recurrence (escapes, non-lattice regimes; 0 on normal data). */
uint64_t umcg_kernel_launches(void);
uint64_t umcg_serial_fallbacks(void);
/* Per-kernel timing with CUDA events on the launching stream (hot kernels
 * only). Enable, run, then dump "name total_ms launches" lines into buf;
 * returns the full text length. */
void umcg_profile_enable(int on);
uint64_t umcg_profile_dump(char* buf, uint64_t cap);
const char* umcg_last_error(void);
const char* umcg_version(void);

#ifdef __cplusplus
}
#endif
#endif /* UMCG_H */
