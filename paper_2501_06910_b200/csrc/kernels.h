// Host-side launchers for the umcg kernels (one declaration per kernel family).
#pragma once

#include <vector>

#include "common.cuh"

namespace umcg {

// ---- stream.cu: zero-RLE varint stream encode / decode --------------------
constexpr int ENC_THREADS = 256;
constexpr int ENC_ITEMS = 8;  // <= 9 so a thread opens at most one literal
constexpr uint64_t ENC_TILE = ENC_THREADS * ENC_ITEMS;

struct StreamEncScratch {
    RleSum* csum = nullptr;         // [T/256] chunk aggregates -> exclusive prefixes
    RleSum* sums = nullptr;         // [T]   tile summaries
    RleState* states = nullptr;     // [T+1] entry state per tile (+ final)
    uint64_t* lit_total = nullptr;  // [T]   literal byte totals, keyed by opening tile
    uint64_t* pos = nullptr;        // [T+1] stream position of each tile's first byte (writers)
    uint32_t* glist = nullptr;      // [T]   tiles for the general writer (count in ctl->aux[4+comp])
    uint32_t* n_redo = nullptr;     // [1]   tiles whose summary needs the exact reduction (list in glist)
};
size_t stream_enc_scratch_bytes(uint64_t n);
StreamEncScratch stream_enc_carve(void* base, uint64_t n);

// Encode codes[0..n) (u32 or u64 varint values) as the zero-RLE token stream.
// Writes ctl->stream_len[comp]; output at dst + ctl->stream_off[comp] when
// dst_off_from_ctl, else at dst.
void stream_encode_u32(const uint32_t* codes, uint64_t n, const StreamEncScratch& s, DevCtl* ctl,
                       int comp, uint8_t* dst, bool dst_off_from_ctl, cudaStream_t st);
void stream_encode_u64(const uint64_t* codes, uint64_t n, const StreamEncScratch& s, DevCtl* ctl,
                       int comp, uint8_t* dst, bool dst_off_from_ctl, cudaStream_t st);
// Phase split used by the pipeline (summaries/scan first, layout, then write).
void stream_plan_u32(const uint32_t* codes, uint64_t n, const StreamEncScratch& s, DevCtl* ctl,
                     int comp, cudaStream_t st, bool fast = false);
// fast: tile summaries by k_rle_tiles_fast (pays when zero codes are rare --
// fine residual bounds; token-dense streams are faster with k_rle_tiles)
void stream_plan_u16(const uint16_t* codes, uint64_t n, const StreamEncScratch& s, DevCtl* ctl, int comp,
                     cudaStream_t st, bool fast = false);
void stream_plan_u64(const uint64_t* codes, uint64_t n, const StreamEncScratch& s, DevCtl* ctl,
                     int comp, cudaStream_t st);
// Phases 2-4 only, when the tile summaries (s.sums) were produced by a fused
// code kernel (partition.cu).
void stream_plan_from_sums(uint64_t n, const StreamEncScratch& s, DevCtl* ctl, int comp, cudaStream_t st);
// u16 codes (narrow residual path)
void stream_write_u16(const uint16_t* codes, uint64_t n, const StreamEncScratch& s, DevCtl* ctl, int comp,
                      uint8_t* dst, bool dst_off_from_ctl, cudaStream_t st);
// Raw bytes as codes (lossless_compress of a byte buffer, lossless.hpp:24-51).
void stream_plan_u8(const uint8_t* bytes, uint64_t n, const StreamEncScratch& s, DevCtl* ctl, int comp,
                    cudaStream_t st);
void stream_write_u8(const uint8_t* bytes, uint64_t n, const StreamEncScratch& s, DevCtl* ctl, int comp,
                     uint8_t* dst, bool dst_off_from_ctl, cudaStream_t st);
void stream_write_u32(const uint32_t* codes, uint64_t n, const StreamEncScratch& s, DevCtl* ctl,
                      int comp, uint8_t* dst, bool dst_off_from_ctl, cudaStream_t st);
void stream_write_u64(const uint64_t* codes, uint64_t n, const StreamEncScratch& s, DevCtl* ctl,
                      int comp, uint8_t* dst, bool dst_off_from_ctl, cudaStream_t st);

// Decode: zero-RLE token stream -> varint codes (u64 values) [n].
struct StreamDecScratch {
    DevBuf tokens;   // token table
    DevBuf unpacked; // expanded byte stream
    DevBuf counts;   // per-tile code-end counts
    DevBuf parse;    // parallel token parse: exit table, chunk entries
};
// Returns on host after a synchronization: fills codes[0..n). Throws corrupt_payload.
void stream_decode(const uint8_t* d_stream, uint64_t len, uint64_t n, uint64_t* d_codes,
                   StreamDecScratch& s, DevCtl* ctl, cudaStream_t st);

// Raw byte RLE (umcg_rle_compress): bytes -> codes u64 view is not needed;
// treated as 1-byte "codes" where zero bytes are zero codes.
void rle_bytes_encode(const uint8_t* d_in, uint64_t n, const StreamEncScratch& s, DevCtl* ctl,
                      uint8_t* dst, cudaStream_t st);

// ---- gridinit.cu: umc::grid_init (grid_builder.hpp:201-282) ----------------
void grid_init_gpu(int D, uint64_t n_v, const double* d_xyz, int arity, uint64_t n_cells, const uint64_t* d_cells,
                   double percentile_k, uint64_t g_max, double delta, double seed_threshold,
                   std::vector<std::vector<double>>& axes, cudaStream_t st);

// ---- codes.cu: quantization codes (lattice fast path) + exact serial path --
struct NdShape {
    int D;
    uint64_t dims[8];
    uint64_t strides[8];
};
NdShape make_shape(int D, const uint64_t* dims);

// lossy codes of a values array. pred 0 none, 1 lorenzo_1d, 2 lorenzo_nd.
// Reads bin/tau from ctl->bin[comp]/tau_c[comp]. Flags ctl->need_serial[comp]
// when the lattice formulation may differ from the serial reference chain.
// k_ready: kbuf already holds the N-D lattice indices (fused upstream).
void codes_lossy_values(const double* v, uint64_t n, int pred, const NdShape& sh, DevCtl* ctl,
                        int comp, uint32_t* codes, int32_t* kbuf, cudaStream_t st, bool k_ready = false);
// lossless (tau == 0) XOR codes (codec.hpp:276-294); always exact.
void codes_lossless_values(const double* v, uint64_t n, int pred, const NdShape& sh,
                           uint64_t* codes, cudaStream_t st);

// Residual component (pipeline.hpp:140-146): r_i = x_i - g(x1)_i, lorenzo_1d.
struct ResidualSrc {
    const void* x;        // fp64 or fp32 field
    int x_f32;
    const uint32_t* node; // slot per vertex (nearest)
    const double* x1;     // grid component (exact cluster means)
    int g_kind;           // 0 nearest, 1 multilinear
    const double* coords; // [n*D] (multilinear)
    const double* axes;   // concatenated axes (multilinear)
    const uint64_t* axis_off;  // [D] offsets into axes
    const double* inv_cell;    // RN(1 / cell width), like axes (multilinear)
    double scale[3];           // index-guess scale per axis (multilinear)
    uint64_t shape[3];
    int D;
};
void codes_lossy_residual(const ResidualSrc& src, uint64_t n, DevCtl* ctl, uint32_t* codes,
                          cudaStream_t st);
void codes_lossless_residual(const ResidualSrc& src, uint64_t n, uint64_t* codes, cudaStream_t st);
void materialize_residual(const ResidualSrc& src, uint64_t n, double* out, cudaStream_t st);

// Exact serial replica of the reference predictor loop (codec.hpp:306-326):
// codes (u64) + escape records; n_esc -> ctl->n_esc[comp]. One GPU thread.
void serial_encode(const double* v, uint64_t n, int pred, const NdShape& sh, double tau,
                   uint64_t* codes, double* recon_scratch, uint64_t* esc_idx, double* esc_val,
                   DevCtl* ctl, int comp, cudaStream_t st);
// Escapes in parallel (escape.cu). lorenzo_1d: segmented lattice, fixed point
// over the escape set; false -> the caller takes the serial replica (non-lattice
// regime / no fixed point). Codes u64 (0 at escapes), records in index order.
size_t esc_scratch_bytes(uint64_t n);
bool seg_encode_1d(const double* v, uint64_t n, double tau, uint64_t* codes, uint64_t* esc_idx, double* esc_val,
                   void* scratch, DevCtl* ectl, DevCtl* hctl, uint64_t* n_esc, cudaStream_t st);
bool seg_decode_1d(const uint64_t* codes, uint64_t n, double tau, const uint64_t* esc_idx, const double* esc_val,
                   uint64_t n_esc, int64_t* K, int64_t* scratch, double* out, DevCtl* ectl, DevCtl* hctl,
                   cudaStream_t st);
// Stable compaction of flagged elements into (index, value) records; returns
// the count (host synchronization). tile_off: cdiv(n, 2048) u64 scratch.
uint64_t compact_flags(const uint8_t* F, const double* v, uint64_t n, uint64_t* idx, double* val, uint64_t* tile_off,
                       uint64_t* d_total, uint64_t* h_total, cudaStream_t st);
// N-D Lorenzo (D = 2, 3) with escapes: exact hyperplane wavefront of the
// reference loop (codes.cu). F: per-element escape flags (encode).
bool wave_encode_nd(const double* v, uint64_t n, const NdShape& sh, double tau, uint64_t* codes, double* recon,
                    uint8_t* F, cudaStream_t st);
bool wave_decode_nd(const uint64_t* codes, uint64_t n, const NdShape& sh, double tau, const uint64_t* esc_idx,
                    const double* esc_val, uint64_t n_esc, int32_t* eslot, double* out, cudaStream_t st);
// Exact serial replica of decode (codec.hpp:422-437).
// N-D lossless decode by hyperplane wavefront (D = 2, 3); false otherwise.
bool lossless_nd_wavefront(const uint64_t* codes, uint64_t n, const NdShape& sh, double* out, cudaStream_t st);
void serial_decode(const uint64_t* codes, uint64_t n, int pred, const NdShape& sh, double tau,
                   const uint64_t* esc_idx, const double* esc_val, uint64_t n_esc, double* out,
                   cudaStream_t st);

// Lattice reconstruction (decode fast path). recon = fl(K * bin), K the
// (N-D) prefix sum of zigzag-decoded codes. Writes max|K| key into
// ctl->max_abs_k[0]. out may be a grid array; for the residual component
// the recompose epilogue adds g(x1')_i.
void recon_lossy(const uint64_t* codes, uint64_t n, int pred, const NdShape& sh, double bin,
                 int64_t* kbuf, double* out, DevCtl* ctl, cudaStream_t st);
void recon_lossless(const uint64_t* codes, uint64_t n, int pred, double* out, uint64_t* scratch,
                    cudaStream_t st);
constexpr uint64_t RECON_TILE = 2048;  // scratch for recon_lossless / recon_lossy: cdiv(n, RECON_TILE)+1
// out[i] = g(x1')_i + recon2[i] (pipeline.hpp:206-208), in place on out.
void recompose(const ResidualSrc& src, uint64_t n, double* inout, cudaStream_t st);

// ---- interp.cu: range, budget, cluster mean, fill --------------------------
void minmax(const void* x, int x_f32, uint64_t n, DevCtl* ctl, cudaStream_t st);
struct BudgetArgs {
    double tau, rho, coeff_abs_sum;
    int bound_kind;
    uint64_t n;
};
void budget(const BudgetArgs& a, DevCtl* ctl, cudaStream_t st);
void cluster_mean(const void* x, int x_f32, const uint32_t* perm, const uint32_t* seg_off,
                  uint64_t n_slots, double* x1, cudaStream_t st);
void fill_nearest_visited(const uint32_t* seg_off, uint64_t n_slots, uint64_t row, double* x1,
                          cudaStream_t st);

}  // namespace umcg
