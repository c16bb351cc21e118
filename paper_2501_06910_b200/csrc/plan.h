// The immutable per-mesh device plan + per-call workspace.
#pragma once

#include <atomic>
#include <mutex>

#include "kernels.h"

struct umcg_plan {
    int device = 0;
    int dim = 2;
    int mode = 0;                 // 0 dense, 1 seed
    uint64_t n = 0;               // vertices
    uint64_t n_slots = 0;         // grid-component length
    uint64_t node_count = 0;      // coarse grid nodes
    uint64_t n_visited = 0;
    uint64_t shape[3] = {1, 1, 1};
    double visited_fraction = 0.0;
    uint64_t digest = 0;
    std::vector<double> axes;        // concatenated coarse axes (host copy)
    std::vector<uint64_t> axis_off;  // [dim]
    // device-resident static inputs
    umcg::DevBuf d_node;     // u32 [n]   slot of each vertex (dense node / seed position)
    umcg::DevBuf d_perm;     // u32 [n]   vertices stably sorted by slot
    umcg::DevBuf d_seg;      // u32 [n_slots+1] segment offsets into perm
    umcg::DevBuf d_visited;  // u64 [n_visited] visited linear node ids (seed mode)
    umcg::DevBuf d_axes;     // f64 concatenated axes
    umcg::DevBuf d_axis_off; // u64 [dim]
    umcg::DevBuf d_inv_cell; // f64, like d_axes: RN(1 / cell width) per axis cell
    double axis_scale[3] = {0, 0, 0};  // (m - 1) / (a[m-1] - a[0]): index guess
    umcg::DevBuf d_coords;   // f64 [n*dim] (multilinear g), optional
    bool has_coords = false;
    // multilinear g, layout E (built on first multilinear use, partition.cu
    // ml_prep): the per-axis cell fractions t_d of every vertex (they depend
    // only on the static coordinates and axes) and its cell bits
    umcg::DevBuf d_mlT;      // f64 [dim*n] structure of arrays
    umcg::DevBuf d_mlB;      // u8  [n] bit d: cell lower index = slot index - 1 along d; 0x80: no slot hint
    bool has_mlprep = false;
    // bucketed layout for the partitioned compress path (partition.cu):
    // buckets are contiguous slot ranges holding <= kBucketCap vertices
    // (a heavier slot gets a bucket of its own).
    // Physical layout "E": epochs of kEpoch consecutive vertices; inside an
    // epoch, vertices grouped by bucket (ascending vertex within a group).
    // Both directions of the permutation are then gathers inside one
    // epoch's window (L2 resident).
    uint64_t n_buckets = 0;
    uint64_t n_epochs = 0;
    uint32_t bucket_cap = 4096, bucket_nodes = 1016;  // kBucketCap / kBucketCapL (and slots)
    umcg::DevBuf d_srcE;     // u32 [n]    vertex at layout-E position p
    umcg::DevBuf d_dstE;     // u32 [n]    layout-E position of vertex i
    umcg::DevBuf d_ech;      // u32 [E*(B+1)] offset of bucket b inside epoch e's block
    umcg::DevBuf d_bct;      // uint2 [B*(E+1)] per bucket: (first bucket-local index, layout-E base) per epoch
    umcg::DevBuf d_regular;  // u32 [n_regular] buckets with <= kBucketCap vertices (pipelined kernel)
    uint64_t n_regular = 0;
    umcg::DevBuf d_lnode;    // u16 [n]    bucket-local slot of bucket-order element
    umcg::DevBuf d_lperm;    // u16 [n]    bucket-local element of node-sorted position
    umcg::DevBuf d_lslot;    // u16 [n]    shared-memory slot of node-sorted position (TMA staging)
    umcg::DevBuf d_bk;       // u32 [2*(B+1)] bucket start (vertex) and first slot
    // vertex tiles of kRTile consecutive vertices (k_resid_codes): the
    // layout-E positions of a tile's vertices in ascending order -- runs of
    // consecutive positions, one per bucket chunk the tile meets -- and the
    // tile-local vertex of each
    umcg::DevBuf d_rPt;      // u32 [n]
    umcg::DevBuf d_rLt;      // u16 [n]
    // clones (umcg_plan_clone) alias the static arrays above of their origin;
    // the origin is freed when it and all of its clones are destroyed
    umcg_plan* origin = nullptr;
    std::atomic<int> refs{1};
    // workspace (serialized by mu; a clone has its own)
    std::mutex mu;
    umcg::DevBuf ctl, x1, codes1, codes2, kbuf, enc1, enc2, hdr, scratch_a, scratch_b, scratch_c,
        scratch_d, dx1, dcodes, esc_aux, esc_ctl;
    umcg::StreamDecScratch dec, dec2;
    umcg::SideStream side;  // grid component's chain runs beside the residual's
    umcg::PinnedBuf hctl, hstage;
    umcg::Mailbox mail;  // small device -> host results (control block, headers, verdict)
};

namespace umcg {

// Host-side FNV-1a-64 of serialize_mapping bytes (serialize.hpp:255-267, 300-303).
uint64_t mapping_digest_host(int mode, uint64_t n, const uint64_t* assign, uint64_t n_visited,
                             const uint64_t* visited);
// The same digest from the device-resident mapping (digest.cu: FNV-1a chained
// in parallel through per-chunk affine maps keyed by the hash's low byte).
// UMCG_DIGEST_HOST=1 keeps the byte-serial host loop; UMCG_DIGEST_CHECK=1
// computes both and fails on a difference.
uint64_t mapping_digest_device(int mode, uint64_t n, const uint32_t* d_assign, uint64_t n_visited,
                               const uint64_t* d_visited, umcg::DevBuf& scratch, cudaStream_t st);
// Same digest with u32 assignments (widened to u64 LE bytes as the reference writes them).
uint64_t mapping_digest_host32(int mode, uint64_t n, const uint32_t* assign, uint64_t n_visited,
                               const uint64_t* visited);

// Stable LSD radix sort of (u32 key, u32 value) pairs on key bits
// [begin_bit, end_bit) and an in-place exclusive u32 scan (radix.cu; plan-time).
// vals_in == nullptr sorts the indices 0..n-1. keys_in / vals_in are not
// modified and must not alias the outputs.
void radix_sort_pairs_u32(const uint32_t* keys_in, uint32_t* keys_out, const uint32_t* vals_in, uint32_t* vals_out,
                          uint64_t n, int begin_bit, int end_bit, umcg::DevBuf& tmp_pairs, umcg::DevBuf& tmp_hist,
                          umcg::DevBuf& tmp_scan, cudaStream_t st);
// u64 keys; vals_out == nullptr sorts the keys alone.
void radix_sort_u64(const uint64_t* keys_in, uint64_t* keys_out, const uint32_t* vals_in, uint32_t* vals_out,
                    uint64_t n, int begin_bit, int end_bit, umcg::DevBuf& tmp_pairs, umcg::DevBuf& tmp_hist,
                    umcg::DevBuf& tmp_scan, cudaStream_t st);
void exclusive_scan_u32(uint32_t* d_a, uint64_t n, umcg::DevBuf& scratch, cudaStream_t st);

// Build perm / seg_off from d_node on the plan (stable radix sort by slot),
// then the bucketed layout (plan_build_buckets).
void plan_build_segments(umcg_plan* p, cudaStream_t st);
constexpr uint32_t kBucketCap = 4096;   // vertices per bucket (smem staging; two 512-thread CTAs per SM)
#ifndef UMCG_EPOCH_BITS
#define UMCG_EPOCH_BITS 22
#endif
constexpr uint64_t kEpoch = 1ull << UMCG_EPOCH_BITS;  // vertices per epoch of layout E
constexpr uint32_t kMaxEpochs = 2048;    // k_bucket stages per-epoch chunk prefixes
constexpr uint32_t kBucketNodes = 1016; // slots per bucket
// Large buckets for big uniform meshes: 8192 vertices / 2032 slots, one
// 1024-thread CTA per SM (A/B, config 3: k_bucket_tma 0.696 -> 0.665 ms and,
// through the longer runs of a vertex tile in a bucket chunk,
// k_resid_codes_sr 0.455 -> 0.387 ms; compress 2.415 -> 2.328 ms). Meshes
// with heavy clusters lose with one CTA per SM (a long ordered sum stalls the
// whole CTA: config 2 0.48 -> 0.57 ms), and so do smaller fields and
// multilinear plans (wider x1 bands per bucket): plan_build_buckets picks.
constexpr uint32_t kBucketCapL = 8192;
constexpr uint32_t kBucketNodesL = 2032;
#ifndef UMCG_RTILE_BITS
#define UMCG_RTILE_BITS 15
#endif
constexpr uint32_t kRTileBits = UMCG_RTILE_BITS;
constexpr uint32_t kRTile = 1u << kRTileBits;  // vertices per k_resid_codes tile (a multiple of ENC_TILE)
void plan_build_buckets(umcg_plan* p, cudaStream_t st);

// Component payload decode (codec.hpp:364-441) of a payload in device memory
// into d_out [n]; header already parsed. Throws the reference's error kinds.
struct CompHeader {
    int codec, pred, backend, D;
    double tau;
    uint64_t n, dims[8];
    uint64_t n_esc;
    uint64_t esc_off;     // byte offset of the escape records in the payload
    uint64_t stream_off;  // byte offset of the RLE stream in the payload
    uint64_t stream_len;
};
void decode_component(umcg_plan* ws, const CompHeader& h, const uint8_t* d_payload, double* d_out,
                      cudaStream_t st);

}  // namespace umcg

namespace umcg {
// partition.cu: the partitioned (bucketed) compress path for nearest g.
void partition_values(const void* x, int x_f32, umcg_plan* p, double* xp, DevCtl* ctl, cudaStream_t st);
// narrow: KE int16 and residual codes u16 (the caller guarantees
// |K2| <= 16383 from the budget: |x - x1| <= range, see api.cu).
// K1 (optional): the dense N-D grid component's lattice indices of x1,
// fused (D1 = grid rank).
void bucket_means_residuals(umcg_plan* p, const double* xp, DevCtl* ctl, double* x1, void* Kp, bool narrow,
                            int32_t* K1, int D1, cudaStream_t st);
// Returns whether the RLE tile summaries were written too (else the caller
// runs the stream plan over the codes).
// fine: a fine relative bound (zero codes rare): the run-sorted kernel, summaries by the fast pass.
bool resid_codes_tiles(umcg_plan* p, const void* Kp, void* codes, bool narrow, bool fine, const StreamEncScratch& s,
                       const DevCtl* ctl, cudaStream_t st);
// Multilinear g in bucket order (layout E): residual lattice indices KE
// (compress) and the recomposition x' = g + x2' (decompress, gE [n] scratch).
void ml_residuals(umcg_plan* p, const double* xE, const double* x1, DevCtl* ctl, void* KE, bool narrow,
                  cudaStream_t st);
void ml_recompose(umcg_plan* p, const double* x1, double* gE, double* d_out, cudaStream_t st);
// g in layout E only (the fused residual decode gathers it back, DEC_RECOMPOSE_GE).
void ml_layout_g(umcg_plan* p, const double* x1, double* gE, cudaStream_t st);
}  // namespace umcg
