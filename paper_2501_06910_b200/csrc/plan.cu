// Plan construction: device-resident mapping, stable slot sort, digest, and
// the GPU grid_coarsen (grid_builder.hpp:286-421).

#include <algorithm>
#include <cmath>

#include "plan.h"

namespace umcg {

namespace {

constexpr int THREADS = 256;
inline unsigned blocks(uint64_t n) { return (unsigned)cdiv(n, THREADS); }

struct Fnv {
    uint64_t h = 0xcbf29ce484222325ull;
    void byte(uint8_t b) { h ^= b; h *= 0x100000001b3ull; }
    void le(uint64_t v, int k) { for (int i = 0; i < k; ++i) byte((uint8_t)(v >> (8 * i))); }
};

__global__ void k_iota(uint32_t* __restrict__ v, uint64_t n) {
    const uint64_t i = blockIdx.x * (uint64_t)THREADS + threadIdx.x;
    if (i < n) v[i] = (uint32_t)i;
}

__global__ void k_count(const uint32_t* __restrict__ node, uint64_t n, uint32_t* __restrict__ cnt) {
    const uint64_t i = blockIdx.x * (uint64_t)THREADS + threadIdx.x;
    if (i < n) atomicAdd(&cnt[node[i]], 1u);
}

__global__ void k_count_visited(const uint32_t* __restrict__ seg, uint64_t n_slots,
                                unsigned long long* __restrict__ out) {
    const uint64_t j = blockIdx.x * (uint64_t)THREADS + threadIdx.x;
    const int v = (j < n_slots && seg[j + 1] > seg[j]) ? 1 : 0;
    const int w = __syncthreads_count(v);
    if (threadIdx.x == 0 && w) atomicAdd(out, (unsigned long long)w);
}

// map_vertex (grid_builder.hpp:286-305): nearest node per axis, ties to the
// lower index, outside points clamp; per-axis plane index.
__global__ void k_map_axes(const double* __restrict__ coords, uint64_t n, int D,
                           const double* __restrict__ axes, const uint64_t* __restrict__ off,
                           const uint64_t* __restrict__ sizes, uint32_t* __restrict__ idx) {
    const uint64_t i = blockIdx.x * (uint64_t)THREADS + threadIdx.x;
    if (i >= n) return;
    for (int d = 0; d < D; ++d) {
        const double* a = axes + off[d];
        const uint64_t m = sizes[d];
        const double x = coords[i * D + d];
        uint64_t lo = 0, hi = m;  // std::lower_bound
        while (lo < hi) {
            const uint64_t mid = lo + (hi - lo) / 2;
            if (a[mid] < x) lo = mid + 1; else hi = mid;
        }
        uint64_t k;
        if (lo == 0) k = 0;
        else if (lo == m) k = m - 1;
        else k = (__dsub_rn(x, a[lo - 1]) <= __dsub_rn(a[lo], x)) ? lo - 1 : lo;
        idx[(uint64_t)d * n + i] = (uint32_t)k;
    }
}

__global__ void k_plane_flags(const uint32_t* __restrict__ idx, uint64_t n, int D,
                              const uint64_t* __restrict__ foff, uint8_t* __restrict__ flags) {
    const uint64_t i = blockIdx.x * (uint64_t)THREADS + threadIdx.x;
    if (i >= n) return;
    for (int d = 0; d < D; ++d) flags[foff[d] + idx[(uint64_t)d * n + i]] = 1;
}

// remap_after_coarsen (grid_builder.hpp:313-354)
__global__ void k_remap(const uint32_t* __restrict__ idx, uint64_t n, int D,
                        const int64_t* __restrict__ o2n, const uint64_t* __restrict__ foff,
                        const uint64_t* __restrict__ new_size, uint64_t* __restrict__ lin) {
    const uint64_t i = blockIdx.x * (uint64_t)THREADS + threadIdx.x;
    if (i >= n) return;
    uint64_t l = 0;
    for (int d = 0; d < D; ++d) l = l * new_size[d] + (uint64_t)o2n[foff[d] + idx[(uint64_t)d * n + i]];
    lin[i] = l;
}

// seed mode: position of each assignment in the sorted visited list.
__global__ void k_rank(const uint64_t* __restrict__ lin, uint64_t n, const uint64_t* __restrict__ vis,
                       uint64_t nv, uint32_t* __restrict__ out) {
    const uint64_t i = blockIdx.x * (uint64_t)THREADS + threadIdx.x;
    if (i >= n) return;
    const uint64_t x = lin[i];
    uint64_t lo = 0, hi = nv;
    while (lo < hi) {
        const uint64_t mid = lo + (hi - lo) / 2;
        if (vis[mid] < x) lo = mid + 1; else hi = mid;
    }
    out[i] = (uint32_t)lo;
}

__global__ void k_u64_to_u32(const uint64_t* __restrict__ a, uint64_t n, uint32_t* __restrict__ b) {
    const uint64_t i = blockIdx.x * (uint64_t)THREADS + threadIdx.x;
    if (i < n) b[i] = (uint32_t)a[i];
}

// ---- bucketed layout -------------------------------------------------------
__global__ void k_slot_bucket(const uint32_t* __restrict__ bnode, uint64_t B, uint32_t* __restrict__ sb) {
    const uint64_t b = blockIdx.x * (uint64_t)THREADS + threadIdx.x;
    if (b >= B) return;
    for (uint32_t j = bnode[b]; j < bnode[b + 1]; ++j) sb[j] = (uint32_t)b;
}

__global__ void k_bucket_keys(const uint32_t* __restrict__ node, uint64_t n, const uint32_t* __restrict__ sb,
                              uint32_t* __restrict__ keys) {
    const uint64_t i = blockIdx.x * (uint64_t)THREADS + threadIdx.x;
    if (i < n) keys[i] = sb[node[i]];
}

__global__ void k_dst_lnode(const uint32_t* __restrict__ L, const uint32_t* __restrict__ kb, uint64_t n,
                            const uint32_t* __restrict__ node, const uint32_t* __restrict__ bnode,
                            uint32_t* __restrict__ dst, uint16_t* __restrict__ lnode) {
    const uint64_t k = blockIdx.x * (uint64_t)THREADS + threadIdx.x;
    if (k >= n) return;
    const uint32_t v = L[k];
    dst[v] = (uint32_t)k;
    lnode[k] = (uint16_t)(node[v] - bnode[kb[k]]);
}

__global__ void k_epoch_keys(const uint32_t* __restrict__ node, uint64_t n, const uint32_t* __restrict__ sb,
                             uint64_t B, uint32_t* __restrict__ keys, uint32_t* __restrict__ cnt) {
    const uint64_t i = blockIdx.x * (uint64_t)THREADS + threadIdx.x;
    if (i >= n) return;
    const uint32_t k = (uint32_t)((i / kEpoch) * B + sb[node[i]]);
    keys[i] = k;
    atomicAdd(&cnt[k], 1u);
}

__global__ void k_dstE(const uint32_t* __restrict__ L, uint64_t n, uint32_t* __restrict__ dstE) {
    const uint64_t p = blockIdx.x * (uint64_t)THREADS + threadIdx.x;
    if (p < n) dstE[L[p]] = (uint32_t)p;
}

__global__ void k_rlt(const uint32_t* __restrict__ keys, uint64_t n, uint16_t* __restrict__ rLt) {
    const uint64_t k = blockIdx.x * (uint64_t)THREADS + threadIdx.x;
    if (k < n) rLt[k] = (uint16_t)(keys[k] & (kRTile - 1));
}

// per-epoch exclusive scan of bucket counts (one thread per epoch; E*B small)
__global__ void k_epoch_offsets(const uint32_t* __restrict__ cnt, uint64_t E, uint64_t B, uint32_t* __restrict__ ech) {
    const uint64_t e = blockIdx.x * (uint64_t)THREADS + threadIdx.x;
    if (e >= E) return;
    uint32_t acc = 0;
    for (uint64_t b = 0; b < B; ++b) {
        ech[e * (B + 1) + b] = acc;
        acc += cnt[e * B + b];
    }
    ech[e * (B + 1) + B] = acc;
}

// bucket-major chunk table: for bucket b, epoch e: x = first bucket-local
// index of the epoch-e chunk (x of e = E is the bucket size), y = its layout-E
// position. One thread per bucket (E is small).
__global__ void k_bucket_chunks(const uint32_t* __restrict__ ech, uint64_t E, uint64_t B, uint2* __restrict__ bct) {
    const uint64_t b = blockIdx.x * (uint64_t)THREADS + threadIdx.x;
    if (b >= B) return;
    uint32_t acc = 0;
    for (uint64_t e = 0; e < E; ++e) {
        const uint32_t o = ech[e * (B + 1) + b];
        bct[b * (E + 1) + e] = make_uint2(acc, (uint32_t)(e * kEpoch + o));
        acc += ech[e * (B + 1) + b + 1] - o;
    }
    bct[b * (E + 1) + E] = make_uint2(acc, 0u);
}

__global__ void k_lperm(const uint32_t* __restrict__ perm, uint64_t n, const uint32_t* __restrict__ dst,
                        const uint32_t* __restrict__ node, const uint32_t* __restrict__ sb,
                        const uint32_t* __restrict__ bstart, uint16_t* __restrict__ lperm) {
    const uint64_t k = blockIdx.x * (uint64_t)THREADS + threadIdx.x;
    if (k >= n) return;
    const uint32_t v = perm[k];
    lperm[k] = (uint16_t)(dst[v] - bstart[sb[node[v]]]);
}

// Shared-memory slot of each node-sorted element for the TMA bucket kernel
// (partition.cu k_bucket_tma): chunk e of a bucket is staged at slot base
// c0.x + 2e + phase_e, phase_e chosen so the slot and the layout-E position
// have the same parity (16-byte aligned bulk copies of 8-byte values).
__global__ void k_lslot(const uint32_t* __restrict__ perm, uint64_t n, const uint32_t* __restrict__ node,
                        const uint32_t* __restrict__ sb, const uint16_t* __restrict__ lperm,
                        const uint2* __restrict__ bct, uint64_t E, uint16_t* __restrict__ lslot) {
    const uint64_t q = blockIdx.x * (uint64_t)THREADS + threadIdx.x;
    if (q >= n) return;
    const uint32_t b = sb[node[perm[q]]];
    const uint32_t l = lperm[q];
    const uint2* c = bct + b * (E + 1);
    uint32_t lo = 0, hi = (uint32_t)E;  // last chunk with first index <= l
    while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) >> 1;
        if (c[mid].x <= l) lo = mid; else hi = mid;
    }
    const uint32_t e = lo;
    const uint32_t phase = (c[e].y - c[e].x - 2 * e) & 1u;
    lslot[q] = (uint16_t)(l + 2 * e + phase);
}

// Run heads of a sorted key array (1 where a new key starts), and the
// compaction of the heads through the exclusive scan of those flags.
__global__ void k_run_heads(const uint64_t* __restrict__ s, uint64_t n, uint32_t* __restrict__ f) {
    const uint64_t i = blockIdx.x * (uint64_t)THREADS + threadIdx.x;
    if (i < n) f[i] = (i == 0 || s[i] != s[i - 1]) ? 1u : 0u;
}
__global__ void k_unique_out(const uint64_t* __restrict__ s, uint64_t n, const uint32_t* __restrict__ pos,
                             uint64_t* __restrict__ out, unsigned long long* __restrict__ count) {
    const uint64_t i = blockIdx.x * (uint64_t)THREADS + threadIdx.x;
    if (i >= n) return;
    const bool head = i == 0 || s[i] != s[i - 1];
    if (head) out[pos[i]] = s[i];
    if (i == n - 1) *count = (unsigned long long)pos[i] + (head ? 1u : 0u);
}

}  // namespace

uint64_t mapping_digest_host(int mode, uint64_t n, const uint64_t* assign, uint64_t nv, const uint64_t* vis) {
    Fnv f;
    f.byte('U'); f.byte('M'); f.byte('C'); f.byte('P');
    f.le(1, 2);
    f.byte((uint8_t)mode);
    f.le(n, 8);
    for (uint64_t i = 0; i < n; ++i) f.le(assign[i], 8);
    if (mode == 1) {
        f.le(nv, 8);
        for (uint64_t i = 0; i < nv; ++i) f.le(vis[i], 8);
    }
    return f.h;
}

uint64_t mapping_digest_host32(int mode, uint64_t n, const uint32_t* assign, uint64_t nv, const uint64_t* vis) {
    Fnv f;
    f.byte('U'); f.byte('M'); f.byte('C'); f.byte('P');
    f.le(1, 2);
    f.byte((uint8_t)mode);
    f.le(n, 8);
    for (uint64_t i = 0; i < n; ++i) f.le(assign[i], 8);
    if (mode == 1) {
        f.le(nv, 8);
        for (uint64_t i = 0; i < nv; ++i) f.le(vis[i], 8);
    }
    return f.h;
}

void plan_build_segments(umcg_plan* p, cudaStream_t st) {
    // u32 layout positions (and the sorts' u32 ranks) bound a plan's size
    if (p->n > (uint64_t)INT32_MAX) fail(UMCG_INVALID_ARGUMENT, "more than 2^31-1 vertices per plan");
    const uint64_t n = p->n, ns = p->n_slots;
    uint32_t* node = p->d_node.as<uint32_t>(n ? n : 1);
    uint32_t* perm = p->d_perm.as<uint32_t>(n ? n : 1);
    uint32_t* seg = p->d_seg.as<uint32_t>(ns + 8);  // + padding for 16-byte bulk copies
    DevBuf tmp_keys, tmp_vals, cnt, scratch, rs_hist, rs_scan;
    uint32_t* keys_out = tmp_keys.as<uint32_t>(n ? n : 1);
    uint32_t* iota = tmp_vals.as<uint32_t>(n ? n : 1);
    uint32_t* c = cnt.as<uint32_t>(ns + 1);
    UMCG_CUDA(cudaMemsetAsync(c, 0, (ns + 1) * 4, st));
    if (n) {
        k_iota<<<blocks(n), THREADS, 0, st>>>(iota, n);
        UMCG_LAUNCHED();
        k_count<<<blocks(n), THREADS, 0, st>>>(node, n, c);
        UMCG_LAUNCHED();
        int end_bit = 1;
        while (end_bit < 32 && (1ull << end_bit) < ns) ++end_bit;
        // K0: vertices stably sorted by slot (radix.cu)
        radix_sort_pairs_u32(node, keys_out, iota, perm, n, 0, end_bit, scratch, rs_hist, rs_scan, st);
    }
    // seg = exclusive scan of the slot counts
    UMCG_CUDA(cudaMemcpyAsync(seg, c, (ns + 1) * 4, cudaMemcpyDeviceToDevice, st));
    exclusive_scan_u32(seg, ns + 1, rs_scan, st);
    // visited count (dense info)
    DevBuf vc;
    auto* v = vc.as<unsigned long long>(1);
    UMCG_CUDA(cudaMemsetAsync(v, 0, 8, st));
    k_count_visited<<<blocks(ns), THREADS, 0, st>>>(seg, ns, v);
    UMCG_LAUNCHED();
    unsigned long long hv = 0;
    UMCG_CUDA(cudaMemcpyAsync(&hv, v, 8, cudaMemcpyDeviceToHost, st));
    UMCG_CUDA(cudaStreamSynchronize(st));
    if (p->mode == 0) {
        p->n_visited = hv;
        p->visited_fraction = p->node_count ? (double)hv / (double)p->node_count : 0.0;
    }
    plan_build_buckets(p, st);
}

// Bucketed layout for the partitioned compress path: greedy contiguous slot
// ranges with <= kBucketCap vertices and <= kBucketNodes slots (a heavier
// slot forms its own bucket). dst = stable (by vertex) sort of vertices by
// bucket, so each bucket holds its vertices in ascending vertex order; lperm
// maps the node-sorted order (perm) into that bucket-local order.
void plan_build_buckets(umcg_plan* p, cudaStream_t st) {
    const uint64_t n = p->n, ns = p->n_slots;
    std::vector<uint32_t> seg(ns + 1);
    UMCG_CUDA(cudaMemcpyAsync(seg.data(), p->d_seg.get(), (ns + 1) * 4, cudaMemcpyDeviceToHost, st));
    UMCG_CUDA(cudaStreamSynchronize(st));
    // bucket size (plan.h kBucketCapL): large buckets for big fields without heavy clusters
    uint32_t max_slot = 0;
    for (uint64_t k = 0; k < ns; ++k) max_slot = std::max(max_slot, seg[k + 1] - seg[k]);
    const bool large = n >= (1ull << 26) && !p->has_coords && max_slot <= 64;
    p->bucket_cap = large ? kBucketCapL : kBucketCap;
    p->bucket_nodes = large ? kBucketNodesL : kBucketNodes;
    const uint32_t cap = p->bucket_cap, cap_nodes = p->bucket_nodes;
    std::vector<uint32_t> bnode;
    uint64_t j = 0;
    while (j < ns) {
        const uint64_t j0 = j;
        bnode.push_back((uint32_t)j0);
        if (seg[j0 + 1] - seg[j0] > cap) { j = j0 + 1; continue; }
        ++j;
        while (j < ns && j - j0 < cap_nodes && seg[j + 1] - seg[j0] <= cap) ++j;
    }
    const uint64_t B = bnode.size();
    bnode.push_back((uint32_t)ns);
    std::vector<uint32_t> tab(2 * (B + 1));
    for (uint64_t b = 0; b <= B; ++b) {
        tab[b] = seg[bnode[b]];
        tab[B + 1 + b] = bnode[b];
    }
    p->n_buckets = B;
    {
        std::vector<uint32_t> reg;
        for (uint64_t b = 0; b < B; ++b)
            if (tab[b + 1] - tab[b] <= cap) reg.push_back((uint32_t)b);
        p->n_regular = reg.size();
        uint32_t* dr = p->d_regular.as<uint32_t>(reg.size() + 1);
        if (!reg.empty()) UMCG_CUDA(cudaMemcpyAsync(dr, reg.data(), reg.size() * 4, cudaMemcpyHostToDevice, st));
        UMCG_CUDA(cudaStreamSynchronize(st));
    }
    uint32_t* dbk = p->d_bk.as<uint32_t>(tab.size());
    UMCG_CUDA(cudaMemcpyAsync(dbk, tab.data(), tab.size() * 4, cudaMemcpyHostToDevice, st));
    const uint32_t* bstart = dbk;
    const uint32_t* dbn = dbk + B + 1;
    DevBuf dstbuf;
    uint32_t* dst = dstbuf.as<uint32_t>(n ? n : 1);  // bucket-order position (temporary)
    uint16_t* lnode = p->d_lnode.as<uint16_t>(n + 16);  // + padding: 16-byte bulk copies may overrun
    uint16_t* lperm = p->d_lperm.as<uint16_t>(n + 16);
    if (!n || !B) { UMCG_CUDA(cudaStreamSynchronize(st)); return; }
    DevBuf sbuf, keys, keys_s, iota, L, scratch;
    uint32_t* sb = sbuf.as<uint32_t>(ns);
    k_slot_bucket<<<blocks(B), THREADS, 0, st>>>(dbn, B, sb);
    UMCG_LAUNCHED();
    uint32_t* kk = keys.as<uint32_t>(n);
    uint32_t* ks = keys_s.as<uint32_t>(n);
    uint32_t* io = iota.as<uint32_t>(n);
    uint32_t* Lv = L.as<uint32_t>(n);
    k_bucket_keys<<<blocks(n), THREADS, 0, st>>>(p->d_node.as<uint32_t>(1), n, sb, kk);
    UMCG_LAUNCHED();
    k_iota<<<blocks(n), THREADS, 0, st>>>(io, n);
    UMCG_LAUNCHED();
    int end_bit = 1;
    while (end_bit < 32 && (1ull << end_bit) < B) ++end_bit;
    DevBuf rs_hist, rs_scan;
    radix_sort_pairs_u32(kk, ks, io, Lv, n, 0, end_bit, scratch, rs_hist, rs_scan, st);
    k_dst_lnode<<<blocks(n), THREADS, 0, st>>>(Lv, ks, n, p->d_node.as<uint32_t>(1), dbn, dst, lnode);
    UMCG_LAUNCHED();
    k_lperm<<<blocks(n), THREADS, 0, st>>>(p->d_perm.as<uint32_t>(1), n, dst, p->d_node.as<uint32_t>(1), sb,
                                           bstart, lperm);
    UMCG_LAUNCHED();
    // layout E: stable sort by (epoch, bucket)
    const uint64_t E = cdiv(n, kEpoch);
    if (E > kMaxEpochs) fail(UMCG_INVALID_ARGUMENT, "too many vertices for layout E");
    p->n_epochs = E;
    DevBuf ecnt;
    uint32_t* ec = ecnt.as<uint32_t>(E * B + 1);
    UMCG_CUDA(cudaMemsetAsync(ec, 0, (E * B + 1) * 4, st));
    k_epoch_keys<<<blocks(n), THREADS, 0, st>>>(p->d_node.as<uint32_t>(1), n, sb, B, kk, ec);
    UMCG_LAUNCHED();
    k_iota<<<blocks(n), THREADS, 0, st>>>(io, n);
    UMCG_LAUNCHED();
    uint32_t* srcE = p->d_srcE.as<uint32_t>(n);
    end_bit = 1;
    while (end_bit < 32 && (1ull << end_bit) < E * B) ++end_bit;
    radix_sort_pairs_u32(kk, ks, io, srcE, n, 0, end_bit, scratch, rs_hist, rs_scan, st);
    k_dstE<<<blocks(n), THREADS, 0, st>>>(srcE, n, p->d_dstE.as<uint32_t>(n));
    UMCG_LAUNCHED();
    // vertex tiles: stable sort of the layout-E positions by the tile of their
    // vertex (bits kRTileBits.. of srcE) keeps each tile's positions ascending
    {
        k_iota<<<blocks(n), THREADS, 0, st>>>(io, n);
        UMCG_LAUNCHED();
        int hi = kRTileBits + 1;
        while (hi < 32 && (1ull << hi) < n) ++hi;
        uint32_t* rPt = p->d_rPt.as<uint32_t>(n);
        radix_sort_pairs_u32(srcE, ks, io, rPt, n, (int)kRTileBits, hi, scratch, rs_hist, rs_scan, st);
        k_rlt<<<blocks(n), THREADS, 0, st>>>(ks, n, p->d_rLt.as<uint16_t>(n));
        UMCG_LAUNCHED();
    }
    k_epoch_offsets<<<blocks(E), THREADS, 0, st>>>(ec, E, B, p->d_ech.as<uint32_t>(E * (B + 1)));
    UMCG_LAUNCHED();
    k_bucket_chunks<<<blocks(B), THREADS, 0, st>>>(p->d_ech.as<uint32_t>(1), E, B, p->d_bct.as<uint2>(B * (E + 1)));
    UMCG_LAUNCHED();
    k_lslot<<<blocks(n), THREADS, 0, st>>>(p->d_perm.as<uint32_t>(1), n, p->d_node.as<uint32_t>(1), sb, lperm,
                                           p->d_bct.as<uint2>(1), E, p->d_lslot.as<uint16_t>(n + 16));
    UMCG_LAUNCHED();
    UMCG_CUDA(cudaStreamSynchronize(st));
}

static void upload_grid(umcg_plan* p, const umcg_grid_desc* g) {
    if (!g || !g->axis_sizes || !g->axes) fail(UMCG_INVALID_ARGUMENT, "grid descriptor is NULL");
    if (g->dim != 2 && g->dim != 3) fail(UMCG_MALFORMED_FILE, "grid dimension must be 2 or 3");
    p->dim = g->dim;
    p->axes.clear();
    p->axis_off.assign(g->dim, 0);
    p->node_count = 1;
    for (int d = 0; d < g->dim; ++d) {
        const uint64_t m = g->axis_sizes[d];
        if (m == 0) fail(UMCG_MALFORMED_FILE, "empty grid axis");
        p->axis_off[d] = p->axes.size();
        p->shape[d] = m;
        p->node_count *= m;
        // validate_grid (grid.hpp:34-47)
        const double* a = g->axes + p->axis_off[d];
        for (uint64_t i = 0; i < m; ++i) {
            if (!std::isfinite(a[i])) fail(UMCG_NON_FINITE_VALUE, "non-finite axis coordinate");
            if (i > 0 && !(a[i] > a[i - 1])) fail(UMCG_MALFORMED_FILE, "grid axis not strictly increasing");
        }
        p->axes.insert(p->axes.end(), a, a + m);
    }
    for (int d = g->dim; d < 3; ++d) p->shape[d] = 1;
    double* da = p->d_axes.as<double>(p->axes.size());
    UMCG_CUDA(cudaMemcpy(da, p->axes.data(), p->axes.size() * 8, cudaMemcpyHostToDevice));
    // multilinear helpers: RN(1 / (a[l+1] - a[l])) per cell (correctly rounded
    // division by one fma correction, multilinear.cuh) and an index-guess scale
    std::vector<double> inv(p->axes.size(), 0.0);
    for (int d = 0; d < g->dim; ++d) {
        const double* a = p->axes.data() + p->axis_off[d];
        const uint64_t m = p->shape[d];
        for (uint64_t l = 0; l + 1 < m; ++l) inv[p->axis_off[d] + l] = 1.0 / (a[l + 1] - a[l]);
        p->axis_scale[d] = m > 1 ? (double)(m - 1) / (a[m - 1] - a[0]) : 0.0;
    }
    double* dinv = p->d_inv_cell.as<double>(inv.size());
    UMCG_CUDA(cudaMemcpy(dinv, inv.data(), inv.size() * 8, cudaMemcpyHostToDevice));
    uint64_t* doff = p->d_axis_off.as<uint64_t>(3);
    UMCG_CUDA(cudaMemcpy(doff, p->axis_off.data(), p->dim * 8, cudaMemcpyHostToDevice));
}

umcg_plan* plan_create_host(const umcg_grid_desc* g, const umcg_mapping_desc* m, int mesh_dim,
                            const double* coords) {
    if (!m) fail(UMCG_INVALID_ARGUMENT, "mapping descriptor is NULL");
    auto* p = new umcg_plan;
    try {
        UMCG_CUDA(cudaGetDevice(&p->device));
        upload_grid(p, g);
        p->mode = m->mode ? 1 : 0;
        p->n = m->n_vertices;
        if (p->n > (uint64_t)INT32_MAX) fail(UMCG_INVALID_ARGUMENT, "more than 2^31-1 vertices per plan");
        if (p->mode == 1) {
            p->n_slots = m->n_visited;
            p->n_visited = m->n_visited;
            // validate_mapping (grid.hpp:94-110)
            for (uint64_t i = 0; i < m->n_visited; ++i) {
                if (m->visited_nodes[i] >= p->node_count) fail(UMCG_INDEX_OUT_OF_RANGE, "visited node out of grid range");
                if (i > 0 && !(m->visited_nodes[i] > m->visited_nodes[i - 1]))
                    fail(UMCG_MALFORMED_FILE, "visited node list not strictly increasing");
            }
            p->visited_fraction = p->node_count ? (double)m->n_visited / (double)p->node_count : 0.0;
            uint64_t* dv = p->d_visited.as<uint64_t>(m->n_visited ? m->n_visited : 1);
            if (m->n_visited)
                UMCG_CUDA(cudaMemcpy(dv, m->visited_nodes, m->n_visited * 8, cudaMemcpyHostToDevice));
        } else {
            p->n_slots = p->node_count;
        }
        if (p->n_slots >= (1ull << 32)) fail(UMCG_INVALID_ARGUMENT, "grid component longer than 2^32-1");
        std::vector<uint32_t> a32(p->n);
        for (uint64_t i = 0; i < p->n; ++i) {
            const uint64_t a = m->assignments[i];
            if (a >= p->n_slots)
                fail(UMCG_INDEX_OUT_OF_RANGE, p->mode ? "seed assignment out of visited list range"
                                                     : "dense assignment out of grid range");
            a32[i] = (uint32_t)a;
        }
        uint32_t* dn = p->d_node.as<uint32_t>(p->n ? p->n : 1);
        if (p->n) UMCG_CUDA(cudaMemcpy(dn, a32.data(), p->n * 4, cudaMemcpyHostToDevice));
        if (coords && p->n) {
            if (mesh_dim != p->dim) fail(UMCG_MALFORMED_FILE, "mesh dimension does not match grid");
            double* dc = p->d_coords.as<double>(p->n * p->dim);
            UMCG_CUDA(cudaMemcpy(dc, coords, p->n * p->dim * 8, cudaMemcpyHostToDevice));
            p->has_coords = true;
        }
        plan_build_segments(p, 0);
        static const bool dig_host = std::getenv("UMCG_DIGEST_HOST") != nullptr;
        static const bool dig_check = std::getenv("UMCG_DIGEST_CHECK") != nullptr;
        if (dig_host) {
            p->digest = mapping_digest_host(p->mode, p->n, m->assignments, m->n_visited, m->visited_nodes);
        } else {
            p->digest = mapping_digest_device(p->mode, p->n, dn, m->n_visited,
                                              p->mode == 1 ? p->d_visited.as<uint64_t>(1) : nullptr, p->scratch_a, 0);
            if (dig_check &&
                p->digest != mapping_digest_host(p->mode, p->n, m->assignments, m->n_visited, m->visited_nodes))
                fail(UMCG_INTERNAL_INCONSISTENCY, "device mapping digest differs from the host digest");
        }
    } catch (...) {
        delete p;
        throw;
    }
    return p;
}

// GPU grid_coarsen (grid_builder.hpp:365-421).
umcg_plan* plan_build_gpu(const umcg_grid_desc* g0, uint64_t n, const double* d_coords, double thr,
                          int keep_coords) {
    if (!g0 || !d_coords) fail(UMCG_INVALID_ARGUMENT, "NULL argument");
    if (!(thr > 0.0) || thr > 1.0) fail(UMCG_ERROR, "seed mode threshold must be in (0, 1]");
    if (n > (uint64_t)INT32_MAX) fail(UMCG_INVALID_ARGUMENT, "more than 2^31-1 vertices per plan");
    const int D = g0->dim;
    if (D != 2 && D != 3) fail(UMCG_MALFORMED_FILE, "grid dimension must be 2 or 3");
    cudaStream_t st = 0;
    std::vector<uint64_t> sizes(D), off(D);
    uint64_t tot = 0;
    for (int d = 0; d < D; ++d) { sizes[d] = g0->axis_sizes[d]; off[d] = tot; tot += sizes[d]; }
    DevBuf axes, doff, dsz, idx, flags, o2n, nsz, lin, lin_sorted, uniq, nuniq, scratch;
    double* da = axes.as<double>(tot);
    UMCG_CUDA(cudaMemcpy(da, g0->axes, tot * 8, cudaMemcpyHostToDevice));
    uint64_t* dof = doff.as<uint64_t>(D);
    UMCG_CUDA(cudaMemcpy(dof, off.data(), D * 8, cudaMemcpyHostToDevice));
    uint64_t* dsize = dsz.as<uint64_t>(D);
    UMCG_CUDA(cudaMemcpy(dsize, sizes.data(), D * 8, cudaMemcpyHostToDevice));
    uint32_t* didx = idx.as<uint32_t>(D * (n ? n : 1));
    uint8_t* dfl = flags.as<uint8_t>(tot);
    UMCG_CUDA(cudaMemset(dfl, 0, tot));
    if (n) {
        k_map_axes<<<blocks(n), THREADS, 0, st>>>(d_coords, n, D, da, dof, dsize, didx);
        UMCG_LAUNCHED();
        k_plane_flags<<<blocks(n), THREADS, 0, st>>>(didx, n, D, dof, dfl);
        UMCG_LAUNCHED();
    }
    std::vector<uint8_t> hfl(tot);
    UMCG_CUDA(cudaMemcpy(hfl.data(), dfl, tot, cudaMemcpyDeviceToHost));
    // coarse axes + old->new plane maps
    std::vector<int64_t> ho2n(tot, -1);
    std::vector<uint64_t> nsize(D, 0);
    std::vector<double> caxes;
    std::vector<uint64_t> csizes(D);
    for (int d = 0; d < D; ++d) {
        int64_t next = 0;
        for (uint64_t k = 0; k < sizes[d]; ++k)
            if (hfl[off[d] + k]) {
                ho2n[off[d] + k] = next++;
                caxes.push_back(g0->axes[off[d] + k]);
            }
        nsize[d] = (uint64_t)next;
        csizes[d] = (uint64_t)next;
    }
    int64_t* do2n = o2n.as<int64_t>(tot);
    UMCG_CUDA(cudaMemcpy(do2n, ho2n.data(), tot * 8, cudaMemcpyHostToDevice));
    uint64_t* dnsz = nsz.as<uint64_t>(D);
    UMCG_CUDA(cudaMemcpy(dnsz, nsize.data(), D * 8, cudaMemcpyHostToDevice));
    uint64_t* dlin = lin.as<uint64_t>(n ? n : 1);
    if (n) {
        k_remap<<<blocks(n), THREADS, 0, st>>>(didx, n, D, do2n, dof, dnsz, dlin);
        UMCG_LAUNCHED();
    }
    // visited = sort + unique of assignments
    uint64_t* dsorted = lin_sorted.as<uint64_t>(n ? n : 1);
    uint64_t* duniq = uniq.as<uint64_t>(n ? n : 1);
    auto* dnu = nuniq.as<unsigned long long>(1);
    uint64_t nv = 0;
    if (n) {
        // (radix.cu) keys below the coarse grid's node count; then the heads
        // of the runs of equal keys, compacted through a scan of their flags
        uint64_t nodes = 1;
        for (int d = 0; d < D; ++d) nodes *= std::max<uint64_t>(csizes[d], 1);
        int end_bit = 1;
        while (end_bit < 64 && (1ull << end_bit) < nodes) ++end_bit;
        DevBuf rs_hist, rs_scan, heads;
        radix_sort_u64(dlin, dsorted, nullptr, nullptr, n, 0, end_bit, scratch, rs_hist, rs_scan, st);
        uint32_t* hp = heads.as<uint32_t>(n);
        k_run_heads<<<blocks(n), THREADS, 0, st>>>(dsorted, n, hp);
        UMCG_LAUNCHED();
        exclusive_scan_u32(hp, n, rs_scan, st);
        k_unique_out<<<blocks(n), THREADS, 0, st>>>(dsorted, n, hp, duniq, dnu);
        UMCG_LAUNCHED();
        unsigned long long h = 0;
        UMCG_CUDA(cudaMemcpy(&h, dnu, 8, cudaMemcpyDeviceToHost));
        nv = h;
    }
    uint64_t survivors = 1;
    for (int d = 0; d < D; ++d) survivors *= csizes[d];
    const double frac = (double)nv / (double)survivors;

    auto* p = new umcg_plan;
    try {
        UMCG_CUDA(cudaGetDevice(&p->device));
        std::vector<uint64_t> csz(csizes);
        umcg_grid_desc cg{D, csz.data(), caxes.data()};
        upload_grid(p, &cg);
        p->n = n;
        p->n_visited = nv;
        p->visited_fraction = frac;
        p->mode = frac < thr ? 1 : 0;
        uint32_t* dn = p->d_node.as<uint32_t>(n ? n : 1);
        std::vector<uint64_t> hvis;
        if (p->mode == 1) {
            p->n_slots = nv;
            uint64_t* dv = p->d_visited.as<uint64_t>(nv ? nv : 1);
            if (nv) UMCG_CUDA(cudaMemcpy(dv, duniq, nv * 8, cudaMemcpyDeviceToDevice));
            if (n) {
                k_rank<<<blocks(n), THREADS, 0, st>>>(dlin, n, dv, nv, dn);
                UMCG_LAUNCHED();
            }
            hvis.resize(nv);
            if (nv) UMCG_CUDA(cudaMemcpy(hvis.data(), dv, nv * 8, cudaMemcpyDeviceToHost));
        } else {
            p->n_slots = p->node_count;
            if (p->n_slots >= (1ull << 32)) fail(UMCG_INVALID_ARGUMENT, "grid component longer than 2^32-1");
            if (n) {
                k_u64_to_u32<<<blocks(n), THREADS, 0, st>>>(dlin, n, dn);
                UMCG_LAUNCHED();
            }
        }
        if (keep_coords && n) {
            double* dc = p->d_coords.as<double>(n * D);
            UMCG_CUDA(cudaMemcpy(dc, d_coords, n * D * 8, cudaMemcpyDeviceToDevice));
            p->has_coords = true;
        }
        plan_build_segments(p, st);
        static const bool dig_host = std::getenv("UMCG_DIGEST_HOST") != nullptr;
        static const bool dig_check = std::getenv("UMCG_DIGEST_CHECK") != nullptr;
        if (!dig_host)
            p->digest = mapping_digest_device(p->mode, n, dn, nv, p->mode == 1 ? p->d_visited.as<uint64_t>(1) : nullptr,
                                              p->scratch_a, st);
        if (dig_host || dig_check) {
            std::vector<uint32_t> h32(n);
            if (n) UMCG_CUDA(cudaMemcpy(h32.data(), dn, n * 4, cudaMemcpyDeviceToHost));
            const uint64_t hd = mapping_digest_host32(p->mode, n, h32.data(), nv, hvis.data());
            if (dig_check && !dig_host && hd != p->digest)
                fail(UMCG_INTERNAL_INCONSISTENCY, "device mapping digest differs from the host digest");
            p->digest = hd;
        }
        if (p->mode == 0) {
            p->n_visited = nv;
            p->visited_fraction = frac;
        }
    } catch (...) {
        delete p;
        throw;
    }
    return p;
}

}  // namespace umcg
