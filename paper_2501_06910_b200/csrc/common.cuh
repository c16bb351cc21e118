// Shared host/device helpers for the umcg sm_100a kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <mutex>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/umcg.h"

namespace umcg {

// ---------------------------------------------------------------------------
// Host-side error plumbing: internal code throws Error; the C ABI catches it
// and returns the status (include/umcg.h).
// ---------------------------------------------------------------------------
struct Error : std::runtime_error {
    umcg_status status;
    Error(umcg_status s, const std::string& m) : std::runtime_error(m), status(s) {}
};

[[noreturn]] inline void fail(umcg_status s, const std::string& m) { throw Error(s, m); }

inline void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) fail(UMCG_CUDA_ERROR, std::string(what) + ": " + cudaGetErrorString(e));
}
#define UMCG_CUDA(x) ::umcg::cuda_check((x), #x)

extern std::atomic<uint64_t> g_launches;
// exact-serial fallbacks taken (encode / decode): should stay 0 on normal data
extern std::atomic<uint64_t> g_serial_fallbacks;
inline void count_launch(uint64_t k = 1) { g_launches.fetch_add(k, std::memory_order_relaxed); }
#define UMCG_LAUNCHED()                                  \
    do {                                                 \
        ::umcg::count_launch();                          \
        ::umcg::cuda_check(cudaGetLastError(), "launch"); \
    } while (0)

inline uint64_t cdiv(uint64_t a, uint64_t b) { return (a + b - 1) / b; }

// Optional per-kernel timing (umcg_profile): CUDA events recorded on the
// launching stream around the hot kernels; off by default (no cost).
extern std::atomic<int> g_profile_on;
void prof_record(const char* name, cudaEvent_t a, cudaEvent_t b);
struct ProfScope {
    const char* name;
    cudaStream_t st;
    cudaEvent_t a = nullptr, b = nullptr;
    ProfScope(const char* n, cudaStream_t s) : name(n), st(s) {
        if (g_profile_on.load(std::memory_order_relaxed)) {
            cudaEventCreate(&a);
            cudaEventCreate(&b);
            cudaEventRecord(a, st);
        }
    }
    ~ProfScope() {
        if (a) {
            cudaEventRecord(b, st);
            prof_record(name, a, b);
        }
    }
};

// Error codes raised on the device land in DevCtl::err (first writer wins).
enum DevErr : int {
    DE_NONE = 0,
    DE_CORRUPT_END = 1,       // unexpected end of data
    DE_CORRUPT_VARINT = 2,    // varint exceeds 64 bits
    DE_CORRUPT_TOKEN = 3,     // unknown token in lossless stream
    DE_CORRUPT_TRAILING = 4,  // trailing bytes in quantized stream
    DE_CORRUPT_ESCAPE = 5,    // bad escape index sequence
};

// ---------------------------------------------------------------------------
// varint / zig-zag (reference common.hpp:60-66, 99-107, 129-135)
// ---------------------------------------------------------------------------
__host__ __device__ __forceinline__ uint32_t vlen64(uint64_t v) {
    // bytes of ByteWriter::varint(v): 1 + floor(log128(v))
    uint32_t bits = v ? 64u - (uint32_t)
#ifdef __CUDA_ARCH__
                                  __clzll((long long)v)
#else
                                  __builtin_clzll(v)
#endif
                      : 1u;
    return (bits + 6u) / 7u;
}

__host__ __device__ __forceinline__ uint64_t zz_enc(int64_t v) {
    return ((uint64_t)v << 1) ^ (uint64_t)(v >> 63);
}
__host__ __device__ __forceinline__ int64_t zz_dec(uint64_t v) {
    return (int64_t)(v >> 1) ^ -(int64_t)(v & 1);
}

// ---------------------------------------------------------------------------
// Zero-RLE stream structure (reference lossless.hpp:24-51).
//
// The byte stream is the concatenation of varint(code_i). A 0x00 byte occurs
// exactly when code_i == 0 (every byte of a multi-byte varint is nonzero), so
// the RLE token structure is decided at code granularity: maximal runs of
// >= 8 zero codes become Z tokens, everything between becomes literal
// tokens. RleSum summarizes a contiguous chunk of codes so that chunks
// compose associatively (used for block- and grid-level scans).
// ---------------------------------------------------------------------------
constexpr uint64_t kMinZeroRun = 8;     // lossless.hpp:13 (detail::kMinZeroRun)
constexpr uint32_t kNoOrigin = 0xffffffffu;

__host__ __device__ __forceinline__ uint64_t lit_size(uint64_t b) { return 1 + vlen64(b) + b; }
__host__ __device__ __forceinline__ uint64_t z_size(uint64_t r) { return 1 + vlen64(r); }

struct RleSum {
    uint64_t lz;      // leading zero codes (== chunk length when allzero)
    uint64_t tz;      // trailing zero codes (0 when allzero)
    uint64_t fb;      // bytes of the first core segment
    uint64_t lb;      // bytes of the last core segment (valid when has_int)
    uint64_t mid;     // output bytes of complete pieces between first and last segment
    uint32_t origin;  // chunk id where the last segment started
    uint32_t flags;   // bit0 allzero, bit1 has_int
    __host__ __device__ bool allzero() const { return flags & 1u; }
    __host__ __device__ bool has_int() const { return flags & 2u; }
};

__host__ __device__ __forceinline__ RleSum rle_identity() {
    RleSum s;
    s.lz = s.tz = s.fb = s.lb = s.mid = 0;
    s.origin = kNoOrigin;
    s.flags = 1u;
    return s;
}

__host__ __device__ __forceinline__ RleSum rle_leaf(uint64_t code_bytes, bool zero, uint32_t origin) {
    RleSum s;
    s.tz = s.lb = s.mid = 0;
    if (zero) {
        s.lz = 1; s.fb = 0; s.origin = kNoOrigin; s.flags = 1u;
    } else {
        s.lz = 0; s.fb = code_bytes; s.origin = origin; s.flags = 0u;
    }
    return s;
}

// Summary of A followed by B.
__host__ __device__ __forceinline__ RleSum rle_compose(const RleSum& A, const RleSum& B) {
    if (A.allzero()) {
        RleSum r = B;
        r.lz += A.lz;
        return r;
    }
    if (B.allzero()) {
        RleSum r = A;
        r.tz += B.lz;
        return r;
    }
    RleSum r;
    r.lz = A.lz;
    r.tz = B.tz;
    const uint64_t J = A.tz + B.lz;
    const bool ah = A.has_int(), bh = B.has_int();
    if (J >= kMinZeroRun) {
        r.fb = A.fb;
        r.lb = bh ? B.lb : B.fb;
        r.mid = (ah ? A.mid + lit_size(A.lb) : 0) + z_size(J) + (bh ? lit_size(B.fb) + B.mid : 0);
        r.origin = B.origin;
        r.flags = 2u;
    } else {
        if (!ah && !bh) {
            r.fb = A.fb + J + B.fb; r.lb = 0; r.mid = 0; r.flags = 0u; r.origin = A.origin;
        } else if (ah && !bh) {
            r.fb = A.fb; r.mid = A.mid; r.lb = A.lb + J + B.fb; r.flags = 2u; r.origin = A.origin;
        } else if (!ah && bh) {
            r.fb = A.fb + J + B.fb; r.mid = B.mid; r.lb = B.lb; r.flags = 2u; r.origin = B.origin;
        } else {
            r.fb = A.fb; r.mid = A.mid + lit_size(A.lb + J + B.fb) + B.mid; r.lb = B.lb;
            r.flags = 2u; r.origin = B.origin;
        }
    }
    return r;
}

// Sequential encoder state between chunks: C = output bytes of closed pieces
// (== header position of the open literal), Lb = bytes in the open literal,
// Zp = pending (unclassified) zero codes, origin = chunk id of the open literal.
struct RleState {
    uint64_t C, Lb, Zp;
    uint32_t origin;
    uint32_t has;
};

__host__ __device__ __forceinline__ RleState rle_state0() {
    RleState s;
    s.C = s.Lb = s.Zp = 0;
    s.origin = kNoOrigin;
    s.has = 0;
    return s;
}

// Advance a state over a summarized chunk. Reports the close of the literal
// that was open on entry (only if one was open and it closes in the chunk).
__host__ __device__ __forceinline__ RleState rle_apply(RleState st, const RleSum& S, bool* closed,
                                                       uint64_t* closed_total) {
    *closed = false;
    if (S.allzero()) {
        st.Zp += S.lz;
        return st;
    }
    const bool entry_open = st.has != 0;
    const uint64_t J = st.Zp + S.lz;
    if (J >= kMinZeroRun) {
        if (entry_open) {
            *closed = true;
            *closed_total = st.Lb;
            st.C += lit_size(st.Lb);
        }
        st.C += z_size(J);
        st.Lb = S.fb;
        st.origin = S.origin;
    } else {
        if (!entry_open) st.origin = S.origin;
        st.Lb = (entry_open ? st.Lb : 0) + J + S.fb;
        if (entry_open && S.has_int()) {
            *closed = true;          // entry literal closes at the first interior run
            *closed_total = st.Lb;
        }
    }
    st.has = 1;
    if (S.has_int()) {
        st.C += lit_size(st.Lb) + S.mid;
        st.Lb = S.lb;
        st.origin = S.origin;
    }
    st.Zp = S.tz;
    return st;
}

// Final close: total stream bytes given the state after the last code.
__host__ __device__ __forceinline__ uint64_t rle_finish(const RleState& st, bool* closes,
                                                        uint64_t* total_lit) {
    *closes = false;
    if (st.Zp >= kMinZeroRun) {
        uint64_t c = st.C;
        if (st.has) { c += lit_size(st.Lb); *closes = true; *total_lit = st.Lb; }
        return c + z_size(st.Zp);
    }
    const uint64_t lb = st.Lb + st.Zp;
    if (st.has || st.Zp > 0) {
        *closes = true;
        *total_lit = lb;
        return st.C + lit_size(lb);
    }
    return st.C;
}

// ---------------------------------------------------------------------------
// L2 eviction-priority hints (PTX createpolicy + .L2::cache_hint): streaming
// traffic is marked evict_first so gathered tables stay resident.
// ---------------------------------------------------------------------------
#ifdef __CUDACC__
__device__ __forceinline__ uint64_t l2_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t l2_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint32_t ld_u32_hint(const uint32_t* a, uint64_t pol) {
    uint32_t v;
    asm volatile("ld.global.nc.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(v) : "l"(a), "l"(pol));
    return v;
}
// cp.async (LDGSTS) helpers: global -> shared copies that complete
// asynchronously; _hint takes an L2 cache policy (createpolicy).
__device__ __forceinline__ void cp_async(void* smem_dst, const void* gmem_src, int bytes) {
    const uint32_t d = (uint32_t)__cvta_generic_to_shared(smem_dst);
    if (bytes == 8)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(gmem_src) : "memory");
    else
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(d), "l"(gmem_src) : "memory");
}
__device__ __forceinline__ void cp_async4_hint(void* smem_dst, const void* gmem_src, uint64_t pol) {
    const uint32_t d = (uint32_t)__cvta_generic_to_shared(smem_dst);
    asm volatile("cp.async.ca.shared.global.L2::cache_hint [%0], [%1], 4, %2;" ::"r"(d), "l"(gmem_src), "l"(pol)
                 : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

__device__ __forceinline__ int32_t ld_s32_hint(const int32_t* a, uint64_t pol) {
    int32_t v;
    asm volatile("ld.global.nc.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(v) : "l"(a), "l"(pol));
    return v;
}
__device__ __forceinline__ int32_t ld_s16_hint(const int16_t* a, uint64_t pol) {
    int16_t v;
    asm volatile("ld.global.nc.L2::cache_hint.s16 %0, [%1], %2;" : "=h"(v) : "l"(a), "l"(pol));
    return v;
}
__device__ __forceinline__ uint4 ld_v4_hint(const void* a, uint64_t pol) {
    uint4 v;
    asm volatile("ld.global.nc.L2::cache_hint.v4.u32 {%0, %1, %2, %3}, [%4], %5;"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(a), "l"(pol));
    return v;
}
__device__ __forceinline__ void st_f64_hint(double* a, double v, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(a), "d"(v), "l"(pol) : "memory");
}
#endif

// ---------------------------------------------------------------------------
// Per-call device control block: scalars produced and consumed by kernels so
// that a compress call needs a single host synchronization at the end.
// ---------------------------------------------------------------------------
struct DevCtl {
    // value range / validation (pipeline.hpp:31-41, mesh.hpp:58-64)
    unsigned long long min_key, max_key;  // order-preserving integer keys of min/max
    int nonfinite;
    int err;                              // DevErr, first writer wins
    // budget (pipeline.hpp:43-57, 94)
    double tau_abs, tau1, tau2;           // unshaved split
    double tau_c[2];                      // shaved per component
    double bin[2];                        // 2 * tau_c
    double inv_bin[2];                    // fl(1 / bin) for round_div
    int lossless;                         // tau_abs == 0
    // per-component fast-path verdicts
    int need_serial[2];                   // escape / regime violation: redo exactly
    int need_wide;                        // narrow (int16) residual path overflowed: redo in int32
    int skip;                             // a rerun is certain: the rest of this pass returns at once
    unsigned long long max_abs_k[2];      // |K| maxima (decode regime check)
    // stream lengths and archive layout
    uint64_t stream_len[2];
    uint64_t n_esc[2];
    uint64_t payload_len[2];
    uint64_t stream_off[2];               // byte offset of each stream in the output buffer
    uint64_t archive_len;
    uint64_t count;                       // generic counter (code ends etc.)
    uint64_t aux[8];
};

__device__ __forceinline__ void set_err(DevCtl* c, int e) { atomicCAS(&c->err, 0, e); }
// The kernels after the bucket pass return at once when its verdicts make a
// rerun certain (api.cu k_gate; escapes, int16 overflow): nothing they would
// write is used, and their inputs may be incomplete.
__device__ __forceinline__ bool pass_skipped(const DevCtl* c) { return c && c->skip; }

// Lattice index + bound check in one step (codec.hpp:305-314 on the
// lattice): K = round(fl(r / bin)) and err = |r - K*bin|, bin = 2*tau.
// K comes from q = fl(r * inv); it can differ from the reference's only when
// fl(r / bin) lies within a few ulp of a half-integer, and then err sits
// within ~5 ulp(r) of bin/2 = tau. That band (widened to 2^-45 |r|) takes the
// IEEE divide, so K and err are exactly the reference's everywhere.
__device__ __forceinline__ double lattice_round(double r, double bin, double inv, double tau, double* err) {
    double K = round(__dmul_rn(r, inv));
    double e = fabs(__dsub_rn(r, __dmul_rn(K, bin)));
    if (fabs(__dsub_rn(e, tau)) <= __dmul_rn(fabs(r), 0x1p-45)) {
        K = round(__ddiv_rn(r, bin));
        e = fabs(__dsub_rn(r, __dmul_rn(K, bin)));
    }
    *err = e;
    return K;
}

// round(fl(r / bin)) (the reference's std::round(r / bin), codec.hpp:307)
// without the IEEE divide on the common path: q = fl(r * inv), inv =
// fl(1 / bin), lies within 3 ulp of fl(r / bin), so unless q is within
// 8 ulp of a half-integer both round (half away from zero) to the same
// integer. The ambiguous band and non-finite q take the exact divide.
__device__ __forceinline__ double round_div(double r, double bin, double inv) {
    const double q = __dmul_rn(r, inv);
    const double f = fabs(__dsub_rn(q, trunc(q)));
    if (!(fabs(__dsub_rn(f, 0.5)) > __dmul_rn(fabs(q), 0x1p-49))) return round(__ddiv_rn(r, bin));
    return round(q);
}

// Order-preserving map double -> u64 (for atomicMin/Max over doubles).
__host__ __device__ __forceinline__ unsigned long long dkey(double v) {
    unsigned long long u;
#ifdef __CUDA_ARCH__
    u = (unsigned long long)__double_as_longlong(v);
#else
    std::memcpy(&u, &v, 8);
#endif
    return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}
__host__ __device__ __forceinline__ double dkey_inv(unsigned long long k) {
    unsigned long long u = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
    double v;
#ifdef __CUDA_ARCH__
    v = __longlong_as_double((long long)u);
#else
    std::memcpy(&v, &u, 8);
#endif
    return v;
}

// ---------------------------------------------------------------------------
// Growable device scratch buffers (per plan / per thread).
// ---------------------------------------------------------------------------
class DevBuf {
public:
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf() { release(); }
    void* reserve(size_t bytes) {
        if (bytes > cap_) {
            release();
            size_t c = bytes < 256 ? 256 : bytes;
            UMCG_CUDA(cudaMalloc(&p_, c));
            cap_ = c;
        }
        return p_;
    }
    template <class T> T* as(size_t n) { return static_cast<T*>(reserve(n * sizeof(T))); }
    void release() {
        if (p_ && owned_) cudaFree(p_);
        p_ = nullptr;
        cap_ = 0;
        owned_ = true;
    }
    // Non-owning view of another buffer's memory (plan clones share the
    // static mapping arrays of their origin, which outlives them).
    void alias(const DevBuf& o) {
        release();
        p_ = o.p_;
        cap_ = o.cap_;
        owned_ = false;
    }
    void* get() const { return p_; }
    size_t capacity() const { return cap_; }

private:
    void* p_ = nullptr;
    size_t cap_ = 0;
    bool owned_ = true;
};

// Per-device bookkeeping: cudaFuncSetAttribute, streams, events and device
// buffers belong to one device, so process- or thread-wide "done" flags and
// thread-local resources are kept per device (plans may live on different
// devices; calls set the plan's device first).
constexpr int kMaxDevices = 16;
inline int current_device() {
    int d = 0;
    UMCG_CUDA(cudaGetDevice(&d));
    if (d < 0 || d >= kMaxDevices) fail(UMCG_ERROR, "device index beyond the per-device tables");
    return d;
}
// Runs f() once per device, serialized (a concurrent first call waits until
// the attributes are set before it launches).
class DeviceOnce {
public:
    template <class F>
    void operator()(F&& f) {
        const int d = current_device();
        if (done_.load(std::memory_order_acquire) >> d & 1ull) return;
        std::lock_guard<std::mutex> lock(mu_);
        if (done_.load(std::memory_order_relaxed) >> d & 1ull) return;
        f();
        done_.fetch_or(1ull << d, std::memory_order_release);
    }

private:
    std::mutex mu_;
    std::atomic<uint64_t> done_{0};
};

// A side stream + fork/join events, created on first use (non-blocking, so a
// caller on the legacy default stream is not serialized against it).
struct SideStream {
    cudaStream_t s = nullptr, hi = nullptr;
    cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
    ~SideStream() {
        for (auto& e : ev) if (e) cudaEventDestroy(e);
        if (s) cudaStreamDestroy(s);
        if (hi) cudaStreamDestroy(hi);
    }
    cudaStream_t get() {
        if (!s) {
            UMCG_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
            for (auto& e : ev) UMCG_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        }
        return s;
    }
    // Highest-priority side stream: a latency-bound chain (few CTAs per
    // kernel) keeps its SMs while a throughput-bound kernel on a normal
    // stream fills the rest.
    cudaStream_t get_hi() {
        get();
        if (!hi) {
            int lo = 0, top = 0;
            UMCG_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &top));
            UMCG_CUDA(cudaStreamCreateWithPriority(&hi, cudaStreamNonBlocking, top));
        }
        return hi;
    }
    // `to` waits for all work queued so far on `from` (event slot k)
    void link(cudaStream_t from, cudaStream_t to, int k) {
        UMCG_CUDA(cudaEventRecord(ev[k], from));
        UMCG_CUDA(cudaStreamWaitEvent(to, ev[k], 0));
    }
};

struct PinnedBuf {
    void* p = nullptr;
    size_t cap = 0;
    ~PinnedBuf() { if (p) cudaFreeHost(p); }
    void* reserve(size_t bytes) {
        if (bytes > cap) {
            if (p) cudaFreeHost(p);
            p = nullptr;
            UMCG_CUDA(cudaMallocHost(&p, bytes < 64 ? 64 : bytes));
            cap = bytes;
        }
        return p;
    }
};

// Device -> host hand-off without a copy operation or a stream
// synchronization: the last kernel of a phase writes its small result into
// pinned host memory (unified addressing: the same pointer on the device),
// then a ticket; the host polls the ticket. A posted PCIe write reaches the
// host in ~1-2 us, against ~10 us for cudaMemcpyAsync + cudaStreamSynchronize
// (UMCG_DEC_TRACE: headers on the device at +13 us, on the host at +24 us).
// UMCG_NO_MAILBOX=1 keeps the copy + synchronize hand-off (A/B knob).
struct Mailbox {
    static constexpr size_t kData = 64;  // payload offset: the ticket has its own cache line
    PinnedBuf buf;
    uint64_t seq = 0;
    uint8_t* base = nullptr;
    // payload of >= bytes; call before every use (the buffer only grows)
    uint8_t* data(size_t bytes) {
        if (!base || bytes + kData > buf.cap) {
            base = static_cast<uint8_t*>(buf.reserve(bytes + kData < 4096 ? 4096 : bytes + kData));
            *reinterpret_cast<volatile uint64_t*>(base) = 0;
            seq = 0;
        }
        return base + kData;
    }
    volatile uint64_t* ticket() { return reinterpret_cast<volatile uint64_t*>(base); }
    uint64_t next() { return ++seq; }
    static bool enabled() {
        static const bool on = std::getenv("UMCG_NO_MAILBOX") == nullptr;
        return on;
    }
    // Poll until the ticket shows seq (a pause per poll: the sibling
    // hyperthread and the other host threads' driver calls are not starved).
    // Every 16k polls (~1 ms) the stream is queried, so a failed launch or a
    // faulted kernel surfaces as its CUDA error instead of an endless wait.
    void wait(cudaStream_t st) {
        const volatile uint64_t* t = ticket();
        for (uint32_t spins = 1;; ++spins) {
            if (*t == seq) break;
#if defined(__x86_64__) || defined(__i386__)
            __builtin_ia32_pause();
#endif
            if ((spins & 0x3fffu) == 0) {
                const cudaError_t q = cudaStreamQuery(st);
                if (q == cudaSuccess) {
                    if (*t == seq) break;
                    throw umcg::Error(UMCG_INTERNAL_INCONSISTENCY, "mailbox ticket missing after the stream finished");
                }
                if (q != cudaErrorNotReady) UMCG_CUDA(q);
            }
        }
        std::atomic_thread_fence(std::memory_order_acquire);
    }
};

#ifdef __CUDACC__
// Post a ticket after the payload stores of this thread (and, after a
// __syncthreads(), of its CTA: each writer fences first).
__device__ __forceinline__ void mailbox_post(volatile uint64_t* ticket, uint64_t seq) {
    __threadfence_system();
    *ticket = seq;
}
#endif

}  // namespace umcg
