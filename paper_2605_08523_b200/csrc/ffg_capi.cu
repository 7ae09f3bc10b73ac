// Host side of the fermiforge B200 C ABI (include/fermiforge/ffg.h).
//
// Validation mirrors the reference (ModelCoefficients::validate
// scalar_models.cpp:133-171, FermiParams::validate :27-34); then the device
// pipeline  reset -> K1 rescale_tiles -> K2 mlsp2_pair_kernel (all layers) -> K3 finalize
// is enqueued on the caller's stream, with K2 forked to the device's K2 stream (DevState).  No CPU fallback: without an sm_100 device every
// compute entry point fails with FFG_ERR_CUDA.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include <cublas_v2.h>
#include <dlfcn.h>
#include <nvtx3/nvToolsExt.h>

#include "fermiforge/ffg.h"
#include "k2_pair.cuh"
#include "k2_wide.cuh"
#include "direct.cuh"

using namespace ffg;

namespace {

thread_local std::string g_err;

// NVTX range over an entry point or a pipeline stage (header-only NVTX3: a no-op unless a tool such
// as Nsight Systems is attached)
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};

int set_err(int code, const char* fmt, ...) {
    char buf[1024];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

#define CK(x)                                                                                  \
    do {                                                                                       \
        cudaError_t e_ = (x);                                                                  \
        if (e_ != cudaSuccess)                                                                 \
            return set_err(FFG_ERR_CUDA, "%s: %s (%s:%d)", #x, cudaGetErrorString(e_), __FILE__, \
                           __LINE__);                                                          \
    } while (0)

// --------------------------------------------------------------------- validation
int validate_model(const ffg_model* m) {
    if (!m || !m->abcd) return set_err(FFG_ERR_VALIDATION, "ModelCoefficients: model is null");
    if (!(m->beta0 > 0.0) || !std::isfinite(m->beta0))
        return set_err(FFG_ERR_VALIDATION, "FermiParams: beta must be positive and finite");
    if (!std::isfinite(m->mu0)) return set_err(FFG_ERR_VALIDATION, "FermiParams: mu must be finite");
    if (!(m->mu0 > 0.0 && m->mu0 < 1.0))
        return set_err(FFG_ERR_VALIDATION, "ModelCoefficients: mu0 must lie in (0,1)");
    if (m->n_layers < 1)
        return set_err(FFG_ERR_VALIDATION, "ModelCoefficients: MLSP2 needs at least one layer");
    for (int i = 0; i < 4 * m->n_layers; ++i)
        if (!std::isfinite(m->abcd[i]))
            return set_err(FFG_ERR_VALIDATION, "ModelCoefficients: MLSP2 coefficients must be finite");
    return FFG_OK;
}

int mode_to_internal(int32_t mode, int* out) {
    switch (mode) {
        case FFG_MODE_MIXED_EMULATED: *out = kModeF32E; return FFG_OK;
        case FFG_MODE_FP16: *out = kModeF16; return FFG_OK;
        case FFG_MODE_BF16: *out = kModeBF16; return FFG_OK;
        case FFG_MODE_DOUBLE: *out = kModeF64; return FFG_OK;
        case FFG_MODE_SINGLE: *out = kModeF32; return FFG_OK;
        default: return set_err(FFG_ERR_VALIDATION, "unknown PrecisionMode %d", mode);
    }
}

int validate_n(int64_t n) {
    if (n < 1) return set_err(FFG_ERR_DIMENSION, "matrix dimension must be >= 1 (got %lld)", (long long)n);
    if (n > 65536) return set_err(FFG_ERR_DIMENSION, "matrix dimension %lld exceeds 65536", (long long)n);
    return FFG_OK;
}

int check_device(int* dev_out) {
    int dev = 0, count = 0;
    cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess || count == 0)
        return set_err(FFG_ERR_CUDA, "no CUDA device: %s", cudaGetErrorString(e));
    CK(cudaGetDevice(&dev));
    int major = 0;
    CK(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev));
    if (major != 10)
        return set_err(FFG_ERR_CUDA, "device %d is sm_%d0; this library is built for sm_100a only", dev, major);
    *dev_out = dev;
    return FFG_OK;
}

// --------------------------------------------------------------------- tensor maps
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(p);
    });
    return fn;
}

// Row-major matrix [rows][np] of 16-bit (elem=2) or fp32 (elem=4) values viewed by TMA as
// box_rows x box_cols boxes with a 128-byte (box_cols * elem == 128) or 64-byte swizzle.
int make_map(CUtensorMap* tm, void* base, int64_t rows, int64_t np, int elem, int box_cols,
             int box_rows, CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B) {
    EncodeTiledFn enc = encode_fn();
    if (!enc) return set_err(FFG_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    cuuint64_t dims[2] = {(cuuint64_t)np, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)np * elem};
    cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(tm, elem == 2 ? CU_TENSOR_MAP_DATA_TYPE_UINT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                     2, base, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return set_err(FFG_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
    return FFG_OK;
}

// --------------------------------------------------------------------- workspace
// Per-matrix record read back by the host paths: stats {Tr D, Tr D^2}, widened bounds
// {eps_min, eps_max, x_min, x_max}, status, flags {non-finite layer, half-range layer}, products.
constexpr size_t kRecordBytes = 2 * 8 + 4 * 8 + 4 + 2 * 4 + 4;

// One in-flight batch of the host-buffer path: device staging, pinned per-matrix records,
// events, and the call parameters provenance needs at wait time.
struct HostSlot {
    static constexpr int kMaxChunks = 8;
    double* Hs = nullptr;
    double* Ds = nullptr;
    size_t cap = 0;
    void* host_small = nullptr;
    void* host_small_dev = nullptr;  // its device-mapped address (records_kernel writes there)
    size_t host_small_bytes = 0;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr, ev_d2h = nullptr;
    cudaEvent_t ev_in[kMaxChunks] = {}, ev_done[kMaxChunks] = {};
    bool busy = false;
    int64_t ticket = 0;
    int B = 0;
    int64_t n = 0;
    int PT = 0;
    int mode_api = 0;
    ffg_model model{};
    std::vector<double> mu, kT;
    bool has_mu = false, has_kT = false;
};

struct Workspace {
    int device = -1;
    size_t cap_elems = 0;  // B * np * np
    int cap_B = 0;
    size_t cap_T = 0;      // B * T
    size_t cap_h = 0;      // staging elements (B * n * n)
    float* A = nullptr;
    uint16_t* op[4] = {nullptr, nullptr, nullptr, nullptr};  // hi0, lo0, hi1, lo1
    uint8_t* dX = nullptr;   // DOUBLE / SINGLE modes (direct.cuh): X, Y = X X, A in fp64 or fp32
    uint8_t* dY = nullptr;
    uint8_t* dA = nullptr;
    size_t cap_direct = 0;   // bytes of each
    double* Hs = nullptr;
    double* Ds = nullptr;
    double* params = nullptr;       // [4][cap_B]: alpha, gamma, scale, mu
    double* params_host = nullptr;  // pinned mirror
    unsigned long long* bounds = nullptr;
    int* flags = nullptr;
    uint32_t* products = nullptr;   // [B] instrumented tensor-core product passes (K2 issuer)
    double2* partials = nullptr;
    double* stats = nullptr;
    double* bounds_out = nullptr;
    int* status = nullptr;
    void* host_small = nullptr;     // pinned readback: stats, bounds, status, flags
    size_t host_small_bytes = 0;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;  // K2 runs on the device's K2 stream
    // tensor-map cache over the operand arrays hi0 lo0 hi1 lo1: [0..3] 64x128 operand boxes
    // (SW128), [4..7] 32x32 epilogue pieces (SW64)
    // pair kernel (k2_pair.cuh): panel counters, pair table, per-layer coefficients, maps
    uint32_t* counters = nullptr;
    size_t cap_cnt = 0;
    uint32_t* pairs = nullptr;
    uint8_t* xa_used = nullptr;      // [nb][nb] blocks in the pair table's orientation
    size_t cap_used = 0;
    int64_t pairs_nb = -1;  // key of the cached pair table (nb, row-block rank / world)
    int PT = 0;
    size_t cap_pairs = 0;
    float* coef = nullptr;              // [L][8] hi/lo fp32 coefficients (load_coef)
    size_t cap_coef = 0;
    int pm_B = -1, pm_np = -1;
    PairMaps pmaps;
    // pipelined host path (submit_host / finish_host): copy streams and three in-flight slots
    static constexpr int kMaxChunks = HostSlot::kMaxChunks;
    static constexpr int kSlots = 3;  // a third call in flight keeps both copy engines busy (e2e +~8%)
    cudaStream_t s_h2d = nullptr, s_d2h = nullptr;
    HostSlot slot[kSlots];
    int64_t next_ticket = 0;
    // pinned upload ring for small per-call host data (params, coefficients)
    // (deep enough that the pipelined host path never blocks on a slot whose copy is pending:
    // two uploads per chunk, up to kMaxChunks chunks per call, several calls in flight)
    static constexpr int kRing = 64;
    static constexpr size_t kSlot = 16 * 1024;
    uint8_t* ring = nullptr;
    uint8_t* ring_dev = nullptr;    // the ring's device-mapped address
    cudaEvent_t ring_ev[kRing] = {};
    int ring_next = 0;
    std::mutex mu;
};

std::mutex g_ws_mu;
std::map<std::pair<int, cudaStream_t>, Workspace*> g_ws;

Workspace* get_ws(int dev, cudaStream_t st) {
    std::lock_guard<std::mutex> lk(g_ws_mu);
    auto key = std::make_pair(dev, st);
    auto it = g_ws.find(key);
    if (it != g_ws.end()) return it->second;
    Workspace* w = new Workspace();
    w->device = dev;
    g_ws[key] = w;
    return w;
}

void free_ws(Workspace* w) {
    cudaFree(w->A);
    cudaFree(w->dX);
    cudaFree(w->dY);
    cudaFree(w->dA);
    for (auto& p : w->op) cudaFree(p);
    cudaFree(w->Hs);
    cudaFree(w->Ds);
    cudaFree(w->params);
    cudaFreeHost(w->params_host);
    cudaFree(w->bounds);
    cudaFree(w->flags);
    cudaFree(w->products);
    cudaFree(w->partials);
    cudaFree(w->stats);
    cudaFree(w->bounds_out);
    cudaFree(w->status);
    cudaFreeHost(w->host_small);
    cudaFree(w->counters);
    cudaFree(w->pairs);
    cudaFree(w->xa_used);
    cudaFree(w->coef);
    cudaFreeHost(w->ring);
    if (w->s_h2d) cudaStreamDestroy(w->s_h2d);
    if (w->s_d2h) cudaStreamDestroy(w->s_d2h);
    for (auto& hsl : w->slot) {
        cudaFree(hsl.Hs);
        cudaFree(hsl.Ds);
        cudaFreeHost(hsl.host_small);
        for (cudaEvent_t e : {hsl.ev0, hsl.ev1, hsl.ev_d2h})
            if (e) cudaEventDestroy(e);
        for (auto& e : hsl.ev_in)
            if (e) cudaEventDestroy(e);
        for (auto& e : hsl.ev_done)
            if (e) cudaEventDestroy(e);
    }
    for (auto& e : w->ring_ev)
        if (e) cudaEventDestroy(e);
    for (cudaEvent_t e : {w->ev0, w->ev1, w->ev_fork, w->ev_join})
        if (e) cudaEventDestroy(e);
}

template <typename T>
int grow(T** p, size_t& cap_field_unused, size_t n) {
    (void)cap_field_unused;
    cudaFree(*p);
    *p = nullptr;
    CK(cudaMalloc(reinterpret_cast<void**>(p), std::max<size_t>(n, 1) * sizeof(T)));
    return FFG_OK;
}

int ensure(Workspace& w, int B, int64_t np, int64_t T, bool operands) {
    size_t dummy = 0;
    if (!w.ev0) {
        CK(cudaEventCreate(&w.ev0));
        CK(cudaEventCreate(&w.ev1));
        CK(cudaEventCreateWithFlags(&w.ev_fork, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&w.ev_join, cudaEventDisableTiming));
    }
    const size_t elems = (size_t)B * np * np;
    if (operands && elems > w.cap_elems) {
        int rc;
        if ((rc = grow(&w.A, dummy, elems))) return rc;
        for (auto& p : w.op)
            if ((rc = grow(&p, dummy, elems))) return rc;
        w.cap_elems = elems;
    }
    if (B > w.cap_B) {
        int rc;
        if ((rc = grow(&w.params, dummy, (size_t)4 * B))) return rc;
        cudaFreeHost(w.params_host);
        CK(cudaMallocHost(&w.params_host, sizeof(double) * 4 * B));
        if ((rc = grow(&w.bounds, dummy, (size_t)2 * B))) return rc;
        if ((rc = grow(&w.flags, dummy, (size_t)2 * B))) return rc;
        if ((rc = grow(&w.products, dummy, (size_t)B))) return rc;
        if ((rc = grow(&w.stats, dummy, (size_t)2 * B))) return rc;
        if ((rc = grow(&w.bounds_out, dummy, (size_t)4 * B))) return rc;
        if ((rc = grow(&w.status, dummy, (size_t)B))) return rc;
        cudaFreeHost(w.host_small);
        w.host_small_bytes = (size_t)B * kRecordBytes;
        CK(cudaMallocHost(&w.host_small, w.host_small_bytes));
        w.cap_B = B;
    }
    if ((size_t)B * T > w.cap_T) {
        int rc;
        if ((rc = grow(&w.partials, dummy, (size_t)B * T))) return rc;
        w.cap_T = (size_t)B * T;
    }
    return FFG_OK;
}

int ensure_staging(Workspace& w, size_t elems) {
    size_t dummy = 0;
    if (elems > w.cap_h) {
        int rc;
        if ((rc = grow(&w.Hs, dummy, elems))) return rc;
        if ((rc = grow(&w.Ds, dummy, elems))) return rc;
        w.cap_h = elems;
    }
    return FFG_OK;
}

// Small host<->device transfers as kernels over page-locked, device-mapped host memory: a
// cudaMemcpyAsync of a few hundred bytes is a copy-engine operation and queues behind the
// pipelined host path's 64 MiB matrix transfers (measured 5-25 us each, ~290 us of idle compute
// stream per chunk, scripts/timeline_e2e.py); an SM reads or writes the bytes over PCIe instead.
__global__ void copy_words_kernel(uint32_t* __restrict__ dst, const uint32_t* __restrict__ src, int words) {
    for (int i = threadIdx.x; i < words; i += blockDim.x) dst[i] = src[i];
}
// ... and up to 4 KB carried in the launch itself (kernel parameter space): no PCIe read at all
constexpr int kInlineWords = 1000;
struct InlineBlob {
    uint32_t w[kInlineWords];
};
__global__ void inline_words_kernel(uint32_t* __restrict__ dst, const __grid_constant__ InlineBlob blob, int words) {
    for (int i = threadIdx.x; i < words; i += blockDim.x) dst[i] = blob.w[i];
}
// per-matrix records of matrices [0, mb) of the workspace into the host record block (at m0)
__global__ void records_kernel(uint8_t* host, int B, int m0, int mb, const double* stats, const double* bounds,
                               const int* status, const int* flags, const uint32_t* products) {
    double* h_stats = reinterpret_cast<double*>(host);
    double* h_bounds = h_stats + 2 * B;
    int* h_status = reinterpret_cast<int*>(h_bounds + 4 * B);
    int* h_flags = h_status + B;
    uint32_t* h_prod = reinterpret_cast<uint32_t*>(h_flags + 2 * B);
    for (int m = threadIdx.x; m < mb; m += blockDim.x) {
        h_stats[2 * (m0 + m) + 0] = stats[2 * m + 0];
        h_stats[2 * (m0 + m) + 1] = stats[2 * m + 1];
        for (int k = 0; k < 4; ++k) h_bounds[4 * (m0 + m) + k] = bounds[4 * m + k];
        h_status[m0 + m] = status[m];
        h_flags[2 * (m0 + m) + 0] = flags[2 * m + 0];
        h_flags[2 * (m0 + m) + 1] = flags[2 * m + 1];
        h_prod[m0 + m] = products[m];
    }
    __threadfence_system();
}

// Copy a small host array to the device asynchronously on `st`: up to 4 KB as the parameter block
// of a one-CTA kernel launch, larger (<= 16 KB) through a pinned, device-mapped ring slot read by a
// kernel (the slot is reused only after its previous copy has executed: event), so the caller's
// array may change right after the call.  Neither uses a copy engine (see copy_words_kernel).
int upload_small(Workspace& w, void* dst, const void* src, size_t bytes, cudaStream_t st) {
    if (bytes <= sizeof(uint32_t) * kInlineWords && bytes % 4 == 0) {
        InlineBlob blob;
        memcpy(blob.w, src, bytes);
        inline_words_kernel<<<1, 256, 0, st>>>(static_cast<uint32_t*>(dst), blob, (int)(bytes / 4));
        CK(cudaGetLastError());
        return FFG_OK;
    }
    if (bytes > Workspace::kSlot) {
        CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st));  // pageable: staged
        return FFG_OK;
    }
    if (!w.ring) {
        CK(cudaHostAlloc(&w.ring, Workspace::kRing * Workspace::kSlot, cudaHostAllocMapped));
        CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&w.ring_dev), w.ring, 0));
        for (auto& e : w.ring_ev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    const int k = w.ring_next;
    w.ring_next = (k + 1) % Workspace::kRing;
    CK(cudaEventSynchronize(w.ring_ev[k]));
    uint8_t* slot = w.ring + (size_t)k * Workspace::kSlot;
    memcpy(slot, src, bytes);
    const size_t words = (bytes + 3) / 4;  // (ring slots and device buffers are 4-byte aligned)
    copy_words_kernel<<<1, 256, 0, st>>>(static_cast<uint32_t*>(dst),
                                         reinterpret_cast<const uint32_t*>(w.ring_dev + (size_t)k * Workspace::kSlot),
                                         (int)words);
    CK(cudaGetLastError());
    CK(cudaEventRecord(w.ring_ev[k], st));
    return FFG_OK;
}

// Pair table of the K2 pair kernel (k2_pair.cuh): every block {R, C} (R <= C) of an nb x nb
// block grid exactly once, as pairs of blocks sharing their B panel S.  Column J pairs its
// upper blocks (I, J) over panel J; an odd leftover (the diagonal) takes block {J, J+1} from
// column J+1 in the lower orientation (J+1, J); the last column's leftover gets a dummy
// partner (so at most one dummy per matrix).  Pairs are then ordered row-major by the
// upper-triangle rows of their blocks so that panels complete early in a layer.
std::vector<uint32_t> pair_table(int nb) {
    struct P { int a0, a1, s, d; };
    std::vector<P> v;
    int skip = -1;
    for (int J = 0; J < nb; ++J) {
        std::vector<int> U;
        for (int I = 0; I <= J; ++I)
            if (I != skip) U.push_back(I);
        skip = -1;
        if (U.size() % 2) {
            U.pop_back();  // the diagonal block (J, J)
            if (J + 1 < nb) {
                v.push_back({J, J + 1, J, 0});
                skip = J;
            } else {
                v.push_back({J, J, J, 1});
            }
        }
        for (size_t k = 0; k + 1 < U.size(); k += 2) v.push_back({U[k], U[k + 1], J, 0});
    }
    auto key = [](const P& t) {
        int r = std::min(t.a0, t.s), c = std::max(t.a0, t.s);
        if (!t.d) {
            r = std::max(r, std::min(t.a1, t.s));
            c = std::max(c, std::max(t.a1, t.s));
        }
        return std::make_pair(r, c);
    };
    std::stable_sort(v.begin(), v.end(), [&](const P& x, const P& y) { return key(x) < key(y); });
    std::vector<uint32_t> out;
    for (const P& t : v)
        out.push_back((uint32_t)t.a0 | ((uint32_t)t.a1 << 10) | ((uint32_t)t.s << 20) |
                      ((uint32_t)t.d << 30));
    return out;
}

// Wide kernel (k2_wide.cuh) item table: every super-block (S, T), S <= T, of the upper triangle of
// 256 x 256 super-blocks, row-major (super-rows complete early); entry S | T << 10.
std::vector<uint32_t> wide_table(int nb) {
    std::vector<uint32_t> out;
    const int nsb = nb / 2;
    for (int S = 0; S < nsb; ++S)
        for (int T = S; T < nsb; ++T) out.push_back((uint32_t)S | ((uint32_t)T << 10));
    return out;
}

// The wide kernel runs a batch when its blocks pair up into 256 x 256 super-blocks (nb even) and the
// FP32-emulated scheme is the default one (fixed-point exact layers, no per-2-K16 drain layers);
// the row-block mode keeps the pair kernel.  Default from np >= 2048: below that a matrix has at
// most 10 super-block items per layer and the pair kernel's finer items keep more CTA pairs busy on
// the layer chain (measured, profiles/r2_configs.json: one N=1024 FP32E 1.11 ms wide vs 0.70 pair,
// 16 x N=1024 2.29 vs 2.23, 128 x N=512 3.8 vs 3.1; N=4096 BF16 2.46 vs 3.05, N=8192 FP32E 37.9 vs
// 46.1, N=16384 FP32E 305 vs 407).  The choice depends only on n and the mode -- never on the batch
// size -- so a matrix gets the same bits in every batch and through every entry point.
// FFG_WIDE=0/1 overrides (read on every call).
bool use_wide(int mode, int nb, bool rowblock) {
    const char* e = getenv("FFG_WIDE");
    const bool ok = nb % 2 == 0 && !rowblock && (mode != kModeF32E || FFG_FIXED_SPLIT);
    if (e) return ok && atoi(e) != 0;
    // N >= 4096: below it the 16-worker pair kernel is faster on every shape measured (N=2048 single
    // FP32E 0.84 vs 1.55 ms, N=3072 2.26 vs 2.67 ms, 16 x N=2048 BF16 6.11 vs 6.44 ms); from N=4096 the wide
    // kernel's operand economy wins (N=4096 FP32E 4.93 vs 5.02 ms, BF16 2.42 vs 2.64 ms)
    return ok && nb >= 32;
}

// --------------------------------------------------------------------- small kernels
__global__ void reset_kernel(unsigned long long* bounds, int* flags, int B,
                             uint32_t* counters = nullptr, int n_counters = 0, uint32_t* products = nullptr) {
    const int m = blockIdx.x * blockDim.x + threadIdx.x;
    if (m < n_counters) counters[m] = 0u;
    if (m < B) {
        bounds[2 * m + 0] = ~0ull;
        bounds[2 * m + 1] = 0ull;
        flags[2 * m + 0] = INT_MAX;
        flags[2 * m + 1] = INT_MAX;
        if (products) products[m] = 0u;
    }
}

// Per-row (diag, sum of squares) partials of a full fp64 matrix, one warp per row.
__global__ void row_stats_kernel(const double* D, int n, double2* partials) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int i = blockIdx.x * 8 + warp;
    if (i >= n) return;
    double sq = 0.0, dg = 0.0;
    for (int j = lane; j < n; j += 32) {
        const double v = D[(size_t)i * n + j];
        sq += v * v;
        if (j == i) dg = v;
    }
    for (int o = 16; o > 0; o >>= 1) {
        sq += __shfl_xor_sync(0xffffffffu, sq, o);
        dg += __shfl_xor_sync(0xffffffffu, dg, o);
    }
    if (lane == 0) partials[i] = make_double2(dg, sq);
}

// Per-row (sum_j D_ij A_ij, 0) partials, one warp per row (ffg_expectation).
__global__ void row_dot_kernel(const double* D, const double* A, int n, double2* partials) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int i = blockIdx.x * 8 + warp;
    if (i >= n) return;
    double s = 0.0;
    for (int j = lane; j < n; j += 32) s += D[(size_t)i * n + j] * A[(size_t)i * n + j];
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) partials[i] = make_double2(s, 0.0);
}

// Layers 0..exact-1 drain the hi*hi accumulator after every MMA, later layers once per
// K-block (their rounding is amplified far less by the remaining recursion).
int exact_drain_layers() {
    static int v = [] {
        const char* e = getenv("FFG_EXACT_DRAIN_LAYERS");
        return e ? atoi(e) : 10;
    }();
    return v;
}

// Layers (from the first) whose fixed-point split rounds lo stochastically (kernels.cuh sr_hash)
int sr_layers() {
    static int v = [] {
        const char* e = getenv("FFG_SR_LAYERS");
        return e ? atoi(e) : FFG_SR_LAYERS;
    }();
    return v;
}

// Layers after the exact ones that drain every 2 K16 steps (measurement knob; FFG_SEMI_DRAIN builds)
int semi_drain_layers() {
    static int v = [] {
        const char* e = getenv("FFG_SEMI_DRAIN_LAYERS");
        return (FFG_SEMI_DRAIN && e) ? atoi(e) : 0;
    }();
    return v;
}

// K16 steps per hi*hi chunk after the exact layers: 4, 8 or 16 (one, two or four K-blocks)
int normal_kstep() {
    static int v = [] {
        const char* e = getenv("FFG_NORMAL_KSTEP");
        const int k = e ? atoi(e) : 8;  // measured: 8 as fast as 16, inside the gates with margin
        // any multiple of 4 (whole K-blocks per chunk; >= 4 nk: one chunk) is accepted for measurement
        return (k >= 4 && k % 4 == 0) ? k : 8;
    }();
    return v;
}

// Paired A updates (every other layer reduces d_l X_l + d_{l+1} X_{l+1} into A at L2, epi_sub_mid_red)
bool a_pairing() {
    static bool v = [] {
        const char* e = getenv("FFG_A_PAIR");
        return e ? atoi(e) != 0 : true;
    }();
    return v;
}

int debug_flags() {
    static int v = [] {
        const char* e = getenv("FFG_DEBUG_K2");
        return e ? atoi(e) : 0;
    }();
    return v;
}

// Per-device library state (each entry is set up on first use with that device current):
//  * `lib`  the stream of the host-buffer entry points on this device;
//  * `k2`   the ONE stream every K2 launch of the library on this device goes to.  K2 is a
//           persistent kernel whose CTA pairs wait on each other's layer results, so it needs all
//           of its CTAs co-resident: two K2 grids running side by side (two caller streams, two
//           threads) could each hold part of the SMs and wait forever.  Serialising them on one
//           stream (fork/join events from the caller's stream) makes that impossible;
//  * the pair kernels' shared-memory attribute and co-resident capacity, the SM count and the
//    watchdog buffer, all of which are per-device properties.
struct DevState {
    bool init = false;
    cudaStream_t lib = nullptr, k2 = nullptr;
    int sms = 148;
    int cap[3][4] = {{-1, -1, -1, -1}, {-1, -1, -1, -1}, {-1, -1, -1, -1}};  // [mode][V] co-resident CTA pairs
                                                                       // (V = 3: the wide kernel)
    bool watch = false;
};
std::mutex g_dev_mu;
std::map<int, DevState> g_dev;

// Host-mapped watchdog record (ptx.cuh watchdog_fire): [0] fired count, [1] block,
// [2] thread, [3] site tag, [4..5] site data.  Survives a trapped context.  One host record
// shared by all devices (the first trap wins).
unsigned long long* g_watch_host = nullptr;

int dev_state(DevState** out) {
    int dev = 0;
    CK(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(g_dev_mu);
    DevState& d = g_dev[dev];
    if (!d.init) {
        CK(cudaStreamCreateWithFlags(&d.lib, cudaStreamNonBlocking));
        CK(cudaStreamCreateWithFlags(&d.k2, cudaStreamNonBlocking));
        CK(cudaDeviceGetAttribute(&d.sms, cudaDevAttrMultiProcessorCount, dev));
        d.init = true;
    }
    *out = &d;
    return FFG_OK;
}

int install_watchdog(DevState& d) {
    std::lock_guard<std::mutex> lk(g_dev_mu);
    if (d.watch) return FFG_OK;
    if (!g_watch_host) {
        void* h = nullptr;
        CK(cudaHostAlloc(&h, 16 * sizeof(unsigned long long), cudaHostAllocMapped | cudaHostAllocPortable));
        memset(h, 0, 16 * sizeof(unsigned long long));
        g_watch_host = static_cast<unsigned long long*>(h);
    }
    void* dp = nullptr;
    CK(cudaHostGetDevicePointer(&dp, g_watch_host, 0));
    CK(cudaMemcpyToSymbol(ffg_watch_buf, &dp, sizeof(dp)));
    d.watch = true;
    return FFG_OK;
}

// Optional CUDA-event timing of every K2 launch, for the roofline figure.
struct LayerProfile {
    bool on = false;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev;
    size_t used = 0;
    double flops = 0.0;  // algorithmic flops of the profiled launches
    std::mutex mu;
} g_prof;

int prof_begin(cudaStream_t st, cudaEvent_t* stop, double flops) {
    *stop = nullptr;
    if (!g_prof.on) return FFG_OK;
    std::lock_guard<std::mutex> lk(g_prof.mu);
    if (g_prof.used == g_prof.ev.size()) {
        cudaEvent_t a, b;
        CK(cudaEventCreate(&a));
        CK(cudaEventCreate(&b));
        g_prof.ev.emplace_back(a, b);
    }
    auto& pr = g_prof.ev[g_prof.used++];
    CK(cudaEventRecord(pr.first, st));
    *stop = pr.second;
    g_prof.flops += flops;
    return FFG_OK;
}

unsigned long long* g_prof_buf = nullptr;  // FFG_DEBUG_K2 & 8: per-CTA role wait cycles


// Matrices per L2-resident group of the pair kernel.  Enough pair items per layer
// (G * PT >= 2 * resident pairs) that a layer's first items find their panels complete while
// the rest of the group's layer is still in flight (static round-robin schedule; see the
// schedule simulation in DESIGN.md), and otherwise as many as fit `FFG_GROUP_MB` (default
// 80 MiB of the 126 MB L2) of per-matrix working set (X, A blocks + two hi/lo parities).
int group_size(int B, int64_t np, int PT, int resident_pairs, int mode) {
    const char* e = getenv("FFG_GROUP");
    if (e) return std::max(1, std::min(B, atoi(e)));
    const char* mb = getenv("FFG_GROUP_MB");
    const double budget = (mb ? atof(mb) : 80.0) * 1048576.0;
    const double per = (double)np * np * (8.0 * 0.5625 + (mode == kModeF32E ? 8.0 : 4.0));
    const int fit = (int)(budget / per);
    const int fill = (2 * resident_pairs + PT - 1) / PT;
    const int g = std::max(1, std::min(B, std::max(fit, fill)));
    // equal groups: a small remainder group would run its layers with most pairs idle and
    // every item on the dependency chain (measured: 64 x N=512, groups 30+30+4 vs 22+22+20)
    const int ng = (B + g - 1) / g;
    return (B + ng - 1) / ng;
}

// Co-resident CTA pairs of the pair kernel on the current device (all pairs must be resident:
// the layer dependencies are waited for inside the kernel).
template <int MODE, int V>
int pair_capacity(int* out) {
    DevState* d;
    int rc;
    if ((rc = dev_state(&d))) return rc;
    int& max_pairs = d->cap[MODE][V];
    if (max_pairs < 0) {
        CK(cudaFuncSetAttribute(mlsp2_pair_kernel<MODE, V>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                PairCfg<MODE, pair_narrow<MODE, V>()>::kSmem));
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(2 * (d->sms / 2));
        cfg.blockDim = dim3(kPairThreads);
        cfg.dynamicSmemBytes = PairCfg<MODE, pair_narrow<MODE, V>()>::kSmem;
        int nc = 0;
        CK(cudaOccupancyMaxActiveClusters(&nc, mlsp2_pair_kernel<MODE, V>, &cfg));
        if (nc < 1) return set_err(FFG_ERR_CUDA, "pair kernel: no co-resident CTA pair fits");
        max_pairs = nc;
    }
    *out = max_pairs;
    return FFG_OK;
}

// Launch on `st`, which must be the device's K2 stream (enqueue forks to it).
template <int MODE, int V>
int launch_pair(const PairMaps& maps, const PairParams& pp, int64_t items, cudaStream_t st) {
    DevState* d;
    int cap, rc;
    if ((rc = pair_capacity<MODE, V>(&cap))) return rc;
    if ((rc = dev_state(&d))) return rc;
    if ((rc = install_watchdog(*d))) return rc;
    // persistent pairs walk all items round-robin
    const int pairs = (int)std::min<int64_t>(cap, items);
    mlsp2_pair_kernel<MODE, V><<<2 * pairs, kPairThreads, PairCfg<MODE, pair_narrow<MODE, V>()>::kSmem, st>>>(maps, pp);
    CK(cudaGetLastError());
    return FFG_OK;
}

// Matrices per L2-resident group of the wide kernel.  Its per-matrix working set is the upper block
// triangle of two hi/lo parities and of A (~6.75 np^2 bytes, half the pair kernel's), and its items
// are four blocks each, so a layer needs more matrices to give every CTA pair work beyond the
// dependency chain: 3 items per resident pair if they fit 1.3x the L2 budget (FFG_GROUP_MB, default
// 100 MiB), else the budget (measured 16 x N=1024: G = 16 -12% vs 8).  Equal groups as above.
int wide_group_size(int B, int64_t np, int PT, int resident_pairs) {
    const char* e = getenv("FFG_GROUP");
    if (e) return std::max(1, std::min(B, atoi(e)));
    const char* mb = getenv("FFG_GROUP_MB");
    const double budget = (mb ? atof(mb) : 100.0) * 1048576.0;
    const double per = 6.75 * (double)np * np;
    const int fit = std::max(1, (int)(budget / per));
    const int fill = (3 * resident_pairs + PT - 1) / PT;
    const int g = std::max(1, std::min(B, std::max(fit, std::min(fill, (int)(1.3 * fit)))));
    const int ng = (B + g - 1) / g;
    return (B + ng - 1) / ng;
}

// Co-resident CTA pairs of the wide kernel (k2_wide.cuh) on the current device.
template <int MODE>
int wide_capacity(int* out) {
    DevState* d;
    int rc;
    if ((rc = dev_state(&d))) return rc;
    int& max_pairs = d->cap[MODE][3];
    if (max_pairs < 0) {
        CK(cudaFuncSetAttribute(mlsp2_wide_kernel<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                WideCfg<MODE>::kSmem));
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(2 * (d->sms / 2));
        cfg.blockDim = dim3(kWideThreads);
        cfg.dynamicSmemBytes = WideCfg<MODE>::kSmem;
        int nc = 0;
        CK(cudaOccupancyMaxActiveClusters(&nc, mlsp2_wide_kernel<MODE>, &cfg));
        if (nc < 1) return set_err(FFG_ERR_CUDA, "wide kernel: no co-resident CTA pair fits");
        max_pairs = nc;
    }
    *out = max_pairs;
    return FFG_OK;
}
template <int MODE>
int launch_wide(const PairMaps& maps, const PairParams& pp, int64_t items, cudaStream_t st) {
    DevState* d;
    int cap, rc;
    if ((rc = wide_capacity<MODE>(&cap))) return rc;
    if ((rc = dev_state(&d))) return rc;
    if ((rc = install_watchdog(*d))) return rc;
    const int pairs = (int)std::min<int64_t>(cap, items);
    mlsp2_wide_kernel<MODE><<<2 * pairs, kWideThreads, WideCfg<MODE>::kSmem, st>>>(maps, pp);
    CK(cudaGetLastError());
    return FFG_OK;
}
int wide_capacity_mode(int mode, int* cap) {
    switch (mode) {
        case kModeF32E: return wide_capacity<kModeF32E>(cap);
        case kModeF16: return wide_capacity<kModeF16>(cap);
        default: return wide_capacity<kModeBF16>(cap);
    }
}
int launch_wide_mode(int mode, const PairMaps& maps, const PairParams& pp, int64_t items, cudaStream_t st) {
    switch (mode) {
        case kModeF32E: return launch_wide<kModeF32E>(maps, pp, items, st);
        case kModeF16: return launch_wide<kModeF16>(maps, pp, items, st);
        default: return launch_wide<kModeBF16>(maps, pp, items, st);
    }
}

// V: 0 streaming, 2 streaming with 16 workers
template <int V>
int pair_capacity_mode(int mode, int* cap) {
    switch (mode) {
        case kModeF32E: return pair_capacity<kModeF32E, V>(cap);
        case kModeF16: return pair_capacity<kModeF16, V>(cap);
        default: return pair_capacity<kModeBF16, V>(cap);
    }
}
template <int V>
int launch_pair_mode(int mode, const PairMaps& maps, const PairParams& pp, int64_t items, cudaStream_t st) {
    switch (mode) {
        case kModeF32E: return launch_pair<kModeF32E, V>(maps, pp, items, st);
        case kModeF16: return launch_pair<kModeF16, V>(maps, pp, items, st);
        default: return launch_pair<kModeBF16, V>(maps, pp, items, st);
    }
}

// np <= 512 (single-product modes: np <= 1024): sixteen drain+epilogue workers, each finishing one
// 32-column piece straight from its registers (Y never holds a TMEM slot).  Measured: 512 x N=512 BF16
// -24%, FP32E -6%; 64 x N=256 FP32E -18%; 16 x N=1024 BF16 -6%, FP32E +13%; 1-4 x N=1024 FP32E -10%,
// BF16 -19%; one N=2048 matrix BF16 -13%, FP32E -4%; 8 x N=1024 FP32E +2%; N=4096 BF16 +10% (the MMA
// starves while all sixteen warps are in the epilogue).  FFG_S16=0/1 overrides.
bool use_s16(int mode, int64_t np, int64_t items_per_layer, int pairs) {
    const char* e = getenv("FFG_S16");
    if (e) return atoi(e) != 0;
    // the 16-worker epilogue (one 32-column piece per warp, sixteen in flight, 64-register control
    // warps) wins wherever measured up to N=2048, batched or not (16 x N=1024 FP32E 1.88 vs 2.12 ms,
    // 64 x N=1024 -9%, N=2048 single -15%; 16 x N=2048 FP32E +2%); beyond that only latency-bound
    // layers (no more items than resident pairs) use it
    (void)mode;
    return np <= 2048 || items_per_layer <= pairs;
}


struct Job {
    int B = 0;
    int64_t n = 0;
    const double* H_dev = nullptr;      // [B][n][n]
    const double* alpha = nullptr;      // host [B]
    const double* gamma = nullptr;      // host [B]
    const double* scale = nullptr;      // host [B] or null (no validity check)
    const double* mu = nullptr;         // host [B] or null
    const ffg_model* model = nullptr;
    int mode = kModeF32E;
    double* D_dev = nullptr;            // [B][n][n] or null
    double* stats_dev = nullptr;        // [B][2] or null (-> workspace)
    int* status_dev = nullptr;          // [B] or null (-> workspace)
    double* bounds_dev = nullptr;       // [B][4] or null (-> workspace)
    int exact_layers = -1;              // fixed-point exact layers (FP32E); -1: the default
    int rb_world = 0, rb_rank = 0;      // row-block mode (B = 1): this rank's block rows of `world`
};

// Block rows [r0, r1) of rank `rank` of `world` (nb % world == 0, checked by the caller).
void rowblock_rows(int nb, int rank, int world, int* r0, int* r1) {
    *r0 = nb / world * rank;
    *r1 = nb / world * (rank + 1);
}

// Row-block table: every block (R, C) of block rows [r0, r1) and ALL columns,
// as pair items (R, R+1, C).  Each block gets exactly the values the symmetric table gives it: a
// block the symmetric table computes in the other orientation, (C, R), is computed here with the
// cross terms in swapped order (bit 31; k2_pair.cuh), which makes it the exact transpose.  A row pair
// whose two blocks disagree on that bit runs as two half items (dummy partner, bit 30).
std::vector<uint32_t> rowblock_table(int nb, int r0, int r1) {
    const std::vector<uint32_t> sym = pair_table(nb);
    std::vector<int> arow((size_t)nb * nb, -1);  // [min * nb + max] -> the A-panel row computing it
    auto key = [nb](int a, int b) { return (size_t)std::min(a, b) * nb + std::max(a, b); };
    for (uint32_t e : sym) {
        const int a0 = e & 1023, a1 = (e >> 10) & 1023, sp = (e >> 20) & 1023;
        arow[key(a0, sp)] = a0;
        if (!((e >> 30) & 1)) arow[key(a1, sp)] = a1;
    }
    auto swp = [&](int R, int C) -> uint32_t { return (R != C && arow[key(R, C)] != R) ? 1u : 0u; };
    std::vector<uint32_t> out;
    for (int R = r0; R < r1; R += 2) {
        const bool two = R + 1 < r1;
        for (int C = 0; C < nb; ++C) {
            const uint32_t s0 = swp(R, C);
            if (two && s0 == swp(R + 1, C)) {
                out.push_back((uint32_t)R | ((uint32_t)(R + 1) << 10) | ((uint32_t)C << 20) | (s0 << 31));
            } else {
                out.push_back((uint32_t)R | ((uint32_t)R << 10) | ((uint32_t)C << 20) | (1u << 30) | (s0 << 31));
                if (two)
                    out.push_back((uint32_t)(R + 1) | ((uint32_t)(R + 1) << 10) | ((uint32_t)C << 20) | (1u << 30) |
                                  (swp(R + 1, C) << 31));
            }
        }
    }
    return out;
}

int ensure_pair(Workspace& w, int B, int64_t np, int nb, int L, int rb_rank = 0, int rb_world = 0,
                bool wide = false) {
    size_t dummy = 0;
    int rc;
    const size_t ncnt = (size_t)B * nb * (1 + nb);  // panel counters, then block flags
    if (ncnt > w.cap_cnt) {
        if ((rc = grow(&w.counters, dummy, ncnt))) return rc;
        w.cap_cnt = ncnt;
    }
    const int64_t pkey = (int64_t)nb | ((int64_t)rb_rank << 24) | ((int64_t)rb_world << 44) | ((int64_t)wide << 62);
    if (w.pairs_nb != pkey) {
        std::vector<uint32_t> t;
        if (wide) {
            t = wide_table(nb);
        } else if (rb_world > 0) {
            int r0, r1;
            rowblock_rows(nb, rb_rank, rb_world, &r0, &r1);
            t = rowblock_table(nb, r0, r1);
        } else {
            t = pair_table(nb);
        }
        if (t.size() > w.cap_pairs) {
            if ((rc = grow(&w.pairs, dummy, t.size()))) return rc;
            w.cap_pairs = t.size();
        }
        CK(cudaMemcpy(w.pairs, t.data(), t.size() * 4, cudaMemcpyHostToDevice));
        std::vector<uint8_t> used((size_t)nb * nb, 0);
        if (wide) {  // the upper block triangle (k2_wide.cuh storage)
            for (int P = 0; P < nb; ++P)
                for (int Q = P; Q < nb; ++Q) used[(size_t)P * nb + Q] = 1;
        } else {
            for (uint32_t e : t) {
                const int a0 = e & 1023, a1 = (e >> 10) & 1023, sp = (e >> 20) & 1023;
                used[(size_t)a0 * nb + sp] = 1;
                if (!((e >> 30) & 1)) used[(size_t)a1 * nb + sp] = 1;
            }
        }
        if (used.size() > w.cap_used) {
            if ((rc = grow(&w.xa_used, dummy, used.size()))) return rc;
            w.cap_used = used.size();
        }
        CK(cudaMemcpy(w.xa_used, used.data(), used.size(), cudaMemcpyHostToDevice));
        w.pairs_nb = pkey;
        w.PT = (int)t.size();
    }
    if ((size_t)8 * L > w.cap_coef) {
        if ((rc = grow(&w.coef, dummy, (size_t)8 * L))) return rc;
        w.cap_coef = (size_t)8 * L;
    }
    if (w.pm_B != B || w.pm_np != (int)np) {
        for (int par = 0; par < 2; ++par) {
            uint16_t* hi = w.op[2 * par + 0];
            uint16_t* lo = w.op[2 * par + 1];
            const int64_t rows = (int64_t)B * np;
            if ((rc = make_map(&w.pmaps.a_hi[par], hi, rows, np, 2, 64, 128))) return rc;
            if ((rc = make_map(&w.pmaps.a_lo[par], lo, rows, np, 2, 64, 128))) return rc;
            if ((rc = make_map(&w.pmaps.b_hi[par], hi, rows, np, 2, 64, kPairHalf))) return rc;
            if ((rc = make_map(&w.pmaps.b_lo[par], lo, rows, np, 2, 64, kPairHalf))) return rc;
            if ((rc = make_map(&w.pmaps.p_hi[par], hi, rows, np, 2, 32, 32, CU_TENSOR_MAP_SWIZZLE_64B)))
                return rc;
            if ((rc = make_map(&w.pmaps.p_lo[par], lo, rows, np, 2, 32, 32, CU_TENSOR_MAP_SWIZZLE_64B)))
                return rc;
        }
        w.pm_B = B;
        w.pm_np = (int)np;
    }
    return FFG_OK;
}

// Enqueue the full pipeline for one batch on `st` (asynchronous; the small per-call host
// arrays go through the pinned upload ring): enqueue_k1 (uploads, reset, K1), enqueue_k2 (layers
// [l0, l1) on the device's K2 stream), enqueue_k3.  The row-block entry points run them separately.
struct EnqueueCtx {
    int64_t np = 0;
    int nb = 0;
    int64_t Tpart = 0;
    int exact_layers = 0;
    bool wide = false;   // k2_wide.cuh kernel (use_wide)
    RegionCheck region{};
};

int enqueue_k1(Workspace& w, const Job& j, cudaStream_t st, EnqueueCtx& cx) {
    NvtxRange nv("ffg K1 enqueue (uploads, reset, rescale)");
    const int B = j.B;
    const int64_t n = j.n;
    const int64_t np = (n + kBM - 1) / kBM * kBM;
    const int nb = (int)(np / kBM);
    const ffg_model& md = *j.model;
    int rc;
    if ((rc = ensure(w, B, np, 0, true))) return rc;
    cx.wide = use_wide(j.mode, nb, j.rb_world > 0);
    if ((rc = ensure_pair(w, B, np, nb, md.n_layers, j.rb_rank, j.rb_world, cx.wide))) return rc;
    const int64_t Tpart = 2 * (int64_t)w.PT;  // statistics partials per matrix
    if ((size_t)B * Tpart > w.cap_T) {
        size_t dummy = 0;
        if ((rc = grow(&w.partials, dummy, (size_t)B * Tpart))) return rc;
        w.cap_T = (size_t)B * Tpart;
    }
    // per-matrix parameters
    std::vector<double> ph((size_t)4 * B);
    for (int m = 0; m < B; ++m) {
        ph[0 * B + m] = j.alpha[m];
        ph[1 * B + m] = j.gamma[m];
        ph[2 * B + m] = j.scale ? j.scale[m] : 0.0;
        ph[3 * B + m] = j.mu ? j.mu[m] : 0.0;
    }
    if ((rc = upload_small(w, w.params, ph.data(), sizeof(double) * 4 * B, st))) return rc;
    // hi/lo fp32 split of a, b, c and the next layer's d per layer (epilogue.cuh load_coef; the
    // paired A updates are derived in the kernel from the same 8-float rows)
    std::vector<float> cf((size_t)8 * md.n_layers);
    auto split = [](double v, float* o) {
        o[0] = (float)v;
        o[1] = (float)(v - (double)o[0]);
    };
    for (int l = 0; l < md.n_layers; ++l) {
        float* o = cf.data() + 8 * l;
        split(md.abcd[4 * l + 0], o + 0);
        split(md.abcd[4 * l + 1], o + 2);
        split(md.abcd[4 * l + 2], o + 4);
        split(l + 1 < md.n_layers ? md.abcd[4 * (l + 1) + 3] : 0.0, o + 6);
    }
    if ((rc = upload_small(w, w.coef, cf.data(), sizeof(float) * cf.size(), st))) return rc;
    const int ncnt = B * nb * (1 + nb);
    reset_kernel<<<(std::max(B, ncnt) + 127) / 128, 128, 0, st>>>(w.bounds, w.flags, B, w.counters, ncnt,
                                                                 w.products);
    CK(cudaGetLastError());
    cx.np = np;
    cx.nb = nb;
    cx.Tpart = Tpart;
    cx.exact_layers = j.exact_layers >= 0 ? j.exact_layers : exact_drain_layers();
    cx.region = RegionCheck{w.bounds, j.scale ? w.params + 2 * B : nullptr, w.params + 3 * B, md.mu0};

    RescaleParams rp{};
    rp.H = j.H_dev;
    rp.alpha = w.params;
    rp.gamma = w.params + B;
    rp.d0 = md.abcd[3];
    rp.A = w.A;
    rp.hi = w.op[0];
    rp.lo = w.op[1];
    rp.bounds = w.bounds;
    rp.flags = w.flags;
    rp.n = (int)n;
    rp.np = (int)np;
    rp.mode = j.mode;
    rp.fixed = (FFG_FIXED_SPLIT && j.mode == kModeF32E && cx.exact_layers > 0) ? 1 : 0;
    rp.sr = (rp.fixed && sr_layers() > 0) ? 1 : 0;
    rp.xa_used = w.xa_used;   // X/A stores only for the blocks K2 reads
    rescale_tiles_kernel<kK1Warps><<<dim3((unsigned)(np / kK1Rows), (unsigned)B), 32 * kK1Warps, 0, st>>>(rp);
    CK(cudaGetLastError());
    return FFG_OK;
}

// K2 over layers [l0, l1): forked from `st` to the device's K2 stream (DevState) and joined back.
int enqueue_k2(Workspace& w, const Job& j, cudaStream_t st, const EnqueueCtx& cx, int l0, int l1) {
    NvtxRange nv("ffg K2 enqueue (recursion layers)");
    const int B = j.B;
    const int64_t n = j.n;
    const ffg_model& md = *j.model;
    const bool rowblock = j.rb_world > 0;
    int rc;
    PairParams pp{};
    pp.ophi[0] = w.op[0];
    pp.oplo[0] = w.op[1];
    pp.ophi[1] = w.op[2];
    pp.oplo[1] = w.op[3];
    pp.A = w.A;
    pp.D = (l1 == md.n_layers) ? j.D_dev : nullptr;
    pp.partials = w.partials;
    pp.flags = w.flags;
    pp.counters = w.counters;
    pp.bflags = w.counters + (size_t)B * cx.nb;
    pp.pairs = w.pairs;
    pp.coef = reinterpret_cast<const float4*>(w.coef);
    pp.a_pair = a_pairing() ? 1 : 0;
    pp.n = (int)n;
    pp.np = (int)cx.np;
    pp.nb = cx.nb;
    pp.PT = w.PT;
    pp.products = w.products;
    pp.region = cx.region;
    pp.l0 = l0;
    pp.l1 = l1;
    pp.n_layers = md.n_layers;
    pp.exact_layers = cx.exact_layers;
    pp.sr_layers = sr_layers();
    pp.semi_layers = semi_drain_layers();
    pp.normal_kstep = normal_kstep();
    pp.rowblock = rowblock ? 1 : 0;
    // algorithmic flops per layer: c N^2 (N+1) for the symmetric square; a row-block
    // rank computes its rows x all columns, 2 c rows N^2
    const double cmode = (j.mode == kModeF32E) ? 3.0 : 1.0;
    double layer_flops = (double)B * cmode * (double)n * n * (n + 1);
    if (rowblock) {
        int r0, r1;
        rowblock_rows(cx.nb, j.rb_rank, j.rb_world, &r0, &r1);
        pp.drow0 = r0 * kBM;
        const double rows = (double)(std::min<int64_t>((int64_t)r1 * kBM, n) - (int64_t)r0 * kBM);
        layer_flops = 2.0 * cmode * rows * (double)n * n;
    }
    pp.dbg = debug_flags();
    if (pp.dbg & 8) {
        // [0, 16 * 1024): per-CTA role wait cycles; then (dbg & 4096) [items][12] event times
        static unsigned long long* prof = nullptr;
        if (!prof) {
            CK(cudaMallocManaged(&prof, sizeof(unsigned long long) * (16 * 1024 + 12 * 131072)));
            CK(cudaMemset(prof, 0, sizeof(unsigned long long) * (16 * 1024 + 12 * 131072)));
        }
        pp.prof = prof;
        if (pp.dbg & 4096) pp.tl = prof + 16 * 1024;  // every launch overwrites its items' entries
        g_prof_buf = prof;
    }
    DevState* d;
    if ((rc = dev_state(&d))) return rc;
    cudaStream_t k2s = d->k2;
    CK(cudaEventRecord(w.ev_fork, st));
    CK(cudaStreamWaitEvent(k2s, w.ev_fork, 0));
    cudaEvent_t stop;
    if ((rc = prof_begin(k2s, &stop, layer_flops * (l1 - l0)))) return rc;
    // one persistent launch per kValidBits matrices (the kernel's validity bitmap)
    for (int m0 = 0; m0 < B; m0 += kValidBits) {
        const int Bl = std::min(B - m0, kValidBits);
        PairParams lp = pp;
        lp.m0 = m0;
        lp.B = Bl;
        int cap = 0;
        if (cx.wide) {
            if ((rc = wide_capacity_mode(j.mode, &cap))) return rc;
            lp.G = wide_group_size(Bl, cx.np, w.PT, cap);
            const char* bdw = getenv("FFG_BLOCKDEPS");
            lp.blockdeps = bdw ? atoi(bdw) : (lp.G == 1 && l1 - l0 > 1);
            const int64_t items = (int64_t)(l1 - l0) * Bl * w.PT;
            if ((rc = launch_wide_mode(j.mode, w.pmaps, lp, items, k2s))) return rc;
            continue;
        }
        if ((rc = pair_capacity_mode<0>(j.mode, &cap))) return rc;
        lp.G = group_size(Bl, cx.np, w.PT, cap, j.mode);
        const bool s16 = use_s16(j.mode, cx.np, (int64_t)lp.G * w.PT, cap);
        if (s16 && (rc = pair_capacity_mode<2>(j.mode, &cap))) return rc;
        // single-matrix groups: a layer is one matrix, so its items wait on each other;
        // block-granular waits let a next-layer item start on its completed blocks
        // (measured: N=4096 -8%; in multi-matrix groups other matrices fill the gaps and
        // the extra polls cost 2-5%)
        const char* bd = getenv("FFG_BLOCKDEPS");
        lp.blockdeps = bd ? atoi(bd) : (lp.G == 1 && l1 - l0 > 1);
        const int64_t items = (int64_t)(l1 - l0) * Bl * w.PT;
        if ((rc = s16 ? launch_pair_mode<2>(j.mode, w.pmaps, lp, items, k2s)
                      : launch_pair_mode<0>(j.mode, w.pmaps, lp, items, k2s)))
            return rc;
    }
    if (stop) CK(cudaEventRecord(stop, k2s));
    CK(cudaEventRecord(w.ev_join, k2s));
    CK(cudaStreamWaitEvent(st, w.ev_join, 0));
    return FFG_OK;
}

// K3: statistics, validity status, NaN D for out-of-region matrices (d_rows: rows of D per matrix
// the kernel owns -- n, or a row-block rank's rows).
int enqueue_k3(Workspace& w, const Job& j, cudaStream_t st, const EnqueueCtx& cx, int64_t d_rows) {
    NvtxRange nv("ffg K3 enqueue (statistics, status)");
    FinalizeParams fp{};
    fp.partials = w.partials;
    fp.flags = w.flags;
    fp.region = cx.region;
    fp.T = (int)cx.Tpart;
    fp.B = j.B;
    fp.D = j.D_dev;
    fp.d_elems = d_rows * j.n;
    fp.stats = j.stats_dev ? j.stats_dev : w.stats;
    fp.bounds_out = j.bounds_dev ? j.bounds_dev : w.bounds_out;
    fp.status = j.status_dev ? j.status_dev : w.status;
    finalize_stats_kernel<<<j.B, 256, 0, st>>>(fp);
    CK(cudaGetLastError());
    return FFG_OK;
}

// ------------------------------------------------------------------ DOUBLE / SINGLE (direct.cuh)
// cuBLAS is loaded on first use of these modes only (dlopen: the tensor-core path never loads it).
struct CublasApi {
    bool tried = false, ok = false;
    cublasStatus_t (*create)(cublasHandle_t*) = nullptr;
    cublasStatus_t (*set_stream)(cublasHandle_t, cudaStream_t) = nullptr;
    cublasStatus_t (*set_math)(cublasHandle_t, cublasMath_t) = nullptr;
    cublasStatus_t (*dgemm)(cublasHandle_t, cublasOperation_t, cublasOperation_t, int, int, int, const double*,
                            const double*, int, long long, const double*, int, long long, const double*, double*,
                            int, long long, int) = nullptr;
    cublasStatus_t (*sgemm)(cublasHandle_t, cublasOperation_t, cublasOperation_t, int, int, int, const float*,
                            const float*, int, long long, const float*, int, long long, const float*, float*,
                            int, long long, int) = nullptr;
};
CublasApi g_cublas;
std::mutex g_cublas_mu;
std::map<int, cublasHandle_t> g_cublas_handle;

int cublas_handle(cudaStream_t st, cublasHandle_t* out) {
    std::lock_guard<std::mutex> lk(g_cublas_mu);
    if (!g_cublas.tried) {
        g_cublas.tried = true;
        // already loaded by the host process (torch) or the CUDA toolkit's copy
        const char* names[] = {"libcublas.so.12", "/usr/local/cuda/lib64/libcublas.so.12", "libcublas.so"};
        void* h = nullptr;
        for (const char* nm : names)
            if ((h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL))) break;
        if (h) {
            g_cublas.create = reinterpret_cast<decltype(g_cublas.create)>(dlsym(h, "cublasCreate_v2"));
            g_cublas.set_stream = reinterpret_cast<decltype(g_cublas.set_stream)>(dlsym(h, "cublasSetStream_v2"));
            g_cublas.set_math = reinterpret_cast<decltype(g_cublas.set_math)>(dlsym(h, "cublasSetMathMode"));
            g_cublas.dgemm = reinterpret_cast<decltype(g_cublas.dgemm)>(dlsym(h, "cublasDgemmStridedBatched"));
            g_cublas.sgemm = reinterpret_cast<decltype(g_cublas.sgemm)>(dlsym(h, "cublasSgemmStridedBatched"));
            g_cublas.ok = g_cublas.create && g_cublas.set_stream && g_cublas.set_math && g_cublas.dgemm &&
                          g_cublas.sgemm;
        }
    }
    if (!g_cublas.ok) return set_err(FFG_ERR_UNSUPPORTED, "DOUBLE/SINGLE modes need cuBLAS (libcublas.so.12 not found)");
    int dev = 0;
    CK(cudaGetDevice(&dev));
    auto it = g_cublas_handle.find(dev);
    if (it == g_cublas_handle.end()) {
        cublasHandle_t hd;
        if (g_cublas.create(&hd) != CUBLAS_STATUS_SUCCESS) return set_err(FFG_ERR_CUDA, "cublasCreate failed");
        g_cublas.set_math(hd, CUBLAS_PEDANTIC_MATH);  // true fp32 / fp64 arithmetic (no TF32)
        it = g_cublas_handle.emplace(dev, hd).first;
    }
    if (g_cublas.set_stream(it->second, st) != CUBLAS_STATUS_SUCCESS)
        return set_err(FFG_ERR_CUDA, "cublasSetStream failed");
    *out = it->second;
    return FFG_OK;
}

// The recursion in fp64 (DOUBLE) / fp32 (SINGLE) arithmetic: bounds, X0 / A, L x (GEMM + fused layer
// update), D + row partials, K3.  Y = X X as a column-major GEMM of the row-major X: X is exactly
// symmetric, and the layer update reads only upper-triangle entries of Y.
template <typename T>
int enqueue_direct(Workspace& w, const Job& j, cudaStream_t st) {
    NvtxRange nv("ffg direct enqueue (DOUBLE/SINGLE)");
    const int B = j.B;
    const int n = (int)j.n;
    const ffg_model& md = *j.model;
    const size_t nn = (size_t)n * n;
    int rc;
    if ((rc = ensure(w, B, 0, n, false))) return rc;
    const size_t bytes = (size_t)B * nn * sizeof(T);
    if (bytes > w.cap_direct) {
        size_t dummy = 0;
        if ((rc = grow(&w.dX, dummy, bytes))) return rc;
        if ((rc = grow(&w.dY, dummy, bytes))) return rc;
        if ((rc = grow(&w.dA, dummy, bytes))) return rc;
        w.cap_direct = bytes;
    }
    cublasHandle_t hd;
    if ((rc = cublas_handle(st, &hd))) return rc;
    std::vector<double> ph((size_t)4 * B);
    for (int m = 0; m < B; ++m) {
        ph[0 * B + m] = j.alpha[m];
        ph[1 * B + m] = j.gamma[m];
        ph[2 * B + m] = j.scale ? j.scale[m] : 0.0;
        ph[3 * B + m] = j.mu ? j.mu[m] : 0.0;
    }
    if ((rc = upload_small(w, w.params, ph.data(), sizeof(double) * 4 * B, st))) return rc;
    reset_kernel<<<(B + 127) / 128, 128, 0, st>>>(w.bounds, w.flags, B, nullptr, 0, w.products);
    CK(cudaGetLastError());
    gershgorin_kernel<<<dim3((unsigned)((n + 7) / 8), (unsigned)B), 256, 0, st>>>(j.H_dev, n, w.bounds);
    CK(cudaGetLastError());
    T* X = reinterpret_cast<T*>(w.dX);
    T* Y = reinterpret_cast<T*>(w.dY);
    T* A = reinterpret_cast<T*>(w.dA);
    const unsigned eb = (unsigned)std::min<size_t>((nn + 255) / 256, 1024);
    direct_init_kernel<T><<<dim3(eb, (unsigned)B), 256, 0, st>>>(j.H_dev, w.params, w.params + B, md.abcd[3], X, A,
                                                                 n, w.flags);
    CK(cudaGetLastError());
    const int nt = (n + 31) / 32;
    const unsigned tiles = (unsigned)(nt * (nt + 1) / 2);
    const T one = (T)1, zero = (T)0;
    for (int l = 0; l < md.n_layers; ++l) {
        cublasStatus_t cs;
        if constexpr (std::is_same<T, double>::value)
            cs = g_cublas.dgemm(hd, CUBLAS_OP_N, CUBLAS_OP_N, n, n, n, &one, X, n, (long long)nn, X, n, (long long)nn,
                                &zero, Y, n, (long long)nn, B);
        else
            cs = g_cublas.sgemm(hd, CUBLAS_OP_N, CUBLAS_OP_N, n, n, n, &one, X, n, (long long)nn, X, n, (long long)nn,
                                &zero, Y, n, (long long)nn, B);
        if (cs != CUBLAS_STATUS_SUCCESS) return set_err(FFG_ERR_CUDA, "cuBLAS gemm failed (%d)", (int)cs);
        DirectLayer<T> dl;
        dl.Y = Y;
        dl.X = X;
        dl.A = A;
        dl.a = md.abcd[4 * l + 0];
        dl.b = md.abcd[4 * l + 1];
        dl.c = md.abcd[4 * l + 2];
        dl.d_next = l + 1 < md.n_layers ? md.abcd[4 * (l + 1) + 3] : 0.0;
        dl.n = n;
        dl.flags = w.flags;
        dl.layer = l;
        direct_layer_kernel<T><<<dim3(tiles, (unsigned)B), 256, 0, st>>>(dl);
        CK(cudaGetLastError());
    }
    RegionCheck region{w.bounds, j.scale ? w.params + 2 * B : nullptr, w.params + 3 * B, md.mu0};
    direct_final_kernel<T><<<dim3((unsigned)((n + 7) / 8), (unsigned)B), 256, 0, st>>>(
        X, A, j.D_dev, n, w.partials, region, md.n_layers, w.products);
    CK(cudaGetLastError());
    EnqueueCtx cx;
    cx.Tpart = n;
    cx.region = region;
    return enqueue_k3(w, j, st, cx, j.n);
}

int enqueue(Workspace& w, const Job& j, cudaStream_t st) {
    if (j.mode == kModeF64) return enqueue_direct<double>(w, j, st);
    if (j.mode == kModeF32) return enqueue_direct<float>(w, j, st);
    EnqueueCtx cx;
    int rc;
    if ((rc = enqueue_k1(w, j, st, cx))) return rc;
    if ((rc = enqueue_k2(w, j, st, cx, 0, j.model->n_layers))) return rc;
    return enqueue_k3(w, j, st, cx, j.n);
}

// The host-buffer entry points' stream on the current device (null on failure: ffg_last_error).
cudaStream_t lib_stream() {
    DevState* d;
    return dev_state(&d) == FFG_OK ? d->lib : nullptr;
}

// products: the K2 issuer's instrumented count of product passes for this matrix (all layers, all
// pair items); PT: pair items per layer, so products / PT = tensor-core products per square summed
// over the layers (SPEC.md:404 multiplication accounting; each product covers the upper-triangle
// blocks: 3 per FP32-emulated square, 4 in the fixed-point exact layers, 1 in BF16/FP16).
void fill_prov(ffg_provenance* pv, const double* bnd, const double* kT, double mu, int status,
               const int* flags, const ffg_model* md, int mode_api, int n, double ms, uint32_t products,
               int PT) {
    pv->eps_min = bnd[0];
    pv->eps_max = bnd[1];
    pv->x_min = bnd[2];
    pv->x_max = bnd[3];
    const double W = bnd[1] - bnd[0];
    pv->beta_prime = kT ? W / *kT : 0.0;
    pv->mu_prime = W > 0 ? (bnd[1] - mu) / W : 0.0;
    pv->mode = mode_api;
    pv->n_layers = md->n_layers;
    pv->half_products = PT > 0 ? (int64_t)(products / (uint32_t)PT) : 0;
    pv->diverged_layer = flags[0] == INT_MAX ? -1 : flags[0];
    pv->half_range_layer = flags[1] == INT_MAX ? -1 : flags[1];
    pv->status = status;
    pv->n = n;
    pv->device_ms = ms;
}

const char* status_text(int st) {
    switch (st) {
        case FFG_ERR_OUT_OF_REGION: return "out of region of validity";
        case FFG_ERR_DIVERGED: return "non-finite entry mid-recursion";
        case FFG_ERR_HALF_RANGE: return "binary16 split overflow";
        default: return "error";
    }
}

// Chunks of the pipelined host path (smaller chunks overlap more transfer but shrink each K2
// launch below its dependency slack).  Measured at N=1024, B=16: one synchronous call, 1 / 2 /
// 4 chunks -> e2e 1990 / 2795 / 3041 matrices/s (default B/4); two async calls in flight ->
// 3647 / 4507 / 3797 (default B/8: the neighbouring call already covers the edges).
// FFG_E2E_CHUNKS overrides.
int e2e_chunks(int B, bool async) {
    const char* e = getenv("FFG_E2E_CHUNKS");
    const int c = e ? atoi(e) : B / (async ? 8 : 4);
    return std::max(1, std::min({c, B, (int)Workspace::kMaxChunks}));
}

// Host-buffer driver shared by density_matrix(ces) / apply_model / mixed_square.
// Submit the pipelined host path for one batch into a free pipeline slot (no host sync): the
// batch runs in chunks; chunk k's H2D (copy stream) overlaps the compute of chunk k-1 and its
// D2H (second copy stream) the compute of chunk k+1.  All kernels stay on the library stream
// (K2 needs every CTA of its launch co-resident).  Three slots: a call may be submitted while
// the previous two are still in flight; slot buffers (H/D staging, pinned records) are per slot,
// the K2 workspace is shared in stream order.
int submit_host(Workspace& w, cudaStream_t st, int B, const double* const* H, int64_t n, const double* alpha,
                const double* gamma, const double* scale, const double* mu, const double* kT,
                const ffg_model* md, int mode_api, int mode, double* const* D_out, int* slot_out,
                bool async = false, int exact_layers = -1) {
    int rc;
    int si = -1;
    for (int k = 0; k < Workspace::kSlots; ++k)
        if (!w.slot[k].busy && (si < 0 || w.slot[k].ticket < w.slot[si].ticket)) si = k;
    if (si < 0) return set_err(FFG_ERR_VALIDATION, "three calls already in flight: ffg_wait one first");
    HostSlot& hsl = w.slot[si];
    const size_t nn = (size_t)n * n;
    size_t dummy = 0;
    if ((size_t)B * nn > hsl.cap) {
        if ((rc = grow(&hsl.Hs, dummy, (size_t)B * nn))) return rc;
        if ((rc = grow(&hsl.Ds, dummy, (size_t)B * nn))) return rc;
        hsl.cap = (size_t)B * nn;
    }
    const size_t small = (size_t)B * kRecordBytes;
    if (small > hsl.host_small_bytes) {
        cudaFreeHost(hsl.host_small);
        CK(cudaHostAlloc(&hsl.host_small, small, cudaHostAllocMapped));
        CK(cudaHostGetDevicePointer(&hsl.host_small_dev, hsl.host_small, 0));
        hsl.host_small_bytes = small;
    }
    if (!hsl.ev0) {
        CK(cudaEventCreate(&hsl.ev0));
        CK(cudaEventCreate(&hsl.ev1));
        CK(cudaEventCreateWithFlags(&hsl.ev_d2h, cudaEventDisableTiming));
        for (int k = 0; k < Workspace::kMaxChunks; ++k) {
            CK(cudaEventCreateWithFlags(&hsl.ev_in[k], cudaEventDisableTiming));
            CK(cudaEventCreateWithFlags(&hsl.ev_done[k], cudaEventDisableTiming));
        }
    }
    if (!w.s_h2d) {
        CK(cudaStreamCreateWithFlags(&w.s_h2d, cudaStreamNonBlocking));
        CK(cudaStreamCreateWithFlags(&w.s_d2h, cudaStreamNonBlocking));
    }
    const int64_t np = (n + kBM - 1) / kBM * kBM;
    const int64_t T = (np / kBM) * (np / kBM + 1) / 2;
    if ((rc = ensure(w, B, np, T, true))) return rc;
    bool want_D = false;
    if (D_out)
        for (int m = 0; m < B; ++m) want_D |= D_out[m] != nullptr;
    uint8_t* hs = static_cast<uint8_t*>(hsl.host_small);
    double* h_stats = reinterpret_cast<double*>(hs);
    double* h_bounds = h_stats + 2 * B;
    int* h_status = reinterpret_cast<int*>(h_bounds + 4 * B);
    int* h_flags = h_status + B;
    uint32_t* h_prod = reinterpret_cast<uint32_t*>(h_flags + 2 * B);
    const int nchunk = e2e_chunks(B, async);
    auto chunk_range = [&](int k, int& m0, int& mb) {
        m0 = (int)((int64_t)B * k / nchunk);
        mb = (int)((int64_t)B * (k + 1) / nchunk) - m0;
    };
    for (int k = 0; k < nchunk; ++k) {
        int m0, mb;
        chunk_range(k, m0, mb);
        for (int m = m0; m < m0 + mb; ++m)
            CK(cudaMemcpyAsync(hsl.Hs + m * nn, H[m], nn * sizeof(double), cudaMemcpyHostToDevice, w.s_h2d));
        CK(cudaEventRecord(hsl.ev_in[k], w.s_h2d));
    }
    CK(cudaEventRecord(hsl.ev0, st));
    for (int k = 0; k < nchunk; ++k) {
        int m0, mb;
        chunk_range(k, m0, mb);
        CK(cudaStreamWaitEvent(st, hsl.ev_in[k], 0));
        Job j;
        j.B = mb;
        j.n = n;
        j.H_dev = hsl.Hs + m0 * nn;
        j.alpha = alpha + m0;
        j.gamma = gamma + m0;
        j.scale = scale ? scale + m0 : nullptr;
        j.mu = mu ? mu + m0 : nullptr;
        j.model = md;
        j.mode = mode;
        j.D_dev = want_D ? hsl.Ds + m0 * nn : nullptr;
        j.exact_layers = exact_layers;
        if ((rc = enqueue(w, j, st))) return rc;
        // per-matrix records of this chunk (the next chunk's reset reuses the workspace), written
        // into the mapped record block by a kernel (no copy engine: see copy_words_kernel)
        records_kernel<<<1, 128, 0, st>>>(static_cast<uint8_t*>(hsl.host_small_dev), B, m0, mb, w.stats,
                                          w.bounds_out, w.status, w.flags, w.products);
        CK(cudaGetLastError());
        CK(cudaEventRecord(hsl.ev_done[k], st));
        if (want_D) {
            CK(cudaStreamWaitEvent(w.s_d2h, hsl.ev_done[k], 0));
            for (int m = m0; m < m0 + mb; ++m)
                if (D_out[m])
                    CK(cudaMemcpyAsync(D_out[m], hsl.Ds + m * nn, nn * sizeof(double), cudaMemcpyDeviceToHost,
                                       w.s_d2h));
        }
    }
    CK(cudaEventRecord(hsl.ev1, st));
    CK(cudaEventRecord(hsl.ev_d2h, w.s_d2h));
    hsl.busy = true;
    hsl.ticket = ++w.next_ticket;
    hsl.B = B;
    hsl.n = n;
    hsl.PT = (mode == kModeF64 || mode == kModeF32) ? 1 : w.PT;  // direct modes count squarings directly
    hsl.mode_api = mode_api;
    hsl.model = *md;
    hsl.mu.assign(mu ? mu : alpha, (mu ? mu : alpha) + B);
    hsl.has_mu = mu != nullptr;
    hsl.kT.assign(kT ? kT : alpha, (kT ? kT : alpha) + B);
    hsl.has_kT = kT != nullptr;
    *slot_out = si;
    return FFG_OK;
}

// Wait for a submitted batch and deliver its statistics / provenance / status.
int finish_host(Workspace& w, int si, double* stats_out, ffg_provenance* prov) {
    HostSlot& hsl = w.slot[si];
    hsl.busy = false;
    CK(cudaEventSynchronize(hsl.ev1));
    CK(cudaEventSynchronize(hsl.ev_d2h));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, hsl.ev0, hsl.ev1));
    const int B = hsl.B;
    uint8_t* hs = static_cast<uint8_t*>(hsl.host_small);
    double* h_stats = reinterpret_cast<double*>(hs);
    double* h_bounds = h_stats + 2 * B;
    int* h_status = reinterpret_cast<int*>(h_bounds + 4 * B);
    int* h_flags = h_status + B;
    const uint32_t* h_prod = reinterpret_cast<const uint32_t*>(h_flags + 2 * B);
    int first = FFG_OK, first_m = -1;
    for (int m = 0; m < B; ++m) {
        if (stats_out) {
            stats_out[2 * m + 0] = h_stats[2 * m + 0];
            stats_out[2 * m + 1] = h_stats[2 * m + 1];
        }
        if (prov)
            fill_prov(&prov[m], h_bounds + 4 * m, hsl.has_kT ? &hsl.kT[m] : nullptr,
                      hsl.has_mu ? hsl.mu[m] : 0.0, h_status[m], h_flags + 2 * m, &hsl.model, hsl.mode_api,
                      (int)hsl.n, ms, h_prod[m], hsl.PT);
        if (h_status[m] != FFG_OK && first == FFG_OK) {
            first = h_status[m];
            first_m = m;
        }
    }
    if (first != FFG_OK) {
        const double* b = h_bounds + 4 * first_m;
        if (first == FFG_ERR_OUT_OF_REGION)
            return set_err(first, "matrix %d: out of region of validity: %s (x_min=%.17g, x_max=%.17g; "
                           "eps=[%.17g, %.17g])", first_m,
                           !(b[2] >= 0.0) ? "mu0 + (beta/beta0)(eps_min - mu) >= 0 violated"
                                          : "mu0 + (beta/beta0)(eps_max - mu) <= 1 violated",
                           b[2], b[3], b[0], b[1]);
        const int* f = h_flags + 2 * first_m;
        return set_err(first, "matrix %d: %s at layer %d", first_m, status_text(first),
                       first == FFG_ERR_DIVERGED ? f[0] : f[1]);
    }
    return FFG_OK;
}

int validate_host_call(int B, const double* const* H, int64_t n, const ffg_model* md, int mode_api, int* mode,
                       int* dev) {
    int rc;
    if ((rc = validate_model(md))) return rc;
    if ((rc = mode_to_internal(mode_api, mode))) return rc;
    if ((rc = validate_n(n))) return rc;
    if (B < 1) return set_err(FFG_ERR_DIMENSION, "batch must be >= 1");
    for (int m = 0; m < B; ++m)
        if (!H[m]) return set_err(FFG_ERR_VALIDATION, "H[%d] is null", m);
    return check_device(dev);
}

// Host-buffer driver shared by density_matrix(ces) / apply_model / mixed_square: submit + wait.
int run_host(int B, const double* const* H, int64_t n, const double* alpha, const double* gamma,
             const double* scale, const double* mu, const double* kT, const ffg_model* md,
             int mode_api, double* const* D_out, double* stats_out, ffg_provenance* prov,
             int exact_layers = -1) {
    int rc, dev, mode;
    if ((rc = validate_host_call(B, H, n, md, mode_api, &mode, &dev))) return rc;
    cudaStream_t st = lib_stream();
    if (!st) return FFG_ERR_CUDA;
    Workspace& w = *get_ws(dev, st);
    std::lock_guard<std::mutex> lk(w.mu);
    int si;
    if ((rc = submit_host(w, st, B, H, n, alpha, gamma, scale, mu, kT, md, mode_api, mode, D_out, &si, false,
                          exact_layers)))
        return rc;
    return finish_host(w, si, stats_out, prov);
}

int check_mu_kT(int B, const double* mu, const double* kT) {
    if (!mu || !kT) return set_err(FFG_ERR_VALIDATION, "mu / kT arrays are null");
    for (int m = 0; m < B; ++m) {
        if (!(kT[m] > 0.0) || !std::isfinite(kT[m]))
            return set_err(FFG_ERR_VALIDATION, "kT[%d] must be positive and finite", m);
        if (!std::isfinite(mu[m])) return set_err(FFG_ERR_VALIDATION, "mu[%d] must be finite", m);
    }
    return FFG_OK;
}

void rescale_coeffs(int B, const double* mu, const double* kT, const ffg_model* md,
                    std::vector<double>& alpha, std::vector<double>& gamma,
                    std::vector<double>& scale) {
    alpha.resize(B);
    gamma.resize(B);
    scale.resize(B);
    for (int m = 0; m < B; ++m) {
        const double s = (1.0 / kT[m]) / md->beta0;
        scale[m] = s;
        alpha[m] = -s;
        gamma[m] = (1.0 - md->mu0) + s * mu[m];
    }
}

// One K1 -> K2 -> K3 run of a single device-resident matrix (workspace staging) and its
// per-matrix records: stats {Tr D, Tr D^2}, widened bounds {eps_min, eps_max, x_min, x_max},
// status, flags.  D goes to w.Ds when want_D.
int eval_single(Workspace& w, cudaStream_t st, int64_t n, double alpha, double gamma, double scale,
                double mu, const ffg_model* md, int mode, bool want_D, double stats[2], double bounds[4],
                int* status, int flags[2], uint32_t* products = nullptr) {
    Job j;
    j.B = 1;
    j.n = n;
    j.H_dev = w.Hs;
    j.alpha = &alpha;
    j.gamma = &gamma;
    j.scale = &scale;
    j.mu = &mu;
    j.model = md;
    j.mode = mode;
    j.D_dev = want_D ? w.Ds : nullptr;
    int rc;
    if ((rc = enqueue(w, j, st))) return rc;
    uint8_t* hs = static_cast<uint8_t*>(w.host_small);
    CK(cudaMemcpyAsync(hs, w.stats, 16, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(hs + 16, w.bounds_out, 32, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(hs + 48, w.status, 4, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(hs + 52, w.flags, 8, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(hs + 60, w.products, 4, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    memcpy(stats, hs, 16);
    memcpy(bounds, hs + 16, 32);
    memcpy(status, hs + 48, 4);
    memcpy(flags, hs + 52, 8);
    if (products) memcpy(products, hs + 60, 4);
    return FFG_OK;
}

// Row-block session (ffg_rowblock_*): one rank's own workspace and job over the whole run.
struct RowBlockState {
    Workspace* w = nullptr;
    int device = -1;
    Job job;
    EnqueueCtx cx;
    std::vector<double> abcd;
    ffg_model model{};
    double alpha = 0, gamma = 0, scale = 0, mu = 0, kT = 0;
    int mode_api = 0;
    int64_t n = 0, np = 0;
    int nb = 0, rank = 0, world = 1, r0 = 0, r1 = 0;
    int next_layer = 0;
};

int status_error(int code, const double* b, const int* f) {
    if (code == FFG_ERR_OUT_OF_REGION)
        return set_err(code, "out of region of validity: x in [%.17g, %.17g] (eps=[%.17g, %.17g])", b[2], b[3],
                       b[0], b[1]);
    return set_err(code, "%s at layer %d", status_text(code), code == FFG_ERR_DIVERGED ? f[0] : f[1]);
}

}  // namespace

struct ffg_rowblock {
    RowBlockState s;
};

// ===================================================================== C ABI
extern "C" {

int ffg_abi_version(void) { return FFG_ABI_VERSION; }
const char* ffg_last_error(void) { return g_err.c_str(); }

int ffg_device_available(void) {
    int dev;
    return check_device(&dev) == FFG_OK ? 1 : 0;
}

int ffg_in_region_of_validity(double beta_prime, double mu_prime, double beta0, double mu0) {
    if (!(mu_prime > 0.0 && mu_prime < 1.0)) return 0;
    return (mu0 / mu_prime) * beta0 >= beta_prime &&
                   ((1.0 - mu0) / (1.0 - mu_prime)) * beta0 >= beta_prime
               ? 1
               : 0;
}

int ffg_spectral_bounds(const double* H, int64_t n, double* eps_min, double* eps_max) {
    NvtxRange nv("ffg_spectral_bounds");
    int rc, dev;
    if ((rc = validate_n(n))) return rc;
    if (!H || !eps_min || !eps_max) return set_err(FFG_ERR_VALIDATION, "null argument");
    if ((rc = check_device(&dev))) return rc;
    cudaStream_t st = lib_stream();
    if (!st) return FFG_ERR_CUDA;
    Workspace& w = *get_ws(dev, st);
    std::lock_guard<std::mutex> lk(w.mu);
    const size_t nn = (size_t)n * n;
    if ((rc = ensure_staging(w, nn))) return rc;
    if ((rc = ensure(w, 1, 128, 1, false))) return rc;
    CK(cudaMemcpyAsync(w.Hs, H, nn * 8, cudaMemcpyHostToDevice, st));
    reset_kernel<<<1, 32, 0, st>>>(w.bounds, w.flags, 1);
    gershgorin_kernel<<<dim3((unsigned)((n + 7) / 8), 1), 256, 0, st>>>(w.Hs, (int)n, w.bounds);
    CK(cudaGetLastError());
    unsigned long long k[2];
    CK(cudaMemcpyAsync(k, w.bounds, 16, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    double lo = key_to_double(k[0]), hi = key_to_double(k[1]);
    const double wd = 1e-12 * (hi - lo);
    *eps_min = lo - wd;
    *eps_max = hi + wd;
    return FFG_OK;
}

int ffg_apply_model(const double* H0, int64_t n, const ffg_model* model, int32_t mode,
                    double* D_out, ffg_provenance* prov) {
    NvtxRange nv("ffg_apply_model");
    const double alpha = -1.0, gamma = 1.0;  // X0 = I - H0 (scalar_models.cpp:333)
    double* Dp[1] = {D_out};
    return run_host(1, &H0, n, &alpha, &gamma, nullptr, nullptr, nullptr, model, mode, Dp,
                    nullptr, prov);
}

// X0 = half(X), X1 = half(X - X0), Y = X0 X0 + X0 X1 + (X0 X1)^T accumulated in
// single precision, over the whole binary16 range.  The kernels split x * 2^14; a call picks the
// power of two 2^e that puts max|X| just below 65504 (e <= 40: small inputs keep their lo parts out
// of the binary16 subnormals) and feeds X * 2^(e-14), then scales Y back by 2^(28-2e) -- exact
// power-of-two scalings, so the split is that of X at scale 2^e.  One layer of the identity model
// (a=1, b=c=d=0) on the floating split (no fixed-point exact layer): the three upper-triangle
// products hi*hi + hi*lo + lo*hi of Eq. 48, i.e. 1.5 full-GEMM equivalents against SPEC's "2 half
// multiplications".  |X| beyond the binary16 range -> FFG_ERR_HALF_RANGE (overflow error).
int ffg_mixed_square(const float* X, int64_t n, float* Y_out) {
    NvtxRange nv("ffg_mixed_square");
    int rc;
    if ((rc = validate_n(n))) return rc;
    if (!X || !Y_out) return set_err(FFG_ERR_VALIDATION, "null argument");
    const size_t nn = (size_t)n * n;
    float amax = 0.0f;
    for (size_t e = 0; e < nn; ++e) {
        if (!std::isfinite(X[e])) return set_err(FFG_ERR_VALIDATION, "mixed_square: non-finite entry %zu", e);
        amax = std::max(amax, std::fabs(X[e]));
    }
    if (!(amax < 65504.0f))
        return set_err(FFG_ERR_HALF_RANGE, "mixed_square: max|X| = %.9g exceeds the binary16 range (65504)",
                       (double)amax);
    int e = 40;
    if (amax > 0.0f) {
        e = std::min(40, (int)std::floor(std::log2(65504.0 / (double)amax)));
        while (e > -30 && !((double)amax * std::ldexp(1.0, e) < 65504.0)) --e;
    }
    std::vector<double> Xd(nn), Yd(nn);
    for (size_t k = 0; k < nn; ++k) Xd[k] = (double)std::ldexp(X[k], e - 14);  // exact in fp32 and fp64
    const double abcd[4] = {1.0, 0.0, 0.0, 0.0};
    ffg_model m{abcd, 1, 1.0, 0.5};
    const double alpha = 1.0, gamma = 0.0;
    const double* Hp[1] = {Xd.data()};
    double* Dp[1] = {Yd.data()};
    rc = run_host(1, Hp, n, &alpha, &gamma, nullptr, nullptr, nullptr, &m, FFG_MODE_MIXED_EMULATED, Dp, nullptr,
                  nullptr, /*exact_layers=*/0);
    if (rc) return rc;
    for (size_t k = 0; k < nn; ++k) Y_out[k] = (float)std::ldexp(Yd[k], 28 - 2 * e);
    return FFG_OK;
}

int ffg_expectation(const double* D, const double* A, int64_t n, double* out) {
    NvtxRange nv("ffg_expectation");
    int rc, dev;
    if ((rc = validate_n(n))) return rc;
    if (!D || !A || !out) return set_err(FFG_ERR_VALIDATION, "null argument");
    if ((rc = check_device(&dev))) return rc;
    cudaStream_t st = lib_stream();
    if (!st) return FFG_ERR_CUDA;
    Workspace& w = *get_ws(dev, st);
    std::lock_guard<std::mutex> lk(w.mu);
    const size_t nn = (size_t)n * n;
    if ((rc = ensure_staging(w, nn))) return rc;
    if ((rc = ensure(w, 1, 128, n, false))) return rc;
    CK(cudaMemcpyAsync(w.Hs, A, nn * 8, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(w.Ds, D, nn * 8, cudaMemcpyHostToDevice, st));
    row_dot_kernel<<<(unsigned)((n + 7) / 8), 256, 0, st>>>(w.Ds, w.Hs, (int)n, w.partials);
    reset_kernel<<<1, 32, 0, st>>>(w.bounds, w.flags, 1);
    FinalizeParams fp{};
    fp.partials = w.partials;
    fp.region = RegionCheck{w.bounds, nullptr, nullptr, 0.0};
    fp.flags = w.flags;
    fp.T = (int)n;
    fp.B = 1;
    fp.stats = w.stats;
    fp.bounds_out = w.bounds_out;
    fp.status = w.status;
    finalize_stats_kernel<<<1, 256, 0, st>>>(fp);
    CK(cudaGetLastError());
    double r[2];
    CK(cudaMemcpyAsync(r, w.stats, 16, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    *out = r[0];
    return FFG_OK;
}

int ffg_entropy_trace(const double* H, int64_t n, double mu, double kT, const ffg_entropy_model* em,
                      int32_t mode_api, double* entropy_trace, ffg_provenance* prov) {
    NvtxRange nv("ffg_entropy_trace");
    int rc, dev, mode;
    if (!em) return set_err(FFG_ERR_VALIDATION, "entropy model is null");
    if ((rc = validate_model(&em->inner))) return rc;
    if (!(em->alpha > 0.0 && em->alpha < 1.0) || !std::isfinite(em->alpha))
        return set_err(FFG_ERR_VALIDATION, "EntropyModelCoefficients: alpha must lie in (0,1)");
    if ((rc = mode_to_internal(mode_api, &mode))) return rc;
    if ((rc = validate_n(n))) return rc;
    if ((rc = check_mu_kT(1, &mu, &kT))) return rc;
    if (!H || !entropy_trace) return set_err(FFG_ERR_VALIDATION, "null argument");
    if ((rc = check_device(&dev))) return rc;
    cudaStream_t st = lib_stream();
    if (!st) return FFG_ERR_CUDA;
    Workspace& w = *get_ws(dev, st);
    std::lock_guard<std::mutex> lk(w.mu);
    const size_t nn = (size_t)n * n;
    if ((rc = ensure_staging(w, nn))) return rc;
    CK(cudaMemcpyAsync(w.Hs, H, nn * 8, cudaMemcpyHostToDevice, st));
    // model frame x = mu0 + s (H - mu), x0 = alpha (x - mu0) + mu0 = alpha s (H - mu) + mu0
    const double s = (1.0 / kT) / em->inner.beta0;
    const double a = em->alpha * s, g = em->inner.mu0 - em->alpha * s * mu;
    double stats[2], bounds[4];
    int status, flags[2];
    uint32_t products = 0;
    if ((rc = eval_single(w, st, n, a, g, s, mu, &em->inner, mode, false, stats, bounds, &status, flags,
                          &products)))
        return rc;
    if (prov) fill_prov(prov, bounds, &kT, mu, status, flags, &em->inner, mode_api, (int)n, 0.0, products, w.PT);
    if (status != FFG_OK) return status_error(status, bounds, flags);
    *entropy_trace = 4.0 * std::log(2.0) * (stats[0] - stats[1]);
    return FFG_OK;
}

int ffg_solve_chemical_potential(const double* H, int64_t n, double kT, double n_occ, double mu_guess,
                                 const ffg_model* md, int32_t mode_api, double tol, int32_t max_iter,
                                 double* D_out, double* stats_out, double* history, ffg_mu_report* report) {
    NvtxRange nv("ffg_solve_chemical_potential");
    int rc, dev, mode;
    if ((rc = validate_model(md))) return rc;
    if ((rc = mode_to_internal(mode_api, &mode))) return rc;
    if ((rc = validate_n(n))) return rc;
    if (!H) return set_err(FFG_ERR_VALIDATION, "H is null");
    if (!(kT > 0.0) || !std::isfinite(kT)) return set_err(FFG_ERR_VALIDATION, "kT must be positive and finite");
    if (!(n_occ > 0.0 && n_occ < (double)n))
        return set_err(FFG_ERR_VALIDATION, "n_occ must lie in (0, N) (got %.17g)", n_occ);
    if (!std::isfinite(mu_guess)) return set_err(FFG_ERR_VALIDATION, "mu_guess must be finite");
    if (!(tol > 0.0) || max_iter < 1) return set_err(FFG_ERR_VALIDATION, "tol > 0 and max_iter >= 1 required");
    if ((rc = check_device(&dev))) return rc;
    cudaStream_t st = lib_stream();
    if (!st) return FFG_ERR_CUDA;
    Workspace& w = *get_ws(dev, st);
    std::lock_guard<std::mutex> lk(w.mu);
    const size_t nn = (size_t)n * n;
    if ((rc = ensure_staging(w, nn))) return rc;
    CK(cudaMemcpyAsync(w.Hs, H, nn * 8, cudaMemcpyHostToDevice, st));
    const double beta = 1.0 / kT, s = beta / md->beta0;
    auto eval = [&](double mu, double* stats, double* bounds, int* status, int* flags) {
        return eval_single(w, st, n, -s, (1.0 - md->mu0) + s * mu, s, mu, md, mode, true, stats, bounds, status,
                           flags);
    };
    double mu = mu_guess, stats[2], bounds[4];
    int status, flags[2];
    if ((rc = eval(mu, stats, bounds, &status, flags))) return rc;
    // bracket: mu for which the model's region of validity holds (x_min >= 0, x_max <= 1) and
    // Tr D is monotone in mu (Eq. 43: dTr D / dmu = beta Tr D(I - D) >= 0)
    const double W = bounds[1] - bounds[0];
    double lo = std::max(bounds[0], bounds[1] - (1.0 - md->mu0) / s);
    double hi = std::min(bounds[1], bounds[0] + md->mu0 / s);
    if (!(lo < hi))
        return set_err(FFG_ERR_OUT_OF_REGION, "no chemical potential keeps beta'=%.6g inside the model's region "
                       "of validity (beta0=%.6g)", beta * W, md->beta0);
    if (status == FFG_ERR_OUT_OF_REGION) {  // cold start outside the region: restart mid-bracket
        mu = 0.5 * (lo + hi);
        if ((rc = eval(mu, stats, bounds, &status, flags))) return rc;
    }
    if (status != FFG_OK) return status_error(status, bounds, flags);
    int it = 1, bis = 0;
    bool conv = false;
    double g = stats[0] - n_occ;
    for (;;) {
        if (history) {
            history[2 * (it - 1) + 0] = mu;
            history[2 * (it - 1) + 1] = g;
        }
        if (std::fabs(g) <= tol) {
            conv = true;
            break;
        }
        if (it >= max_iter) break;
        if (g > 0.0) hi = std::min(hi, mu); else lo = std::max(lo, mu);
        const double gp = beta * (stats[0] - stats[1]);   // Eq. 44
        double next;
        if (gp > 1e-14 * beta * (double)n) {
            double dmu = -g / gp;                             // Eq. 45
            dmu = std::max(-0.5 * W, std::min(0.5 * W, dmu)); // clamp: half the spectral width
            next = mu + dmu;
            if (!(next > lo && next < hi)) {                  // safeguard: leave the bracket -> bisect
                next = 0.5 * (lo + hi);
                ++bis;
            }
        } else {                                              // flat derivative: bisection fallback
            next = 0.5 * (lo + hi);
            ++bis;
        }
        mu = next;
        if ((rc = eval(mu, stats, bounds, &status, flags))) return rc;
        if (status != FFG_OK) return status_error(status, bounds, flags);
        g = stats[0] - n_occ;
        ++it;
    }
    if (D_out) {
        CK(cudaMemcpyAsync(D_out, w.Ds, nn * 8, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
    }
    if (stats_out) {
        stats_out[0] = stats[0];
        stats_out[1] = stats[1];
    }
    if (report) {
        report->mu = mu;
        report->residual = g;
        report->iterations = it;
        report->converged = conv ? 1 : 0;
        report->bisections = bis;
    }
    if (!conv)
        return set_err(FFG_ERR_DIVERGED, "chemical potential not converged after %d evaluations "
                       "(|Tr D - n_occ| = %.3g > tol %.3g)", it, std::fabs(g), tol);
    return FFG_OK;
}

int ffg_density_statistics(const double* D, int64_t n, double* stats_out) {
    NvtxRange nv("ffg_density_statistics");
    int rc, dev;
    if ((rc = validate_n(n))) return rc;
    if (!D || !stats_out) return set_err(FFG_ERR_VALIDATION, "null argument");
    if ((rc = check_device(&dev))) return rc;
    cudaStream_t st = lib_stream();
    if (!st) return FFG_ERR_CUDA;
    Workspace& w = *get_ws(dev, st);
    std::lock_guard<std::mutex> lk(w.mu);
    const size_t nn = (size_t)n * n;
    if ((rc = ensure_staging(w, nn))) return rc;
    if ((rc = ensure(w, 1, 128, n, false))) return rc;
    CK(cudaMemcpyAsync(w.Hs, D, nn * 8, cudaMemcpyHostToDevice, st));
    row_stats_kernel<<<(unsigned)((n + 7) / 8), 256, 0, st>>>(w.Hs, (int)n, w.partials);
    reset_kernel<<<1, 32, 0, st>>>(w.bounds, w.flags, 1);
    FinalizeParams fp{};
    fp.partials = w.partials;
    fp.region = RegionCheck{w.bounds, nullptr, nullptr, 0.0};
    fp.flags = w.flags;
    fp.T = (int)n;
    fp.B = 1;
    fp.stats = w.stats;
    fp.bounds_out = w.bounds_out;
    fp.status = w.status;
    finalize_stats_kernel<<<1, 256, 0, st>>>(fp);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(stats_out, w.stats, 16, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    return FFG_OK;
}

int ffg_density_matrix(const double* H, int64_t n, double mu, double kT, const ffg_model* model,
                       int32_t mode, double* D_out, double* stats_out, ffg_provenance* prov) {
    NvtxRange nv("ffg_density_matrix");
    double* Dp[1] = {D_out};
    return ffg_density_matrices(1, &H, n, &mu, &kT, model, mode, Dp, stats_out, prov);
}

int ffg_density_matrices(int32_t batch, const double* const* H, int64_t n, const double* mu,
                         const double* kT, const ffg_model* model, int32_t mode,
                         double* const* D_out, double* stats_out, ffg_provenance* prov) {
    NvtxRange nv("ffg_density_matrices");
    int rc;
    if (batch < 1) return set_err(FFG_ERR_DIMENSION, "batch must be >= 1");
    if (!H) return set_err(FFG_ERR_VALIDATION, "H is null");
    if ((rc = validate_model(model))) return rc;
    if ((rc = check_mu_kT(batch, mu, kT))) return rc;
    std::vector<double> alpha, gamma, scale;
    rescale_coeffs(batch, mu, kT, model, alpha, gamma, scale);
    return run_host(batch, H, n, alpha.data(), gamma.data(), scale.data(), mu, kT, model, mode,
                    D_out, stats_out, prov);
}

int ffg_density_matrices_async(int32_t batch, const double* const* H, int64_t n, const double* mu,
                               const double* kT, const ffg_model* model, int32_t mode_api,
                               double* const* D_out, int64_t* ticket) {
    NvtxRange nv("ffg_density_matrices_async");
    int rc, dev, mode;
    if (!H || !ticket) return set_err(FFG_ERR_VALIDATION, "H / ticket is null");
    if ((rc = validate_host_call(batch, H, n, model, mode_api, &mode, &dev))) return rc;
    if ((rc = check_mu_kT(batch, mu, kT))) return rc;
    std::vector<double> alpha, gamma, scale;
    rescale_coeffs(batch, mu, kT, model, alpha, gamma, scale);
    cudaStream_t st = lib_stream();
    if (!st) return FFG_ERR_CUDA;
    Workspace& w = *get_ws(dev, st);
    std::lock_guard<std::mutex> lk(w.mu);
    int si;
    if ((rc = submit_host(w, st, batch, H, n, alpha.data(), gamma.data(), scale.data(), mu, kT, model, mode_api,
                          mode, D_out, &si, true)))
        return rc;
    *ticket = w.slot[si].ticket;
    return FFG_OK;
}

int ffg_wait(int64_t ticket, double* stats_out, ffg_provenance* prov) {
    NvtxRange nv("ffg_wait");
    int rc, dev;
    if ((rc = check_device(&dev))) return rc;
    cudaStream_t st = lib_stream();
    if (!st) return FFG_ERR_CUDA;
    Workspace& w = *get_ws(dev, st);
    std::lock_guard<std::mutex> lk(w.mu);
    for (int k = 0; k < Workspace::kSlots; ++k)
        if (w.slot[k].busy && w.slot[k].ticket == ticket) return finish_host(w, k, stats_out, prov);
    return set_err(FFG_ERR_VALIDATION, "ffg_wait: unknown or already completed ticket %lld", (long long)ticket);
}

int ffg_density_matrices_dev(int32_t batch, const double* H_dev, int64_t n, const double* mu,
                             const double* kT, const ffg_model* model, int32_t mode,
                             double* D_dev, double* stats_dev, int32_t* status_dev,
                             double* bounds_dev, void* stream) {
    NvtxRange nv("ffg_density_matrices_dev");
    int rc, dev, imode;
    if (batch < 1) return set_err(FFG_ERR_DIMENSION, "batch must be >= 1");
    if (!H_dev) return set_err(FFG_ERR_VALIDATION, "H_dev is null");
    if ((rc = validate_model(model))) return rc;
    if ((rc = mode_to_internal(mode, &imode))) return rc;
    if ((rc = validate_n(n))) return rc;
    if ((rc = check_mu_kT(batch, mu, kT))) return rc;
    if ((rc = check_device(&dev))) return rc;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    Workspace& w = *get_ws(dev, st);
    std::lock_guard<std::mutex> lk(w.mu);
    std::vector<double> alpha, gamma, scale;
    rescale_coeffs(batch, mu, kT, model, alpha, gamma, scale);
    Job j;
    j.B = batch;
    j.n = n;
    j.H_dev = H_dev;
    j.alpha = alpha.data();
    j.gamma = gamma.data();
    j.scale = scale.data();
    j.mu = mu;
    j.model = model;
    j.mode = imode;
    j.D_dev = D_dev;
    j.stats_dev = stats_dev;
    j.status_dev = status_dev;
    j.bounds_dev = bounds_dev;
    return enqueue(w, j, st);
}

int32_t ffg_k2_kernel(int64_t n, int32_t mode) {
    int m;
    if (n < 1 || mode_to_internal(mode, &m)) return -1;
    if (m == kModeF64 || m == kModeF32) return 2;  // library GEMM + direct.cuh layer kernels
    const int64_t np = (n + kBM - 1) / kBM * kBM;
    return use_wide(m, (int)(np / kBM), false) ? 1 : 0;
}

int64_t ffg_kernel_launches(int32_t batch, int64_t n, const ffg_model* model, int32_t mode) {
    int m;
    if (!model || batch < 1 || n < 1 || mode_to_internal(mode, &m)) return 0;
    if (m == kModeF64 || m == kModeF32)  // upload, reset, bounds, init, L layer updates, final, K3
        return 6 + model->n_layers;      // (+ L library GEMMs, not counted: not our kernels)
    // two parameter uploads (launch-carried, upload_small), reset, K1, K2 (all layers; one persistent
    // launch per kValidBits matrices), K3
    return 5 + (batch + kValidBits - 1) / kValidBits;
}

int ffg_profile_layers(int enable) {
    std::lock_guard<std::mutex> lk(g_prof.mu);
    g_prof.on = enable != 0;
    g_prof.used = 0;
    g_prof.flops = 0.0;
    return FFG_OK;
}

int ffg_profile_read_ex(double* total_ms, int64_t* launches, double* algorithmic_flops) {
    std::lock_guard<std::mutex> lk(g_prof.mu);
    double t = 0.0;
    for (size_t i = 0; i < g_prof.used; ++i) {
        CK(cudaEventSynchronize(g_prof.ev[i].second));
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, g_prof.ev[i].first, g_prof.ev[i].second));
        t += ms;
    }
    if (total_ms) *total_ms = t;
    if (launches) *launches = (int64_t)g_prof.used;
    if (algorithmic_flops) *algorithmic_flops = g_prof.flops;
    g_prof.used = 0;
    g_prof.flops = 0.0;
    return FFG_OK;
}

int ffg_profile_read(double* total_ms, int64_t* launches) {
    return ffg_profile_read_ex(total_ms, launches, nullptr);
}

// Measurement only (FFG_DEBUG_K2 & 8): per-CTA role wait cycles of the last pair launch.
int ffg_debug_role_cycles(uint64_t* out, int32_t ctas) {
    if (!g_prof_buf) return set_err(FFG_ERR_VALIDATION, "no profile (set FFG_DEBUG_K2 & 8)");
    CK(cudaDeviceSynchronize());
    memcpy(out, g_prof_buf, sizeof(uint64_t) * 16 * ctas);
    return FFG_OK;
}

// Measurement/debug: the watchdog record (see install_watchdog); returns fired count.
int64_t ffg_debug_watchdog(uint64_t* out6) {
    if (!g_watch_host) return 0;
    for (int i = 0; i < 6; ++i) out6[i] = g_watch_host[i];
    return (int64_t)g_watch_host[0];
}

int32_t ffg_rowblock_table(int32_t nb, int32_t rank, int32_t world, uint32_t* out, int32_t capacity) {
    if (nb < 1 || nb > 1023 || world < 1 || rank < 0 || rank >= world || nb % world) return -1;
    int r0, r1;
    rowblock_rows(nb, rank, world, &r0, &r1);
    const std::vector<uint32_t> t = rowblock_table(nb, r0, r1);
    if (out)
        for (int32_t i = 0; i < (int32_t)t.size() && i < capacity; ++i) out[i] = t[i];
    return (int32_t)t.size();
}

int ffg_rowblock_begin(const double* H_dev, int64_t n, double mu, double kT, const ffg_model* model,
                       int32_t mode_api, int32_t rank, int32_t world, void* stream, ffg_rowblock** handle) {
    NvtxRange nv("ffg_rowblock_begin");
    int rc, dev, mode;
    if (!H_dev || !handle) return set_err(FFG_ERR_VALIDATION, "H_dev / handle is null");
    *handle = nullptr;
    if ((rc = validate_model(model))) return rc;
    if ((rc = mode_to_internal(mode_api, &mode))) return rc;
    if (mode == kModeF64 || mode == kModeF32)
        return set_err(FFG_ERR_UNSUPPORTED, "row-block sharding runs the tensor-core modes (MIXED_EMULATED, BF16, FP16)");
    if ((rc = validate_n(n))) return rc;
    if ((rc = check_mu_kT(1, &mu, &kT))) return rc;
    if (world < 1 || rank < 0 || rank >= world)
        return set_err(FFG_ERR_VALIDATION, "row-block rank %d of world %d", rank, world);
    const int nb = (int)((n + kBM - 1) / kBM);
    if (nb % world)
        return set_err(FFG_ERR_DIMENSION, "row-block sharding needs the %d blocks of 128 rows to divide evenly "
                       "over %d ranks (n = %lld)", nb, world, (long long)n);
    if ((rc = check_device(&dev))) return rc;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    ffg_rowblock* h = new ffg_rowblock();
    RowBlockState& S = h->s;
    S.w = new Workspace();
    S.w->device = dev;
    S.device = dev;
    S.abcd.assign(model->abcd, model->abcd + 4 * model->n_layers);
    S.model = *model;
    S.model.abcd = S.abcd.data();
    S.kT = kT;
    S.mu = mu;
    S.scale = (1.0 / kT) / model->beta0;
    S.alpha = -S.scale;
    S.gamma = (1.0 - model->mu0) + S.scale * mu;
    S.mode_api = mode_api;
    S.n = n;
    S.nb = nb;
    S.np = (int64_t)nb * kBM;
    S.rank = rank;
    S.world = world;
    rowblock_rows(nb, rank, world, &S.r0, &S.r1);
    Job& j = S.job;
    j.B = 1;
    j.n = n;
    j.H_dev = H_dev;
    j.alpha = &S.alpha;
    j.gamma = &S.gamma;
    j.scale = &S.scale;
    j.mu = &S.mu;
    j.model = &S.model;
    j.mode = mode;
    j.rb_world = world;
    j.rb_rank = rank;
    if ((rc = enqueue_k1(*S.w, j, st, S.cx))) {
        free_ws(S.w);
        delete S.w;
        delete h;
        return rc;
    }
    *handle = h;
    return FFG_OK;
}

int ffg_rowblock_rows(const ffg_rowblock* h, int64_t* row0, int64_t* rows, int64_t* np) {
    if (!h) return set_err(FFG_ERR_VALIDATION, "null handle");
    const RowBlockState& S = h->s;
    if (row0) *row0 = (int64_t)S.r0 * kBM;
    if (rows) *rows = (int64_t)(S.r1 - S.r0) * kBM;
    if (np) *np = S.np;
    return FFG_OK;
}

int ffg_rowblock_operands(ffg_rowblock* h, int32_t parity, void** hi, void** lo) {
    if (!h || parity < 0 || parity > 1) return set_err(FFG_ERR_VALIDATION, "bad handle / parity");
    RowBlockState& S = h->s;
    if (hi) *hi = S.w->op[2 * parity];
    if (lo) *lo = S.job.mode == kModeF32E ? S.w->op[2 * parity + 1] : nullptr;
    return FFG_OK;
}

int ffg_rowblock_layer(ffg_rowblock* h, int32_t layer, double* D_rows, void* stream) {
    NvtxRange nv("ffg_rowblock_layer");
    if (!h) return set_err(FFG_ERR_VALIDATION, "null handle");
    RowBlockState& S = h->s;
    if (layer != S.next_layer || layer >= S.model.n_layers)
        return set_err(FFG_ERR_VALIDATION, "row-block layer %d out of order (next %d of %d)", layer, S.next_layer,
                       S.model.n_layers);
    int cur = -1;
    CK(cudaGetDevice(&cur));
    if (cur != S.device) return set_err(FFG_ERR_VALIDATION, "row-block handle belongs to device %d", S.device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const bool last = layer + 1 == S.model.n_layers;
    S.job.D_dev = last ? D_rows : nullptr;
    int rc;
    if ((rc = enqueue_k2(*S.w, S.job, st, S.cx, layer, layer + 1))) return rc;
    if (last) {
        const int64_t d_rows = std::min<int64_t>((int64_t)S.r1 * kBM, S.n) - (int64_t)S.r0 * kBM;
        if ((rc = enqueue_k3(*S.w, S.job, st, S.cx, std::max<int64_t>(d_rows, 0)))) return rc;
    }
    ++S.next_layer;
    return FFG_OK;
}

int ffg_rowblock_end(ffg_rowblock* h, double* partial_stats, int32_t* status, ffg_provenance* prov,
                     void* stream) {
    NvtxRange nv("ffg_rowblock_end");
    if (!h) return set_err(FFG_ERR_VALIDATION, "null handle");
    RowBlockState& S = h->s;
    Workspace& w = *S.w;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    int rc = FFG_OK;
    if (S.next_layer != S.model.n_layers) {
        rc = set_err(FFG_ERR_VALIDATION, "row-block ended after %d of %d layers", S.next_layer, S.model.n_layers);
    } else {
        double stats[2], bounds[4];
        int st_code = 0, flags[2];
        uint32_t products = 0;
        cudaError_t e = cudaSuccess;
        e = e ? e : cudaMemcpyAsync(stats, w.stats, 16, cudaMemcpyDeviceToHost, st);
        e = e ? e : cudaMemcpyAsync(bounds, w.bounds_out, 32, cudaMemcpyDeviceToHost, st);
        e = e ? e : cudaMemcpyAsync(&st_code, w.status, 4, cudaMemcpyDeviceToHost, st);
        e = e ? e : cudaMemcpyAsync(flags, w.flags, 8, cudaMemcpyDeviceToHost, st);
        e = e ? e : cudaMemcpyAsync(&products, w.products, 4, cudaMemcpyDeviceToHost, st);
        e = e ? e : cudaStreamSynchronize(st);
        if (e != cudaSuccess) {
            rc = set_err(FFG_ERR_CUDA, "row-block readback: %s", cudaGetErrorString(e));
        } else {
            if (partial_stats) {
                partial_stats[0] = stats[0];
                partial_stats[1] = stats[1];
            }
            if (status) *status = st_code;
            if (prov)
                fill_prov(prov, bounds, &S.kT, S.mu, st_code, flags, &S.model, S.mode_api, (int)S.n, 0.0, products,
                          w.PT);
            if (st_code != FFG_OK) rc = status_error(st_code, bounds, flags);
        }
    }
    cudaStreamSynchronize(st);
    free_ws(S.w);
    delete S.w;
    delete h;
    return rc;
}

int32_t ffg_pair_table(int32_t nb, uint32_t* out, int32_t capacity) {
    if (nb < 1 || nb > 1023) return -1;
    const std::vector<uint32_t> t = pair_table(nb);
    if (out)
        for (int32_t i = 0; i < (int32_t)t.size() && i < capacity; ++i) out[i] = t[i];
    return (int32_t)t.size();
}

void ffg_release_workspaces(void) {
    std::lock_guard<std::mutex> lk(g_ws_mu);
    for (auto& kv : g_ws) {
        free_ws(kv.second);
        delete kv.second;
    }
    g_ws.clear();
}

}  // extern "C"
