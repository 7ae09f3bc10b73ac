// MLSP2 density-matrix kernels for sm_100a: shared definitions, K1 and K3.
//
//   K1  rescale_tiles        H (fp64) -> X0 = alpha H + gamma I (fp32), A1 = d0 X0,
//                            binary16 hi/lo split of X0 * 2^14 (or bf16 hi/lo), Gershgorin bounds.
//                            One HBM pass; HBM-bound.
//                            (gershgorin_kernel: bounds only, the spectral_bounds API)
//   K2  mlsp2_pair_kernel    all recursion layers on tcgen05 CTA pairs (k2_pair.cuh, epilogue in
//                            epilogue.cuh): (scalar_models.cpp:243-252 lifted to matrices;
//                            SPEC.md:359-377)
//   K3  finalize_stats       fixed-order reduction of the per-block partials, validity
//                            status per matrix.
//
// Data layout in HBM (per batch of B matrices, padded size np = ceil(n/128)*128):
//   A     fp32, tile-interleaved 128x128 blocks (xa_tile_base / xa_off), the blocks K2 touches
//   hi/lo binary16 (or bf16) [2 parities][B][np][np], full symmetric storage: layer l reads parity
//      l&1 (TMA operands, and the epilogue's X_l = (hi + lo) / scale), writes parity (l+1)&1.
//      There is no fp32 copy of X.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <cfloat>
#include <climits>

#include "ptx.cuh"

namespace ffg {

enum Mode : int { kModeF32E = 0, kModeF16 = 1, kModeBF16 = 2 };

constexpr int kBM = 128;            // tile rows   (UMMA M)
constexpr int kBN = 128;            // tile cols   (UMMA N)
constexpr int kBK = 64;             // K per stage (one 128-byte swizzle atom of 16-bit values)
constexpr int kUK = 16;             // K per UMMA instruction (kind::f16)
constexpr int kOpBytes = kBM * kBK * 2;  // one 128x64 16-bit operand tile = 16 KB
constexpr float kHalfScale = 16384.0f;   // global 2^14 pre-scale before the binary16 split
constexpr float kHalfMax = 65504.0f;
constexpr int kEpiWarps = 8;            // accumulator-drain / epilogue warps
constexpr int kEpiCols = kBN / (kEpiWarps / 4);  // tile columns per epilogue warp

template <int MODE>
struct ModeTraits;
template <>
struct ModeTraits<kModeF32E> {  // FP32-emulated: hi*hi + hi*lo + lo*hi (+ lo*lo in exact layers)
    static constexpr int kProducts = 3, kFmt = 0, kHasLo = 1;
    static constexpr float kScale = kHalfScale;
};
template <>
struct ModeTraits<kModeF16> {
    static constexpr int kProducts = 1, kFmt = 0, kHasLo = 0;
    static constexpr float kScale = kHalfScale;
};
template <>
struct ModeTraits<kModeBF16> {
    static constexpr int kProducts = 1, kFmt = 1, kHasLo = 0;
    static constexpr float kScale = 1.0f;
};

// 16-bit operand encodings (raw bits) -------------------------------------------------
#ifndef FFG_FIXED_SPLIT
#define FFG_FIXED_SPLIT 1  // FP32E exact layers: fixed-point hi instead of per-K16 drains (k2_pair.cuh)
#endif
#ifndef FFG_SR_LO
#define FFG_SR_LO 1  // fixed-point split: stochastic (hash) rounding of the lo part
#endif

// Stochastic rounding of the fixed-point split's lo part.  The residual x 2^14 - hi is exact in
// fp32; rounding it to nearest binary16 gives IDENTICAL errors to identical matrix entries (a
// tight-binding X_0 has one hopping value on every bond), and the recursion turns that correlated
// error into a systematic shift of the electron count (~1e-6 relative, measured; the first layers'
// errors are amplified ~beta0/4).  Rounding up with probability (distance to the lower binary16
// neighbour) / ulp instead -- the random draw a hash of the element's unordered index pair and the
// layer, so it is symmetric, deterministic and independent of batch position -- makes the error
// zero-mean and uncorrelated; the trace error drops ~10x.  Only the first
// `sr_layers` layers' operands (default 3: the layers whose errors the recursion amplifies most)
// are rounded this way.  Normal binary16 range: add 13 random bits below the binary16 precision of
// the fp32 pattern and truncate; residuals in the binary16 subnormal range (< 2^-38 in X units)
// then round to nearest in the conversion.
#ifndef FFG_SR_LAYERS
#define FFG_SR_LAYERS 3
#endif
__device__ __forceinline__ uint32_t sr_mix(uint32_t key, uint32_t layer) {
    uint32_t x = key + layer * 0x9E3779B9u;
    x *= 0x85EBCA77u;
    x ^= x >> 13;
    x *= 0xC2B2AE3Du;
    x ^= x >> 16;
    return x;
}
// key of the unordered pair {i, j} (indices < 65536)
__device__ __forceinline__ uint32_t sr_hash(uint32_t i, uint32_t j, uint32_t layer) {
    return sr_mix((min(i, j) << 16) | max(i, j), layer);
}
__device__ __forceinline__ float sr_f16_grid(float r, uint32_t h) {
    return __uint_as_float((__float_as_uint(r) + (h & 0x1FFFu)) & ~0x1FFFu);
}

template <int MODE>
__device__ __forceinline__ void split16(float x, uint16_t& hi, uint16_t& lo, bool fixed = false, bool sr = false,
                                        uint32_t h = 0) {
    // every mode writes lo: K2's epilogue rebuilds X_0 from hi + lo (there is no fp32 copy of X)
    if constexpr (MODE == kModeBF16) {
        const __nv_bfloat16 hb = __float2bfloat16_rn(x);
        hi = __bfloat16_as_ushort(hb);
        lo = __bfloat16_as_ushort(__float2bfloat16_rn(x - __bfloat162float(hb)));
    } else {
        const float xs = x * kHalfScale;
        const __half hh = __float2half_rn((MODE == kModeF32E && fixed) ? rintf(xs * 0.125f) * 8.0f : xs);
        hi = __half_as_ushort(hh);
        const float r = xs - __half2float(hh);
        lo = __half_as_ushort(__float2half_rn((MODE == kModeF32E && FFG_SR_LO && fixed && sr) ? sr_f16_grid(r, h) : r));
    }
}
template <int MODE>
__device__ __forceinline__ bool half_range_bad(float x) {
    if constexpr (MODE == kModeBF16) return false;
    return fabsf(x * kHalfScale) >= kHalfMax;
}

// X and A live in a tile-interleaved layout: tile (I,J) of matrix m is a contiguous
// 128x128 fp32 block stored as [32 column-quads][128 rows][4]; element (r, c) of the tile
// at ((c/4)*128 + r)*4 + c%4.  A warp whose lanes own consecutive rows then reads/writes
// 512 contiguous bytes per float4 access.
__host__ __device__ __forceinline__ size_t xa_tile_base(int m, int I, int J, int nb) {
    return (((size_t)m * nb + I) * nb + J) * (size_t)(kBM * kBN);
}
__host__ __device__ __forceinline__ uint32_t xa_off(int r, int c4) {  // float offset of quad c4, row r
    return ((uint32_t)c4 * kBM + (uint32_t)r) * 4u;
}
// ===================================================================================== K1
struct RescaleParams {
    const double* H;            // [B][n][n] row-major, exactly symmetric
    const double* alpha;        // [B] X0 = alpha_m H + gamma_m I
    const double* gamma;        // [B]
    double d0;                  // first accumulator weight: A1 = d0 X0
    float* A;                   // [B][np][np] tile-interleaved (xa_tile_base)
    uint16_t* hi;               // [B][np][np] parity 0, row-major
    uint16_t* lo;               // [B][np][np] parity 0
    unsigned long long* bounds; // [B][2] ordered keys of (eps_min, eps_max) before widening
    int* flags;                 // [B][2] first bad X_k index: [0] non-finite, [1] half range
    int n, np, mode;
    const uint8_t* xa_used;     // [nb][nb] blocks whose X/A K2 reads (null: all blocks)
    int fixed;                  // FP32E: fixed-point hi split of X0 (layer 0 is an exact layer)
    int sr;                     // ... with the stochastically rounded lo (sr_layers > 0)
};

// Gershgorin bounds only (the spectral_bounds entry): one warp per row, 8 rows per
// CTA, grid (ceil(n/8), B); per-row radius in a fixed-order warp tree, exact min/max through
// order-preserving integer atomics (deterministic).
__global__ void __launch_bounds__(256) gershgorin_kernel(const double* __restrict__ H, int n,
                                                         unsigned long long* bounds) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int m = blockIdx.y;
    const int i = blockIdx.x * 8 + warp;
    __shared__ double s_lo[8], s_hi[8];
    double rlo = DBL_MAX, rhi = -DBL_MAX;
    if (i < n) {
        const double* hrow = H + ((size_t)m * n + i) * n;
        double radius = 0.0, hii = 0.0;
        // the column order of K1's per-lane sums (128-column tiles, 4 consecutive columns per lane),
        // so both kernels produce bit-identical bounds
        for (int c0 = 4 * lane; c0 < n; c0 += 128)
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int j = c0 + e;
                const double h = j < n ? hrow[j] : 0.0;
                if (j == i) hii = h; else radius += fabs(h);
            }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            radius += __shfl_xor_sync(0xffffffffu, radius, o);
            hii += __shfl_xor_sync(0xffffffffu, hii, o);  // exactly one lane holds H_ii
        }
        rlo = hii - radius;
        rhi = hii + radius;
    }
    if (lane == 0) {
        s_lo[warp] = rlo;
        s_hi[warp] = rhi;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double lo = s_lo[0], hi = s_hi[0];
        for (int w = 1; w < 8; ++w) {
            lo = fmin(lo, s_lo[w]);
            hi = fmax(hi, s_hi[w]);
        }
        if (lo <= hi) {
            atomicMin(&bounds[2 * m + 0], ordered_key(lo));
            atomicMax(&bounds[2 * m + 1], ordered_key(hi));
        }
    }
}

// K1 (tiled): one CTA = 32 consecutive rows of one matrix (a quarter of block row I), all
// columns, 128-column tiles.  Each warp streams 4 rows per tile (coalesced double2 loads, 1 KB
// per row), writes the binary16 split row-major (256 B per row), and stages A1 = d0 X0 in shared
// memory so that the block-interleaved [c4][row][4] layout is written with 512-byte contiguous
// runs (the row-per-lane K1 above stored 2 KB apart per lane).  Blocks K2 never reads
// (xa_used) skip the A stores.  Gershgorin radii: fixed-order per-row warp trees.
// (template: WARPS warps = 4 WARPS rows per CTA.  Measured under ncu, 16 x N=1024: 8 warps / 32 rows
// 97 us (512 CTAs: 68 SMs with four, 80 with three), 4 warps 79 us, 2 warps / 8 rows 74 us (2048 CTAs,
// ~14 per SM, one wave))
#ifndef FFG_K1_WARPS
#define FFG_K1_WARPS 2
#endif
constexpr int kK1Warps = FFG_K1_WARPS;
constexpr int kK1Rows = 4 * kK1Warps;
constexpr int kK1Pad = 132;  // padded fp32 row stride of the staging tiles (conflict-free float4)
template <int WARPS>
__global__ void __launch_bounds__(32 * WARPS) rescale_tiles_kernel(const __grid_constant__ RescaleParams p) {
    constexpr int kRows = 4 * WARPS;
    __shared__ __align__(16) float sA[kRows * kK1Pad];
    __shared__ double s_lo[WARPS], s_hi[WARPS];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int m = blockIdx.y;
    const int n = p.n, np = p.np, nb = np / 128;
    const int row0 = blockIdx.x * kRows;            // first row of this CTA
    const int I = row0 / 128, q = (row0 & 127) / kRows;
    const double alpha = p.alpha[m], gamma = p.gamma[m];
    double radius[4] = {0.0, 0.0, 0.0, 0.0}, hii[4] = {0.0, 0.0, 0.0, 0.0};
    bool bad_nf = false, bad_hr = false;
    // the four rows of tile J (this lane's 4 columns); tile J+1 is requested before tile J is
    // processed, so the loads overlap the stores and barriers of the previous tile
    auto load_tile = [&](int J, double (&hk)[4][4]) {
        const int c0 = J * 128 + 4 * lane;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int i = row0 + warp * 4 + k;
#pragma unroll
            for (int e = 0; e < 4; ++e) hk[k][e] = 0.0;
            if (i < n) {
                const double* hrow = p.H + ((size_t)m * n + i) * n;
                if ((n & 3) == 0 && c0 + 3 < n) {
                    const double2 v0 = __ldcs(reinterpret_cast<const double2*>(hrow + c0));
                    const double2 v1 = __ldcs(reinterpret_cast<const double2*>(hrow + c0 + 2));
                    hk[k][0] = v0.x; hk[k][1] = v0.y; hk[k][2] = v1.x; hk[k][3] = v1.y;
                } else {
#pragma unroll
                    for (int e = 0; e < 4; ++e) hk[k][e] = (c0 + e < n) ? hrow[c0 + e] : 0.0;
                }
            }
        }
    };
    double hnext[4][4];
    load_tile(0, hnext);
    for (int J = 0; J < nb; ++J) {
        const int c0 = J * 128 + 4 * lane;           // this lane's 4 columns
        double hk[4][4];
#pragma unroll
        for (int k = 0; k < 4; ++k)
#pragma unroll
            for (int e = 0; e < 4; ++e) hk[k][e] = hnext[k][e];
        if (J + 1 < nb) load_tile(J + 1, hnext);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int rl = warp * 4 + k;              // local row 0..kRows-1
            const int i = row0 + rl;
            const double* h = hk[k];
            float x[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int j = c0 + e;
                if (j == i) hii[k] = h[e]; else radius[k] += fabs(h[e]);
                double v = alpha * h[e];
                if (j == i && i < n) v += gamma;
                x[e] = (float)v;
                bad_nf |= !isfinite(x[e]);
            }
            {
                float a[4];
#pragma unroll
                for (int e = 0; e < 4; ++e) a[e] = (float)(p.d0 * (double)x[e]);
                *reinterpret_cast<float4*>(&sA[rl * kK1Pad + 4 * lane]) = make_float4(a[0], a[1], a[2], a[3]);
                uint16_t hb[4], lb[4];
                if (p.mode == kModeBF16) {
#pragma unroll
                    for (int e = 0; e < 4; ++e) split16<kModeBF16>(x[e], hb[e], lb[e]);
                } else if (p.mode == kModeF16) {
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        split16<kModeF16>(x[e], hb[e], lb[e]);
                        bad_hr |= half_range_bad<kModeF16>(x[e]);
                    }
                } else {
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        split16<kModeF32E>(x[e], hb[e], lb[e], p.fixed != 0, p.sr != 0,
                                           p.sr ? sr_hash((uint32_t)i, (uint32_t)(c0 + e), 0u) : 0u);
                        bad_hr |= half_range_bad<kModeF32E>(x[e]);
                    }
                }
                const size_t orow = ((size_t)m * np + row0 + rl) * np;
                uint2 hv, lv;
                hv.x = hb[0] | ((uint32_t)hb[1] << 16); hv.y = hb[2] | ((uint32_t)hb[3] << 16);
                lv.x = lb[0] | ((uint32_t)lb[1] << 16); lv.y = lb[2] | ((uint32_t)lb[3] << 16);
                *reinterpret_cast<uint2*>(p.hi + orow + c0) = hv;
                *reinterpret_cast<uint2*>(p.lo + orow + c0) = lv;
            }
        }
        if (!p.xa_used || p.xa_used[I * nb + J]) {
            __syncthreads();
            // block (I, J), rows q kRows .. +kRows-1: [c4][row][4]; thread t -> c4 = t / (kRows/4),
            // rows 4 (t % (kRows/4)) .. +3
            const size_t tb = xa_tile_base(m, I, J, nb);
            const int c4 = threadIdx.x / (kRows / 4), r4 = (threadIdx.x % (kRows / 4)) * 4;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int rl = r4 + k;
                const float4 av = *reinterpret_cast<const float4*>(&sA[rl * kK1Pad + 4 * c4]);
                *reinterpret_cast<float4*>(p.A + tb + xa_off(q * kRows + rl, c4)) = av;
            }
        }
        __syncthreads();
    }
    // per-row Gershgorin intervals (fixed-order warp trees), CTA min/max, ordered-key atomics
    double rlo = DBL_MAX, rhi = -DBL_MAX;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        double r = radius[k], d = hii[k];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            r += __shfl_xor_sync(0xffffffffu, r, o);
            d += __shfl_xor_sync(0xffffffffu, d, o);  // exactly one lane holds H_ii
        }
        if (row0 + warp * 4 + k < n) {
            rlo = fmin(rlo, d - r);
            rhi = fmax(rhi, d + r);
        }
    }
    if (lane == 0) {
        s_lo[warp] = rlo;
        s_hi[warp] = rhi;
    }
    const bool any_nf = __any_sync(0xffffffffu, bad_nf);
    const bool any_hr = __any_sync(0xffffffffu, bad_hr);
    if (lane == 0 && any_nf) atomicMin(&p.flags[2 * m + 0], 0);
    if (lane == 0 && any_hr) atomicMin(&p.flags[2 * m + 1], 0);
    __syncthreads();
    if (threadIdx.x == 0) {
        double lo = s_lo[0], hi = s_hi[0];
        for (int w = 1; w < WARPS; ++w) {
            lo = fmin(lo, s_lo[w]);
            hi = fmax(hi, s_hi[w]);
        }
        if (lo <= hi) {
            atomicMin(&p.bounds[2 * m + 0], ordered_key(lo));
            atomicMax(&p.bounds[2 * m + 1], ordered_key(hi));
        }
    }
}

// ===================================================================================== K2 shared
// byte offset of 16-byte chunk c of row r in a tile of 64-byte rows, 64B swizzle
__device__ __forceinline__ uint32_t sw64(uint32_t r, uint32_t c) {
    return r * 64u + ((c ^ ((r >> 1) & 3u)) << 4);
}

constexpr int kEpiWarps2 = 8;                                       // epilogue warps
constexpr int kPieceBytes = 32 * 64;                                // 32x32 binary16 piece

// Region of validity of each matrix (Eq. 41 in the model's un-flipped frame,
// SURVEY.md 0.4): x = mu0 + (beta/beta0)(eps - mu) must lie in [0, 1] at both Gershgorin bounds,
// widened by 1e-12 W.  K2 skips matrices that fail it (rescale_to_model fails before
// apply_model) and K3 reports the status; both evaluate this one function.
struct RegionCheck {
    const unsigned long long* bounds;  // [B][2] ordered keys of (eps_min, eps_max) from K1
    const double* scale;               // [B] beta/beta0, or null: no check (apply_model, mixed_square)
    const double* mu;                  // [B]
    double mu0;
};
__device__ __forceinline__ void widened_bounds(const RegionCheck& rc, int m, double& lo, double& hi) {
    lo = key_to_double(rc.bounds[2 * m + 0]);
    hi = key_to_double(rc.bounds[2 * m + 1]);
    const double w = 1e-12 * (hi - lo);
    lo -= w;
    hi += w;
}
__device__ __forceinline__ bool matrix_in_region(const RegionCheck& rc, int m, double* xmin = nullptr,
                                                 double* xmax = nullptr) {
    if (!rc.scale) return true;
    double lo, hi;
    widened_bounds(rc, m, lo, hi);
    const double x0 = rc.mu0 + rc.scale[m] * (lo - rc.mu[m]);
    const double x1 = rc.mu0 + rc.scale[m] * (hi - rc.mu[m]);
    if (xmin) *xmin = x0;
    if (xmax) *xmax = x1;
    return x0 >= 0.0 && x1 <= 1.0;  // (false for NaN)
}

struct FinalizeParams {
    const double2* partials;          // [B][T]
    const int* flags;                 // [B][2]
    RegionCheck region;               // bounds + validity inputs (scale null: no check)
    double* D;                        // [B][d_elems] or null: an out-of-region matrix's D is set to NaN
    int64_t d_elems;                  // elements of D per matrix (n * n, or a row-block rank's rows * n)
    int T, B;
    double* stats;                    // [B][2] (Tr D, Tr D^2)
    double* bounds_out;               // [B][4] (eps_min, eps_max, x_min, x_max) widened
    int* status;                      // [B]
};

// status codes mirror ffg_status (include/fermiforge/ffg.h)
__global__ void __launch_bounds__(256) finalize_stats_kernel(const __grid_constant__ FinalizeParams p) {
    const int m = blockIdx.x;
    if (p.D && !matrix_in_region(p.region, m)) {
        // K2 skipped this matrix (no recursion outside the region): its D is NaN,
        // never a stale or plausible-looking matrix in the caller's buffer
        double* Dm = p.D + (size_t)m * p.d_elems;
        for (int64_t i = threadIdx.x; i < p.d_elems; i += blockDim.x) Dm[i] = __longlong_as_double(0x7ff8000000000000ll);
    }
    __shared__ double s0[256], s1[256];
    double a = 0.0, b = 0.0;
    for (int t = threadIdx.x; t < p.T; t += 256) {
        const double2 v = p.partials[(size_t)m * p.T + t];
        a += v.x;
        b += v.y;
    }
    s0[threadIdx.x] = a;
    s1[threadIdx.x] = b;
    __syncthreads();
    for (int w = 128; w > 0; w >>= 1) {
        if (threadIdx.x < w) {
            s0[threadIdx.x] += s0[threadIdx.x + w];
            s1[threadIdx.x] += s1[threadIdx.x + w];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        p.stats[2 * m + 0] = s0[0];
        p.stats[2 * m + 1] = s1[0];
        double lo, hi;
        widened_bounds(p.region, m, lo, hi);
        int st = 0;
        double xmin = 0.0, xmax = 0.0;
        if (!matrix_in_region(p.region, m, &xmin, &xmax)) st = 2;  // FFG_ERR_OUT_OF_REGION
        // the earlier event wins (a binary16 split overflow at X_k precedes a non-finite X_{k+1});
        // a non-finite X_k also overflows its split, so ties report divergence
        const int nf = p.flags[2 * m + 0], hr = p.flags[2 * m + 1];
        if (st == 0 && nf != INT_MAX && nf <= hr) st = 3;       // FFG_ERR_DIVERGED
        if (st == 0 && hr != INT_MAX) st = 4;                    // FFG_ERR_HALF_RANGE
        p.status[m] = st;
        p.bounds_out[4 * m + 0] = lo;
        p.bounds_out[4 * m + 1] = hi;
        p.bounds_out[4 * m + 2] = xmin;
        p.bounds_out[4 * m + 3] = xmax;
    }
}

}  // namespace ffg
