// MLSP2 density-matrix kernels for sm_100a.
//
//   K1  rescale_gershgorin   H (fp64) -> X0 = alpha H + gamma I (fp32 master), A1 = d0 X0,
//                            binary16 hi/lo split of X0 * 2^14 (or bf16), Gershgorin bounds.
//                            One HBM pass; HBM-bound.
//   K2  mlsp2_layer<MODE>    one recursion layer on the tcgen05 tensor cores:
//                            Y = X^2 from TMA-fed SMEM tiles into a TMEM accumulator;
//                            epilogue fuses X' = aY + bX + cI, A += d' X', the split of
//                            X' for the next layer (direct + mirrored store), the
//                            non-finite / half-range flags and, on the last layer,
//                            D = A + X_L plus the per-tile (Tr D, sum D^2) partials.
//                            (scalar_models.cpp:243-252 lifted to matrices)
//   K3  finalize_stats       fixed-order reduction of the per-tile partials, validity
//                            status per matrix.
//
// Data layout in HBM (per batch of B matrices, padded size np = ceil(n/128)*128):
//   X  fp32 [B][np][np]   only upper-triangular tiles are live after K1
//   A  fp32 [B][np][np]   idem
//   hi/lo binary16 (or bf16 hi) [2 parities][B][np][np], full symmetric storage:
//      layer l reads parity l&1 through TMA, writes parity (l+1)&1.
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
constexpr int kLayerThreads = 64 + kEpiWarps * 32;

template <int MODE>
struct ModeTraits;
template <>
#ifndef FFG_F32E_STAGES
#define FFG_F32E_STAGES 3
#endif
struct ModeTraits<kModeF32E> {  // FP32-emulated: hi*hi + hi*lo + lo*hi, one accumulator
    static constexpr int kProducts = 3, kFmt = 0, kHasLo = 1, kStages = FFG_F32E_STAGES;
    static constexpr float kScale = kHalfScale;
};
template <>
struct ModeTraits<kModeF16> {
    static constexpr int kProducts = 1, kFmt = 0, kHasLo = 0, kStages = 6;
    static constexpr float kScale = kHalfScale;
};
template <>
struct ModeTraits<kModeBF16> {
    static constexpr int kProducts = 1, kFmt = 1, kHasLo = 0, kStages = 6;
    static constexpr float kScale = 1.0f;
};

template <int MODE>
constexpr int stage_bytes() {
    return (ModeTraits<MODE>::kHasLo ? 4 : 2) * kOpBytes;
}
template <int MODE>
constexpr int layer_pipe_bytes() {  // pipeline stages; reused as epilogue staging (192 KB)
    return ModeTraits<MODE>::kStages * stage_bytes<MODE>() > 192 * 1024
               ? ModeTraits<MODE>::kStages * stage_bytes<MODE>()
               : 192 * 1024;
}
template <int MODE>
constexpr int layer_smem_bytes() {
    return layer_pipe_bytes<MODE>() + 1024 /*barriers, scratch*/ + 1024 /*alignment slack*/;
}

// 16-bit operand encodings (raw bits) -------------------------------------------------
#ifndef FFG_FIXED_SPLIT
#define FFG_FIXED_SPLIT 1  // FP32E exact layers: fixed-point hi instead of per-K16 drains (k2_pair.cuh)
#endif
template <int MODE>
__device__ __forceinline__ void split16(float x, uint16_t& hi, uint16_t& lo, bool fixed = false) {
    if constexpr (MODE == kModeBF16) {
        hi = __bfloat16_as_ushort(__float2bfloat16_rn(x));
        lo = 0;
    } else {
        const float xs = x * kHalfScale;
        const __half h = __float2half_rn((MODE == kModeF32E && fixed) ? rintf(xs * 0.125f) * 8.0f : xs);
        hi = __half_as_ushort(h);
        if constexpr (MODE == kModeF32E) {
            lo = __half_as_ushort(__float2half_rn(xs - __half2float(h)));
        } else {
            lo = 0;
        }
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
    float* X;                   // [B][np][np] tile-interleaved (xa_tile_base)
    float* A;                   // [B][np][np] tile-interleaved
    uint16_t* hi;               // [B][np][np] parity 0, row-major
    uint16_t* lo;               // [B][np][np] parity 0 (F32E only)
    unsigned long long* bounds; // [B][2] ordered keys of (eps_min, eps_max) before widening
    int* flags;                 // [B][2] first bad X_k index: [0] non-finite, [1] half range
    int n, np, mode, write_operands;
    const uint8_t* xa_used;     // [nb][nb] blocks whose X/A K2 reads (null: all blocks)
    int fixed;                  // FP32E: fixed-point hi split of X0 (layer 0 is an exact layer)
};

// One warp per row; 8 rows per CTA; grid (np/8, B).
__global__ void __launch_bounds__(256) rescale_gershgorin_kernel(const __grid_constant__ RescaleParams p) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int m = blockIdx.y;
    const int i = blockIdx.x * 8 + warp;
    const int n = p.n, np = p.np;
    __shared__ double s_lo[8], s_hi[8];
    double rlo = DBL_MAX, rhi = -DBL_MAX;
    bool bad_nf = false, bad_hr = false;
    if (i < np) {
        const double alpha = p.alpha[m], gamma = p.gamma[m];
        const size_t orow = ((size_t)m * np + i) * np;
        const double* hrow = p.H + ((size_t)m * n + (i < n ? i : 0)) * n;
        double radius = 0.0, hii = 0.0;
        const bool vec = ((n & 3) == 0);
        // columns in groups of 4 per lane: j = 4*lane + 128*t
        for (int j0 = 4 * lane; j0 < np; j0 += 128) {
            double h[4];
            if (i < n && vec && j0 + 3 < n) {
                const double2 v0 = *reinterpret_cast<const double2*>(hrow + j0);
                const double2 v1 = *reinterpret_cast<const double2*>(hrow + j0 + 2);
                h[0] = v0.x; h[1] = v0.y; h[2] = v1.x; h[3] = v1.y;
            } else {
#pragma unroll
                for (int e = 0; e < 4; ++e) h[e] = (i < n && j0 + e < n) ? hrow[j0 + e] : 0.0;
            }
            float x[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int j = j0 + e;
                if (j == i) {
                    hii = h[e];
                } else {
                    radius += fabs(h[e]);
                }
                double v = alpha * h[e];
                if (j == i && i < n) v += gamma;
                x[e] = (float)v;
                bad_nf |= !isfinite(x[e]);
            }
            if (p.write_operands) {
                // X / A: tile-interleaved layout (see xa_tile_base); hi / lo: row-major
                const size_t xo = ((((size_t)m * (np / 128) + i / 128) * (np / 128) + j0 / 128) * 16384) +
                                  ((size_t)((j0 & 127) >> 2) * 128 + (i & 127)) * 4;
                *reinterpret_cast<float4*>(p.X + xo) = make_float4(x[0], x[1], x[2], x[3]);
                const float d0 = (float)p.d0;
                float a[4];
#pragma unroll
                for (int e = 0; e < 4; ++e) a[e] = (float)(p.d0 * (double)x[e]);
                (void)d0;
                *reinterpret_cast<float4*>(p.A + xo) = make_float4(a[0], a[1], a[2], a[3]);
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
                        split16<kModeF32E>(x[e], hb[e], lb[e], p.fixed != 0);
                        bad_hr |= half_range_bad<kModeF32E>(x[e]);
                    }
                }
                uint2 hv, lv;
                hv.x = hb[0] | ((uint32_t)hb[1] << 16); hv.y = hb[2] | ((uint32_t)hb[3] << 16);
                lv.x = lb[0] | ((uint32_t)lb[1] << 16); lv.y = lb[2] | ((uint32_t)lb[3] << 16);
                *reinterpret_cast<uint2*>(p.hi + orow + j0) = hv;
                if (p.mode == kModeF32E) *reinterpret_cast<uint2*>(p.lo + orow + j0) = lv;
            }
        }
        // fixed-order warp tree (deterministic for a given n)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            radius += __shfl_xor_sync(0xffffffffu, radius, o);
            hii += __shfl_xor_sync(0xffffffffu, hii, o);  // exactly one lane holds H_ii
        }
        if (i < n) {
            rlo = hii - radius;
            rhi = hii + radius;
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
        for (int w = 1; w < 8; ++w) {
            lo = fmin(lo, s_lo[w]);
            hi = fmax(hi, s_hi[w]);
        }
        if (lo <= hi) {
            atomicMin(&p.bounds[2 * m + 0], ordered_key(lo));
            atomicMax(&p.bounds[2 * m + 1], ordered_key(hi));
        }
    }
}

// K1 (tiled): one CTA = 32 consecutive rows of one matrix (a quarter of block row I), all
// columns, 128-column tiles.  Each warp streams 4 rows per tile (coalesced double2 loads, 1 KB
// per row), writes the binary16 split row-major (256 B per row), and stages X0 / A1 in shared
// memory so that the block-interleaved [c4][row][4] layout is written with 512-byte contiguous
// runs (the row-per-lane K1 above stored 2 KB apart per lane).  Blocks K2 never reads
// (xa_used) skip the X/A stores.  Gershgorin radii: fixed-order per-row warp trees.
constexpr int kK1Rows = 32;
constexpr int kK1Pad = 132;  // padded fp32 row stride of the staging tiles (conflict-free float4)
__global__ void __launch_bounds__(256) rescale_tiles_kernel(const __grid_constant__ RescaleParams p) {
    __shared__ __align__(16) float sX[kK1Rows * kK1Pad];
    __shared__ __align__(16) float sA[kK1Rows * kK1Pad];
    __shared__ double s_lo[8], s_hi[8];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int m = blockIdx.y;
    const int n = p.n, np = p.np, nb = np / 128;
    const int row0 = blockIdx.x * kK1Rows;          // first row of this CTA
    const int I = row0 / 128, q = (row0 & 127) / kK1Rows;
    const double alpha = p.alpha[m], gamma = p.gamma[m];
    const float d0f = (float)p.d0;
    (void)d0f;
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
            const int rl = warp * 4 + k;              // local row 0..31
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
            if (p.write_operands) {
                float a[4];
#pragma unroll
                for (int e = 0; e < 4; ++e) a[e] = (float)(p.d0 * (double)x[e]);
                *reinterpret_cast<float4*>(&sX[rl * kK1Pad + 4 * lane]) = make_float4(x[0], x[1], x[2], x[3]);
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
                        split16<kModeF32E>(x[e], hb[e], lb[e], p.fixed != 0);
                        bad_hr |= half_range_bad<kModeF32E>(x[e]);
                    }
                }
                const size_t orow = ((size_t)m * np + row0 + rl) * np;
                uint2 hv, lv;
                hv.x = hb[0] | ((uint32_t)hb[1] << 16); hv.y = hb[2] | ((uint32_t)hb[3] << 16);
                lv.x = lb[0] | ((uint32_t)lb[1] << 16); lv.y = lb[2] | ((uint32_t)lb[3] << 16);
                *reinterpret_cast<uint2*>(p.hi + orow + c0) = hv;
                if (p.mode == kModeF32E) *reinterpret_cast<uint2*>(p.lo + orow + c0) = lv;
            }
        }
        if (p.write_operands && (!p.xa_used || p.xa_used[I * nb + J])) {
            __syncthreads();
            // block (I, J), rows 32q .. 32q+31: [c4][row][4]; thread t -> c4 = t / 8, rows 4(t%8)..+3
            const size_t tb = xa_tile_base(m, I, J, nb);
            const int c4 = threadIdx.x >> 3, r4 = (threadIdx.x & 7) * 4;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int rl = r4 + k;
                const float4 xv = *reinterpret_cast<const float4*>(&sX[rl * kK1Pad + 4 * c4]);
                const float4 av = *reinterpret_cast<const float4*>(&sA[rl * kK1Pad + 4 * c4]);
                const size_t o = tb + xa_off(q * kK1Rows + rl, c4);
                *reinterpret_cast<float4*>(p.X + o) = xv;
                *reinterpret_cast<float4*>(p.A + o) = av;
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
        for (int w = 1; w < 8; ++w) {
            lo = fmin(lo, s_lo[w]);
            hi = fmax(hi, s_hi[w]);
        }
        if (lo <= hi) {
            atomicMin(&p.bounds[2 * m + 0], ordered_key(lo));
            atomicMax(&p.bounds[2 * m + 1], ordered_key(hi));
        }
    }
}

// ===================================================================================== K2
struct LayerParams {
    float* X;             // [B][np][np] in/out (upper tiles)
    float* A;             // [B][np][np] in/out (upper tiles)
    uint16_t* hi_dst;     // [B][np][np] next parity (unused on the last layer)
    uint16_t* lo_dst;
    double* D;            // last layer: [B][n][n] row-major fp64 output (full storage)
    double2* partials;    // last layer: [B][T] per-tile (sum diag, sum sq)
    int* flags;           // [B][2]
    double a, b, c, d_next;
    int n, np, nb, T;     // nb = np/128 tile rows, T = nb(nb+1)/2 upper tiles
    int layer, last;      // layer index l (produces X_{l+1})
    int n_layers;
    int exact_layers;     // layers draining hi*hi after every MMA (the rest: per K-block)
    int B;                // matrices in this launch
    int dbg;              // measurement only: 1 = skip epilogue work, 2 = skip loads/MMAs/drain
};

__device__ __forceinline__ void decode_upper_tile(int t, int nb, int& I, int& J) {
    int I_ = 0;
    int rowlen = nb;
    while (t >= rowlen) {
        t -= rowlen;
        ++I_;
        --rowlen;
    }
    I = I_;
    J = I_ + t;
}

struct LayerMaps {
    CUtensorMap hi, lo;      // operand source (parity l&1): box 64 x 128, SW128
    CUtensorMap hip, lop;    // destination (parity (l+1)&1): 32 x 32 pieces, SW64
};

// byte offset of 16-byte chunk c of row r in a tile of 64-byte rows, 64B swizzle
__device__ __forceinline__ uint32_t sw64(uint32_t r, uint32_t c) {
    return r * 64u + ((c ^ ((r >> 1) & 3u)) << 4);
}

constexpr int kEpiWarps2 = 8;                                       // epilogue warps
constexpr int kPersistThreads = 128 + kEpiWarps * 32 + kEpiWarps2 * 32;  // 640
constexpr int kPipeStages = 2;                                      // 2 x 64 KB operand stages
constexpr int kStageBytes = 4 * kOpBytes;
constexpr int kStagingOff = kPipeStages * kStageBytes;              // 128 KB
constexpr int kPieceBytes = 32 * 64;                                // 32x32 binary16 piece
constexpr int kStagingBytes = kEpiWarps2 * 4 * kPieceBytes;         // 64 KB
constexpr int kPersistSmem = kStagingOff + kStagingBytes + 1024 + 1024;
// setmaxnreg budgets: they can only redistribute the launch allocation (640 threads x 96)
constexpr int kRegsCtl = 32, kRegsDrain = 104, kRegsEpi = 120;
static_assert(128 * kRegsCtl + kEpiWarps * 32 * kRegsDrain + kEpiWarps2 * 32 * kRegsEpi <= 640 * 96,
              "setmaxnreg targets exceed the CTA register allocation (would deadlock)");

// Persistent, warp-specialised MLSP2 layer.  One CTA per SM walks the (matrix, upper tile)
// list; per tile the tensor core squares a 128x128 block while the epilogue of the previous
// tile runs:
//   warp 0        TMA producer of the hi/lo operand panels (2 x 64 KB stages)
//   warp 1        TMEM allocator + UMMA issuer            (warps 2,3 idle; warpgroup 0)
//   warps 4-11    drain the hi*hi TMEM ring into fp32 registers (round-to-nearest adds) and
//                 form Y = (hi*hi + cross terms)/scale^2 in the tile's TMEM accumulator
//   warps 12-19   epilogue: X' = aY + bX + cI, A += d'X', binary16 split.  X/A are read
//                 and written in place (coalesced, tile-interleaved layout); the split
//                 leaves as 32x32 direct and mirrored pieces through per-warp SMEM staging
//                 and TMA stores.  Last layer: D = A + X_L and the statistics.
// TMEM: [0,256) hi*hi ring (2 x 128), [256,384) / [384,512) per-tile accumulators (cross
// terms, then Y), double-buffered across tiles.
//
// Accumulation precision: tcgen05 FP32 accumulation truncates inside every MMA.  Cross
// terms (2^-11 smaller) have their own accumulator; hi*hi is drained after every MMA for the
// first `exact_layers` layers (their errors are amplified by all later layers, up to
// beta0/4) and after every K-block afterwards ("accumulation precision").
template <int MODE>
__global__ void __launch_bounds__(kPersistThreads, 1)
    mlsp2_layer_persistent(const __grid_constant__ LayerMaps tm, const __grid_constant__ LayerParams p) {
    using Tr = ModeTraits<MODE>;
    constexpr bool kDrain = Tr::kProducts == 3;
    constexpr int NHB = 2;
    constexpr uint32_t kAcc0 = 256;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                               ~uintptr_t(1023));
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kStagingOff + kStagingBytes);
    uint64_t* full = bars;                // [2]
    uint64_t* empty = bars + 2;           // [2]
    uint64_t* hh_full = bars + 4;         // [2]
    uint64_t* hh_empty = bars + 6;        // [2]
    uint64_t* acc_full = bars + 8;        // [2]
    uint64_t* y_full = bars + 10;         // [2]
    uint64_t* acc_empty = bars + 12;      // [2]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 14);
    double* red = reinterpret_cast<double*>(bars + 16);  // [8][2]

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int total = p.B * p.T;
    const int nk = p.np / kBK;
    const int drain_dr = (p.layer < p.exact_layers) ? 1 : 4;  // K16 MMAs per hi*hi fill

    if (threadIdx.x == 0) {
        for (int i = 0; i < 2; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], 1);
            mbar_init(&hh_full[i], 1);
            mbar_init(&hh_empty[i], kEpiWarps);
            mbar_init(&acc_full[i], 1);
            mbar_init(&y_full[i], kEpiWarps);
            mbar_init(&acc_empty[i], kEpiWarps2);
        }
        fence_barrier_init();
        tma_prefetch_desc(&tm.hi);
        if (Tr::kHasLo) tma_prefetch_desc(&tm.lo);
    }
    if (warp == 1) tmem_alloc(tmem_slot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp < 4) {
        asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(kRegsCtl) : "memory");
        if (warp == 0 && lane == 0) {
            // ============================================= TMA producer
            int it = 0;
            for (int tile = blockIdx.x; tile < total; tile += gridDim.x) {
                const int m = tile / p.T;
                int I, J;
                decode_upper_tile(tile - m * p.T, p.nb, I, J);
                const bool diag = I == J;
                const int rowI = m * p.np + I * kBM, rowJ = m * p.np + J * kBN;
                if (!(p.dbg & 1)) {  // warm L2 with this tile's X / A for the epilogue
                    const size_t tb = xa_tile_base(m, I, J, p.nb);
                    tma_prefetch_l2_bulk(p.X + tb, kBM * kBN * 4);
                    tma_prefetch_l2_bulk(p.A + tb, kBM * kBN * 4);
                }
                const uint32_t bytes = (diag ? (Tr::kHasLo ? 2 : 1) : (Tr::kHasLo ? 4 : 2)) * kOpBytes;
                for (int kb = 0; kb < ((p.dbg & 2) ? 0 : nk); ++kb, ++it) {
                    const int s = it & 1;
                    mbar_wait(&empty[s], ((it >> 1) & 1) ^ 1);
                    mbar_expect_tx(&full[s], bytes);
                    uint8_t* st = smem + s * kStageBytes;
                    tma_load_2d(st, &tm.hi, &full[s], kb * kBK, rowI);
                    if (Tr::kHasLo) tma_load_2d(st + kOpBytes, &tm.lo, &full[s], kb * kBK, rowI);
                    if (!diag) {
                        tma_load_2d(st + 2 * kOpBytes, &tm.hi, &full[s], kb * kBK, rowJ);
                        if (Tr::kHasLo) tma_load_2d(st + 3 * kOpBytes, &tm.lo, &full[s], kb * kBK, rowJ);
                    }
                }
            }
        } else if (warp == 1 && lane == 0) {
            // ============================================= UMMA issuer
            constexpr uint32_t idesc = umma_idesc_f16(Tr::kFmt, kBM, kBN);
            int it = 0, g = 0, u = 0;
            for (int tile = blockIdx.x; tile < total; tile += gridDim.x, ++u) {
                const int m = tile / p.T;
                int I, J;
                decode_upper_tile(tile - m * p.T, p.nb, I, J);
                const bool diag = I == J;
                const int ab = u & 1;
                const uint32_t t_acc = tmem + kAcc0 + ab * 128;
                mbar_wait(&acc_empty[ab], ((u >> 1) & 1) ^ 1);  // epilogue of tile u-2 read Y
                tc_fence_after();
                for (int kb = 0; kb < ((p.dbg & 2) ? 0 : nk); ++kb, ++it) {
                    const int s = it & 1;
                    mbar_wait(&full[s], (it >> 1) & 1);
                    tc_fence_after();
                    const uint32_t base = smem_u32(smem + s * kStageBytes);
                    const uint32_t a_hi = base, a_lo = base + kOpBytes;
                    const uint32_t ob = diag ? 0 : 2 * kOpBytes;
                    const uint32_t b_hi = base + ob, b_lo = base + ob + kOpBytes;
#pragma unroll
                    for (int kk = 0; kk < kBK / kUK; ++kk) {
                        const uint32_t koff = kk * kUK * 2;
                        if (!kDrain) {
                            umma_f16(t_acc, umma_desc_sw128(a_hi + koff), umma_desc_sw128(b_hi + koff),
                                     idesc, (kb | kk) != 0);
                        } else {
                            const int hb = g % NHB;
                            if (kk % drain_dr == 0) {
                                mbar_wait(&hh_empty[hb], ((g / NHB) & 1) ^ 1);
                                tc_fence_after();
                            }
                            umma_f16(tmem + hb * 128, umma_desc_sw128(a_hi + koff),
                                     umma_desc_sw128(b_hi + koff), idesc, (kk % drain_dr) != 0);
                            if (kk % drain_dr == drain_dr - 1) {
                                umma_commit(&hh_full[hb]);
                                ++g;
                            }
                            umma_f16(t_acc, umma_desc_sw128(a_hi + koff), umma_desc_sw128(b_lo + koff),
                                     idesc, (kb | kk) != 0);
                            umma_f16(t_acc, umma_desc_sw128(a_lo + koff), umma_desc_sw128(b_hi + koff),
                                     idesc, 1u);
                        }
                    }
                    umma_commit(&empty[s]);
                }
                umma_commit(&acc_full[ab]);
            }
        }
        __syncwarp();
    } else if (warp < 4 + kEpiWarps) {
        asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(kRegsDrain) : "memory");
        // ================================================= hi*hi drain -> Y
        const int q = warp & 3;
        const int hc = (warp - 4) >> 2;
        const uint32_t tlane = tmem + ((uint32_t)(q * 32) << 16);
        const float inv_s2 = 1.0f / (Tr::kScale * Tr::kScale);
        int g = 0, u = 0;
        for (int tile = blockIdx.x; tile < total; tile += gridDim.x, ++u) {
            const int ab = u & 1;
            float yacc[kEpiCols];
#pragma unroll
            for (int e = 0; e < kEpiCols; ++e) yacc[e] = 0.0f;
            if (kDrain && !(p.dbg & 2)) {
                const int fills = nk * (kBK / kUK) / drain_dr;
#pragma unroll 1
                for (int f = 0; f < fills; ++f, ++g) {
                    const int hb = g % NHB;
                    mbar_wait(&hh_full[hb], (g / NHB) & 1);
                    tc_fence_after();
#pragma unroll
                    for (int ch = 0; ch < 2; ++ch) {
                        uint32_t v[32];
                        tmem_ld_32x32b_x32(tlane + hb * 128 + hc * kEpiCols + ch * 32, v);
                        tmem_ld_wait();
                        if (ch == 1) {
                            tc_fence_before();
                            __syncwarp();
                            if (lane == 0) mbar_arrive(&hh_empty[hb]);
                        }
#pragma unroll
                        for (int e = 0; e < 32; e += 2) {
                            const float2 acc = add_f32x2(
                                make_float2(yacc[32 * ch + e], yacc[32 * ch + e + 1]),
                                make_float2(__uint_as_float(v[e]), __uint_as_float(v[e + 1])));
                            yacc[32 * ch + e] = acc.x;
                            yacc[32 * ch + e + 1] = acc.y;
                        }
                    }
                }
            }
            mbar_wait(&acc_full[ab], (u >> 1) & 1);
            tc_fence_after();
#pragma unroll
            for (int ch = 0; ch < kEpiCols / 32; ++ch) {
                const uint32_t ta = tlane + kAcc0 + ab * 128 + hc * kEpiCols + ch * 32;
                uint32_t v[32];
                tmem_ld_32x32b_x32(ta, v);
                tmem_ld_wait();
#pragma unroll
                for (int e = 0; e < 32; ++e) {
                    const float y = kDrain ? yacc[ch * 32 + e] + __uint_as_float(v[e]) : __uint_as_float(v[e]);
                    v[e] = __float_as_uint(y * inv_s2);
                }
                tmem_st_32x32b_x32(ta, v);
            }
            tmem_st_wait();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&y_full[ab]);
        }
    } else {
        asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(kRegsEpi) : "memory");
        // ================================================= epilogue (8 warps)
        const int q = warp & 3;            // TMEM lane quarter = 32-row block of the tile
        const int s = (warp - 12) >> 2;    // handles column quarters s and s + 2
        const int ew = warp - 12;          // epilogue warp index 0..7
        const int r = q * 32 + lane;       // tile row of this thread
        const uint32_t tlane = tmem + ((uint32_t)(q * 32) << 16);
        const int np = p.np, n = p.n;
        uint8_t* stg = smem + kStagingOff + ew * 4 * kPieceBytes;  // hi, lo, hiT, loT pieces
        int u = 0;
        for (int tile = blockIdx.x; tile < total; tile += gridDim.x, ++u) {
            const int ab = u & 1;
            const int m = tile / p.T;
            const int t = tile - m * p.T;
            int I, J;
            decode_upper_tile(t, p.nb, I, J);
            const bool diag = I == J;
            const int gi = I * kBM + r;
            const uint32_t tacc = tlane + kAcc0 + ab * 128;
            float* Xt = p.X + xa_tile_base(m, I, J, p.nb);
            float* At = p.A + xa_tile_base(m, I, J, p.nb);
            bool bad_nf = false, bad_hr = false;
            double tr = 0.0, sq = 0.0;
            mbar_wait(&y_full[ab], (u >> 1) & 1);
            tc_fence_after();
            for (int qi = 0; qi < 2; ++qi) {
                const int qc = s + 2 * qi;  // column quarter (32 columns)
                if (diag && qc < q) continue;  // lower block of a diagonal tile: mirrored elsewhere
                if (p.dbg & 1) continue;
                if (!p.last && lane == 0) tma_store_wait_read();  // staging pieces free again
                __syncwarp();
#pragma unroll
                for (int sub = 0; sub < 2; ++sub) {
                    const int c0 = 32 * qc + 16 * sub;  // first tile column of this pass
                    uint32_t v[16];
                    tmem_ld_32x32b_x16(tacc + c0, v);
                    float4 xq[4], aq[4];
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        xq[k] = *reinterpret_cast<const float4*>(Xt + xa_off(r, c0 / 4 + k));
                        aq[k] = *reinterpret_cast<const float4*>(At + xa_off(r, c0 / 4 + k));
                    }
                    tmem_ld_wait();
                    uint16_t hb[16], lb[16];
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        float xs[4] = {xq[k].x, xq[k].y, xq[k].z, xq[k].w};
                        float as[4] = {aq[k].x, aq[k].y, aq[k].z, aq[k].w};
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            const int cl = c0 + 4 * k + e;
                            const int gj = J * kBN + cl;
                            double xd = p.a * (double)__uint_as_float(v[4 * k + e]) + p.b * (double)xs[e];
                            if (gi == gj && gi < n) xd += p.c;
                            const float xn = (float)xd;
                            const bool own = !diag || cl >= r;
                            bad_nf |= own && !isfinite(xn);
                            if (!p.last) {
                                bad_hr |= own && half_range_bad<MODE>(xn);
                                as[e] = (float)((double)as[e] + p.d_next * (double)xn);
                                xs[e] = xn;
                                split16<MODE>(xn, hb[4 * k + e], lb[4 * k + e]);
                            } else if (own && gi < n && gj < n) {
                                const double dv = (double)as[e] + (double)xn;
                                if (p.D) {
                                    double* Dm = p.D + (size_t)m * n * n;
                                    Dm[(size_t)gi * n + gj] = dv;
                                    if (gi != gj) Dm[(size_t)gj * n + gi] = dv;
                                }
                                if (gi != gj) {
                                    sq += 2.0 * dv * dv;
                                } else {
                                    tr += dv;
                                    sq += dv * dv;
                                }
                            }
                        }
                        if (!p.last) {
                            *reinterpret_cast<float4*>(Xt + xa_off(r, c0 / 4 + k)) = make_float4(xs[0], xs[1], xs[2], xs[3]);
                            *reinterpret_cast<float4*>(At + xa_off(r, c0 / 4 + k)) = make_float4(as[0], as[1], as[2], as[3]);
                        }
                    }
                    if (!p.last) {
                        // direct piece: row lane, columns 16*sub .. +15 of the 32x32 block
                        uint4 hv0, hv1, lv0, lv1;
                        hv0.x = hb[0] | ((uint32_t)hb[1] << 16);   hv0.y = hb[2] | ((uint32_t)hb[3] << 16);
                        hv0.z = hb[4] | ((uint32_t)hb[5] << 16);   hv0.w = hb[6] | ((uint32_t)hb[7] << 16);
                        hv1.x = hb[8] | ((uint32_t)hb[9] << 16);   hv1.y = hb[10] | ((uint32_t)hb[11] << 16);
                        hv1.z = hb[12] | ((uint32_t)hb[13] << 16); hv1.w = hb[14] | ((uint32_t)hb[15] << 16);
                        lv0.x = lb[0] | ((uint32_t)lb[1] << 16);   lv0.y = lb[2] | ((uint32_t)lb[3] << 16);
                        lv0.z = lb[4] | ((uint32_t)lb[5] << 16);   lv0.w = lb[6] | ((uint32_t)lb[7] << 16);
                        lv1.x = lb[8] | ((uint32_t)lb[9] << 16);   lv1.y = lb[10] | ((uint32_t)lb[11] << 16);
                        lv1.z = lb[12] | ((uint32_t)lb[13] << 16); lv1.w = lb[14] | ((uint32_t)lb[15] << 16);
                        const bool dblk = diag && qc == q;  // 32x32 block on the tile diagonal
                        if (!dblk) {
                            *reinterpret_cast<uint4*>(stg + sw64(lane, 2 * sub + 0)) = hv0;
                            *reinterpret_cast<uint4*>(stg + sw64(lane, 2 * sub + 1)) = hv1;
                            if (Tr::kHasLo) {
                                *reinterpret_cast<uint4*>(stg + kPieceBytes + sw64(lane, 2 * sub + 0)) = lv0;
                                *reinterpret_cast<uint4*>(stg + kPieceBytes + sw64(lane, 2 * sub + 1)) = lv1;
                            }
                        }
                        // mirrored piece (or, on the diagonal block, the symmetric completion):
                        // element (lane, 16*sub + e) -> row 16*sub + e, column lane
                        uint8_t* mh = dblk ? stg : stg + 2 * kPieceBytes;
                        uint8_t* ml = dblk ? stg + kPieceBytes : stg + 3 * kPieceBytes;
#pragma unroll
                        for (int e = 0; e < 16; ++e) {
                            const uint32_t col = 16 * sub + e;
                            const uint32_t off = sw64(col, lane >> 3) + (lane & 7) * 2;
                            if (!dblk || (int)col >= lane) {
                                *reinterpret_cast<uint16_t*>(mh + off) = hb[e];
                                if (Tr::kHasLo) *reinterpret_cast<uint16_t*>(ml + off) = lb[e];
                            }
                            if (dblk && (int)col >= lane) {
                                const uint32_t doff = sw64(lane, col >> 3) + (col & 7) * 2;
                                *reinterpret_cast<uint16_t*>(stg + doff) = hb[e];
                                if (Tr::kHasLo) *reinterpret_cast<uint16_t*>(stg + kPieceBytes + doff) = lb[e];
                            }
                        }
                    }
                }
                if (!p.last) {
                    fence_proxy_async_smem();
                    __syncwarp();
                    if (lane == 0) {
                        const int prow = m * np + I * kBM + 32 * q;   // direct piece origin
                        const int pcol = J * kBN + 32 * qc;
                        tma_store_2d(&tm.hip, stg, pcol, prow);
                        if (Tr::kHasLo) tma_store_2d(&tm.lop, stg + kPieceBytes, pcol, prow);
                        if (!(diag && qc == q)) {
                            const int mrow = m * np + J * kBN + 32 * qc;
                            const int mcol = I * kBM + 32 * q;
                            tma_store_2d(&tm.hip, stg + 2 * kPieceBytes, mcol, mrow);
                            if (Tr::kHasLo) tma_store_2d(&tm.lop, stg + 3 * kPieceBytes, mcol, mrow);
                        }
                        tma_store_commit();
                    }
                }
            }
            // this warp's Y reads for the tile are done: release the TMEM accumulator
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&acc_empty[ab]);
            const bool any_nf = __any_sync(0xffffffffu, bad_nf);
            const bool any_hr = __any_sync(0xffffffffu, bad_hr);
            if (lane == 0 && any_nf) atomicMin(&p.flags[2 * m + 0], p.layer + 1);
            if (lane == 0 && any_hr) atomicMin(&p.flags[2 * m + 1], p.layer + 1);
            if (p.last) {
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    tr += __shfl_xor_sync(0xffffffffu, tr, o);
                    sq += __shfl_xor_sync(0xffffffffu, sq, o);
                }
                named_bar_sync(3, kEpiWarps2 * 32);  // previous tile's partial consumed
                if (lane == 0) {
                    red[2 * ew + 0] = tr;
                    red[2 * ew + 1] = sq;
                }
                named_bar_sync(3, kEpiWarps2 * 32);
                if (ew == 0 && lane == 0) {
                    double T0 = 0.0, T1 = 0.0;
                    for (int w = 0; w < kEpiWarps2; ++w) {  // fixed order
                        T0 += red[2 * w + 0];
                        T1 += red[2 * w + 1];
                    }
                    p.partials[(size_t)m * p.T + t] = make_double2(T0, T1);
                }
            }
        }
        if (lane == 0) tma_store_wait_all();
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

// ===================================================================================== K3
struct FinalizeParams {
    const double2* partials;          // [B][T]
    const unsigned long long* bounds; // [B][2]
    const int* flags;                 // [B][2]
    const double* scale;              // [B] beta/beta0 (validity check), may be null
    const double* mu;                 // [B]
    double mu0;
    int T, B;
    double* stats;                    // [B][2] (Tr D, Tr D^2)
    double* bounds_out;               // [B][4] (eps_min, eps_max, x_min, x_max) widened
    int* status;                      // [B]
};

// status codes mirror ffg_status (include/fermiforge/ffg.h)
__global__ void __launch_bounds__(256) finalize_stats_kernel(const __grid_constant__ FinalizeParams p) {
    const int m = blockIdx.x;
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
        double lo = key_to_double(p.bounds[2 * m + 0]);
        double hi = key_to_double(p.bounds[2 * m + 1]);
        const double w = 1e-12 * (hi - lo);
        lo -= w;
        hi += w;
        int st = 0;
        double xmin = 0.0, xmax = 0.0;
        if (p.scale) {
            xmin = p.mu0 + p.scale[m] * (lo - p.mu[m]);
            xmax = p.mu0 + p.scale[m] * (hi - p.mu[m]);
            if (!(xmin >= 0.0) || !(xmax <= 1.0)) st = 2;  // FFG_ERR_OUT_OF_REGION
        }
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
