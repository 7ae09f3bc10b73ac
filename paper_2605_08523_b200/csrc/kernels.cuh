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
template <int MODE>
__device__ __forceinline__ void split16(float x, uint16_t& hi, uint16_t& lo) {
    if constexpr (MODE == kModeBF16) {
        hi = __bfloat16_as_ushort(__float2bfloat16_rn(x));
        lo = 0;
    } else {
        const float xs = x * kHalfScale;
        const __half h = __float2half_rn(xs);
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

// ===================================================================================== K1
struct RescaleParams {
    const double* H;            // [B][n][n] row-major, exactly symmetric
    const double* alpha;        // [B] X0 = alpha_m H + gamma_m I
    const double* gamma;        // [B]
    double d0;                  // first accumulator weight: A1 = d0 X0
    float* X;                   // [B][np][np]
    float* A;                   // [B][np][np]
    uint16_t* hi;               // [B][np][np] parity 0
    uint16_t* lo;               // [B][np][np] parity 0 (F32E only)
    unsigned long long* bounds; // [B][2] ordered keys of (eps_min, eps_max) before widening
    int* flags;                 // [B][2] first bad X_k index: [0] non-finite, [1] half range
    int n, np, mode, write_operands;
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
                *reinterpret_cast<float4*>(p.X + orow + j0) = make_float4(x[0], x[1], x[2], x[3]);
                const float d0 = (float)p.d0;
                float a[4];
#pragma unroll
                for (int e = 0; e < 4; ++e) a[e] = (float)(p.d0 * (double)x[e]);
                (void)d0;
                *reinterpret_cast<float4*>(p.A + orow + j0) = make_float4(a[0], a[1], a[2], a[3]);
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
                        split16<kModeF32E>(x[e], hb[e], lb[e]);
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
    int dbg;              // measurement only: bit0 skip epilogue memory traffic, bit1 skip drain
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
    CUtensorMap hid, lod;    // operand destination (parity (l+1)&1): box 64 x 128, SW128
    CUtensorMap him, lom;    // mirrored destination: box 64 x 64, SW128
    CUtensorMap x, a;        // fp32 master X / accumulator A: box 32 x 128, SW128
};

// byte offset of 16-byte chunk `c` of row `r` in a 128-byte-row tile with the TMA/UMMA
// 128B swizzle (tile base 1024-aligned)
__device__ __forceinline__ uint32_t sw128(uint32_t r, uint32_t c) {
    return r * 128u + ((c ^ (r & 7u)) << 4);
}

// Warp roles: 0 = TMA producer (+ epilogue TMA issue), 1 = TMEM allocator + UMMA issuer,
// 2..9 = accumulator-drain / epilogue warps (warp w reads TMEM lanes 32*(w%4)..+31; its
// column half during the drain is (w-2)/4).  One 128x128 upper-triangular tile per CTA.
//
// Accumulation precision.  tcgen05 FP32 accumulation truncates inside every MMA.  Summing
// hi*lo terms into the large hi*hi accumulator, or letting hi*hi accumulate over the whole
// K extent, biases Tr D by ~3e-6 (measured on B200, reproduced by emulation).
// So hi*lo + lo*hi go to their own TMEM accumulator (2^-11 smaller, its truncation is
// negligible) and every hi*hi MMA (DR=1) lands in a fresh buffer of a 3-deep TMEM ring that
// the epilogue warps drain into fp32 registers with round-to-nearest adds (FADD2) while the
// tensor core fills the next buffer.
// TMEM columns: [0,384) hi*hi ring, [384,512) cross terms, then the final Y.
//
// Epilogue (layers 0..L-2): Y = drained hi*hi + cross terms is written back to TMEM; X and A
// tiles come in by TMA into the (now idle) pipeline SMEM; X' = aY + bX + cI, A += d' X' and
// the split of X' are computed in swizzled SMEM and leave by TMA bulk stores: X, A and the
// direct hi/lo tile at (I,J), the transposed hi/lo tile at (J,I) (for a diagonal tile one
// symmetric 128x128 tile assembled from its upper triangle).  Last layer: D = A + X_L with
// direct fp64 stores and the per-tile statistics.
template <int MODE, int DR>
__global__ void __launch_bounds__(kLayerThreads, 1)
    mlsp2_layer_kernel(const __grid_constant__ LayerMaps tm, const __grid_constant__ LayerParams p) {
    using Tr = ModeTraits<MODE>;
    constexpr int S = Tr::kStages;
    constexpr int SB = stage_bytes<MODE>();
    constexpr uint32_t kHL = 384;  // TMEM column of the cross-term accumulator / final Y
    constexpr int NHB = 3;         // hi*hi accumulator ring
    static_assert(DR == 1 || DR == 2 || DR == 4, "drain granularity");
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                               ~uintptr_t(1023));
    constexpr int kPipe = layer_pipe_bytes<MODE>();
    constexpr bool kDrain = Tr::kProducts == 3;  // single-product modes accumulate in TMEM
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + kPipe);
    uint64_t* empty = full + S;
    uint64_t* hh_full = empty + S;       // [NHB]
    uint64_t* hh_empty = hh_full + NHB;  // [NHB]
    uint64_t* hl_full = hh_empty + NHB;
    uint64_t* xa_full = hl_full + 1;     // X/A tiles landed in smem
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(xa_full + 1);
    double* red = reinterpret_cast<double*>(smem + kPipe + 512);

    // epilogue staging inside the pipeline smem (valid once the mainloop is done)
    uint8_t* sX = smem;                  // [half][box 0..1] 128 rows x 32 fp32, 16 KB boxes
    uint8_t* sA = smem + 64 * 1024;
    uint8_t* sHi = smem + 128 * 1024;    // off-diag: direct 128x64 (16 KB); diag: 2 boxes 128x64
    uint8_t* sLo = smem + 144 * 1024;
    uint8_t* sHiT = smem + 160 * 1024;   // off-diag: mirrored 64x128 as 2 boxes 64x64 (8 KB)
    uint8_t* sLoT = smem + 176 * 1024;
    uint8_t* sHiD = smem + 128 * 1024;   // diag: symmetric 128x128 hi as 2 boxes 128x64 (32 KB)
    uint8_t* sLoD = smem + 160 * 1024;   // diag: symmetric 128x128 lo

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int m = blockIdx.x / p.T;
    const int t = blockIdx.x - m * p.T;
    int I, J;
    decode_upper_tile(t, p.nb, I, J);
    const bool diag = (I == J);
    const int nk = p.np / kBK;
    const bool tma_epi = !p.last && !(p.dbg & 1);
    const int rowI = m * p.np + I * kBM;
    const int rowJ = m * p.np + J * kBN;

    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < NHB; ++b) {
            mbar_init(&hh_full[b], 1);
            mbar_init(&hh_empty[b], kEpiWarps);  // one arrive per epilogue warp
        }
        mbar_init(hl_full, 1);
        mbar_init(xa_full, 1);
        fence_barrier_init();
        tma_prefetch_desc(&tm.hi);
        if (Tr::kHasLo) tma_prefetch_desc(&tm.lo);
    }
    if (warp == 1) tmem_alloc(tmem_slot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        // ------------------------------------------------ TMA producer
        if (lane == 0) {
            if (tma_epi) {  // warm L2 with this tile's X / A for the epilogue
                for (int b = 0; b < 4; ++b) {
                    tma_prefetch_l2_2d(&tm.x, J * kBN + 32 * b, rowI);
                    tma_prefetch_l2_2d(&tm.a, J * kBN + 32 * b, rowI);
                }
            }
            const uint32_t bytes = (diag ? (Tr::kHasLo ? 2 : 1) : (Tr::kHasLo ? 4 : 2)) * kOpBytes;
            for (int kb = 0; kb < nk; ++kb) {
                const int s = kb % S;
                const uint32_t ph = (kb / S) & 1;
                mbar_wait(&empty[s], ph ^ 1);
                mbar_expect_tx(&full[s], bytes);
                uint8_t* st = smem + s * SB;
                tma_load_2d(st + 0 * kOpBytes, &tm.hi, &full[s], kb * kBK, rowI);
                if (Tr::kHasLo) tma_load_2d(st + 1 * kOpBytes, &tm.lo, &full[s], kb * kBK, rowI);
                if (!diag) {
                    const int ob = Tr::kHasLo ? 2 : 1;
                    tma_load_2d(st + ob * kOpBytes, &tm.hi, &full[s], kb * kBK, rowJ);
                    if (Tr::kHasLo)
                        tma_load_2d(st + (ob + 1) * kOpBytes, &tm.lo, &full[s], kb * kBK, rowJ);
                }
            }
            if (tma_epi) {
                // all MMAs retired -> every pipeline stage is free: bring X, A (both halves)
                mbar_wait(hl_full, 0);
                mbar_expect_tx(xa_full, 128 * 1024);
                for (int b = 0; b < 4; ++b) {
                    tma_load_2d(sX + b * 16384, &tm.x, xa_full, J * kBN + 32 * b, rowI);
                    tma_load_2d(sA + b * 16384, &tm.a, xa_full, J * kBN + 32 * b, rowI);
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------ UMMA issuer (one thread)
        if (lane == 0) {
            constexpr uint32_t idesc = umma_idesc_f16(Tr::kFmt, kBM, kBN);
            int g = 0;  // index of the current hi*hi fill (DR K16 steps each)
            for (int kb = 0; kb < nk; ++kb) {
                const int s = kb % S;
                const uint32_t ph = (kb / S) & 1;
                mbar_wait(&full[s], ph);
                tc_fence_after();
                const uint32_t base = smem_u32(smem + s * SB);
                const uint32_t a_hi = base;
                const uint32_t a_lo = base + kOpBytes;
                const uint32_t ob = diag ? 0 : (Tr::kHasLo ? 2 : 1) * kOpBytes;
                const uint32_t b_hi = base + ob;
                const uint32_t b_lo = base + ob + kOpBytes;
#pragma unroll
                for (int kk = 0; kk < kBK / kUK; ++kk) {
                    const uint32_t koff = kk * kUK * 2;  // bytes along K inside the atom
                    const int hb = g % NHB;
                    if (!kDrain) {
                        umma_f16(tmem + kHL, umma_desc_sw128(a_hi + koff),
                                 umma_desc_sw128(b_hi + koff), idesc, (kb | kk) != 0);
                    } else {
                        if (kk % DR == 0 && !(p.dbg & 2)) {
                            mbar_wait(&hh_empty[hb], ((g / NHB) & 1) ^ 1);  // drained by the epilogue
                            tc_fence_after();
                        }
                        umma_f16(tmem + hb * 128, umma_desc_sw128(a_hi + koff),
                                 umma_desc_sw128(b_hi + koff), idesc, (kk % DR) != 0);
                        if (kk % DR == DR - 1) {
                            if (!(p.dbg & 2)) umma_commit(&hh_full[hb]);
                            ++g;
                        }
                    }
                    if (Tr::kProducts == 3) {
                        umma_f16(tmem + kHL, umma_desc_sw128(a_hi + koff),
                                 umma_desc_sw128(b_lo + koff), idesc, (kb | kk) != 0);
                        umma_f16(tmem + kHL, umma_desc_sw128(a_lo + koff),
                                 umma_desc_sw128(b_hi + koff), idesc, 1u);
                    }
                }
                umma_commit(&empty[s]);  // frees the smem stage once these MMAs retire
            }
            umma_commit(hl_full);
        }
        __syncwarp();
    } else {
        // ------------------------------------------------ accumulator drain
        const int q = warp & 3;
        const int hc = (warp - 2) >> 2;  // column half owned during the drain
        const int r = q * 32 + lane;     // tile row of this thread
        const int gi = I * kBM + r;
        const int np = p.np, n = p.n;
        const uint32_t tlane = tmem + ((uint32_t)(q * 32) << 16);
        const float inv_s2 = 1.0f / (Tr::kScale * Tr::kScale);

        float yacc[kEpiCols];
#pragma unroll
        for (int e = 0; e < kEpiCols; ++e) yacc[e] = 0.0f;
        static_assert(kEpiCols == 64, "drain loads two 32-column chunks");
#pragma unroll 1
        for (int g = 0; g < ((p.dbg & 2) || !kDrain ? 0 : nk * (kBK / kUK) / DR); ++g) {
            const int hb = g % NHB;
            mbar_wait(&hh_full[hb], (g / NHB) & 1);
            tc_fence_after();
            uint32_t v0[32], v1[32];
            tmem_ld_32x32b_x32(tlane + hb * 128 + hc * kEpiCols, v0);
            tmem_ld_32x32b_x32(tlane + hb * 128 + hc * kEpiCols + 32, v1);
            tmem_ld_wait();
#pragma unroll
            for (int e = 0; e < 32; e += 2) {
                float2 acc = make_float2(yacc[e], yacc[e + 1]);
                acc = add_f32x2(acc, make_float2(__uint_as_float(v0[e]), __uint_as_float(v0[e + 1])));
                yacc[e] = acc.x;
                yacc[e + 1] = acc.y;
                acc = make_float2(yacc[32 + e], yacc[32 + e + 1]);
                acc = add_f32x2(acc, make_float2(__uint_as_float(v1[e]), __uint_as_float(v1[e + 1])));
                yacc[32 + e] = acc.x;
                yacc[32 + e + 1] = acc.y;
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&hh_empty[hb]);
        }
        // Y = (hi*hi + cross terms) / scale^2, written over the cross-term columns
        mbar_wait(hl_full, 0);
        tc_fence_after();
#pragma unroll
        for (int ch = 0; ch < kEpiCols / 32; ++ch) {
            const uint32_t ta = tlane + kHL + hc * kEpiCols + ch * 32;
            uint32_t v[32];
            tmem_ld_32x32b_x32(ta, v);
            tmem_ld_wait();
#pragma unroll
            for (int e = 0; e < 32; ++e) {
                const float y = kDrain ? yacc[ch * 32 + e] + __uint_as_float(v[e]) : __uint_as_float(v[e]);
                v[e] = __float_as_uint(y * inv_s2);
            }
            if (p.dbg & 2) {  // measurement only: no drain -> Y is the cross-term accumulator
                tmem_ld_32x32b_x32(ta, v);
                tmem_ld_wait();
            }
            tmem_st_32x32b_x32(ta, v);
        }
        tmem_st_wait();
        tc_fence_before();
        named_bar_sync(2, kEpiWarps * 32);  // all of Y is in TMEM
        tc_fence_after();

        double tr = 0.0, sq = 0.0;
        bool bad_nf = false, bad_hr = false;
        const size_t mat = (size_t)m * np * np;
        if (p.dbg & 1) {
            // measurement only: no epilogue memory traffic
        } else if (!p.last) {
            // ============================== TMA epilogue (layers 0..L-2)
            const int sub = hc;  // 32-column block of the current half handled by this warp
            mbar_wait(xa_full, 0);
            for (int h = 0; h < 2; ++h) {
                const int cl0 = h * 64 + sub * 32;  // first tile column of this warp's block
                uint32_t v[32];
                tmem_ld_32x32b_x32(tlane + kHL + cl0, v);
                uint8_t* bx = sX + (h * 2 + sub) * 16384;
                uint8_t* ba = sA + (h * 2 + sub) * 16384;
                tmem_ld_wait();
                uint16_t hb[32], lb[32];
#pragma unroll
                for (int c4 = 0; c4 < 8; ++c4) {
                    float4* px = reinterpret_cast<float4*>(bx + sw128(r, c4));
                    float4* pa = reinterpret_cast<float4*>(ba + sw128(r, c4));
                    float4 xv = *px, av = *pa;
                    float xs[4] = {xv.x, xv.y, xv.z, xv.w};
                    float as[4] = {av.x, av.y, av.z, av.w};
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const int cl = cl0 + c4 * 4 + e;
                        const int gj = J * kBN + cl;
                        const float y = __uint_as_float(v[c4 * 4 + e]);
                        double xd = p.a * (double)y + p.b * (double)xs[e];
                        if (gi == gj && gi < n) xd += p.c;
                        const float xn = (float)xd;
                        const bool own = !diag || cl >= r;
                        bad_nf |= own && !isfinite(xn);
                        bad_hr |= own && half_range_bad<MODE>(xn);
                        as[e] = (float)((double)as[e] + p.d_next * (double)xn);
                        xs[e] = xn;
                        split16<MODE>(xn, hb[c4 * 4 + e], lb[c4 * 4 + e]);
                    }
                    *px = make_float4(xs[0], xs[1], xs[2], xs[3]);
                    *pa = make_float4(as[0], as[1], as[2], as[3]);
                }
                if (!diag) {
                    // direct tile (rows I, 64 columns of half h): row r, 16-B chunks 4*sub..
#pragma unroll
                    for (int c8 = 0; c8 < 4; ++c8) {
                        uint4 hv, lv;
                        hv.x = hb[c8 * 8 + 0] | ((uint32_t)hb[c8 * 8 + 1] << 16);
                        hv.y = hb[c8 * 8 + 2] | ((uint32_t)hb[c8 * 8 + 3] << 16);
                        hv.z = hb[c8 * 8 + 4] | ((uint32_t)hb[c8 * 8 + 5] << 16);
                        hv.w = hb[c8 * 8 + 6] | ((uint32_t)hb[c8 * 8 + 7] << 16);
                        *reinterpret_cast<uint4*>(sHi + sw128(r, sub * 4 + c8)) = hv;
                        if (Tr::kHasLo) {
                            lv.x = lb[c8 * 8 + 0] | ((uint32_t)lb[c8 * 8 + 1] << 16);
                            lv.y = lb[c8 * 8 + 2] | ((uint32_t)lb[c8 * 8 + 3] << 16);
                            lv.z = lb[c8 * 8 + 4] | ((uint32_t)lb[c8 * 8 + 5] << 16);
                            lv.w = lb[c8 * 8 + 6] | ((uint32_t)lb[c8 * 8 + 7] << 16);
                            *reinterpret_cast<uint4*>(sLo + sw128(r, sub * 4 + c8)) = lv;
                        }
                    }
                    // mirrored tile (rows = 64 columns of half h, cols = 128 rows of I):
                    // element (r, cl) -> row cl - 64h, col r; box r/64 of 64x64
                    uint8_t* mh = sHiT + (r >> 6) * 8192;
                    uint8_t* ml = sLoT + (r >> 6) * 8192;
                    const uint32_t cb = (uint32_t)(r & 63);
#pragma unroll
                    for (int e = 0; e < 32; ++e) {
                        const uint32_t mr = sub * 32 + e;
                        const uint32_t off = sw128(mr, cb >> 3) + (cb & 7) * 2;
                        *reinterpret_cast<uint16_t*>(mh + off) = hb[e];
                        if (Tr::kHasLo) *reinterpret_cast<uint16_t*>(ml + off) = lb[e];
                    }
                } else {
                    // diagonal tile: symmetric 128x128 assembled from the upper triangle,
                    // 2 boxes of 128 rows x 64 cols
#pragma unroll
                    for (int e = 0; e < 32; ++e) {
                        const uint32_t cl = cl0 + e;
                        if ((int)cl >= r) {
                            uint32_t off = (cl >> 6) * 16384 + sw128(r, (cl & 63) >> 3) + (cl & 7) * 2;
                            *reinterpret_cast<uint16_t*>(sHiD + off) = hb[e];
                            if (Tr::kHasLo) *reinterpret_cast<uint16_t*>(sLoD + off) = lb[e];
                            off = (r >> 6) * 16384 + sw128(cl, (r & 63) >> 3) + (r & 7) * 2;
                            *reinterpret_cast<uint16_t*>(sHiD + off) = hb[e];
                            if (Tr::kHasLo) *reinterpret_cast<uint16_t*>(sLoD + off) = lb[e];
                        }
                    }
                }
                fence_proxy_async_smem();
                named_bar_sync(2, kEpiWarps * 32);
                if (warp == 2 && lane == 0) {
                    for (int b = 0; b < 2; ++b) {
                        tma_store_2d(&tm.x, sX + (h * 2 + b) * 16384, J * kBN + h * 64 + 32 * b, rowI);
                        tma_store_2d(&tm.a, sA + (h * 2 + b) * 16384, J * kBN + h * 64 + 32 * b, rowI);
                    }
                    if (!diag) {
                        tma_store_2d(&tm.hid, sHi, J * kBN + h * 64, rowI);
                        if (Tr::kHasLo) tma_store_2d(&tm.lod, sLo, J * kBN + h * 64, rowI);
                        for (int b = 0; b < 2; ++b) {
                            tma_store_2d(&tm.him, sHiT + b * 8192, I * kBM + 64 * b, rowJ + h * 64);
                            if (Tr::kHasLo)
                                tma_store_2d(&tm.lom, sLoT + b * 8192, I * kBM + 64 * b, rowJ + h * 64);
                        }
                    } else if (h == 1) {
                        for (int b = 0; b < 2; ++b) {
                            tma_store_2d(&tm.hid, sHiD + b * 16384, I * kBM + 64 * b, rowI);
                            if (Tr::kHasLo) tma_store_2d(&tm.lod, sLoD + b * 16384, I * kBM + 64 * b, rowI);
                        }
                    }
                    tma_store_commit();
                    tma_store_wait_read();  // staging reusable for the next half
                }
                named_bar_sync(2, kEpiWarps * 32);
            }
            if (warp == 2 && lane == 0) tma_store_wait_all();
        } else {
            // ============================== last layer: D = A + X_L, statistics
#pragma unroll
            for (int ch = 0; ch < kEpiCols / 16; ++ch) {
                uint32_t v[16];
                tmem_ld_32x32b_x16(tlane + kHL + hc * kEpiCols + ch * 16, v);
                const int gj0 = J * kBN + hc * kEpiCols + ch * 16;
                const size_t off = mat + (size_t)gi * np + gj0;
                float xo[16], ao[16];
#pragma unroll
                for (int e = 0; e < 16; e += 4) {
                    const float4 xv = *reinterpret_cast<const float4*>(p.X + off + e);
                    const float4 av = *reinterpret_cast<const float4*>(p.A + off + e);
                    xo[e] = xv.x; xo[e + 1] = xv.y; xo[e + 2] = xv.z; xo[e + 3] = xv.w;
                    ao[e] = av.x; ao[e + 1] = av.y; ao[e + 2] = av.z; ao[e + 3] = av.w;
                }
                tmem_ld_wait();
#pragma unroll
                for (int e = 0; e < 16; ++e) {
                    const int gj = gj0 + e;
                    double xd = p.a * (double)__uint_as_float(v[e]) + p.b * (double)xo[e];
                    if (gi == gj && gi < n) xd += p.c;
                    const float xn = (float)xd;
                    const bool own = !diag || gj >= gi;
                    bad_nf |= own && !isfinite(xn);
                    if (own && gi < n && gj < n) {
                        const double dv = (double)ao[e] + (double)xn;
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
            }
        }
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
            if (lane == 0) {
                red[2 * (warp - 2) + 0] = tr;
                red[2 * (warp - 2) + 1] = sq;
            }
            named_bar_sync(1, kEpiWarps * 32);
            if (warp == 2 && lane == 0) {
                double T0 = 0.0, T1 = 0.0;
                for (int w = 0; w < kEpiWarps; ++w) {  // fixed order
                    T0 += red[2 * w + 0];
                    T1 += red[2 * w + 1];
                }
                p.partials[(size_t)m * p.T + t] = make_double2(T0, T1);
            }
        }
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
        if (st == 0 && p.flags[2 * m + 0] != INT_MAX) st = 3;  // FFG_ERR_DIVERGED
        if (st == 0 && p.flags[2 * m + 1] != INT_MAX) st = 4;  // FFG_ERR_HALF_RANGE
        p.status[m] = st;
        p.bounds_out[4 * m + 0] = lo;
        p.bounds_out[4 * m + 1] = hi;
        p.bounds_out[4 * m + 2] = xmin;
        p.bounds_out[4 * m + 3] = xmax;
    }
}

}  // namespace ffg
