// K2 epilogue arithmetic for one thread's row segment of a 128x128 block:
//   X' = a Y + b X (+ c on the diagonal),  A' = A + d' X',  binary16 hi/lo split of X'
// (scalar_models.cpp:243-252 per element: `acc += d*x` for the next layer, then
// `x = a*x2 + b*x + c`).  The fp64 coefficients enter as hi/lo fp32 pairs, so no layer sees a
// systematically rounded coefficient.  Default: fused FMAs, x' = fma(a_hi, y, fma(b_hi, x,
// a_lo y + b_lo x)) (<= ~1 ulp); FFG_EPI_EFT=1 selects error-free transformations (FMA product
// errors, TwoSum: the fp32 rounding of a ~2^-46-accurate value, as evaluating in fp64 and
// rounding once).  Both measure the same accuracy on the parity sample; neither
// uses fp64 or conversion instructions.  Padded rows/columns (>= n) hold zeros in X and Y, so they stay
// zero (the identity term is only added for rows < n).
#pragma once
#include "kernels.cuh"

namespace ffg {

struct EpiCoef {
    float a_hi, a_lo, b_hi, b_lo, c_hi, c_lo, d_hi, d_lo;
    float dc_hi, dc_lo;  // paired A updates: this layer's d, applied to the input X (0: none)
    bool red;            // this layer adds (dc X + d X') into A
    bool fixed;          // split X' with the fixed-point hi (the next layer accumulates hi*hi exactly)
    bool sr;             // ... and round its lo stochastically (the first sr_layers layers)
    uint32_t layer;      // the layer whose operands the split produces (stochastic-rounding hash)
};

// Layer l's coefficients as hi/lo fp32 pairs, split on the host from the fp64 model (hi = rn_f32(v),
// lo = rn_f32(v - hi)): table row l = {a, b}, {c, d_{l+1}} (d_L = 0).  d' multiplies the layer's output
// X', dc its input X.  With paired A updates only the odd layers reduce into A, adding d_l X_l +
// d_{l+1} X_{l+1} at once (d_l is row l-1's d'); K1 wrote A = d_0 X_0.  The table stays at 8 floats
// per layer (under 1 KB for 30 layers) so its per-call upload travels inline with the launch stream
// instead of queueing on a copy engine behind the host path's matrix transfers.
__device__ __forceinline__ EpiCoef load_coef(const float4* coef, int l, int n_layers, bool paired) {
    const float4 u = __ldg(coef + 2 * l), w = __ldg(coef + 2 * l + 1);
    EpiCoef k{u.x, u.y, u.z, u.w, w.x, w.y, w.z, w.w, 0.0f, 0.0f, l + 1 < n_layers, false, false, (uint32_t)(l + 1)};
    if (paired) {
        if (l & 1) {
            const float4 wp = __ldg(coef + 2 * (l - 1) + 1);
            k.dc_hi = wp.z;
            k.dc_lo = wp.w;
        } else {
            k.d_hi = k.d_lo = 0.0f;
            k.red = false;
        }
    }
    return k;
}

#ifndef FFG_EPI_EFT
#define FFG_EPI_EFT 0  // 1: error-free transformations (~correctly rounded); 0: fused FMAs on hi/lo
                       // coefficients (default: same measured accuracy, 4-7% faster K2)
#endif

// a Y + b X (+ c when with_c), nearly correctly rounded
template <bool WITH_C>
__device__ __forceinline__ float poly_step(float y, float x, const EpiCoef& k) {
#if !FFG_EPI_EFT
    // fp32 FMAs on hi/lo coefficients: no systematic coefficient rounding, <= ~1 ulp
    float t = fmaf(k.a_lo, y, k.b_lo * x);
    if constexpr (WITH_C) t += k.c_hi + k.c_lo;
    return fmaf(k.a_hi, y, fmaf(k.b_hi, x, t));
#else
    const float p = k.a_hi * y;
    const float ep = fmaf(k.a_hi, y, -p);
    const float q = k.b_hi * x;
    const float eq = fmaf(k.b_hi, x, -q);
    float s = p + q;
    float z = s - p;
    float t = (p - (s - z)) + (q - z);
    t += ep + eq;
    t = fmaf(k.a_lo, y, fmaf(k.b_lo, x, t));
    if constexpr (WITH_C) {
        const float s2 = s + k.c_hi;
        const float z2 = s2 - s;
        t += ((s - (s2 - z2)) + (k.c_hi - z2)) + k.c_lo;
        s = s2;
    }
    return s + t;
#endif
}

// A + d x, nearly correctly rounded
__device__ __forceinline__ float acc_step(float a, float x, const EpiCoef& k) {
#if !FFG_EPI_EFT
    return fmaf(k.d_hi, x, fmaf(k.d_lo, x, a));
#else
    const float m = k.d_hi * x;
    const float em = fmaf(k.d_hi, x, -m);
    const float s = a + m;
    const float z = s - a;
    const float t = ((a - (s - z)) + (m - z)) + fmaf(k.d_lo, x, em);
    return s + t;
#endif
}

// packed binary16 split of two values: hi = rn(x * 2^14), lo = rn(x * 2^14 - hi)
// (bf16 mode: hi = rn_bf16(x), lo = rn_bf16(x - hi)).  Every mode stores lo: the next layer's
// epilogue rebuilds X from hi + lo (load_xop); only FP32-emulated multiplies with it.  fixed (FP32E, the layers before `exact_layers`): hi is
// rounded to a multiple of 8 in the 2^14-scaled domain (x on a 2^-11 grid, or 2^-10 where binary16
// rounds it again for |x| >= 1), so the next layer's hi*hi products and all their partial sums lie on
// the 2^6 grid and an fp32 accumulator adds them exactly (|sums| < 2^30 for a spectrum in [0, 1]);
// lo is then rounded stochastically with the element hashes h0, h1 (kernels.cuh sr_hash).
template <int MODE>
__device__ __forceinline__ void split2(float x0, float x1, uint32_t& hi, uint32_t& lo, bool fixed = false,
                                       bool sr = false, uint32_t h0 = 0, uint32_t h1 = 0) {
    if constexpr (MODE == kModeBF16) {
        const __nv_bfloat162 h = __floats2bfloat162_rn(x0, x1);
        hi = *reinterpret_cast<const uint32_t*>(&h);
        const float2 f = __bfloat1622float2(h);
        const __nv_bfloat162 r = __floats2bfloat162_rn(x0 - f.x, x1 - f.y);
        lo = *reinterpret_cast<const uint32_t*>(&r);
    } else {
        const float s0 = x0 * kHalfScale, s1 = x1 * kHalfScale;
        const __half2 h = (MODE == kModeF32E && fixed)
                              ? __floats2half2_rn(rintf(s0 * 0.125f) * 8.0f, rintf(s1 * 0.125f) * 8.0f)
                              : __floats2half2_rn(s0, s1);
        hi = *reinterpret_cast<const uint32_t*>(&h);
        const float2 f = __half22float2(h);
        float r0 = s0 - f.x, r1 = s1 - f.y;  // exact
        if (MODE == kModeF32E && FFG_SR_LO && fixed && sr) {
            r0 = sr_f16_grid(r0, h0);
            r1 = sr_f16_grid(r1, h1);
        }
        const __half2 r = __floats2half2_rn(r0, r1);
        lo = *reinterpret_cast<const uint32_t*>(&r);
    }
}

__device__ __forceinline__ void sts_u16(uint32_t addr, uint16_t v) {
    asm volatile("st.shared.u16 [%0], %1;" ::"r"(addr), "h"(v) : "memory");
}
__device__ __forceinline__ void sts_v4(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
    asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d)
                 : "memory");
}

__device__ __forceinline__ void ldsm_x4_trans(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2,
                                              uint32_t& r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0, %1, %2, %3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(addr)
                 : "memory");
}
__device__ __forceinline__ void stsm_x4(uint32_t addr, uint32_t r0, uint32_t r1, uint32_t r2, uint32_t r3) {
    asm volatile("stmatrix.sync.aligned.m8n8.x4.shared.b16 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(r0),
                 "r"(r1), "r"(r2), "r"(r3)
                 : "memory");
}
// Transpose a 32x32 binary16 piece (64-byte rows, SW64) from `src` into `dst` with the warp:
// per 8-row strip rs, ldmatrix.trans reads the four 8x8 matrices (rs, cb) transposed and
// stmatrix writes them as matrices (cb, rs) of dst.
__device__ __forceinline__ void transpose_piece(uint32_t src, uint32_t dst, int lane) {
    const uint32_t j = lane >> 3, rr = lane & 7;
#pragma unroll
    for (uint32_t rs = 0; rs < 4; ++rs) {
        uint32_t r0, r1, r2, r3;
        ldsm_x4_trans(src + sw64(rs * 8 + rr, j), r0, r1, r2, r3);
        stsm_x4(dst + sw64(j * 8 + rr, rs), r0, r1, r2, r3);
    }
}

// In-place transpose of a 32x32 binary16 piece (64-byte rows, SW64): the warp reads all sixteen
// 8x8 matrices transposed into registers, then stores matrix (rs, cb)^T at position (cb, rs).
__device__ __forceinline__ void transpose_piece_inplace(uint32_t buf, int lane) {
    const uint32_t j = lane >> 3, rr = lane & 7;
    uint32_t t[4][4];
#pragma unroll
    for (uint32_t rs = 0; rs < 4; ++rs) ldsm_x4_trans(buf + sw64(rs * 8 + rr, j), t[rs][0], t[rs][1], t[rs][2], t[rs][3]);
    __syncwarp();
#pragma unroll
    for (uint32_t rs = 0; rs < 4; ++rs) stsm_x4(buf + sw64(j * 8 + rr, rs), t[rs][0], t[rs][1], t[rs][2], t[rs][3]);
}

// Per-thread health of the values it produced: z accumulates x*0 (NaN iff any x is
// non-finite), mx the largest |x| (binary16 split range: |x| 2^14 < 65504).
struct EpiHealth {
    float z = 0.0f, mx = 0.0f;
    __device__ __forceinline__ void add(float x) {
        z = fmaf(x, 0.0f, z);
        mx = fmaxf(mx, fabsf(x));
    }
    __device__ __forceinline__ bool nonfinite() const { return z != z; }
    template <int MODE>
    __device__ __forceinline__ bool half_range() const {
        return MODE != kModeBF16 && !(mx * kHalfScale < kHalfMax);
    }
};

// A' = A + d'X' as a fire-and-forget vector reduction at L2 (no read of A, no round trip; every
// element receives at most one add per layer, so the result is deterministic).  The sum d'X' is
// formed in fp32 from the hi/lo coefficient (one more rounding than acc_step's fused form; both
// ~1 ulp).
__device__ __forceinline__ void red_add_v4(float* gp, float a, float b, float c, float d) {
    asm volatile("red.relaxed.gpu.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(gp), "f"(a), "f"(b), "f"(c),
                 "f"(d)
                 : "memory");
}
__device__ __forceinline__ float acc_term(float x, const EpiCoef& k) { return fmaf(k.d_hi, x, k.d_lo * x); }

// X_l of 16 consecutive columns of one row, as the packed binary16 (bf16) hi / lo operands the
// layer multiplies (there is no fp32 master copy of X): one 32-byte load each (256-bit LDG: a warp
// reads 32 whole sectors).  Rebuilt as (hi + lo) / scale -- exact in fp32 -- so b X and the
// paired A term see X to the split's ~22 bits (16 in bf16 mode), measured inside the gates
// (DESIGN.md 3).
struct XOp {
    uint32_t h[8], l[8];
};
__device__ __forceinline__ void ld_cg_v8(const void* p, uint32_t (&v)[8]) {
    asm volatile("ld.global.cg.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "l"(p));
}
// hi / lo: the operand arrays of the layer's input parity at (row, first column) of the 16 values
__device__ __forceinline__ void load_xop(const uint16_t* hi, const uint16_t* lo, XOp& x) {
    ld_cg_v8(hi, x.h);
    ld_cg_v8(lo, x.l);
}
template <int MODE>
__device__ __forceinline__ float2 xop_pair(const XOp& x, int k) {  // elements 2k, 2k+1
    if constexpr (MODE == kModeBF16) {
        const float2 h = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&x.h[k]));
        const float2 l = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&x.l[k]));
        return make_float2(h.x + l.x, h.y + l.y);
    } else {
        const float2 h = __half22float2(*reinterpret_cast<const __half2*>(&x.h[k]));
        const float2 l = __half22float2(*reinterpret_cast<const __half2*>(&x.l[k]));
        constexpr float inv = 1.0f / kHalfScale;
        return make_float2((h.x + l.x) * inv, (h.y + l.y) * inv);
    }
}

// One 16-column sub-block (columns c0..c0+15 of the 128x128 block) of this thread's row r,
// mid-recursion layer, X already in registers: X stored, A updated by reduction, hi/lo into the warp's 32x32 direct staging piece
// (`stg_d`: hi at +0, lo at +kPieceBytes; row = lane).  The mirrored piece is produced
// afterwards by the warp (transpose_piece).  DIAG: the block is on the matrix diagonal; only
// columns >= r are owned (the rest is the mirror of owned values) and the identity term is
// added at column r.  dblk: the 32x32 piece itself is on the diagonal and is completed
// symmetrically in place.
// gi / gj0: global row of this thread and first global column of the block (stochastic-rounding
// hashes of the fixed-point split).
template <int MODE, bool DIAG>
__device__ __forceinline__ void epi_sub_mid_red(const uint32_t (&v)[16], const XOp& xq, float* At,
                                                int r, int c0, int lane, int sub, bool c_on, const EpiCoef& k,
                                                uint32_t stg_d, bool dblk, EpiHealth& hl, int gi, int gj0,
                                                bool nomem = false) {
    using Tr = ModeTraits<MODE>;
    uint32_t hp[8], lp[8];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const float2 x01 = xop_pair<MODE>(xq, 2 * j), x23 = xop_pair<MODE>(xq, 2 * j + 1);
        float xs[4] = {x01.x, x01.y, x23.x, x23.y};
        float ts[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const float y = __uint_as_float(v[4 * j + e]);
            float xn;
            if constexpr (DIAG) {
                const int cl = c0 + 4 * j + e;
                xn = (cl == r && c_on) ? poly_step<true>(y, xs[e], k) : poly_step<false>(y, xs[e], k);
                if (cl >= r) hl.add(xn);
            } else {
                xn = poly_step<false>(y, xs[e], k);
                hl.add(xn);
            }
            ts[e] = acc_term(xn, k) + fmaf(k.dc_hi, xs[e], k.dc_lo * xs[e]);
            xs[e] = xn;
        }
        if (!nomem && k.red)  // (nomem: measurement only, dbg & 64)
            red_add_v4(At + xa_off(r, c0 / 4 + j), ts[0], ts[1], ts[2], ts[3]);
        uint32_t hh[4] = {0u, 0u, 0u, 0u};
        if (MODE == kModeF32E && FFG_SR_LO && k.sr) {
            // sr_hash(gi, gj, layer) incrementally: the key of {i, j} is (min << 16) | max; a block
            // below the diagonal has j < i for all elements (a diagonal block's j < i elements are
            // mirrors, their values unused)
            const bool lower = gi >= gj0 + kBN;
            const uint32_t kb = lower ? ((uint32_t)(gj0 + c0) << 16) + (uint32_t)gi
                                      : ((uint32_t)gi << 16) + (uint32_t)(gj0 + c0);
            const uint32_t ks = lower ? 65536u : 1u;
#pragma unroll
            for (int e = 0; e < 4; ++e) hh[e] = sr_mix(kb + (uint32_t)(4 * j + e) * ks, k.layer);
        }
        split2<MODE>(xs[0], xs[1], hp[2 * j], lp[2 * j], k.fixed, k.sr, hh[0], hh[1]);
        split2<MODE>(xs[2], xs[3], hp[2 * j + 1], lp[2 * j + 1], k.fixed, k.sr, hh[2], hh[3]);
    }
    if (!dblk) {
        sts_v4(stg_d + sw64(lane, 2 * sub + 0), hp[0], hp[1], hp[2], hp[3]);
        sts_v4(stg_d + sw64(lane, 2 * sub + 1), hp[4], hp[5], hp[6], hp[7]);
        sts_v4(stg_d + kPieceBytes + sw64(lane, 2 * sub + 0), lp[0], lp[1], lp[2], lp[3]);
        sts_v4(stg_d + kPieceBytes + sw64(lane, 2 * sub + 1), lp[4], lp[5], lp[6], lp[7]);
    } else {
#pragma unroll
        for (int e = 0; e < 16; ++e) {
            const uint32_t col = 16 * sub + e;
            if ((int)col < lane) continue;
            const uint16_t hb = (uint16_t)(hp[e >> 1] >> (16 * (e & 1)));
            const uint16_t lb = (uint16_t)(lp[e >> 1] >> (16 * (e & 1)));
            const uint32_t off = sw64(col, lane >> 3) + (lane & 7) * 2;
            const uint32_t doff = sw64(lane, col >> 3) + (col & 7) * 2;
            sts_u16(stg_d + off, hb);
            sts_u16(stg_d + doff, hb);
            sts_u16(stg_d + kPieceBytes + off, lb);
            sts_u16(stg_d + kPieceBytes + doff, lb);
        }
    }
}

// Last layer: D = A + X_L (fp64, full symmetric storage) and the statistics of the owned
// elements (Tr D, sum D^2 with off-diagonal elements counted twice); sixteen columns.  mir = false
// (row-block table, off the diagonal blocks): only the direct entry, counted once -- the mirrored
// entry belongs to another rank's rows, which computes it itself.
// The direct entries of an off-diagonal block go out as one 32-byte store per four columns when the
// row slab allows it (n % 4 == 0, all four inside the matrix): a warp then writes 32 whole sectors per
// instruction instead of touching each sector four times with 8-byte stores.
template <int MODE, bool DIAG>
__device__ __forceinline__ void epi_sub_last(const uint32_t (&v)[16], const XOp& xop, const float* At,
                                             int r, int c0, int gi, int gj0, int n, bool c_on,
                                             const EpiCoef& k, double* Dm, EpiHealth& hl, double& tr,
                                             double& sq, bool mir = true) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const float2 x01 = xop_pair<MODE>(xop, 2 * j), x23 = xop_pair<MODE>(xop, 2 * j + 1);
        const float4 aq = __ldcg(reinterpret_cast<const float4*>(At + xa_off(r, c0 / 4 + j)));
        const float xs[4] = {x01.x, x01.y, x23.x, x23.y};
        const float as[4] = {aq.x, aq.y, aq.z, aq.w};
        const int gjq = gj0 + c0 + 4 * j;  // first column of the quad
        const bool vec = !DIAG && Dm && gi < n && gjq + 3 < n && (n & 3) == 0;
        double dq[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const int cl = c0 + 4 * j + e;
            const int gj = gj0 + cl;
            const float y = __uint_as_float(v[4 * j + e]);
            const bool dg = DIAG && cl == r;
            const float xn = (dg && c_on) ? poly_step<true>(y, xs[e], k) : poly_step<false>(y, xs[e], k);
            const bool own = !DIAG || cl >= r;
            if (own) hl.add(xn);
            const double dv = (double)as[e] + (double)fmaf(k.dc_hi, xs[e], k.dc_lo * xs[e]) + (double)xn;
            dq[e] = dv;
            if (own && gi < n && gj < n) {
                if (Dm) {
                    if (!vec) Dm[(size_t)gi * n + gj] = dv;
                    if (!dg && (DIAG || mir)) Dm[(size_t)gj * n + gi] = dv;
                }
                if (dg) {
                    tr += dv;
                    sq += dv * dv;
                } else {
                    sq += ((DIAG || mir) ? 2.0 : 1.0) * dv * dv;
                }
            }
        }
        if (vec)
            asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(Dm + (size_t)gi * n + gjq), "d"(dq[0]),
                         "d"(dq[1]), "d"(dq[2]), "d"(dq[3])
                         : "memory");
    }
}


}  // namespace ffg
