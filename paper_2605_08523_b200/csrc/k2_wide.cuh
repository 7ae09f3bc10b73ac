// K2 (wide form): the MLSP2 recursion layers on CTA pairs with 256 x 256 output tiles
// (tcgen05.mma.cta_group::2, M = 256, N = 256) and each hi/lo block stored ONCE.
//
// Why: the pair kernel (k2_pair.cuh, 256 x 128 tiles) moves ~6200 B/cycle through L2 at the bench
// configuration, 58% of it the operand stream (profiles/r2_*).
// A 256 x 256 tile loads 256 + 256 operand rows per 256 x 256 outputs instead of 256 + 128 per
// 256 x 128: two thirds of the operand bytes per flop.
//
// Item = SUPER-BLOCK (S, T), S <= T, of 2 x 2 blocks of 128 x 128: CTA rank c of the pair computes
// block row P = 2S + c against block columns 2T, 2T + 1 (its TMEM receives 128 rows x 256 columns).
// A diagonal super-block (S, S) also computes the lower block (2S + 1, 2S), which is discarded
// (its values are the mirror of (2S, 2S + 1)): 10 items of 4 blocks for the 36 blocks of N = 1024.
//
// Storage: hi/lo of X_l are written only for blocks (P, Q) with P <= Q (the upper block triangle;
// diagonal blocks in full, exactly symmetric).  An operand tile X[P, K-block kb] of block column
// Kc = kb / 2 is read
//   K-major  from the stored block (P, Kc)        when Kc > 2S   (both rows of the super-row <= Kc)
//   MN-major from the stored block (Kc, P)^T      when Kc <= 2S  (X symmetric; diagonal blocks are
//                                                                 exactly symmetric in storage)
// so both CTAs of a pair always agree on the operand major-ness of a K-block (one UMMA instruction
// descriptor for the pair).  No mirrored pieces are stored except inside diagonal blocks.
//
// Dependencies: counter[m][S] counts, per layer, the items touching super-row S (each CTA of an
// item (S, T) adds 1 to S and T after its stores): 2 nsb per layer when complete.  A layer-(l+1)
// item waits for its super-rows S and T, which also covers the WAR hazard on the parity it writes.
//
// Roles (640 threads): warp 0 TMA producer, warp 1 TMEM allocator / UMMA issuer (leader CTA), warps
// 4-19 sixteen WORKERS: warp w owns TMEM lane quarter w & 3 (32 rows) and a 64-column group
// (w - 4) >> 2 of the 256-column tile.  FP32-emulated: the workers sum the chunks of an item with
// round-to-nearest adds (k2_pair.cuh accumulation scheme: exact fixed-point hi*hi + cross terms in
// the exact layers; chunks of `normal_kstep` K16 steps afterwards), write Y into the item's last
// TMEM slot and run the epilogue from it; single-product modes read the whole-K accumulator.
// TMEM: 2 slots x 256 columns.
#pragma once
#include "k2_pair.cuh"

namespace ffg {

constexpr int kWideBN = 256;                     // tile columns (UMMA N)
constexpr int kWideWorkers = 16;
constexpr int kWideCount = 2;                    // counter increments per item and super-row (per CTA)
template <int MODE>
struct WideCfg {
    static constexpr int kOps = ModeTraits<MODE>::kHasLo ? 4 : 2;   // A_hi (A_lo) B_hi (B_lo)
    static constexpr int kStageBytes = kOps * kOpBytes;              // 64 KB / 32 KB
    static constexpr int kStages = ModeTraits<MODE>::kHasLo ? 3 : 6;
    static constexpr int kBarOff = kStages * kStageBytes;
    static constexpr int kValidOff = kBarOff + 1024;
    static constexpr int kSmem = kValidOff + kValidBits / 8 + 1024;
};
static_assert(WideCfg<kModeF32E>::kSmem <= 227 * 1024, "wide kernel smem");
static_assert(WideCfg<kModeBF16>::kSmem <= 227 * 1024, "wide kernel smem");
// 640 threads: warp 0 producer, warp 1 UMMA issuer, warps 2-3 idle, warps 4-19 workers; setmaxnreg
// moves registers from the control warpgroup to the workers (per SMSP: one control warp + four workers)
constexpr int kWideThreads = 640;
constexpr int kWideWorker0 = 4;
constexpr int kWRegsCtl = 64, kWRegsWork = 104;
static_assert(128 * kWRegsCtl + 512 * kWRegsWork <= kWideThreads * 96, "setmaxnreg budget (wide)");

// K-major SW128 operand descriptor (128 rows x 64 K, 8-row atoms at 1024 B); K16 step = +32 B
__device__ __forceinline__ uint64_t wdesc_k(uint32_t addr) { return umma_desc_sw128(addr); }
// MN-major SW128 operand descriptor: two 64-element MN halves (TMA boxes) 8 KB apart (LBO), 8-K
// atoms of 8 x 128 B (SBO = 1024 B); K16 step = +2048 B
__device__ __forceinline__ uint64_t wdesc_mn(uint32_t addr) {
    return umma_desc_sw128(addr) | (static_cast<uint64_t>(8192u >> 4) << 16);
}

__device__ __forceinline__ void st_v8(void* gp, const uint32_t (&v)[8]) {
    asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(gp), "r"(v[0]), "r"(v[1]), "r"(v[2]),
                 "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
                 : "memory");
}
__device__ __forceinline__ void st_u16(uint16_t* gp, uint16_t v) {
    asm volatile("st.global.u16 [%0], %1;" ::"l"(gp), "h"(v) : "memory");
}
__device__ __forceinline__ void st_v4_f64(double* gp, double a, double b, double c, double d) {
    asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(gp), "d"(a), "d"(b), "d"(c), "d"(d) : "memory");
}

// Packed fp32 pairs (sm_100 FFMA2 / FMUL2 / FADD2): each lane of a pair is rounded exactly like the
// scalar instruction, so the epilogue's results do not change -- only its issue cost halves.
__device__ __forceinline__ uint64_t f2u(float2 a) {
    uint64_t r;
    memcpy(&r, &a, 8);
    return r;
}
__device__ __forceinline__ float2 u2f(uint64_t r) {
    float2 a;
    memcpy(&a, &r, 8);
    return a;
}
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) {
    uint64_t d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(f2u(a)), "l"(f2u(b)), "l"(f2u(c)));
    return u2f(d);
}
__device__ __forceinline__ float2 mul2(float2 a, float2 b) {
    uint64_t d;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(f2u(a)), "l"(f2u(b)));
    return u2f(d);
}
__device__ __forceinline__ float2 bc2(float v) { return make_float2(v, v); }

// 16 consecutive columns (cl .. cl+15 of block (P, Q)) of this thread's row r, mid-recursion layer:
// X' = a Y + b X (+ c), A += d'X' (+ dc X) by L2 reduction, packed binary16 (bf16) split into hp / lp
// -- epilogue.cuh's poly_step / acc_term / split2 arithmetic, two elements per instruction.
// DIAG: only columns >= r are owned (health); the identity term at column r.
template <int MODE, bool DIAG>
__device__ __forceinline__ void wide_mid(const uint32_t (&v)[16], const XOp& xq, float* At, int r, int cl,
                                         bool c_on, const EpiCoef& k, EpiHealth& hl, int gi, int gj0,
                                         uint32_t (&hp)[8], uint32_t (&lp)[8], bool nomem = false) {
    static_assert(FFG_EPI_EFT == 0, "the packed wide epilogue implements the fused-FMA form");
    float2 z2 = make_float2(0.0f, 0.0f);
    float mx = hl.mx;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        float2 x[2], xn[2], ts[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int e = 4 * j + 2 * h;  // elements e, e+1
            x[h] = xop_pair<MODE>(xq, e >> 1);
            const float2 y = make_float2(__uint_as_float(v[e]), __uint_as_float(v[e + 1]));
            // poly_step: t = a_lo y + b_lo x (+ c); x' = a_hi y + (b_hi x + t)
            float2 t = fma2(bc2(k.a_lo), y, mul2(bc2(k.b_lo), x[h]));
            if constexpr (DIAG) {
                if (c_on && (r >> 1) == ((cl + e) >> 1)) {  // the identity term at column r
                    if (cl + e == r) t.x += k.c_hi + k.c_lo;
                    else t.y += k.c_hi + k.c_lo;
                }
            }
            xn[h] = fma2(bc2(k.a_hi), y, fma2(bc2(k.b_hi), x[h], t));
            // acc_term(x') + dc x
            const float2 at = fma2(bc2(k.d_hi), xn[h], mul2(bc2(k.d_lo), xn[h]));
            const float2 dt = fma2(bc2(k.dc_hi), x[h], mul2(bc2(k.dc_lo), x[h]));
            ts[h] = make_float2(at.x + dt.x, at.y + dt.y);
            // health of the owned elements
            if constexpr (DIAG) {
                const int col = cl + e;
                if (col >= r) hl.add(xn[h].x);
                if (col + 1 >= r) hl.add(xn[h].y);
            } else {
                z2 = fma2(xn[h], bc2(0.0f), z2);
                mx = fmaxf(mx, fmaxf(fabsf(xn[h].x), fabsf(xn[h].y)));
            }
        }
        if (k.red && !nomem) red_add_v4(At + xa_off(r, cl / 4 + j), ts[0].x, ts[0].y, ts[1].x, ts[1].y);
        if constexpr (MODE == kModeF32E) {
            if (FFG_SR_LO && k.sr) {
                uint32_t hh[4];
#pragma unroll
                for (int e = 0; e < 4; ++e) hh[e] = sr_hash((uint32_t)gi, (uint32_t)(gj0 + cl + 4 * j + e), k.layer);
                split2<MODE>(xn[0].x, xn[0].y, hp[2 * j], lp[2 * j], k.fixed, true, hh[0], hh[1]);
                split2<MODE>(xn[1].x, xn[1].y, hp[2 * j + 1], lp[2 * j + 1], k.fixed, true, hh[2], hh[3]);
                continue;
            }
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                // split2: hi = rn_f16(x 2^14) (fixed: a multiple of 8), lo = rn_f16(x 2^14 - hi)
                float2 sx = mul2(xn[h], bc2(kHalfScale));
                float2 hv = sx;
                if (k.fixed) {
                    const float2 q8 = mul2(sx, bc2(0.125f));
                    hv = mul2(make_float2(rintf(q8.x), rintf(q8.y)), bc2(8.0f));
                }
                const __half2 hh2 = __floats2half2_rn(hv.x, hv.y);
                const float2 f = __half22float2(hh2);
                const float2 rr = fma2(f, bc2(-1.0f), sx);  // exact
                const __half2 ll2 = __floats2half2_rn(rr.x, rr.y);
                hp[2 * j + h] = *reinterpret_cast<const uint32_t*>(&hh2);
                lp[2 * j + h] = *reinterpret_cast<const uint32_t*>(&ll2);
            }
        } else {
            split2<MODE>(xn[0].x, xn[0].y, hp[2 * j], lp[2 * j], false);
            split2<MODE>(xn[1].x, xn[1].y, hp[2 * j + 1], lp[2 * j + 1], false);
        }
    }
    if constexpr (!DIAG) {
        hl.z = hl.z + (z2.x + z2.y);  // NaN iff any x' is non-finite
        hl.mx = mx;
    }
}

// Last layer, 16 columns: D = A + X_L (fp64) for the owned elements (DIAG: columns >= r), direct and
// mirrored entries, statistics (off-diagonal elements counted twice).  Four columns at a time (the
// worker still holds the rest of its Y in registers).
template <int MODE, bool DIAG>
__device__ __forceinline__ void wide_last(const uint32_t (&v)[16], const XOp& xq, const float* At, int r, int cl,
                                          int gi, int gj0, int n, bool c_on, const EpiCoef& k, double* Dm,
                                          EpiHealth& hl, double& tr, double& sq) {
    const bool vec = !DIAG && Dm && gi < n && gj0 + cl + 15 < n && (n & 3) == 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const float2 x01 = xop_pair<MODE>(xq, 2 * j), x23 = xop_pair<MODE>(xq, 2 * j + 1);
        const float4 aq = __ldcg(reinterpret_cast<const float4*>(At + xa_off(r, cl / 4 + j)));
        const float xs[4] = {x01.x, x01.y, x23.x, x23.y};
        const float as[4] = {aq.x, aq.y, aq.z, aq.w};
        double d[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const int col = cl + 4 * j + e;
            const float y = __uint_as_float(v[4 * j + e]);
            const bool dg = DIAG && col == r;
            const float xn = (dg && c_on) ? poly_step<true>(y, xs[e], k) : poly_step<false>(y, xs[e], k);
            const bool o = (!DIAG || col >= r) && gi < n && gj0 + col < n;
            if (!DIAG || col >= r) hl.add(xn);
            d[e] = (double)as[e] + (double)fmaf(k.dc_hi, xs[e], k.dc_lo * xs[e]) + (double)xn;
            if (o) {
                if (dg) {
                    tr += d[e];
                    sq += d[e] * d[e];
                } else {
                    sq += 2.0 * d[e] * d[e];
                }
                // mirrored entry: for each column the warp's 32 consecutive rows -> 256 contiguous bytes
                if (Dm && !dg) Dm[(size_t)(gj0 + col) * n + gi] = d[e];
                if (Dm && !vec) Dm[(size_t)gi * n + gj0 + col] = d[e];
            }
        }
        if (vec) st_v4_f64(Dm + (size_t)gi * n + gj0 + cl + 4 * j, d[0], d[1], d[2], d[3]);
    }
}

// The 16-column sub-blocks this warp finishes for an item: sub s (columns 64 (cg & 1) + 16 s of block Q)
// unless the block is the redundant (2S+1, 2S) or the 32-column piece lies below a diagonal block's
// diagonal (written as a mirror by the owner of the transposed piece).
__device__ __forceinline__ bool wide_sub_live(bool redundant, bool diag, int cg, int q, int sub) {
    return !redundant && !(diag && ((64 * (cg & 1) + 16 * sub) >> 5) < q);
}

template <int MODE>
__device__ __forceinline__ void wide_workers(const PairParams& p, const MatrixMap& mm, uint32_t tmem, int warp,
                                             int lane, uint32_t rank, int pair_id, int n_pairs, int total, int nk,
                                             int nsb, uint64_t* slot_full, uint64_t* slot_empty, double* red) {
    using Tr = ModeTraits<MODE>;
    constexpr bool kDrain = Tr::kProducts == 3;
    const int wk = warp - kWideWorker0, q = warp & 3, cg = wk >> 2;
    const int r = q * 32 + lane;
    const int nb = p.nb, n = p.n, np = p.np;
    const uint32_t tl = tmem + ((uint32_t)(q * 32) << 16) + 64 * cg;  // + slot * 256
    constexpr float inv_s2 = 1.0f / (Tr::kScale * Tr::kScale);
    const uint32_t slot_empty_l0 = mapa_shared(smem_u32(&slot_empty[0]), 0);  // leader's
    const uint32_t slot_full_a = smem_u32(&slot_full[0]);
    int g = 0;
    unsigned long long w_chunk = 0, w_epi = 0, w_pub = 0, w_dep = 0, w_drain = 0, w_setup = 0;
    for (int item = pair_id; item < total; item += n_pairs) {
        int m, l, pi;
        pair_decode(p, mm, item, m, l, pi);
        const uint32_t pr = __ldg(p.pairs + pi);
        const int S = pr & 1023, T = (pr >> 10) & 1023;
        const long long t_d0 = FFG_ROLE_PROF ? clock64() : 0;
        const int P = 2 * S + (int)rank;
        const int Q = 2 * T + (cg >> 1);
        const bool redundant = S == T && rank == 1 && (cg >> 1) == 0;  // block (2S+1, 2S): mirror of (2S, 2S+1)
        const bool diag = P == Q;
        const bool last = l == p.n_layers - 1;
        const int gi = P * kBM + r;
        const size_t xrow = ((size_t)m * np + gi) * np + (size_t)Q * kBN + 64 * (cg & 1);
        const uint16_t* xh = p.ophi[l & 1] + xrow;
        const uint16_t* xl = p.oplo[l & 1] + xrow;
        // X_l of this block is complete once super-row S is, and every layer-l reader of the parity
        // this item overwrites is done once super-rows S and T are (the producer's dependency wait, or
        // -- block-granular mode -- not yet: re-acquired here for this warp's own loads and stores);
        // the X loads go out before the wait for Y
        if (l > p.l0) {
            if (lane == 0) {
                const uint32_t need = (uint32_t)(kWideCount * nsb * (l - p.l0));
                const long long t0 = FFG_ROLE_PROF ? clock64() : 0;
                while (ld_acquire_gpu(p.counters + (size_t)m * nsb + S) < need) {
                }
                while (ld_acquire_gpu(p.counters + (size_t)m * nsb + T) < need) {
                }
                if (FFG_ROLE_PROF) w_dep += (unsigned long long)(clock64() - t0);
            }
            __syncwarp();
        }
        // X operands of the next live sub-block in flight (issued before the wait for Y)
        XOp xa = {};
        int sa = 0;
        while (sa < 4 && !wide_sub_live(redundant, diag, cg, q, sa)) ++sa;
        if (!kDrain && sa < 4 && !(p.dbg & 128)) load_xop(xh + 16 * sa, xl + 16 * sa, xa);
        int ysl;
        if constexpr (kDrain) {
            const int kst = layer_kstep(l, p.exact_layers, p.semi_layers, p.normal_kstep);
            const int chunks = kst == 0 ? 2 : layer_chunks(MODE, nk, kst);
            float yacc[64];
#pragma unroll
            for (int e = 0; e < 64; ++e) yacc[e] = 0.0f;
#pragma unroll 1
            for (int f = 0; f < chunks; ++f, ++g) {
                const int sl = g & 1;
                FFG_TIMED(w_chunk, mbar_wait_at(slot_full_a + 8 * sl, (g >> 1) & 1));
                tc_fence_after();
                uint32_t dep = 0;
#pragma unroll
                for (int ch = 0; ch < 4; ++ch) {
                    uint32_t v[16];
                    tmem_ld_32x32b_x16(tl + sl * 256 + ch * 16 + dep, v);
                    tmem_ld_wait();
#pragma unroll
                    for (int e = 0; e < 16; e += 2) {
                        const float2 a = add_f32x2(make_float2(yacc[16 * ch + e], yacc[16 * ch + e + 1]),
                                                   make_float2(__uint_as_float(v[e]), __uint_as_float(v[e + 1])));
                        yacc[16 * ch + e] = a.x;
                        yacc[16 * ch + e + 1] = a.y;
                    }
                    // one x16 batch in flight (keeps the sums in registers; see k2_pair.cuh drain)
                    dep = (__float_as_uint(yacc[16 * ch + 15]) | __float_as_uint(yacc[16 * ch])) & p.zero;
                }
                if (f + 1 < chunks) {  // this slot is free again; the last one receives Y
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive_cluster(slot_empty_l0 + 8 * sl);
                }
            }
            ysl = (g - 1) & 1;
#pragma unroll
            for (int ch = 0; ch < 4; ++ch) {
                uint32_t v[16];
#pragma unroll
                for (int e = 0; e < 16; ++e) v[e] = __float_as_uint(yacc[16 * ch + e] * inv_s2);
                tmem_st_32x32b_x16(tl + ysl * 256 + ch * 16, v);
            }
            if (sa < 4 && !(p.dbg & 128)) load_xop(xh + 16 * sa, xl + 16 * sa, xa);
            tmem_st_wait();
        } else {
            ysl = g & 1;
            FFG_TIMED(w_chunk, mbar_wait_at(slot_full_a + 8 * ysl, (g >> 1) & 1));
            tc_fence_after();
            ++g;
        }
        const long long t_e0 = FFG_ROLE_PROF ? clock64() : 0;
        if (FFG_ROLE_PROF) w_drain += (unsigned long long)(t_e0 - t_d0);
        // ------------------------------------------------------------- epilogue of the item
        const bool c_on = gi < n;
        EpiCoef k = load_coef(p.coef, l, p.n_layers, p.a_pair != 0);
        k.fixed = FFG_FIXED_SPLIT && MODE == kModeF32E && l + 1 < p.exact_layers;  // next layer exact
        k.sr = k.fixed && l + 1 < p.sr_layers;
        const int nxt = (l + 1) & 1;
        float* At = p.A + xa_tile_base(m, P, Q, nb);
        uint16_t* oh = const_cast<uint16_t*>(p.ophi[nxt]);
        uint16_t* ol = const_cast<uint16_t*>(p.oplo[nxt]);
        double* Dm = last && p.D ? p.D + (size_t)m * n * n : nullptr;
        EpiHealth hl;
        double tr = 0.0, sq = 0.0;
        // Y of the next sub-block is requested from TMEM before this one is processed
        if (FFG_ROLE_PROF) w_setup += (unsigned long long)(clock64() - t_e0);
        uint32_t vn[16] = {};
        const bool ldy = !(p.dbg & 512);  // (measurement only: dbg & 512 skips the Y reads)
        if (sa < 4 && ldy) tmem_ld_32x32b_x16(tl + ysl * 256 + 16 * sa, vn);
#pragma unroll 1
        for (int sub = sa; sub < 4; ++sub) {  // (sa: first live sub-block; all later ones are live)
            const int cl = 64 * (cg & 1) + 16 * sub;  // first column in block Q
            tmem_ld_wait();
            uint32_t v[16];
#pragma unroll
            for (int e = 0; e < 16; ++e) v[e] = vn[e];
            if (sub + 1 < 4 && ldy) tmem_ld_32x32b_x16(tl + ysl * 256 + 16 * (sub + 1), vn);
            if constexpr (!kDrain && Tr::kScale != 1.0f) {
#pragma unroll
                for (int e = 0; e < 16; ++e) v[e] = __float_as_uint(__uint_as_float(v[e]) * inv_s2);
            }
            const XOp xq = xa;
            if (sub + 1 < 4 && !(p.dbg & 128)) load_xop(xh + 16 * (sub + 1), xl + 16 * (sub + 1), xa);
            if (!last) {
                uint32_t hp[8], lp[8];
                const size_t orow = ((size_t)m * np + gi) * np + (size_t)Q * kBN + cl;
                if (diag) {
                    wide_mid<MODE, true>(v, xq, At, r, cl, c_on, k, hl, gi, Q * kBN, hp, lp, p.dbg & 64);
                    const size_t mrow0 = ((size_t)m * np + Q * kBN + cl) * np + (size_t)P * kBM + r;
                    uint16_t* mh = oh + mrow0;
                    uint16_t* ml = ol + mrow0;
                    // direct row (in a diagonal piece its entries below the diagonal are provisional),
                    // then -- after the warp's direct stores -- the owned entries col > r mirrored to
                    // (col, r), overwriting the provisional ones: a location (c, r), c > r, gets its
                    // provisional value in the sub-block of column r <= the sub-block of column c
                    st_v8(oh + orow, hp);
                    st_v8(ol + orow, lp);
                    __syncwarp();
#pragma unroll
                    for (int e = 0; e < 16; ++e) {
                        if (cl + e > r) {
                            st_u16(mh + (size_t)e * np, (uint16_t)(hp[e >> 1] >> (16 * (e & 1))));
                            st_u16(ml + (size_t)e * np, (uint16_t)(lp[e >> 1] >> (16 * (e & 1))));
                        }
                    }
                } else {
                    wide_mid<MODE, false>(v, xq, At, r, cl, c_on, k, hl, gi, Q * kBN, hp, lp, p.dbg & 64);
                    if (!(p.dbg & 32)) {  // (measurement only: dbg & 32 skips the hi/lo stores)
                        st_v8(oh + orow, hp);
                        st_v8(ol + orow, lp);
                    }
                }
            } else if (diag) {
                wide_last<MODE, true>(v, xq, At, r, cl, gi, Q * kBN, n, c_on, k, Dm, hl, tr, sq);
            } else {
                wide_last<MODE, false>(v, xq, At, r, cl, gi, Q * kBN, n, c_on, k, Dm, hl, tr, sq);
            }
        }
        // this warp's Y reads are done: release the pair's TMEM slot
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(slot_empty_l0 + 8 * ysl);
        const long long t_e1 = FFG_ROLE_PROF ? clock64() : 0;
        if (FFG_ROLE_PROF) w_epi += (unsigned long long)(t_e1 - t_e0);
        if (!redundant) {
            const bool any_nf = __any_sync(0xffffffffu, hl.nonfinite());
            const bool any_hr = !last && __any_sync(0xffffffffu, hl.template half_range<MODE>());
            if (lane == 0 && any_nf) atomicMin(&p.flags[2 * m + 0], l + 1);
            if (lane == 0 && any_hr) atomicMin(&p.flags[2 * m + 1], l + 1);
        }
        if (last) {
            // per-CTA statistics of the item: warp trees, then the 16 warps in fixed order
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                tr += __shfl_xor_sync(0xffffffffu, tr, o);
                sq += __shfl_xor_sync(0xffffffffu, sq, o);
            }
            named_bar_sync(3, kWideWorkers * 32);  // the previous item's partial consumed
            if (lane == 0) {
                red[2 * wk + 0] = tr;
                red[2 * wk + 1] = sq;
            }
            named_bar_sync(3, kWideWorkers * 32);
            if (wk == 0 && lane == 0) {
                double T0 = 0.0, T1 = 0.0;
                for (int w = 0; w < kWideWorkers; ++w) {
                    T0 += red[2 * w + 0];
                    T1 += red[2 * w + 1];
                }
                p.partials[(size_t)m * 2 * p.PT + 2 * pi + rank] = make_double2(T0, T1);
            }
        } else if (l + 1 < p.l1) {
            // publish: this CTA's stores of the item -> super-row counters S and T (one fence for
            // the CTA: per-warp fences measured 1.8x slower on the BF16 dependency chain)
            fence_proxy_async_global();
            __syncwarp();
            named_bar_sync(4, kWideWorkers * 32);
            if (wk == 0 && lane == 0) {
                __threadfence();
                uint32_t* cm = p.counters + (size_t)m * nsb;
                if (p.blockdeps) red_relaxed_gpu_add(p.bflags + ((size_t)m * nsb + S) * nsb + T, 1u);
                red_relaxed_gpu_add(cm + S, 1u);
                if (T != S) red_relaxed_gpu_add(cm + T, 1u);
            }
        }
        if (FFG_ROLE_PROF) w_pub += (unsigned long long)(clock64() - t_e1);
    }
    if (FFG_ROLE_PROF && (p.dbg & 8) && lane == 0 && (wk == 0 || wk == 5)) {
        unsigned long long* o = p.prof + (size_t)blockIdx.x * 16 + (wk == 0 ? 6 : 12);
        o[0] = w_chunk;
        o[1] = w_drain - w_chunk;
        o[2] = w_dep;
        o[3] = w_epi;
        if (wk == 0) {
            o[4] = w_pub;
            o[5] = w_setup;
        }
    }
}

template <int MODE>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kWideThreads, 1)
    mlsp2_wide_kernel(const __grid_constant__ PairMaps tm, const __grid_constant__ PairParams p) {
    constexpr int kSlots = 2;  // TMEM: 2 x 256 columns
    using Tr = ModeTraits<MODE>;
    using Cfg = WideCfg<MODE>;
    constexpr bool kDrain = Tr::kProducts == 3;
    constexpr int S_ = Cfg::kStages;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                               ~uintptr_t(1023));
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Cfg::kBarOff);
    uint64_t* full = bars;                      // [S_] leader: TMA bytes of both CTAs
    uint64_t* empty = bars + S_;                // [S_] both: stage consumed (multicast commit)
    uint64_t* slot_full = bars + 2 * S_;        // [2]  both: chunk accumulated in TMEM slot
    uint64_t* slot_empty = bars + 2 * S_ + 2;   // [2]  leader: slot read by both CTAs' workers
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * S_ + 4);
    double* red = reinterpret_cast<double*>(bars + 2 * S_ + 6);  // [16][2]
    // 32-bit shared addresses of the barriers (the wait loops keep these, not generic pointers)
    const uint32_t full_a = smem_u32(full), empty_a = smem_u32(empty), slot_empty_a = smem_u32(slot_empty);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = cluster_ctarank();
    const bool leader = rank == 0;
    const int pair_id = blockIdx.x >> 1, n_pairs = gridDim.x >> 1;
    uint32_t* valid_bits = reinterpret_cast<uint32_t*>(smem + Cfg::kValidOff);
    const int nk = p.np / kBK;
    const int nsb = p.nb / 2;

    if (threadIdx.x == 0) {
        for (int i = 0; i < S_; ++i) {
            mbar_init(&full[i], (p.dbg & 16) ? 2 : 1);  // (dbg & 16, measurement only: no operand loads)
            mbar_init(&empty[i], 1);
        }
        for (int i = 0; i < kSlots; ++i) {
            mbar_init(&slot_full[i], 1);
            mbar_init(&slot_empty[i], 2 * kWideWorkers);
        }
        fence_barrier_init();
    }
    for (int wd = threadIdx.x; wd < (p.B + 31) / 32; wd += blockDim.x) {
        uint32_t bits = 0u;
        for (int b = 0; b < 32; ++b) {
            const int m = 32 * wd + b;
            if (m < p.B && matrix_in_region(p.region, p.m0 + m)) bits |= 1u << b;
        }
        valid_bits[wd] = bits;
    }
    if (warp == 1) tmem_alloc_pair(tmem_slot, 512);
    tc_fence_before();
    cluster_sync_all();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    MatrixMap mm{valid_bits, 0, false};
    for (int wd = 0; wd < (p.B + 31) / 32; ++wd) mm.nvalid += __popc(valid_bits[wd]);
    mm.remap = mm.nvalid != p.B;
    const int total = (p.l1 - p.l0) * mm.nvalid * p.PT;
    const uint32_t full_l0 = mapa_shared(full_a, 0);  // the leader's full barriers (TMA complete_tx)

    if (warp < kWideWorker0) {
        asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(kWRegsCtl) : "memory");
        if (warp == 0 && lane == 0) {
            // ================================================= TMA producer (both CTAs)
            for (int i = 0; i < 2; ++i) {
                tma_prefetch_desc(&tm.a_hi[i]);
                tma_prefetch_desc(&tm.b_hi[i]);
                if (Tr::kHasLo) {
                    tma_prefetch_desc(&tm.a_lo[i]);
                    tma_prefetch_desc(&tm.b_lo[i]);
                }
            }
            const uint32_t bytes = 2u * Cfg::kStageBytes;  // both CTAs land on the leader's barrier
            int it = 0;
            unsigned long long w_dep = 0, w_empty = 0;
            const long long t_start = clock64();
            for (int item = pair_id; item < total; item += n_pairs) {
                int m, l, pi;
                pair_decode(p, mm, item, m, l, pi);
                const uint32_t pr = __ldg(p.pairs + pi);
                const int S = pr & 1023, T = (pr >> 10) & 1023;
                const uint32_t* cm = p.counters + (size_t)m * nsb;
                const uint32_t need = (uint32_t)(kWideCount * nsb * (l - p.l0));
                // block-granular dependencies (single-matrix groups, p.blockdeps): while super-row S or
                // T is incomplete, each super-column U of the K loop waits for the two super-blocks
                // its operand tiles come from, so the item's first K-blocks overlap the previous
                // layer's tail (the pair kernel's scheme, k2_pair.cuh)
                bool blockwise = false;
                if (l > p.l0) {
                    const long long t0 = clock64();
                    if (p.blockdeps) {
                        blockwise = ld_acquire_gpu(cm + S) < need || ld_acquire_gpu(cm + T) < need;
                    } else {
                        while (ld_acquire_gpu(cm + S) < need)
                            watchdog_check(t0, 13, ((unsigned long long)item << 32) | (uint32_t)(m * 1024 + S), need);
                        while (ld_acquire_gpu(cm + T) < need)
                            watchdog_check(t0, 14, ((unsigned long long)item << 32) | (uint32_t)(m * 1024 + T), need);
                    }
                    if (FFG_ROLE_PROF) w_dep += (unsigned long long)(clock64() - t0);
                    if (!blockwise) fence_proxy_async_global();
                }
                const int par = l & 1;
                const int mrow = m * p.np;
                const int PA = 2 * S + (int)rank, PB = 2 * T + (int)rank;
                for (int kb = 0; kb < nk; ++kb, ++it) {
                    const int s = it % S_;
                    if (blockwise && (kb & 3) == 0) {
                        const int U = kb >> 2;  // super-column of the next four K-blocks
                        const uint32_t needb = (uint32_t)(kWideCount * (l - p.l0));
                        const uint32_t* bf = p.bflags + (size_t)m * nsb * nsb;
                        const uint32_t* fa = bf + min(S, U) * nsb + max(S, U);
                        const uint32_t* fb = bf + min(T, U) * nsb + max(T, U);
                        const long long t0 = clock64();
                        uint32_t va = ld_acquire_gpu(fa), vb = ld_acquire_gpu(fb);
                        if (ld_acquire_gpu(cm + S) >= need && ld_acquire_gpu(cm + T) >= need) blockwise = false;
                        while (va < needb) {
                            watchdog_check(t0, 15, ((unsigned long long)item << 32) | (uint32_t)(S * 1024 + U), needb);
                            va = ld_acquire_gpu(fa);
                        }
                        while (vb < needb) {
                            watchdog_check(t0, 16, ((unsigned long long)item << 32) | (uint32_t)(T * 1024 + U), needb);
                            vb = ld_acquire_gpu(fb);
                        }
                        if (FFG_ROLE_PROF) w_dep += (unsigned long long)(clock64() - t0);
                        fence_proxy_async_global();
                    }
                    FFG_TIMED(w_empty, mbar_wait_at(empty_a + 8 * s, ((it / S_) & 1) ^ 1));
                    const uint32_t fbar = full_l0 + 8 * s;
                    if (p.dbg & 16) {  // measurement: no operand traffic (MMAs on stale smem)
                        mbar_arrive_cluster(fbar);
                        continue;
                    }
                    if (leader) mbar_expect_tx(&full[s], bytes);
                    uint8_t* st = smem + s * Cfg::kStageBytes;
                    const int kc = kb >> 1;
                    // operand tile rows P x K-block kb: K-major from block (P, kc) above the
                    // super-row, else MN-major from the stored transpose (kc, P)
                    auto load = [&](uint8_t* dst, const CUtensorMap* km, const CUtensorMap* mn, int P, int Srow) {
                        if (kc > 2 * Srow) {
                            tma_load_2d_pair(dst, km, fbar, kb * kBK, mrow + P * kBM);
                        } else {
                            tma_load_2d_pair(dst, mn, fbar, P * kBM, mrow + kb * kBK);
                            tma_load_2d_pair(dst + kOpBytes / 2, mn, fbar, P * kBM + 64, mrow + kb * kBK);
                        }
                    };
                    if (Tr::kHasLo) {
                        load(st, &tm.a_hi[par], &tm.b_hi[par], PA, S);
                        load(st + kOpBytes, &tm.a_lo[par], &tm.b_lo[par], PA, S);
                        load(st + 2 * kOpBytes, &tm.a_hi[par], &tm.b_hi[par], PB, T);
                        load(st + 3 * kOpBytes, &tm.a_lo[par], &tm.b_lo[par], PB, T);
                    } else {
                        load(st, &tm.a_hi[par], &tm.b_hi[par], PA, S);
                        load(st + kOpBytes, &tm.a_hi[par], &tm.b_hi[par], PB, T);
                    }
                }
            }
            if (FFG_ROLE_PROF && (p.dbg & 8)) {
                unsigned long long* o = p.prof + (size_t)blockIdx.x * 16;
                o[0] = (unsigned long long)(clock64() - t_start);
                o[1] = w_dep;
                o[2] = w_empty;
            }
        } else if (warp == 1 && leader) {
            // ================================================= UMMA issuer (leader CTA)
            constexpr uint32_t idesc0 = umma_idesc_f16(Tr::kFmt, 2 * kBM, kWideBN);
            constexpr uint32_t offAlo = kOpBytes;
            constexpr uint32_t offBhi = Tr::kHasLo ? 2 * kOpBytes : kOpBytes;
            constexpr uint32_t offBlo = 3 * kOpBytes;
            const uint32_t sbase = smem_u32(smem);
            int it = 0, g = 0;
            unsigned long long w_full = 0, w_slot = 0, w_slot2 = 0;
            for (int item = pair_id; item < total; item += n_pairs) {
                int m, l, pi;
                pair_decode(p, mm, item, m, l, pi);
                const uint32_t pr = __ldg(p.pairs + pi);
                const int S = pr & 1023, T = (pr >> 10) & 1023;
                const int kst = layer_kstep(l, p.exact_layers, p.semi_layers, p.normal_kstep);
                const bool kFixed = kDrain && kst == 0;
                if (p.products && lane == 0)
                    atomicAdd(&p.products[m], (uint32_t)(kFixed ? (FFG_FIXED_LOLO ? 4 : 3) : Tr::kProducts));
                uint32_t t_slot = 0, t_hh = 0, t_x = 0;
                auto open_slot = [&]() {
                    const int sl = g % kSlots;
                    FFG_TIMED(w_slot, mbar_wait_at(slot_empty_a + 8 * sl, ((g / kSlots) & 1) ^ 1));
                    tc_fence_after();
                    t_slot = tmem + sl * kWideBN;
                };
                auto close_slot = [&]() {
                    if (elect_one_sync()) umma_commit_pair(&slot_full[g % kSlots]);
                    __syncwarp();
                    ++g;
                };
                if (kFixed) {
                    const int s0 = g % kSlots, s1 = (g + 1) % kSlots;
                    FFG_TIMED(w_slot2, mbar_wait_at(slot_empty_a + 8 * s0, ((g / kSlots) & 1) ^ 1));
                    FFG_TIMED(w_slot2, mbar_wait_at(slot_empty_a + 8 * s1, (((g + 1) / kSlots) & 1) ^ 1));
                    tc_fence_after();
                    t_hh = tmem + s0 * kWideBN;
                    t_x = tmem + s1 * kWideBN;
                }
                if (!kDrain) open_slot();
                const int kbc = kDrain && !kFixed ? kst / (kBK / kUK) : 1;  // K-blocks per chunk
                for (int kb = 0; kb < nk; ++kb, ++it) {
                    const int s = it % S_;
                    FFG_TIMED(w_full, mbar_wait_at(full_a + 8 * s, (it / S_) & 1));
                    tc_fence_after();
                    const uint32_t st = sbase + s * Cfg::kStageBytes;
                    const bool amn = (kb >> 1) <= 2 * S, bmn = (kb >> 1) <= 2 * T;
                    const uint32_t idesc = idesc0 | ((uint32_t)amn << 15) | ((uint32_t)bmn << 16);
                    const uint64_t dAh = amn ? wdesc_mn(st) : wdesc_k(st);
                    const uint64_t dBh = bmn ? wdesc_mn(st + offBhi) : wdesc_k(st + offBhi);
                    const uint64_t aStep = amn ? 128u : 2u, bStep = bmn ? 128u : 2u;  // K16 (>> 4)
                    constexpr uint64_t kLo = kOpBytes >> 4;                            // hi -> lo
                    if (kFixed) {
                        if (elect_one_sync()) {
#pragma unroll
                            for (int kk = 0; kk < kBK / kUK; ++kk) {
                                const uint64_t da = dAh + kk * aStep, db = dBh + kk * bStep;
                                if (!(p.dbg & 2)) umma_f16_pair(t_x, da, db + kLo, idesc, (kb | kk) != 0);      // hi*lo
                                if (!(p.dbg & 2)) umma_f16_pair(t_x, da + kLo, db, idesc, 1u);                  // lo*hi
                                if (FFG_FIXED_LOLO && !(p.dbg & 2)) umma_f16_pair(t_x, da + kLo, db + kLo, idesc, 1u);
                                if (!(p.dbg & 2)) umma_f16_pair(t_hh, da, db, idesc, (kb | kk) != 0);           // hi*hi (exact)
                            }
                        }
                        __syncwarp();
                    } else if (!kDrain) {
                        if (elect_one_sync()) {
#pragma unroll
                            for (int kk = 0; kk < kBK / kUK; ++kk)
                                if (!(p.dbg & 2)) umma_f16_pair(t_slot, dAh + kk * aStep, dBh + kk * bStep, idesc, (kb | kk) != 0);
                        }
                        __syncwarp();
                    } else {
                        const bool first = kb % kbc == 0;
                        if (first) open_slot();
                        if (elect_one_sync()) {
#pragma unroll
                            for (int kk = 0; kk < kBK / kUK; ++kk) {
                                const uint64_t da = dAh + kk * aStep, db = dBh + kk * bStep;
                                if (!(p.dbg & 2)) umma_f16_pair(t_slot, da, db + kLo, idesc, !(first && kk == 0));
                                if (!(p.dbg & 2)) umma_f16_pair(t_slot, da + kLo, db, idesc, 1u);
                            }
#pragma unroll
                            for (int kk = 0; kk < kBK / kUK; ++kk)
                                if (!(p.dbg & 2)) umma_f16_pair(t_slot, dAh + kk * aStep, dBh + kk * bStep, idesc, 1u);
                        }
                        __syncwarp();
                        if (kb % kbc == kbc - 1 || kb == nk - 1) close_slot();
                    }
                    if (elect_one_sync()) umma_commit_pair(&empty[s]);
                    __syncwarp();
                }
                if (kFixed) {
                    if (elect_one_sync()) {
                        umma_commit_pair(&slot_full[g % kSlots]);
                        umma_commit_pair(&slot_full[(g + 1) % kSlots]);
                    }
                    __syncwarp();
                    g += 2;
                } else if (!kDrain) {
                    close_slot();
                }
            }
            if (FFG_ROLE_PROF && (p.dbg & 8) && lane == 0) {
                unsigned long long* o = p.prof + (size_t)blockIdx.x * 16;
                o[3] = w_full;
                o[4] = w_slot;
                o[5] = w_slot2;
            }
        }
        __syncwarp();
    } else {
        asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(kWRegsWork) : "memory");
        wide_workers<MODE>(p, mm, tmem, warp, lane, rank, pair_id, n_pairs, total, nk, nsb, slot_full, slot_empty,
                           red);
    }
    tc_fence_before();
    __syncthreads();
    cluster_sync_all();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc_pair(tmem, 512);
    }
}

}  // namespace ffg
