// K2 (pair form): the MLSP2 recursion layers on CTA pairs (tcgen05 cta_group::2).
//
// One launch runs layers [l0, l1) of a whole batch.  The unit of work is a PAIR ITEM: two
// 128x128 blocks of Y = X^2 that share their B panel S, computed by one M=256 x N=128 MMA
// over a CTA pair -- CTA rank c computes block (A_c, S) = panel A_c . panel S^T (X is
// symmetric, so every block is a product of two ROW panels and both UMMA operands are
// K-major row panels of the binary16 hi/lo split; no transpose pass).  The pair table
// (host: pair_table()) covers every block {R, C} of the upper triangle exactly once, in the
// orientation (A_c, S) chosen there; at most one dummy block per matrix.
//
// Items are ordered  group -> layer -> matrix in group -> pair  and dealt round-robin to the
// persistent CTA pairs.  A group of G matrices runs all its layers before the next group
// starts, so the group's working set (X, A, two hi/lo parities) stays resident in L2.  A
// layer-(l+1) item waits (producer thread, ld.acquire.gpu) until panels A_c and S of its
// matrix are complete at layer l: every block {P, *} increments counter[m][P] once per layer
// after its hi/lo stores have landed (cp.async.bulk.wait_group 0 + release).  Panel counts
// also order the WAR hazard on the hi/lo parity a layer overwrites: every reader of panels
// A_c and S at layer l-1 is one of the blocks those counters wait for.
//
// Single-matrix groups also track per-block completion (bflags) and a producer whose panels are
// not complete yet waits per 128-column block just before loading it.
//
// Per CTA (640 threads, warp-specialised, setmaxnreg 48/104/112; 16-worker variant 64/104):
//   warp 0        TMA producer: A_hi, A_lo (128 x 64) of panel A_c and this CTA's half
//                 (64 x 64) of B_hi, B_lo of panel S; complete_tx on the LEADER's full barrier
//   warp 1        TMEM allocator (both CTAs) / UMMA issuer (leader only)
//   warps 4-11    drain the chunk ring (round-to-nearest register sums) -> Y in TMEM
//   warps 12-19   epilogue (epilogue.cuh): X' = aY + bX + cI, A += d'X' (L2 reductions, paired
//                 over two layers), binary16 split, direct + mirrored 32x32 pieces by TMA store;
//                 last layer: D = A + X_L and the per-block statistics.
// Variants (template V): 0 the above, 2 sixteen workers that drain and finish one 32-column
// piece each (latency-bound layers; ffg_capi.cu use_s16).
// Matrices outside the model's region of validity (K1's Gershgorin bounds, the K3 formula
// matrix_in_region) never enter the item space: the prologue compacts the launch's matrices to
// the valid ones (MatrixMap) and the items walk only those -- no loads, no MMAs, no epilogue for an
// out-of-region matrix (K3 then writes its D as NaN).  The MMA issuer counts the products it issues
// per matrix (p.products).
// Accumulation precision: in the first `exact_layers` layers hi is a fixed-point split
// and hi*hi accumulates EXACTLY over the whole K in its own TMEM accumulator (cross terms and
// lo*lo in a second); later layers drain every two K-blocks into round-to-nearest registers.
#pragma once
#include <type_traits>

#include "epilogue.cuh"

namespace ffg {

#ifndef FFG_ROLE_PROF
#define FFG_ROLE_PROF 0
#endif
// measurement builds: per-item event times (PairParams::tl)
#define FFG_TL(item_, ev_)                                                                      \
    do {                                                                                        \
        if (FFG_ROLE_PROF && (p.dbg & 4096) && p.tl) {                                          \
            unsigned long long t_;                                                              \
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                              \
            p.tl[(size_t)(item_) * 12 + (ev_)] = t_;                                             \
        }                                                                                       \
    } while (0)
#define FFG_TLV(item_, ev_, v_)                                                                 \
    do {                                                                                        \
        if (FFG_ROLE_PROF && (p.dbg & 4096) && p.tl) p.tl[(size_t)(item_) * 12 + (ev_)] = (v_); \
    } while (0)


constexpr int kPairThreads = 640;
// setmaxnreg budgets per warpgroup (control / drain / epilogue); they only redistribute the
// launch allocation of 640 x 96 registers
#ifndef FFG_DRAIN_BATCH
#define FFG_DRAIN_BATCH 2  // x16 TMEM loads in flight per drain wait (1 or 2; measured: 2)
#endif
#if defined(FFG_P_CTL)
constexpr int kPRegsCtl = FFG_P_CTL, kPRegsDrain = FFG_P_DRAIN, kPRegsEpi = FFG_P_EPI;
#elif FFG_DRAIN_BATCH > 1
constexpr int kPRegsCtl = 48, kPRegsDrain = 104, kPRegsEpi = 112;
#else
constexpr int kPRegsCtl = 48, kPRegsDrain = 96, kPRegsEpi = 120;
#endif
static_assert(128 * kPRegsCtl + 256 * kPRegsDrain + 256 * kPRegsEpi <= 640 * 96, "setmaxnreg budget");
// 16-worker variant: 16 worker warps (drain + epilogue) own 32 columns each of the CTA's block
constexpr int kResWorkers = 16;
#ifndef FFG_R_CTL
// control warps' registers in the 16-worker variant: 64 (the whole 640 x 96 budget) keeps the producer's and
// the MMA issuer's K-loop state out of local memory (measured against 40: N=1024 single -7%, 16 x N=1024
// BF16 -2%)
#define FFG_R_CTL 64
#endif
constexpr int kRRegsCtl = FFG_R_CTL, kRRegsWork = 104;
static_assert(128 * kRRegsCtl + 512 * kRRegsWork <= 640 * 96, "setmaxnreg budget (16 workers)");
constexpr int kPairHalf = kBN / 2;                  // B rows supplied by each CTA
constexpr int kPairOpA = kBM * kBK * 2;             // 16 KB
constexpr int kPairOpB = kPairHalf * kBK * 2;       // 8 KB
// epilogue staging: 64 KB = 8 epilogue warps x four 2 KB pieces (direct + mirrored hi/lo), or
// 16 worker warps x two pieces (mirrors transposed in place)
constexpr int kPairStagingBytes = kEpiWarps2 * 4 * kPieceBytes;

#ifndef FFG_NARROW_STAGING
#define FFG_NARROW_STAGING 1  // streaming FP32E: two staging pieces per epilogue warp (mirrors in place), 4 stages
#endif
// Validity bitmap of a launch's matrices (at most kValidBits per launch; the host splits larger
// batches) in shared memory, filled in the prologue
constexpr int kValidBits = 8192;
// NARROW (streaming kernel, FP32E, FFG_NARROW_STAGING): 32 KB of staging buys a fourth operand stage
template <int MODE, bool NARROW = false>
struct PairCfg {
    static constexpr int kStagingBytes = NARROW ? kPairStagingBytes / 2 : kPairStagingBytes;
    static constexpr int kStageBytes = ModeTraits<MODE>::kHasLo ? 2 * (kPairOpA + kPairOpB)
                                                                : (kPairOpA + kPairOpB);
    static constexpr int kStages = (ModeTraits<MODE>::kHasLo ? 3 : 6) + (NARROW ? 1 : 0);
    static constexpr int kStagingOff = kStages * kStageBytes;
    static constexpr int kBarOff = kStagingOff + kStagingBytes;
    static constexpr int kValidOff = kBarOff + 1024;           // validity bitmap (kValidBits matrices)
    static constexpr int kSmem = kValidOff + kValidBits / 8 + 1024;  // + alignment slack
};
static_assert(PairCfg<kModeF32E>::kSmem <= 227 * 1024, "pair kernel smem");
static_assert(PairCfg<kModeBF16>::kSmem <= 227 * 1024, "pair kernel smem");
static_assert(PairCfg<kModeF32E, true>::kSmem <= 227 * 1024, "pair kernel smem");
template <int MODE, int V>
constexpr bool pair_narrow() { return FFG_NARROW_STAGING && V == 0 && ModeTraits<MODE>::kHasLo; }
static_assert(kEpiWarps == kEpiWarps2, "slot_empty counts drain and epilogue warps alike");

// TMEM: 4 slots x 128 columns.  A CHUNK is accumulated into the next slot of the ring.
// FP32-emulated: in the exact layers two whole-K chunks (hi*hi on the fixed-point split, exact;
// the cross terms), afterwards one chunk per two K-blocks with the cross terms issued first (hi*lo
// with accumulate=0, lo*hi) and hi*hi last (accumulation precision); single-product
// modes: the whole K extent.  The drain warps sum chunks in registers with round-to-nearest adds
// and write Y into the item's LAST slot, which the epilogue frees.
#ifndef FFG_BLOCK_DEPS
#define FFG_BLOCK_DEPS 1  // producer waits per 128-column block when a panel is incomplete (runtime: p.blockdeps)
#endif
#ifndef FFG_EPI_SPIN
#define FFG_EPI_SPIN 0  // epilogue warps spin on y_full instead of sleeping
#endif
#ifndef FFG_DEP_BACKOFF
#define FFG_DEP_BACKOFF 0  // ns of __nanosleep between panel-counter polls (0: tight poll)
#endif
#ifndef FFG_XA_AHEAD
#define FFG_XA_AHEAD 0  // items ahead the producer prefetches the epilogue's X/A block into L2
#endif
#ifndef FFG_DRAIN_SPIN
#define FFG_DRAIN_SPIN 1  // drain warps spin on slot_full (measured faster than sleeping)
#endif
#ifndef FFG_DRAIN_DEP
#define FFG_DRAIN_DEP 1  // order drain batches (see the drain loop)
#endif
#ifndef FFG_FIXED_SPLIT
#define FFG_FIXED_SPLIT 1  // FP32E: fixed-point hi (exact hi*hi accumulation), two accumulators per item
#endif
#ifndef FFG_FIXED_LOLO
#define FFG_FIXED_LOLO 1  // (with FFG_FIXED_SPLIT) the fourth product lo*lo into the cross accumulator
#endif
#ifndef FFG_EXACT_K16
#define FFG_EXACT_K16 1  // K16 steps per chunk in exact-drain layers (1 or 2)
#endif
#ifndef FFG_SEMI_DRAIN
#define FFG_SEMI_DRAIN 0  // compile the drain-every-2-K16 layers (FFG_SEMI_DRAIN_LAYERS, measurement)
#endif
__host__ __device__ constexpr int pair_chunks(int mode, int nk, bool exact) {
    return mode == kModeF32E ? (exact ? nk * (kBK / kUK) / FFG_EXACT_K16 : nk) : 1;
}
// K16 steps per chunk of layer l: FFG_EXACT_K16 in the exact-drain layers, 2 in the following
// `semi_layers`, a whole K-block (4) after that
__host__ __device__ constexpr int layer_kstep(int l, int exact_layers, int semi_layers, int normal_kstep) {
    return l < exact_layers ? (FFG_FIXED_SPLIT ? 0 : FFG_EXACT_K16)
                            : (l < exact_layers + semi_layers ? 2 : normal_kstep);
}
__host__ __device__ constexpr int layer_chunks(int mode, int nk, int kstep) {
    // kstep 0: fixed-point exact layer, two whole-K accumulators (hi*hi, cross terms); a chunk of
    // several K-blocks ends early at the last K-block
    return mode != kModeF32E ? 1
           : kstep == 0      ? 2
           : kstep <= kBK / kUK ? nk * (kBK / kUK) / kstep
                                : (nk + kstep / (kBK / kUK) - 1) / (kstep / (kBK / kUK));
}

struct PairMaps {
    CUtensorMap a_hi[2], a_lo[2];     // operand A boxes 64 x 128 (SW128), per hi/lo parity
    CUtensorMap b_hi[2], b_lo[2];     // operand B half boxes 64 x 64 (SW128)
    CUtensorMap p_hi[2], p_lo[2];     // epilogue store pieces 32 x 32 (SW64)
};

struct PairParams {
    const uint16_t* ophi[2];  // binary16 (bf16) operand arrays [B][np][np] per parity: the epilogue
    const uint16_t* oplo[2];  // rebuilds X_l from them (no fp32 master copy of X)
    float* A;                 // [B][nb][nb] tile-interleaved blocks (the blocks K2 touches)
    double* D;                // last layer: [B][n][n] fp64 (full storage) or null
    double2* partials;        // last layer: [B][2*PT] per block (sum diag, sum sq)
    int* flags;               // [B][2]
    uint32_t* counters;       // [B][nb] panel completion counts (zero at launch)
    uint32_t* bflags;         // [B][nb][nb] block completion counts, index min*nb+max (FFG_BLOCK_DEPS)
    int blockdeps;            // 1: producer waits per block while a panel is incomplete (host: G == 1)
    const uint32_t* pairs;    // [PT]  A0 | A1 << 10 | S << 20 | dummy << 30
    const float4* coef;       // [n_layers][2] hi/lo fp32 a, b, c, d_next (epilogue.cuh load_coef)
    int a_pair;               // paired A updates (odd layers reduce d_l X_l + d_{l+1} X_{l+1})
    int n, np, nb, PT;
    int B, G;                 // matrices, group size
    int l0, l1, n_layers;     // layers of this launch, model depth
    int exact_layers;
    int sr_layers;            // layers whose fixed-point split rounds lo stochastically (kernels.cuh)
    int semi_layers;          // layers after the exact ones draining every 2 K16 steps
    int normal_kstep;         // K16 steps per chunk in the remaining layers (4: one K-block, 8: two)
    int dbg;                  // measurement only: 1 skip epilogue math, 2 skip loads/MMAs,
                              // 4 skip dependency waits, 8 per-role wait cycles -> prof,
                              // 16 skip operand loads, 32 skip hi/lo stores, 64 skip X/A
                              // stores (A: reductions), 128 skip X loads (all measurement only: results are wrong);
                              // FFG_ROLE_PROF builds: 4096 per-item event times -> tl, 8192 16-worker drains
                              // without TMEM reads
    unsigned long long* prof; // [gridDim][16] (dbg & 8)
    unsigned long long* tl;   // [items][12] globaltimer per item (dbg & 4096, FFG_ROLE_PROF builds): producer
                              // start, first operand load issued, last chunk drained, published, first
                              // operands landed (MMA), last MMA issued, epilogue math done (S16), stores issued;
                              // cumulative wait cycles: MMA full at the item's end and after its first stage, producer deps, empty
    int m0;                   // first matrix of this launch
    uint32_t zero;            // always 0: an opaque operand for scheduling dependencies (drain)
    uint32_t* products;       // [B] tensor-core product passes issued per matrix (instrumented count)
    RegionCheck region;       // validity of each matrix from K1's bounds (kernels.cuh)
    int rowblock;             // row-block table (a rank's block rows x all columns): no mirrored
                              // hi/lo pieces or D entries off the diagonal blocks, each element counted once
    int drow0;                // row-block: first global row of D's row slab (D indexed (gi - drow0) * n + gj)
};

// The launch's matrices that are inside the region of validity: nvalid of the B, bit m of `valid`
// set for matrix m0 + m.  All valid (the normal case): item matrix index = position.  Otherwise
// position -> the position-th set bit (every role computes the same map).
struct MatrixMap {
    const uint32_t* valid;
    int nvalid;
    bool remap;
    __device__ __forceinline__ int matrix(int pos) const {
        if (!remap) return pos;
        int w = 0;
        for (;; ++w) {
            const int c = __popc(valid[w]);
            if (pos < c) break;
            pos -= c;
        }
        uint32_t bits = valid[w];
        for (int k = 0; k < pos; ++k) bits &= bits - 1;  // drop the lowest set bits
        return 32 * w + (__ffs(bits) - 1);
    }
};

__device__ __forceinline__ void pair_decode(const PairParams& p, const MatrixMap& mm, int item, int& m, int& l,
                                            int& pi) {
    const int L = p.l1 - p.l0;
    const int per_group = L * p.G * p.PT;
    const int g = item / per_group;
    const int base = g * p.G;
    const int Gg = min(p.G, mm.nvalid - base);
    int r = item - g * per_group;
    const int per_layer = Gg * p.PT;
    const int dl = r / per_layer;
    r -= dl * per_layer;
    const int mi = r / p.PT;
    pi = r - mi * p.PT;
    m = p.m0 + mm.matrix(base + mi);
    l = p.l0 + dl;
}



// Streaming 16-worker epilogue (kernel variant V = 2): warps 4-19 all work on every item.  Warp w:
// TMEM lane quarter q = w & 3 (rows 32q..32q+31), column quarter c = (w - 4) >> 2 (32 columns).
// The warp drains its 32 columns of every chunk into register sums and releases each TMEM slot
// as soon as it is read (Y never holds a slot, so the MMA always has the four-slot ring), then
// runs the epilogue of its 32x32 piece straight from those registers: one piece per warp per item
// instead of two, sixteen in flight per CTA.
template <int MODE>
__device__ __forceinline__ void stream16_workers(const PairMaps& tm, const PairParams& p, uint32_t tmem,
                                                 int warp, int lane, uint32_t rank, int pair_id, int n_pairs,
                                                 int total, int nk, uint64_t* slot_full, uint64_t* slot_empty,
                                                 uint8_t* staging, double* red, const MatrixMap& mm) {
    using Tr = ModeTraits<MODE>;
    const int wk = warp - 4, q = warp & 3, c = wk >> 2;
    const int r = q * 32 + lane;
    const int nb = p.nb, n = p.n, np = p.np;
    const uint32_t tl = tmem + ((uint32_t)(q * 32) << 16) + 32 * c;  // + slot * 128
    const float inv_s2 = 1.0f / (Tr::kScale * Tr::kScale);
    const uint32_t slot_empty_l0 = mapa_shared(smem_u32(&slot_empty[0]), 0);  // leader's
    const uint32_t slot_full_a = smem_u32(&slot_full[0]);
    uint8_t* stg = staging + wk * 2 * kPieceBytes;  // direct hi piece, lo piece (mirrors in place)
    const uint32_t stg_a = smem_u32(stg);
    int g = 0;
    for (int item = pair_id; item < total; item += n_pairs) {
        int m, l, pi;
        pair_decode(p, mm, item, m, l, pi);
        const int chunks = (p.dbg & 2) ? 1 : layer_chunks(MODE, nk, layer_kstep(l, p.exact_layers, p.semi_layers, p.normal_kstep));
        float yacc[32];
#pragma unroll
        for (int e = 0; e < 32; ++e) yacc[e] = 0.0f;
#pragma unroll 1
        for (int f = 0; f < chunks; ++f, ++g) {
            const int sl = g & 3;
            mbar_wait_at(slot_full_a + 8 * sl, (g >> 2) & 1);
            tc_fence_after();
            uint32_t v[32];
            if (FFG_ROLE_PROF && (p.dbg & 8192)) {  // measurement: no TMEM reads (results wrong)
#pragma unroll
                for (int e = 0; e < 32; ++e) v[e] = 0u;
            } else {
                tmem_ld_32x32b_x16(tl + sl * 128, *reinterpret_cast<uint32_t(*)[16]>(&v[0]));
                tmem_ld_32x32b_x16(tl + sl * 128 + 16, *reinterpret_cast<uint32_t(*)[16]>(&v[16]));
                tmem_ld_wait();
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster(slot_empty_l0 + 8 * sl);
#pragma unroll
            for (int e = 0; e < 32; e += 2) {
                const float2 acc = add_f32x2(make_float2(yacc[e], yacc[e + 1]),
                                             make_float2(__uint_as_float(v[e]), __uint_as_float(v[e + 1])));
                yacc[e] = acc.x;
                yacc[e + 1] = acc.y;
            }
        }
        if (wk == 0 && lane == 0 && rank == 0) FFG_TL(item, 2);
        // ------------------------------------------------------------- epilogue of the item
        const uint32_t pr = __ldg(p.pairs + pi);
        const int R = rank ? (pr >> 10) & 1023 : pr & 1023;
        const int C = (pr >> 20) & 1023;
        const bool dummy = rank && ((pr >> 30) & 1);
        const bool last = (l == p.n_layers - 1);
        const bool diag = R == C;
        const bool skip = dummy || (p.dbg & 1) || (diag && c < q);
        const bool dblk = diag && c == q;
        const bool mir = !p.rowblock || diag;  // row-block: no mirror of an off-diagonal block
        const int gi = R * kBM + r;
        const bool c_on = gi < n;
        EpiCoef k = load_coef(p.coef, l, p.n_layers, p.a_pair != 0);
        k.fixed = FFG_FIXED_SPLIT && MODE == kModeF32E && l + 1 < p.exact_layers;  // next layer exact
        k.sr = k.fixed && l + 1 < p.sr_layers;
        const int nxt = (l + 1) & 1;
        float* At = p.A + xa_tile_base(m, R, C, nb);
        // X_l of this thread's row in the block, from the layer's input operands (parity l & 1)
        const size_t xrow = ((size_t)m * np + gi) * np + (size_t)C * kBN;
        const uint16_t* xh = p.ophi[l & 1] + xrow;
        const uint16_t* xl = p.oplo[l & 1] + xrow;
        EpiHealth hl;
        double tr = 0.0, sq = 0.0;
        if (!skip) {
            if (!last) {
                if (lane == 0) tma_store_wait_read();  // the staging pieces are free again
                __syncwarp();
                XOp xq;
                if (!(p.dbg & 128)) load_xop(xh + 32 * c, xl + 32 * c, xq);
#pragma unroll
                for (int sub = 0; sub < 2; ++sub) {
                    const int c0 = 32 * c + 16 * sub;
                    XOp xn;
                    if (sub == 0 && !(p.dbg & 128)) load_xop(xh + c0 + 16, xl + c0 + 16, xn);
                    uint32_t v[16];
#pragma unroll
                    for (int e = 0; e < 16; ++e) v[e] = __float_as_uint(yacc[16 * sub + e] * inv_s2);
                    if (diag)
                        epi_sub_mid_red<MODE, true>(v, xq, At, r, c0, lane, sub, c_on, k, stg_a, dblk, hl,
                                                    gi, C * kBN, p.dbg & 64);
                    else
                        epi_sub_mid_red<MODE, false>(v, xq, At, r, c0, lane, sub, c_on, k, stg_a, false, hl,
                                                     gi, C * kBN, p.dbg & 64);
                    if (sub == 0) xq = xn;
                }
                if (wk == 0 && lane == 0 && rank == 0) FFG_TL(item, 6);
                if (!(p.dbg & 32)) {
                    fence_proxy_async_smem();
                    __syncwarp();
                    if (lane == 0) {
                        const int prow = m * np + R * kBM + 32 * q;  // direct piece origin
                        const int pcol = C * kBN + 32 * c;
                        tma_store_2d(&tm.p_hi[nxt], stg, pcol, prow);
                        tma_store_2d(&tm.p_lo[nxt], stg + kPieceBytes, pcol, prow);
                        tma_store_commit();
                    }
                    if (!dblk && mir) {  // mirrored pieces: transpose in place once the direct stores read them
                        if (lane == 0) tma_store_wait_read();
                        __syncwarp();
                        transpose_piece_inplace(stg_a, lane);
                        transpose_piece_inplace(stg_a + kPieceBytes, lane);
                        fence_proxy_async_smem();
                        __syncwarp();
                        if (lane == 0) {
                            const int mrow = m * np + C * kBN + 32 * c;
                            const int mcol = R * kBM + 32 * q;
                            tma_store_2d(&tm.p_hi[nxt], stg, mcol, mrow);
                            tma_store_2d(&tm.p_lo[nxt], stg + kPieceBytes, mcol, mrow);
                            tma_store_commit();
                        }
                    }
                }
            } else {
                double* Dm = p.D ? p.D + (size_t)m * n * n - (ptrdiff_t)p.drow0 * n : nullptr;
#pragma unroll
                for (int sub = 0; sub < 2; ++sub) {
                    const int c0 = 32 * c + 16 * sub;
                    uint32_t v[16];
#pragma unroll
                    for (int e = 0; e < 16; ++e) v[e] = __float_as_uint(yacc[16 * sub + e] * inv_s2);
                    XOp xo;
                    load_xop(xh + c0, xl + c0, xo);
                    if (diag)
                        epi_sub_last<MODE, true>(v, xo, At, r, c0, gi, C * kBN, n, c_on, k, Dm, hl, tr, sq);
                    else
                        epi_sub_last<MODE, false>(v, xo, At, r, c0, gi, C * kBN, n, c_on, k, Dm, hl, tr, sq, mir);
                }
            }
        }
        if (!dummy) {
            const bool any_nf = __any_sync(0xffffffffu, hl.nonfinite());
            const bool any_hr = !last && __any_sync(0xffffffffu, hl.template half_range<MODE>());
            if (lane == 0 && any_nf) atomicMin(&p.flags[2 * m + 0], l + 1);
            if (lane == 0 && any_hr) atomicMin(&p.flags[2 * m + 1], l + 1);
        }
        if (last) {
            // block statistics: one partial per 32x32 piece (index 4c + q), summed in piece order
            // (the same fixed order as the 8-warp epilogue)
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                tr += __shfl_xor_sync(0xffffffffu, tr, o);
                sq += __shfl_xor_sync(0xffffffffu, sq, o);
            }
            named_bar_sync(3, 16 * 32);  // the previous block's partial consumed
            if (lane == 0) {
                red[2 * wk + 0] = tr;
                red[2 * wk + 1] = sq;
            }
            named_bar_sync(3, 16 * 32);
            if (wk == 0 && lane == 0) {
                double T0 = 0.0, T1 = 0.0;
                for (int w = 0; w < 16; ++w) {  // fixed order
                    T0 += red[2 * w + 0];
                    T1 += red[2 * w + 1];
                }
                p.partials[(size_t)m * 2 * p.PT + 2 * pi + rank] = make_double2(T0, T1);
                if (rank == 0) FFG_TL(item, 3);
            }
        } else if (!dummy && l + 1 < p.l1) {
            // publish the block: hi/lo stores landed, X/A writes ordered -> block / panel counters
            if (wk == 0 && lane == 0 && rank == 0) FFG_TL(item, 7);
            if (lane == 0) {
                tma_store_wait_all();
                fence_proxy_async_global();
            }
            __syncwarp();
            named_bar_sync(4, 16 * 32);
            if (wk == 0 && lane == 0) {
                __threadfence();
                uint32_t* cm = p.counters + (size_t)m * nb;
                if (FFG_BLOCK_DEPS && MODE == kModeF32E && p.blockdeps)
                    red_relaxed_gpu_add(p.bflags + (size_t)m * nb * nb + (R < C ? R * nb + C : C * nb + R), 1u);
                red_relaxed_gpu_add(cm + R, 1u);
                if (C != R) red_relaxed_gpu_add(cm + C, 1u);
                if (rank == 0) FFG_TL(item, 3);
            }
        }
    }
    if (lane == 0) tma_store_wait_all();
}

// dbg & 8: accumulate the cycles a role spends in a wait into a register counter (measurement
// builds only, -DFFG_ROLE_PROF=1: the counters cost registers in roles at the edge of their budget)

#define FFG_TIMED(acc, stmt)                                     \
    do {                                                         \
        if (FFG_ROLE_PROF && (p.dbg & 8)) {                                         \
            const long long t_ = clock64();                      \
            stmt;                                                \
            acc += (unsigned long long)(clock64() - t_);         \
        } else {                                                 \
            stmt;                                                \
        }                                                        \
    } while (0)

#define FFG_TIMED_DRAIN(acc, stmt) FFG_TIMED(acc, stmt)

// V: 0 streaming (drain + epilogue warps), 2 streaming with 16 workers (S16)
template <int MODE, int V = 0>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kPairThreads, 1)
    mlsp2_pair_kernel(const __grid_constant__ PairMaps tm, const __grid_constant__ PairParams p) {
    static_assert(V == 0 || V == 2, "K2 variants: 0 streaming, 2 sixteen workers");
    constexpr bool S16 = V == 2;
    constexpr int kSlots = 4;  // TMEM chunk ring
    using Tr = ModeTraits<MODE>;
    constexpr bool kNarrow = pair_narrow<MODE, V>();
    using Cfg = PairCfg<MODE, kNarrow>;
    // (FP32-emulated only: a K-block pair there is 1.5K MMA cycles, enough to hide the polls)
    constexpr bool kBlockDeps = FFG_BLOCK_DEPS && Tr::kHasLo;
    constexpr bool kDrain = Tr::kProducts == 3;
    // per-K16 / per-2-K16 drain layers: only the FFG_FIXED_SPLIT=0 scheme or FFG_SEMI_DRAIN builds
    constexpr bool kExactPath = !FFG_FIXED_SPLIT || FFG_SEMI_DRAIN;
    constexpr int S = Cfg::kStages;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                               ~uintptr_t(1023));
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Cfg::kBarOff);
    uint64_t* full = bars;                 // [S]  leader: TMA bytes of both CTAs
    uint64_t* empty = bars + S;            // [S]  both: stage consumed (multicast commit)
    uint64_t* slot_full = bars + 2 * S;    // [4]  both: chunk accumulated in TMEM slot
    uint64_t* slot_empty = bars + 2 * S + 4;  // [4] leader: slot read by both CTAs
    uint64_t* y_full = bars + 2 * S + 8;   // [4]  local: Y formed in this slot (last chunk);
                                           //      two groups: [g] = group g drained an item
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * S + 12);
    double* red = reinterpret_cast<double*>(bars + 2 * S + 14);  // [16][2]
    // 32-bit shared addresses of the barriers (wait loops on generic pointers made ptxas
    // rematerialise the dynamic shared-memory base, with a spill, on every iteration)
    const uint32_t full_a = smem_u32(full), empty_a = smem_u32(empty), slot_full_a = smem_u32(slot_full),
                   slot_empty_a = smem_u32(slot_empty), y_full_a = smem_u32(y_full);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = cluster_ctarank();
    const bool leader = rank == 0;
    const int pair_id = blockIdx.x >> 1, n_pairs = gridDim.x >> 1;
    uint32_t* valid_bits = reinterpret_cast<uint32_t*>(smem + Cfg::kValidOff);
    const int nk = p.np / kBK;
    const int nb = p.nb;

    if (threadIdx.x == 0) {
        for (int i = 0; i < S; ++i) {
            mbar_init(&full[i], (p.dbg & 16) ? 2 : 1);
            mbar_init(&empty[i], 1);
        }
        for (int i = 0; i < 4; ++i) {
            mbar_init(&slot_full[i], 1);
            // drain warps, or epilogue warps (Y slot); S16: the 16 worker warps
            mbar_init(&slot_empty[i], S16 ? 2 * kResWorkers : 2 * kEpiWarps);
        }
        for (int i = 0; i < 4; ++i) mbar_init(&y_full[i], kEpiWarps);
        fence_barrier_init();
    }
    // validity bitmap of this launch's matrices (K1's bounds are final: K1 ran before this launch
    // in stream order)
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
    __syncthreads();  // (the cluster barrier already orders the slot write; this makes it visible to racecheck)
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    MatrixMap mm{valid_bits, 0, false};
    for (int wd = 0; wd < (p.B + 31) / 32; ++wd) mm.nvalid += __popc(valid_bits[wd]);
    mm.remap = mm.nvalid != p.B;
    const int total = (p.l1 - p.l0) * mm.nvalid * p.PT;

    if (warp < 4) {
        asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(S16 ? kRRegsCtl : kPRegsCtl) : "memory");
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
                if (rank == 0) FFG_TL(item, 0);
                const uint32_t pr = __ldg(p.pairs + pi);
                const int a0 = pr & 1023, a1 = (pr >> 10) & 1023, sp = (pr >> 20) & 1023;
                const int ap = rank ? a1 : a0;
                // block-granular dependencies: when a panel is not complete yet, each K-block
                // pair (one 128-column block of panels A_c and S) is waited for just before it is
                // loaded, so the item's first K-blocks overlap the previous layer's tail
                bool blockwise = false;
                if (kBlockDeps && p.blockdeps && l > p.l0 && !(p.dbg & 4)) {
                    const uint32_t need = (uint32_t)(nb * (l - p.l0));
                    const uint32_t* cm = p.counters + (size_t)m * nb;
                    blockwise = ld_acquire_gpu(cm + ap) < need || ld_acquire_gpu(cm + sp) < need;
                    if (!blockwise) fence_proxy_async_global();
                } else if (l > p.l0 && !(p.dbg & 4)) {
                    const uint32_t need = (uint32_t)(nb * (l - p.l0));
                    const uint32_t* cm = p.counters + (size_t)m * nb;
                    const long long t0 = clock64();
                    while (ld_acquire_gpu(cm + ap) < need && (FFG_DEP_BACKOFF ? (__nanosleep(FFG_DEP_BACKOFF), 1) : 1))
                        watchdog_check(t0, 3, ((unsigned long long)item << 32) | (uint32_t)(m * 1024 + ap),
                                       ((unsigned long long)need << 32) | ld_acquire_gpu(cm + ap));
                    while (ld_acquire_gpu(cm + sp) < need && (FFG_DEP_BACKOFF ? (__nanosleep(FFG_DEP_BACKOFF), 1) : 1))
                        watchdog_check(t0, 4, ((unsigned long long)item << 32) | (uint32_t)(m * 1024 + sp),
                                       ((unsigned long long)need << 32) | ld_acquire_gpu(cm + sp));
                    if (FFG_ROLE_PROF && (p.dbg & 8)) w_dep += (unsigned long long)(clock64() - t0);
                    fence_proxy_async_global();
                }
                // warm L2 with the X/A block the epilogue of a LATER item of this CTA will read
                // (FFG_XA_AHEAD items ahead; L2 is the coherence point, so an early prefetch
                // cannot serve stale data)
                if (!(p.dbg & 1)) {
                    const int ia = item + FFG_XA_AHEAD * n_pairs;
                    if (ia < total) {
                        int m2, l2, pi2;
                        pair_decode(p, mm, ia, m2, l2, pi2);
                        const uint32_t pr2 = __ldg(p.pairs + pi2);
                        if (!(rank && ((pr2 >> 30) & 1))) {
                            const int ap2 = rank ? (pr2 >> 10) & 1023 : pr2 & 1023;
                            const size_t tb = xa_tile_base(m2, ap2, (pr2 >> 20) & 1023, nb);
                            tma_prefetch_l2_bulk(p.A + tb, kBM * kBN * 4);
                        }
                    }
                }
                const int par = l & 1;
                const int rowA = m * p.np + ap * kBM;
                const int rowB = m * p.np + sp * kBN + (int)rank * kPairHalf;
                for (int kb = 0; kb < ((p.dbg & 2) ? 0 : nk); ++kb, ++it) {
                    const int s = it % S;
                    if (kBlockDeps && blockwise && (kb & 1) == 0) {
                        const int blk = kb >> 1;  // 128-column block of this K-block pair
                        const uint32_t need = (uint32_t)(l - p.l0);
                        const uint32_t* bf = p.bflags + (size_t)m * nb * nb;
                        const uint32_t* fa = bf + (ap < blk ? ap * nb + blk : blk * nb + ap);
                        const uint32_t* fs = bf + (sp < blk ? sp * nb + blk : blk * nb + sp);
                        const uint32_t* cm = p.counters + (size_t)m * nb;
                        const uint32_t needp = (uint32_t)(nb * (l - p.l0));
                        const long long t0 = clock64();
                        // the four polls in flight together; complete panels end the blockwise mode
                        uint32_t va = ld_acquire_gpu(fa), vs = ld_acquire_gpu(fs);
                        const uint32_t pa = ld_acquire_gpu(cm + ap), ps = ld_acquire_gpu(cm + sp);
                        if (pa >= needp && ps >= needp) blockwise = false;
                        while (va < need) {
                            watchdog_check(t0, 5, ((unsigned long long)item << 32) | (uint32_t)(ap * 1024 + blk), need);
                            va = ld_acquire_gpu(fa);
                        }
                        while (vs < need) {
                            watchdog_check(t0, 6, ((unsigned long long)item << 32) | (uint32_t)(sp * 1024 + blk), need);
                            vs = ld_acquire_gpu(fs);
                        }
                        if (FFG_ROLE_PROF && (p.dbg & 8)) w_dep += (unsigned long long)(clock64() - t0);
                        fence_proxy_async_global();
                    }
                    FFG_TIMED(w_empty, mbar_wait_at(empty_a + 8 * s, ((it / S) & 1) ^ 1));
                    const uint32_t fbar = mapa_shared(smem_u32(&full[s]), 0);
                    if (p.dbg & 16) {  // measurement: no operand traffic (MMAs on stale smem);
                        mbar_arrive_cluster(fbar);  // both CTAs arrive, keeping them in step
                        continue;
                    }
                    if (leader) mbar_expect_tx(&full[s], bytes);
                    uint8_t* st = smem + s * Cfg::kStageBytes;
                    tma_load_2d_pair(st, &tm.a_hi[par], fbar, kb * kBK, rowA);
                    if (Tr::kHasLo) {
                        tma_load_2d_pair(st + kPairOpA, &tm.a_lo[par], fbar, kb * kBK, rowA);
                        tma_load_2d_pair(st + 2 * kPairOpA, &tm.b_hi[par], fbar, kb * kBK, rowB);
                        tma_load_2d_pair(st + 2 * kPairOpA + kPairOpB, &tm.b_lo[par], fbar, kb * kBK, rowB);
                    } else {
                        tma_load_2d_pair(st + kPairOpA, &tm.b_hi[par], fbar, kb * kBK, rowB);
                    }
                    if (kb == 0 && rank == 0) FFG_TL(item, 1);
                }
                if (rank == 0) {
                    FFG_TLV(item, 10, w_dep);
                    FFG_TLV(item, 11, w_empty);
                }
            }
            if (FFG_ROLE_PROF && (p.dbg & 8)) {
                unsigned long long* o = p.prof + (size_t)blockIdx.x * 16;
                o[0] = (unsigned long long)(clock64() - t_start);
                o[1] = w_dep;
                o[2] = w_empty;
            }
        } else if (warp == 1 && leader) {
            // ================================================= UMMA issuer (leader CTA, whole
            // warp: descriptors are warp-uniform; one elected lane issues each instruction)
            constexpr uint32_t idesc = umma_idesc_f16(Tr::kFmt, 2 * kBM, kBN);
            constexpr uint32_t offAlo = kPairOpA;
            constexpr uint32_t offBhi = Tr::kHasLo ? 2 * kPairOpA : kPairOpA;
            constexpr uint32_t offBlo = 2 * kPairOpA + kPairOpB;
            const uint64_t desc0 = umma_desc_sw128(smem_u32(smem));  // stage 0, offset 0
            int it = 0, g = 0;
            unsigned long long w_full = 0, w_slot = 0;
            for (int item = pair_id; item < total; item += n_pairs) {
                int m, l, pi;
                pair_decode(p, mm, item, m, l, pi);
                const int kst = layer_kstep(l, p.exact_layers, p.semi_layers, p.normal_kstep);
                const bool exact = kst != 0 && kst < kBK / kUK;
                // cross-term order (pair-table bit 31): hi*lo then lo*hi, or swapped for an item
                // whose blocks are the transposes of blocks computed elsewhere in the other
                // orientation -- element (i, j) then gets exactly the value (j, i) gets there
                // (the products of each sum are the same; only their accumulation order matters)
                const bool swapx = (__ldg(p.pairs + pi) >> 31) & 1u;
                // the item's MMA sequence with the cross-term order fixed at compile time (no extra
                // registers in this 48-register role)
                auto run_item = [&](auto swap_tag) {
                constexpr bool kSwap = decltype(swap_tag)::value;
                constexpr uint32_t x1a = kSwap ? offAlo : 0u, x1b = kSwap ? offBhi : offBlo;
                constexpr uint32_t x2a = kSwap ? 0u : offAlo, x2b = kSwap ? offBlo : offBhi;
                uint32_t t_slot = 0;
                auto open_slot = [&]() {
                    const int sl = g % kSlots;
                    FFG_TIMED(w_slot, mbar_wait_at(slot_empty_a + 8 * sl, ((g / kSlots) & 1) ^ 1));
                    tc_fence_after();
                    t_slot = tmem + sl * 128;
                };
                auto close_slot = [&]() {
                    if (elect_one_sync()) umma_commit_pair(&slot_full[g % kSlots]);
                    __syncwarp();
                    ++g;
                };
                // descriptor of (stage base + byte offset): the start address field is addr>>4
                auto D = [&](uint64_t sbase, uint32_t off) { return sbase + (off >> 4); };
                // FFG_FIXED_SPLIT: hi*hi over the whole K in one accumulator (exact: every product
                // and partial sum lies on the 2^6 grid of the fixed-point hi, |sum| < 2^30), the cross
                // terms in a second; the drain adds the two once
                const bool kFixed = kDrain && kst == 0 && !(p.dbg & 2);
                // instrumented product count: product passes of this item
                if (p.products && lane == 0)
                    atomicAdd(&p.products[m], (uint32_t)(kFixed ? (FFG_FIXED_LOLO ? 4 : 3) : Tr::kProducts));
                uint32_t t_hh = 0, t_x = 0;
                if (kFixed) {
                    const int s0 = g % kSlots, s1 = (g + 1) % kSlots;
                    FFG_TIMED(w_slot, mbar_wait_at(slot_empty_a + 8 * s0, ((g / kSlots) & 1) ^ 1));
                    FFG_TIMED(w_slot, mbar_wait_at(slot_empty_a + 8 * s1, (((g + 1) / kSlots) & 1) ^ 1));
                    tc_fence_after();
                    t_hh = tmem + s0 * 128;
                    t_x = tmem + s1 * 128;
                }
                if (!kDrain) open_slot();
                for (int kb = 0; kb < ((p.dbg & 2) ? 0 : nk); ++kb, ++it) {
                    const int s = it % S;
                    FFG_TIMED(w_full, mbar_wait_at(full_a + 8 * s, (it / S) & 1));
                    if (kb == 0 && lane == 0) {
                        FFG_TL(item, 4);
                        FFG_TLV(item, 9, w_full);
                    }
                    tc_fence_after();
                    const uint64_t sb = desc0 + (uint64_t)((s * Cfg::kStageBytes) >> 4);
                    if (kFixed) {
                        if (elect_one_sync()) {
#pragma unroll
                            for (int kk = 0; kk < kBK / kUK; ++kk) {
                                const uint32_t koff = kk * kUK * 2;
                                umma_f16_pair(t_x, D(sb, x1a + koff), D(sb, x1b + koff), idesc, (kb | kk) != 0);
                                umma_f16_pair(t_x, D(sb, x2a + koff), D(sb, x2b + koff), idesc, 1u);
                                if (FFG_FIXED_LOLO)  // lo*lo: the fixed-point lo is absolute (~2^-12), not negligible
                                    umma_f16_pair(t_x, D(sb, offAlo + koff), D(sb, offBlo + koff), idesc, 1u);
                                umma_f16_pair(t_hh, D(sb, koff), D(sb, offBhi + koff), idesc, (kb | kk) != 0);
                            }
                        }
                        __syncwarp();
                    } else if (!kDrain) {
#pragma unroll
                        for (int kk = 0; kk < kBK / kUK; ++kk) {
                            const uint32_t koff = kk * kUK * 2;
                            if (elect_one_sync())
                                umma_f16_pair(t_slot, D(sb, koff), D(sb, offBhi + koff), idesc, (kb | kk) != 0);
                            __syncwarp();
                        }
                    } else if (kExactPath && exact) {
                        auto issue = [&](auto kc) {
                            constexpr int KST = decltype(kc)::value;
#pragma unroll
                            for (int k0 = 0; k0 < kBK / kUK; k0 += KST) {
                                open_slot();
                                if (elect_one_sync()) {
#pragma unroll
                                    for (int kk = k0; kk < k0 + KST; ++kk) {
                                        const uint32_t koff = kk * kUK * 2;
                                        umma_f16_pair(t_slot, D(sb, x1a + koff), D(sb, x1b + koff), idesc, kk != k0);
                                        umma_f16_pair(t_slot, D(sb, x2a + koff), D(sb, x2b + koff), idesc, 1u);
                                    }
#pragma unroll
                                    for (int kk = k0; kk < k0 + KST; ++kk) {
                                        const uint32_t koff = kk * kUK * 2;
                                        umma_f16_pair(t_slot, D(sb, koff), D(sb, offBhi + koff), idesc, 1u);
                                    }
                                }
                                __syncwarp();
                                close_slot();
                            }
                        };
                        if (kst == FFG_EXACT_K16)
                            issue(std::integral_constant<int, FFG_EXACT_K16>{});
                        else
                            issue(std::integral_constant<int, 2>{});
                    } else {
                        const int kbc = kst / (kBK / kUK);  // K-blocks per chunk
                        const bool first = kb % kbc == 0;
                        if (first) open_slot();
                        if (elect_one_sync()) {
#pragma unroll
                            for (int kk = 0; kk < kBK / kUK; ++kk) {
                                const uint32_t koff = kk * kUK * 2;
                                umma_f16_pair(t_slot, D(sb, x1a + koff), D(sb, x1b + koff), idesc, !(first && kk == 0));
                                umma_f16_pair(t_slot, D(sb, x2a + koff), D(sb, x2b + koff), idesc, 1u);
                            }
#pragma unroll
                            for (int kk = 0; kk < kBK / kUK; ++kk) {
                                const uint32_t koff = kk * kUK * 2;
                                umma_f16_pair(t_slot, D(sb, koff), D(sb, offBhi + koff), idesc, 1u);
                            }
                        }
                        __syncwarp();
                        if (kb % kbc == kbc - 1 || kb == nk - 1) close_slot();
                    }
                    if (elect_one_sync()) umma_commit_pair(&empty[s]);
                    __syncwarp();
                }
                if (lane == 0) {
                    FFG_TL(item, 5);
                    FFG_TLV(item, 8, w_full);
                }
                if (kFixed) {
                    if (elect_one_sync()) {
                        umma_commit_pair(&slot_full[g % kSlots]);
                        umma_commit_pair(&slot_full[(g + 1) % kSlots]);
                    }
                    __syncwarp();
                    g += 2;
                } else if (!kDrain || (p.dbg & 2)) {
                    if (kDrain) open_slot();
                    close_slot();
                }
                            };
                if (swapx)
                    run_item(std::true_type{});
                else
                    run_item(std::false_type{});
}
            if ((FFG_ROLE_PROF && (p.dbg & 8)) && lane == 0) {
                unsigned long long* o = p.prof + (size_t)blockIdx.x * 16;
                o[3] = w_full;
                o[4] = w_slot;
            }
        }
        __syncwarp();
    } else if constexpr (S16) {
        asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(kRRegsWork) : "memory");
        stream16_workers<MODE>(tm, p, tmem, warp, lane, rank, pair_id, n_pairs, total, nk, slot_full,
                               slot_empty, smem + Cfg::kStagingOff, red, mm);
    } else if (warp < 4 + kEpiWarps) {
        asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(kPRegsDrain) : "memory");
        // ===================================================== chunk drain -> Y (both CTAs)
        // (FP32-emulated only: single-product modes hand the accumulator to the epilogue)
        if constexpr (kDrain) {
            const int q = warp & 3;
            const int hc = (warp - 4) >> 2;
            const uint32_t tlane = tmem + ((uint32_t)(q * 32) << 16) + hc * kEpiCols;
            const float inv_s2 = 1.0f / (Tr::kScale * Tr::kScale);
            const uint32_t slot_empty_l0 = mapa_shared(smem_u32(&slot_empty[0]), 0);  // leader's
            int g = 0, u = 0;
            unsigned long long w_sf = 0;
            for (int item = pair_id; item < total; item += n_pairs, ++u) {
                int m, l, pi;
                pair_decode(p, mm, item, m, l, pi);
                const int chunks = (p.dbg & 2) ? 1 : layer_chunks(MODE, nk, layer_kstep(l, p.exact_layers, p.semi_layers, p.normal_kstep));
                float yacc[kEpiCols];
    #pragma unroll
                for (int e = 0; e < kEpiCols; ++e) yacc[e] = 0.0f;
    #pragma unroll 1
                for (int f = 0; f < chunks; ++f, ++g) {
                    const int sl = g & 3;
                    #if FFG_DRAIN_SPIN
                    FFG_TIMED_DRAIN(w_sf, mbar_wait_at(slot_full_a + 8 * sl, (g >> 2) & 1));
    #else
                    FFG_TIMED_DRAIN(w_sf, mbar_wait_at_sleep(slot_full_a + 8 * sl, (g >> 2) & 1));
    #endif
                    tc_fence_after();
                    const bool lastc = f == chunks - 1;
                    // ptxas hoists TMEM loads above the previous batch's adds, and the extra
                    // registers in flight spill two accumulator pairs (local stores to L2 every
                    // chunk); making each batch's load address depend on the previous batch's last
                    // sum (AND with the runtime zero p.zero) keeps one batch in flight
                    uint32_t dep = 0;
    #pragma unroll
                    for (int ch = 0; ch < 4; ch += FFG_DRAIN_BATCH) {
                        uint32_t v[16 * FFG_DRAIN_BATCH];
    #pragma unroll
                        for (int b = 0; b < FFG_DRAIN_BATCH; ++b)
                            tmem_ld_32x32b_x16(tlane + sl * 128 + (ch + b) * 16 + dep,
                                               *reinterpret_cast<uint32_t(*)[16]>(&v[16 * b]));
                        tmem_ld_wait();
                        if (ch + FFG_DRAIN_BATCH == 4 && !lastc) {
                            tc_fence_before();
                            __syncwarp();
                            if (lane == 0) mbar_arrive_cluster(slot_empty_l0 + 8 * sl);
                        }
    #pragma unroll
                        for (int e = 0; e < 16 * FFG_DRAIN_BATCH; e += 2) {
                            const float2 acc = add_f32x2(
                                make_float2(yacc[16 * ch + e], yacc[16 * ch + e + 1]),
                                make_float2(__uint_as_float(v[e]), __uint_as_float(v[e + 1])));
                            yacc[16 * ch + e] = acc.x;
                            yacc[16 * ch + e + 1] = acc.y;
                        }
                        if (FFG_DRAIN_DEP)
                            dep = (__float_as_uint(yacc[16 * ch + 16 * FFG_DRAIN_BATCH - 1]) |
                                   __float_as_uint(yacc[16 * ch])) & p.zero;
                    }
                }
                {  // Y into the item's last slot for the epilogue (which frees the slot); outside
                   // the chunk loop, so the loop keeps its registers for the sums in flight
                    const int sl = (g - 1) & 3;
    #pragma unroll
                    for (int ch = 0; ch < 4; ++ch) {
                        uint32_t v[16];
    #pragma unroll
                        for (int e = 0; e < 16; ++e) v[e] = __float_as_uint(yacc[16 * ch + e] * inv_s2);
                        tmem_st_32x32b_x16(tlane + sl * 128 + ch * 16, v);
                    }
                    tmem_st_wait();
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&y_full[sl]);
                }
            }
            if ((FFG_ROLE_PROF && (p.dbg & 8)) && warp == 4 && lane == 0) p.prof[(size_t)blockIdx.x * 16 + 5] = w_sf;
        }
    } else {
        asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(kPRegsEpi) : "memory");
        // ===================================================== epilogue (both CTAs)
        const int q = warp & 3;            // TMEM lane quarter = 32-row slice of the block
        const int s = (warp - 12) >> 2;    // column quarters s and s + 2
        const int ew = warp - 12;
        const int r = q * 32 + lane;       // block row of this thread
        const uint32_t tlane = tmem + ((uint32_t)(q * 32) << 16);
        const int np = p.np, n = p.n;
        uint8_t* stg = smem + Cfg::kStagingOff + ew * (kNarrow ? 2 : 4) * kPieceBytes;
        const uint32_t stg_a = smem_u32(stg);
        const uint32_t slot_empty_l0 = mapa_shared(smem_u32(&slot_empty[0]), 0);  // leader's
        int g = 0;
        uint32_t yph = 0;  // per-slot phase bits of y_full (a slot holds Y until freed here)
        unsigned long long w_y = 0, w_pub = 0, w_st = 0, w_cmp = 0, w_pc = 0, w_tail = 0, w_item = 0;
        for (int item = pair_id; item < total; item += n_pairs) {
            const long long t_item = (FFG_ROLE_PROF && (p.dbg & 8)) ? clock64() : 0;
            int m, l, pi;
            pair_decode(p, mm, item, m, l, pi);
            const uint32_t pr = __ldg(p.pairs + pi);
            const int R = rank ? (pr >> 10) & 1023 : pr & 1023;  // block rows (A panel)
            const int C = (pr >> 20) & 1023;                     // block cols (B panel)
            const bool dummy = rank && ((pr >> 30) & 1);
            const bool last = (l == p.n_layers - 1);
            EpiCoef k = load_coef(p.coef, l, p.n_layers, p.a_pair != 0);
            k.fixed = FFG_FIXED_SPLIT && MODE == kModeF32E && l + 1 < p.exact_layers;  // next layer exact
        k.sr = k.fixed && l + 1 < p.sr_layers;
            const int nxt = (l + 1) & 1;   // hi/lo parity written by this layer
            g += (p.dbg & 2) ? 1 : layer_chunks(MODE, nk, layer_kstep(l, p.exact_layers, p.semi_layers, p.normal_kstep));
            const int ysl = (g - 1) & 3;   // slot holding this item's Y
            const bool diag = R == C;
            const int gi = R * kBM + r;
            const bool c_on = gi < n;      // identity term only on real rows
            const uint32_t tacc = tlane + ysl * 128;
            float* At = p.A + xa_tile_base(m, R, C, nb);
            // X_l of this thread's row in the block, from the layer's input operands (parity l & 1)
            const size_t xrow = ((size_t)m * np + gi) * np + (size_t)C * kBN;
            const uint16_t* xh = p.ophi[l & 1] + xrow;
            const uint16_t* xl = p.oplo[l & 1] + xrow;
            EpiHealth hl;
            double tr = 0.0, sq = 0.0;
            double t0 = 0.0, s0 = 0.0, t1 = 0.0, s1 = 0.0;  // last layer: statistics per 32x32 piece
            // X of this warp's first sub-block is requested before the wait for Y; every
            // sub-block then requests the next one's X before computing (software pipeline)
            const bool ok0 = !(dummy || (p.dbg & 1) || (diag && s < q));
            const bool ok1 = !(dummy || (p.dbg & 1) || (diag && s + 2 < q));
            XOp xq;
            if (!last && (ok0 || ok1)) {
                // the block's X of layer l is complete once panel R is (the producer's
                // dependency wait; the early read must not rely on the wait for Y)
                if (l > p.l0 && !(p.dbg & 4)) {
                    if (lane == 0) {
                        if (kBlockDeps && p.blockdeps) {  // this block's own X of layer l
                            const uint32_t* f = p.bflags + (size_t)m * nb * nb + (R < C ? R * nb + C : C * nb + R);
                            while (ld_acquire_gpu(f) < (uint32_t)(l - p.l0)) {
                            }
                        } else {
                            const uint32_t need = (uint32_t)(nb * (l - p.l0));
                            while (ld_acquire_gpu(p.counters + (size_t)m * nb + R) < need) {
                            }
                        }
                    }
                    __syncwarp();
                }
                if (!(p.dbg & 128)) {
                    const int cq = 32 * (ok0 ? s : s + 2);
                    load_xop(xh + cq, xl + cq, xq);
                }
            }
            if constexpr (!kDrain) {
                // single-product modes: the slot holds the whole-K accumulator, read directly
                // (no drain pass); the 1/scale^2 is applied as it is loaded
                FFG_TIMED(w_y, mbar_wait_at_sleep(slot_full_a + 8 * ysl, ((g - 1) >> 2) & 1));
            } else {
#if FFG_EPI_SPIN
                FFG_TIMED(w_y, mbar_wait_at(y_full_a + 8 * ysl, (yph >> ysl) & 1));
#else
                FFG_TIMED(w_y, mbar_wait_at_sleep(y_full_a + 8 * ysl, (yph >> ysl) & 1));
#endif
                yph ^= 1u << ysl;
            }
            tc_fence_after();
#pragma unroll 1
            for (int qi = 0; qi < 2; ++qi) {
                const int qc = s + 2 * qi;  // column quarter (32 columns)
                // lower half of a diagonal block is mirrored from the upper half
                if (dummy || (p.dbg & 1) || (diag && qc < q)) {
                    if (lane == 0) tma_store_commit();
                    continue;
                }
                if (!last) {
                    if (lane == 0) FFG_TIMED(w_st, tma_store_wait_read());  // staging free again
                    __syncwarp();
                }
                const bool dblk = diag && qc == q;  // 32x32 piece on the matrix diagonal
                const bool mir = !p.rowblock || diag;  // row-block: no mirror of an off-diagonal block
                const long long t_c0 = (FFG_ROLE_PROF && (p.dbg & 8)) ? clock64() : 0;
#pragma unroll
                for (int sub = 0; sub < 2; ++sub) {
                    const int c0 = 32 * qc + 16 * sub;
                    uint32_t v[16];
                    tmem_ld_32x32b_x16(tacc + c0, v);
                    tmem_ld_wait();
                    if constexpr (!kDrain && Tr::kScale != 1.0f) {
#pragma unroll
                        for (int e = 0; e < 16; ++e)
                            v[e] = __float_as_uint(__uint_as_float(v[e]) * (1.0f / (Tr::kScale * Tr::kScale)));
                    }
                    if (!last) {
                        XOp xn;
                        const bool more = sub == 0 || (qi == 0 && ok1);
                        if (more && !(p.dbg & 128)) {
                            const int cn = sub == 0 ? c0 + 16 : 32 * (s + 2);
                            load_xop(xh + cn, xl + cn, xn);
                        }
                        if (diag)
                            epi_sub_mid_red<MODE, true>(v, xq, At, r, c0, lane, sub, c_on, k, stg_a, dblk, hl,
                                                        gi, C * kBN, p.dbg & 64);
                        else
                            epi_sub_mid_red<MODE, false>(v, xq, At, r, c0, lane, sub, c_on, k, stg_a, false, hl,
                                                         gi, C * kBN, p.dbg & 64);
                        if (more) xq = xn;
                    } else {
                        double* Dm = p.D ? p.D + (size_t)m * n * n - (ptrdiff_t)p.drow0 * n : nullptr;
                        XOp xo;
                        load_xop(xh + c0, xl + c0, xo);
                        if (diag)
                            epi_sub_last<MODE, true>(v, xo, At, r, c0, gi, C * kBN, n, c_on, k, Dm, hl, tr, sq);
                        else
                            epi_sub_last<MODE, false>(v, xo, At, r, c0, gi, C * kBN, n, c_on, k, Dm, hl, tr, sq, mir);
                    }
                }
                const long long t_c1 = (FFG_ROLE_PROF && (p.dbg & 8)) ? clock64() : 0;
                if (FFG_ROLE_PROF && (p.dbg & 8)) w_cmp += (unsigned long long)(t_c1 - t_c0);
                if (last) {  // this piece's statistics over the warp (fixed butterfly)
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) {
                        tr += __shfl_xor_sync(0xffffffffu, tr, o);
                        sq += __shfl_xor_sync(0xffffffffu, sq, o);
                    }
                    if (qi == 0) {
                        t0 = tr;
                        s0 = sq;
                    } else {
                        t1 = tr;
                        s1 = sq;
                    }
                    tr = sq = 0.0;
                }
                if (kNarrow && !last && !(p.dbg & 32)) {
                    // direct pieces out, then the mirrors transposed in place once the direct stores
                    // have read the staging
                    fence_proxy_async_smem();
                    __syncwarp();
                    if (lane == 0) {
                        tma_store_2d(&tm.p_hi[nxt], stg, C * kBN + 32 * qc, m * np + R * kBM + 32 * q);
                        tma_store_2d(&tm.p_lo[nxt], stg + kPieceBytes, C * kBN + 32 * qc, m * np + R * kBM + 32 * q);
                        tma_store_commit();
                    }
                    if (!dblk && mir) {
                        if (lane == 0) tma_store_wait_read();
                        __syncwarp();
                        transpose_piece_inplace(stg_a, lane);
                        transpose_piece_inplace(stg_a + kPieceBytes, lane);
                        fence_proxy_async_smem();
                        __syncwarp();
                        if (lane == 0) {
                            tma_store_2d(&tm.p_hi[nxt], stg, R * kBM + 32 * q, m * np + C * kBN + 32 * qc);
                            tma_store_2d(&tm.p_lo[nxt], stg + kPieceBytes, R * kBM + 32 * q, m * np + C * kBN + 32 * qc);
                        }
                    }
                } else if (!last) {
                    if (!dblk && mir) {  // mirrored pieces: warp transpose of the direct pieces
                        __syncwarp();
                        transpose_piece(stg_a, stg_a + 2 * kPieceBytes, lane);
                        transpose_piece(stg_a + kPieceBytes, stg_a + 3 * kPieceBytes, lane);
                    }
                    fence_proxy_async_smem();
                    __syncwarp();
                    if (lane == 0 && !(p.dbg & 32)) {
                        const int prow = m * np + R * kBM + 32 * q;   // direct piece origin
                        const int pcol = C * kBN + 32 * qc;
                        tma_store_2d(&tm.p_hi[nxt], stg, pcol, prow);
                        tma_store_2d(&tm.p_lo[nxt], stg + kPieceBytes, pcol, prow);
                        if (!dblk && mir) {
                            const int mrow = m * np + C * kBN + 32 * qc;
                            const int mcol = R * kBM + 32 * q;
                            tma_store_2d(&tm.p_hi[nxt], stg + 2 * kPieceBytes, mcol, mrow);
                            tma_store_2d(&tm.p_lo[nxt], stg + 3 * kPieceBytes, mcol, mrow);
                        }
                    }
                }
                if (lane == 0) tma_store_commit();  // one bulk group per quarter, possibly empty
                if (FFG_ROLE_PROF && (p.dbg & 8)) w_pc += (unsigned long long)(clock64() - t_c1);
            }
            const long long t_tail = (FFG_ROLE_PROF && (p.dbg & 8)) ? clock64() : 0;
            // this warp's Y reads are done: release the pair's TMEM slot
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster(slot_empty_l0 + 8 * ysl);
            if (!dummy) {
                const bool any_nf = __any_sync(0xffffffffu, hl.nonfinite());
                const bool any_hr = !last && __any_sync(0xffffffffu, hl.template half_range<MODE>());
                if (lane == 0 && any_nf) atomicMin(&p.flags[2 * m + 0], l + 1);
                if (lane == 0 && any_hr) atomicMin(&p.flags[2 * m + 1], l + 1);
            }
            if (last) {
                // block statistics: the 16 piece partials (index 4 * quarter + lane quarter) summed in
                // piece order -- the same fixed order as the 16-worker epilogue
                named_bar_sync(3, kEpiWarps2 * 32);  // previous block's partial consumed
                if (lane == 0) {
                    red[2 * (4 * s + q) + 0] = t0;
                    red[2 * (4 * s + q) + 1] = s0;
                    red[2 * (4 * (s + 2) + q) + 0] = t1;
                    red[2 * (4 * (s + 2) + q) + 1] = s1;
                }
                named_bar_sync(3, kEpiWarps2 * 32);
                if (ew == 0 && lane == 0) {
                    double T0 = 0.0, T1 = 0.0;
                    for (int w = 0; w < 16; ++w) {  // fixed order
                        T0 += red[2 * w + 0];
                        T1 += red[2 * w + 1];
                    }
                    p.partials[(size_t)m * 2 * p.PT + 2 * pi + rank] = make_double2(T0, T1);
                }
            } else if (!dummy && l + 1 < p.l1) {
                // publish the block: hi/lo stores landed, X/A stores visible -> panel counters
                const long long tp = clock64();
                if (lane == 0 && !(p.dbg & 256)) {  // dbg & 256: measurement only, no wait
                    tma_store_wait_all();
                    fence_proxy_async_global();
                }
                __syncwarp();
                if (p.dbg & 256) {
                    if (ew == 0 && lane == 0) {
                        uint32_t* cm = p.counters + (size_t)m * nb;
                        red_relaxed_gpu_add(cm + R, 1u);
                        if (C != R) red_relaxed_gpu_add(cm + C, 1u);
                    }
                } else {
                    named_bar_sync(4, kEpiWarps2 * 32);
                    if (ew == 0 && lane == 0) {
                        __threadfence();
                        uint32_t* cm = p.counters + (size_t)m * nb;
                        // the fence above orders this block's writes before all three increments
                        if (kBlockDeps && p.blockdeps)
                            red_relaxed_gpu_add(p.bflags + (size_t)m * nb * nb + (R < C ? R * nb + C : C * nb + R), 1u);
                        red_relaxed_gpu_add(cm + R, 1u);
                        if (C != R) red_relaxed_gpu_add(cm + C, 1u);
                    }
                }
                if (FFG_ROLE_PROF && (p.dbg & 8)) w_pub += (unsigned long long)(clock64() - tp);
            }
            if (FFG_ROLE_PROF && (p.dbg & 8)) {
                const long long te = clock64();
                w_tail += (unsigned long long)(te - t_tail);
                w_item += (unsigned long long)(te - t_item);
            }
        }
        if (lane == 0) tma_store_wait_all();
        if ((FFG_ROLE_PROF && (p.dbg & 8)) && warp == 12 && lane == 0) {
            unsigned long long* o = p.prof + (size_t)blockIdx.x * 16;
            o[6] = w_y;
            o[7] = w_pub;
            o[8] = w_st;
            o[9] = w_cmp;
            o[10] = w_pc;
            o[11] = w_tail;
            o[12] = w_item;
        }
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
