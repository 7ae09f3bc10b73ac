/*
 * fermiforge B200 C ABI -- the drop-in boundary of the finite-temperature
 * density-matrix builder (MLSP2 recursion) on sm_100a.
 *
 * Plain C: pointers, sizes, doubles.  No C++ or CUDA types in any signature
 * (streams are passed as `void*` = cudaStream_t).  Implemented by
 * paper_2605_08523_b200/lib/libfermiforge_b200.so (hand-written sm_100a CUDA,
 * no CPU fallback: every compute entry point returns FFG_ERR_CUDA when no
 * sm_100 device is present).
 *
 * Each entry point replaces a reference interface.  The reference specifies the
 * matrix path in SPEC.md (module matrix_engine / workflow) on top of the
 * proj/core types; citations are file:line relative to the reference root:
 *
 *   ffg_spectral_bounds        SPEC.md:319-327  spectral_bounds(H) -> SpectralBounds
 *   ffg_in_region_of_validity  SPEC.md:349-357  in_region_of_validity(beta', mu', beta0, mu0)
 *   ffg_apply_model            SPEC.md:359-367  apply_model(H0, m, mode)
 *   ffg_mixed_square           SPEC.md:369-377  mixed_square(X)
 *   ffg_density_statistics     SPEC.md:389-397  density_statistics(D)
 *   ffg_density_matrix         SPEC.md:458-462  compute_density_matrix(H, beta, mu, lib, mode)
 *                              (model already selected; the B200 north-star entry
 *                              "H, mu, kT, coefficients -> D, Tr D")
 *   ffg_density_matrices       batched compute_density_matrix (no reference
 *                              counterpart)
 *   ffg_density_matrices_dev   the same on device-resident buffers, asynchronous
 *                              on a caller stream
 *   ffg_rowblock_*             one large H row-block sharded over `world` GPUs, one rank per
 *                              process (the reference permits data-parallel
 *                              matmul with deterministic reductions)
 *
 * Coefficients are the reference's Mlsp2Coefficients rows
 * (proj/core/include/fermiforge/scalar_models.hpp:80-88: a, b, c, d per layer)
 * with ModelCoefficients::trained_at = (beta0, mu0) (scalar_models.hpp:173-183).
 * The model is evaluated exactly as evaluate_model (scalar_models.cpp:330-333,
 * 243-252): X0 = (1 - mu0) I - (beta/beta0)(H - mu I); per layer
 * A += d X; X = a X^2 + b X + c I; D = A + X.
 *
 * Errors: every function returns an ffg_status; ffg_last_error() gives a
 * thread-local message naming the violated condition, mirroring the reference
 * exceptions (ValidationError scalar_models.hpp:21-24, out-of-region SPEC.md:343,
 * DivergedEvaluationError trainer.hpp:20-25, HalfRangeError half_precision.hpp:13-16,
 * std::invalid_argument on dimension mismatch symmetric_matrix.cpp:31).
 *
 * Threading: every entry point is re-entrant; device workspaces are cached
 * per (device, stream) under a mutex.  All reductions are fixed-order, so
 * results are bit-reproducible for a given device, n and batch.
 */
#ifndef FERMIFORGE_FFG_H
#define FERMIFORGE_FFG_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FFG_ABI_VERSION 1

typedef enum ffg_status {
    FFG_OK = 0,
    FFG_ERR_VALIDATION = 1,    /* ValidationError: bad coefficients / kT / mode / sizes   */
    FFG_ERR_OUT_OF_REGION = 2, /* rescale_to_model: (beta', mu') outside Eq. 41            */
    FFG_ERR_DIVERGED = 3,      /* non-finite entry mid-recursion (layer in provenance)     */
    FFG_ERR_HALF_RANGE = 4,    /* binary16 split overflow (HalfRangeError)                 */
    FFG_ERR_UNSUPPORTED = 5,   /* a mode an entry point does not run (e.g. row-block DOUBLE) */
    FFG_ERR_DIMENSION = 6,     /* std::invalid_argument: dimension mismatch                */
    FFG_ERR_CUDA = 7,          /* no sm_100 device, launch or allocation failure           */
    FFG_ERR_NCCL = 8
} ffg_status;

/* PrecisionMode plus the two north-star low-precision modes. */
typedef enum ffg_mode {
    FFG_MODE_DOUBLE = 0,          /* fp64 recursion: library DGEMM + our layer kernels       */
    FFG_MODE_SINGLE = 1,          /* fp32 recursion: library SGEMM (no TF32) + our kernels   */
    FFG_MODE_MIXED_EMULATED = 2,  /* FP32-emulated: binary16 hi/lo split (x 2^14 pre-scale),
                                     hi*hi + hi*lo + lo*hi with FP32 accumulation (Eq. 48) */
    FFG_MODE_BF16 = 3,            /* one bf16 product per square, FP32 accumulation          */
    FFG_MODE_FP16 = 4             /* one binary16 product per square (x 2^14), FP32 accum.   */
} ffg_mode;

/* An MLSP2 ModelCoefficients, borrowed for the duration of a call. */
typedef struct ffg_model {
    const double* abcd; /* n_layers rows of {a, b, c, d}                          */
    int32_t n_layers;   /* >= 1                                                   */
    double beta0;       /* trained_at.beta  (> 0, finite)                         */
    double mu0;         /* trained_at.mu    (in (0, 1))                           */
} ffg_model;

/* Provenance record. */
typedef struct ffg_provenance {
    double eps_min, eps_max;  /* widened Gershgorin bounds of H                         */
    double beta_prime;        /* SPEC normalize_problem: beta' = (eps_max - eps_min) beta */
    double mu_prime;          /* SPEC (flipped) mu' = (eps_max - mu) / (eps_max - eps_min) */
    double x_min, x_max;      /* bounds mapped into the model's un-flipped frame:
                                 x = mu0 + (beta/beta0)(eps - mu); valid iff in [0,1]    */
    int32_t mode;
    int32_t n_layers;
    int64_t half_products;    /* tensor-core products per square summed over the layers,
                                 counted by the K2 issuer: each covers the
                                 upper-triangle blocks; FP32-emulated 3 per square (4 in the
                                 fixed-point exact layers), BF16/FP16 1; 0 when no recursion
                                 ran (out of region)                                     */
    int32_t diverged_layer;   /* first X_k (k = 0..L) non-finite, -1 if none              */
    int32_t half_range_layer; /* first X_k whose binary16 split overflowed, -1 if none    */
    int32_t status;           /* ffg_status of this matrix                                */
    int32_t n;
    double device_ms;         /* device time: rescale + L layers + statistics            */
} ffg_provenance;

int ffg_abi_version(void);
const char* ffg_last_error(void);
/* 1 when an sm_100 device is usable, else 0 (ffg_last_error says why). */
int ffg_device_available(void);

/* SPEC.md:349-357, Eq. 41: (mu0/mu')beta0 >= beta' and ((1-mu0)/(1-mu'))beta0 >= beta',
 * with mu' in the reference model's UN-flipped frame (mu' = (mu - eps_min)/W).
 * Returns 1 valid / 0 not valid.  Pure host function. */
int ffg_in_region_of_validity(double beta_prime, double mu_prime, double beta0, double mu0);

/* Gershgorin bounds of a host matrix, computed on the device (K1). */
int ffg_spectral_bounds(const double* H, int64_t n, double* eps_min, double* eps_max);

/* D = p(H0) for H0 already in the model frame (SPEC apply_model).  D_out n*n. */
int ffg_apply_model(const double* H0, int64_t n, const ffg_model* model, int32_t mode,
                    double* D_out, ffg_provenance* prov);

/* Y = mixed_square(X) on the tensor cores (one FP32-emulated square, fp32 in/out). */
int ffg_mixed_square(const float* X, int64_t n, float* Y_out);

/* (Tr D, sum_ij D_ij^2) of a host matrix (fixed-order device reduction). */
int ffg_density_statistics(const double* D, int64_t n, double* stats_out);

/* North-star entry: H (n*n row-major fp64, exactly symmetric), mu, kT -> D, stats.
 * D_out may be NULL (statistics only).  stats_out = {Tr D, Tr D^2}, may be NULL. */
int ffg_density_matrix(const double* H, int64_t n, double mu, double kT, const ffg_model* model,
                       int32_t mode, double* D_out, double* stats_out, ffg_provenance* prov);

/* Batched: `batch` independent H (host pointers), per-matrix mu / kT.
 * D_out may be NULL or hold NULL entries; stats_out batch*2; prov batch entries or NULL.
 * Returns FFG_OK when every matrix succeeded, else the first failing status.  A matrix outside
 * the region of validity runs no recursion and its D is NaN. */
int ffg_density_matrices(int32_t batch, const double* const* H, int64_t n, const double* mu,
                         const double* kT, const ffg_model* model, int32_t mode,
                         double* const* D_out, double* stats_out, ffg_provenance* prov);

/* Asynchronous form of ffg_density_matrices for pipelined callers (a serving loop): enqueues
 * the chunked H2D / compute / D2H pipeline and returns a ticket at once; at most three calls may
 * be in flight, so a caller overlaps step k's transfers with the neighbouring steps' compute.  H and D_out
 * must stay valid (page-locked for overlap) until ffg_wait(ticket) returns; stats / prov /
 * status are delivered by ffg_wait. */
int ffg_density_matrices_async(int32_t batch, const double* const* H, int64_t n, const double* mu,
                               const double* kT, const ffg_model* model, int32_t mode,
                               double* const* D_out, int64_t* ticket);
int ffg_wait(int64_t ticket, double* stats_out, ffg_provenance* prov);

/* Device-resident batch, asynchronous on `stream` (cudaStream_t, NULL = default):
 * H_dev [batch][n][n] fp64; mu / kT host arrays (copied at call time);
 * D_dev [batch][n][n] fp64 or NULL; stats_dev [batch][2]; status_dev [batch] int32
 * (ffg_status per matrix); bounds_dev [batch][4] (eps_min, eps_max, x_min, x_max)
 * or NULL.  Returns after enqueueing; host-side validation errors are synchronous. */
int ffg_density_matrices_dev(int32_t batch, const double* H_dev, int64_t n, const double* mu,
                             const double* kT, const ffg_model* model, int32_t mode,
                             double* D_dev, double* stats_dev, int32_t* status_dev,
                             double* bounds_dev, void* stream);

/* ---------------------------------------------------------------- row-block sharding
 * One H of size n split by block rows (128-row blocks, nb = ceil(n/128), nb % world == 0) over
 * `world` ranks, one process per GPU.  Rank r owns block rows [r nb/world, (r+1) nb/world) of X,
 * A and D and computes those rows against ALL columns each layer; between layers every rank needs
 * every rank's rows of the binary16 operands X_{l+1} (hi / lo): the caller all-gathers them
 * in place (NCCL) -- the operand buffers are [np][np] row-major with this rank's rows at
 * [row0, row0 + rows) and the same layout on every rank.  Each block is computed with the exact
 * arithmetic of the single-GPU path (pair-table cross-order bit), so the assembled D equals the
 * single-GPU D bit for bit.
 *
 *   h = ffg_rowblock_begin(...)        K1 on the whole (replicated) H: operands of X_0 for every
 *                                      row, X_0 / A_1 for this rank's rows, Gershgorin bounds
 *   for l in 0 .. L-1:
 *       ffg_rowblock_layer(h, l, ...)  layer l on this rank's rows (reads operand parity l & 1,
 *                                      writes this rank's rows of parity (l + 1) & 1; the last
 *                                      layer writes D_rows and the statistics partials)
 *       all-gather parity (l + 1) & 1  (caller; not after the last layer)
 *   ffg_rowblock_end(h, ...)           this rank's partial {sum_i D_ii, sum_ij D_ij^2} over its
 *                                      rows, status; frees the handle
 * All calls are asynchronous on `stream` except end (synchronises). */
typedef struct ffg_rowblock ffg_rowblock;
int ffg_rowblock_begin(const double* H_dev, int64_t n, double mu, double kT, const ffg_model* model,
                       int32_t mode, int32_t rank, int32_t world, void* stream, ffg_rowblock** handle);
/* this rank's element rows [row0, row0 + rows) (rows of D_rows: min(row0 + rows, n) - row0), np */
int ffg_rowblock_rows(const ffg_rowblock* h, int64_t* row0, int64_t* rows, int64_t* np);
/* device pointers of operand parity `parity` (0/1): hi and lo ([np][np] uint16; lo NULL in
 * BF16 / FP16 mode) */
int ffg_rowblock_operands(ffg_rowblock* h, int32_t parity, void** hi, void** lo);
/* layer `layer` (0 .. n_layers-1, in order); D_rows [rows][n] fp64 device, used by the last layer */
int ffg_rowblock_layer(ffg_rowblock* h, int32_t layer, double* D_rows, void* stream);
/* partial_stats: {sum over this rank's rows of D_ii, of D_ij^2}; status: ffg_status of the matrix
 * (out of region, diverged, half range); prov may be NULL. */
int ffg_rowblock_end(ffg_rowblock* h, double* partial_stats, int32_t* status, ffg_provenance* prov,
                     void* stream);

/* ---------------------------------------------------------------- workflow
 * Callers of the density-matrix path built on the same pipeline: every call below runs
 * K1 -> K2 -> K3 only; the statistics (Tr D, Tr D^2) that K3 already produces supply the
 * Newton derivative and the entropy trace, so none needs an extra matrix multiply. */

/* An entropy model (Architecture::Entropy, scalar_models.hpp:150-156; evaluate_entropy
 * scalar_models.cpp:320-326): inner MLSP2 rows evaluated at x0 = alpha (x - mu0) + mu0 with
 * no spectrum flip, s = (4 ln 2) y (1 - y).  inner.beta0 / inner.mu0 are the trained_at of
 * the Fermi model it pairs with (pairing by exact (beta0, mu0)). */
typedef struct ffg_entropy_model {
    ffg_model inner;
    double alpha;       /* in (0, 1) */
} ffg_entropy_model;

/* SPEC thermodynamics: entropy_trace = Tr s(H) for the Fermi function at
 * (mu, kT), computed as (4 ln 2)(Tr Y - Tr Y^2) with Y the inner recursion's output (the
 * fused statistics of K3: no extra GEMM for the final (4 ln 2) Y (I - Y) layer). */
int ffg_entropy_trace(const double* H, int64_t n, double mu, double kT, const ffg_entropy_model* em,
                      int32_t mode, double* entropy_trace, ffg_provenance* prov);

/* SPEC expectation (Eq. 9): <A> = Tr(D A) = sum_ij D_ij A_ij for symmetric
 * D, A (fixed-order device reduction).  Band energy = expectation(D, H - mu I). */
int ffg_expectation(const double* D, const double* A, int64_t n, double* out);

/* SPEC solve_chemical_potential (Eqs. 42-45): Newton iteration on
 * g(mu) = Tr D(mu) - n_occ with g'(mu) = beta (Tr D - Tr D^2) (Eq. 44, from the fused
 * statistics), steps clamped to half the spectral width, safeguarded by a bracket of the
 * model's region of validity; bisection when g' < 1e-14 beta n (flat derivative).  One
 * K1 -> K2 -> K3 run per iteration on the device-resident H. */
typedef struct ffg_mu_report {
    double mu;            /* final chemical potential (energy units of H)            */
    double residual;      /* Tr D(mu) - n_occ                                       */
    int32_t iterations;   /* density-matrix evaluations                             */
    int32_t converged;    /* |residual| <= tol                                      */
    int32_t bisections;   /* steps taken by bisection instead of Newton             */
} ffg_mu_report;
/* D_out (n*n) and stats_out ({Tr D, Tr D^2}) are for the final mu and may be NULL;
 * history (2*max_iter doubles: mu_k, residual_k) may be NULL. */
int ffg_solve_chemical_potential(const double* H, int64_t n, double kT, double n_occ, double mu_guess,
                                 const ffg_model* model, int32_t mode, double tol, int32_t max_iter,
                                 double* D_out, double* stats_out, double* history,
                                 ffg_mu_report* report);

/* Number of kernels ffg_density_matrices_dev launches for one call (for accounting). */
int64_t ffg_kernel_launches(int32_t batch, int64_t n, const ffg_model* model, int32_t mode);

/* Which recursion kernel (K2) computes matrices of order n in `mode` (the choice depends only on
 * n and the mode; FFG_WIDE=0/1 overrides): 0 = mlsp2_pair_kernel (256 x 128 pair items),
 * 1 = mlsp2_wide_kernel (256 x 256 super-block items), 2 = DOUBLE / SINGLE (cuBLAS {D,S}gemm for the
 * square + direct.cuh layer kernels), negative = unsupported mode / size. */
int32_t ffg_k2_kernel(int64_t n, int32_t mode);

/* Measurement hooks (bench.py): when enabled, every recursion-kernel (K2) launch is
 * bracketed by CUDA events on its stream; ffg_profile_read() synchronises them and
 * returns the summed device time and launch count since the last read. */
int ffg_profile_layers(int enable);
int ffg_profile_read(double* total_ms, int64_t* launches);
/* The same, plus the algorithmic flops (L * c * N^2 (N+1) per matrix) of
 * the profiled launches. */
int ffg_profile_read_ex(double* total_ms, int64_t* launches, double* algorithmic_flops);
/* Introspection of the K2 work decomposition (pure host): the pair table for an nb x nb
 * grid of 128-blocks, entries A0 | A1 << 10 | S << 20 | dummy << 30 | swap << 31 (blocks
 * (A0,S) and (A1,S) share B panel S; swap: cross terms in swapped order).  Writes
 * min(count, capacity) entries; returns count, -1 on bad arguments.  ffg_rowblock_table: rank
 * `rank` of `world`'s row-block table. */
int32_t ffg_pair_table(int32_t nb, uint32_t* out, int32_t capacity);
int32_t ffg_rowblock_table(int32_t nb, int32_t rank, int32_t world, uint32_t* out, int32_t capacity);

/* Release cached device workspaces of the calling process. */
void ffg_release_workspaces(void);

#ifdef __cplusplus
}
#endif
#endif /* FERMIFORGE_FFG_H */
