/*
 * TEST INFRASTRUCTURE ONLY -- the CPU oracle.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load this library, and
 * only as the checker (or the timed CPU baseline), never as the product path.
 *
 * Plain-C restatement of the reference's arithmetic for the MLSP2 density-matrix
 * path.  Every function cites the reference file:line (relative to the reference
 * root) it restates.  The matrix functions are unblocked triple loops: they are
 * meant for the small parity sizes (N <= 256); oracle/oracle.py carries the
 * BLAS-backed fp64 recursion used at N >= 1024.
 *
 * Pinning: tests/test_oracle.py checks ffo_evaluate_model bit-for-bit against the
 * compiled reference evaluate_model (oracle/_ref, and the committed golden table
 * tests/golden/scalar_*.json), ffo_pairwise_sum against the reference
 * pairwise_sum, and the matrix recursion against the spectral-mapping oracle
 * D = V diag(evaluate_model(lambda0)) V^T built from the reference's own
 * evaluate_model.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------- scalar model */

/* evaluate_mlsp2: proj/core/src/scalar_models.cpp:243-252.  Operation order is
 * part of the contract: acc += d*x BEFORE the square, then x = a*x2 + b*x + c. */
double ffo_evaluate_mlsp2(const double* abcd, int L, double x0) {
    double x = x0;
    double acc = 0.0;
    for (int i = 0; i < L; ++i) {
        const double a = abcd[4 * i + 0], b = abcd[4 * i + 1];
        const double c = abcd[4 * i + 2], d = abcd[4 * i + 3];
        acc += d * x;
        const double x2 = x * x;
        x = a * x2 + b * x + c;
    }
    return acc + x;
}

/* evaluate_model for the MLSP2 architecture: the Fermi-family spectrum flip
 * x0 = 1 - x (proj/core/src/scalar_models.cpp:330-337). */
double ffo_evaluate_model(const double* abcd, int L, double x) {
    return ffo_evaluate_mlsp2(abcd, L, 1.0 - x);
}

/* fermi: proj/core/src/scalar_models.cpp:36-43 (sign-branched, never overflows). */
double ffo_fermi(double x, double beta, double mu) {
    const double t = beta * (x - mu);
    if (t > 0.0) {
        const double e = exp(-t);
        return e / (1.0 + e);
    }
    return 1.0 / (1.0 + exp(t));
}

/* ---------------------------------------------------------------- reductions */

/* pairwise_sum: proj/core/src/symmetric_matrix.cpp:12-20 (leaf <= 8, split at
 * size/2, left + right). */
double ffo_pairwise_sum(const double* v, int64_t n) {
    if (n <= 8) {
        double s = 0.0;
        for (int64_t i = 0; i < n; ++i) s += v[i];
        return s;
    }
    const int64_t half = n / 2;
    return ffo_pairwise_sum(v, half) + ffo_pairwise_sum(v + half, n - half);
}

/* density_statistics: trace = pairwise sum of the diagonal
 * (symmetric_matrix.cpp:57-61), trace_square = pairwise sum of all squared
 * entries in row-major order (symmetric_matrix.cpp:63-67). */
void ffo_density_statistics(const double* D, int64_t n, double* stats) {
    double* tmp = (double*)malloc(sizeof(double) * (size_t)(n * n > n ? n * n : n));
    for (int64_t i = 0; i < n; ++i) tmp[i] = D[i * n + i];
    stats[0] = ffo_pairwise_sum(tmp, n);
    for (int64_t i = 0; i < n * n; ++i) tmp[i] = D[i] * D[i];
    stats[1] = ffo_pairwise_sum(tmp, n * n);
    free(tmp);
}

/* ---------------------------------------------------------------- bounds / rescale */

/* spectral_bounds: Gershgorin discs, widened by 1e-12 * width.
 * The off-diagonal radius is summed left to right over j != i. */
void ffo_gershgorin(const double* H, int64_t n, double* eps_min, double* eps_max) {
    double lo = INFINITY, hi = -INFINITY;
    for (int64_t i = 0; i < n; ++i) {
        double r = 0.0;
        for (int64_t j = 0; j < n; ++j)
            if (j != i) r += fabs(H[i * n + j]);
        const double hii = H[i * n + i];
        if (hii - r < lo) lo = hii - r;
        if (hii + r > hi) hi = hii + r;
    }
    const double w = 1e-12 * (hi - lo);
    *eps_min = lo - w;
    *eps_max = hi + w;
}

/* in_region_of_validity (Eq. 41) written in
 * the reference model's UN-flipped frame: the model approximates
 * fermi(x; beta0, mu0) for x in [0,1] (scalar_models.cpp:330-333, trainer pivot
 * 1 - mu0 at trainer.cpp:986-991), so every eigenvalue must map to
 *   x = mu0 + (beta/beta0) (lambda - mu)  in [0, 1].
 * Returns 1 when valid, 0 when the lower inequality fails, -1 when the upper
 * one fails. */
int ffo_region_check(double eps_min, double eps_max, double mu, double kT, double beta0,
                     double mu0) {
    const double s = (1.0 / kT) / beta0;
    if (!(mu0 + s * (eps_min - mu) >= 0.0)) return 0;
    if (!(mu0 + s * (eps_max - mu) <= 1.0)) return -1;
    return 1;
}

/* rescale into the model frame, closed form of SPEC normalize_problem ->
 * rescale_to_model composed with the model's flip
 * (scalar_models.cpp:333):  X0 = (1 - mu0) I - (beta/beta0) (H - mu I). */
void ffo_rescale(const double* H, int64_t n, double mu, double kT, double beta0, double mu0,
                 double* X0) {
    const double s = (1.0 / kT) / beta0;
    for (int64_t i = 0; i < n; ++i)
        for (int64_t j = 0; j < n; ++j) {
            double v = -s * H[i * n + j];
            if (i == j) v += (1.0 - mu0) + s * mu;
            X0[i * n + j] = v;
        }
}

/* ---------------------------------------------------------------- matrix recursion */

static void matsq_f64(const double* X, int64_t n, double* Y) {
    memset(Y, 0, sizeof(double) * (size_t)(n * n));
    for (int64_t i = 0; i < n; ++i)
        for (int64_t k = 0; k < n; ++k) {
            const double xik = X[i * n + k];
            const double* xr = X + k * n;
            double* yr = Y + i * n;
            for (int64_t j = 0; j < n; ++j) yr[j] += xik * xr[j];
        }
    /* exact symmetry, as SymmetricMatrix maintains it (symmetric_matrix.hpp:3-5) */
    for (int64_t i = 0; i < n; ++i)
        for (int64_t j = i + 1; j < n; ++j) Y[j * n + i] = Y[i * n + j];
}

/* apply_model in DOUBLE mode: the matrix lift of
 * evaluate_mlsp2 (scalar_models.cpp:243-252) starting from X0 (already in the
 * model's flipped frame):  for each layer  A += d X;  X = a X^2 + b X + c I;
 * D = A + X.  n <= a few hundred. */
void ffo_mlsp2_from_x0(const double* X0, int64_t n, const double* abcd, int L, double* D) {
    const size_t nn = (size_t)(n * n);
    double* X = (double*)malloc(sizeof(double) * nn);
    double* Y = (double*)malloc(sizeof(double) * nn);
    memcpy(X, X0, sizeof(double) * nn);
    memset(D, 0, sizeof(double) * nn); /* D doubles as the accumulator A */
    for (int l = 0; l < L; ++l) {
        const double a = abcd[4 * l + 0], b = abcd[4 * l + 1];
        const double c = abcd[4 * l + 2], d = abcd[4 * l + 3];
        for (size_t e = 0; e < nn; ++e) D[e] += d * X[e];
        matsq_f64(X, n, Y);
        for (int64_t i = 0; i < n; ++i)
            for (int64_t j = 0; j < n; ++j) {
                const size_t e = (size_t)(i * n + j);
                X[e] = a * Y[e] + b * X[e] + (i == j ? c : 0.0);
            }
    }
    for (size_t e = 0; e < nn; ++e) D[e] += X[e];
    free(X);
    free(Y);
}

/* compute_density_matrix in DOUBLE mode with the closed-form
 * rescale above.  Returns the region status of ffo_region_check; D is written
 * only when valid. */
int ffo_density_matrix_f64(const double* H, int64_t n, double mu, double kT, const double* abcd,
                           int L, double beta0, double mu0, double* D, double* stats,
                           double* bounds) {
    double lo, hi;
    ffo_gershgorin(H, n, &lo, &hi);
    if (bounds) {
        bounds[0] = lo;
        bounds[1] = hi;
    }
    const int ok = ffo_region_check(lo, hi, mu, kT, beta0, mu0);
    if (ok != 1) return ok;
    double* X0 = (double*)malloc(sizeof(double) * (size_t)(n * n));
    ffo_rescale(H, n, mu, kT, beta0, mu0, X0);
    ffo_mlsp2_from_x0(X0, n, abcd, L, D);
    free(X0);
    if (stats) ffo_density_statistics(D, n, stats);
    return 1;
}

/* ---------------------------------------------------------------- binary16 */

/* IEEE binary16 from float, round-to-nearest-even with subnormals; the semantics
 * declared (never defined) at proj/core/include/fermiforge/half_precision.hpp:3-22.
 * Returns 0 and sets *overflow when |x| rounds beyond the finite half range. */
uint16_t ffo_float_to_half_bits(float x, int* overflow) {
    uint32_t u;
    memcpy(&u, &x, 4);
    const uint32_t sign = (u >> 16) & 0x8000u;
    const uint32_t ax = u & 0x7fffffffu;
    if (overflow) *overflow = 0;
    if (ax >= 0x7f800000u) { /* inf / nan */
        if (overflow) *overflow = 1;
        return (uint16_t)(sign | 0x7c00u | (ax > 0x7f800000u ? 0x200u : 0u));
    }
    if (ax >= 0x477ff000u) { /* >= 65520 rounds to inf */
        if (overflow) *overflow = 1;
        return (uint16_t)(sign | 0x7c00u);
    }
    if (ax < 0x33000000u) return (uint16_t)sign; /* < 2^-25 rounds to zero */
    const int32_t e = (int32_t)(ax >> 23) - 127;
    uint32_t mant = (ax & 0x7fffffu) | 0x800000u; /* 24-bit significand */
    if (e < -14) {                                  /* subnormal half */
        const int shift = -14 - e + 13;             /* 14..24 */
        const uint32_t q = mant >> shift;
        const uint32_t rem = mant & ((1u << shift) - 1u);
        const uint32_t halfway = 1u << (shift - 1);
        uint32_t r = q + ((rem > halfway || (rem == halfway && (q & 1u))) ? 1u : 0u);
        return (uint16_t)(sign | r); /* r may carry into the smallest normal: correct */
    }
    uint32_t q = mant >> 13;
    const uint32_t rem = mant & 0x1fffu;
    if (rem > 0x1000u || (rem == 0x1000u && (q & 1u))) q += 1u;
    uint32_t he = (uint32_t)(e + 15);
    if (q == 0x800u) { /* mantissa carry */
        q = 0x400u;
        he += 1u;
    }
    return (uint16_t)(sign | (he << 10) | (q & 0x3ffu));
}

float ffo_half_bits_to_float(uint16_t h) {
    const uint32_t sign = ((uint32_t)h & 0x8000u) << 16;
    const uint32_t e = ((uint32_t)h >> 10) & 0x1fu;
    const uint32_t m = (uint32_t)h & 0x3ffu;
    uint32_t u;
    if (e == 0) {
        if (m == 0) {
            u = sign;
        } else { /* subnormal: m * 2^-24 */
            const float f = (float)m * 5.9604644775390625e-8f;
            memcpy(&u, &f, 4);
            u |= sign;
        }
    } else if (e == 31) {
        u = sign | 0x7f800000u | (m << 13);
    } else {
        u = sign | ((e - 15 + 127) << 23) | (m << 13);
    }
    float f;
    memcpy(&f, &u, 4);
    return f;
}

/* ---------------------------------------------------------------- mixed precision */

/* Split of X (fp32) into binary16 hi/lo after a global power-of-two pre-scale:
 * hi = fp16(X * scale), lo = fp16(X * scale - hi).  mixed_square semantics
 * (Eq. 48) with the pre-scale documented in
 * DESIGN.md.  Returns the number of entries that overflowed binary16. */
int64_t ffo_split_half(const float* X, int64_t count, float scale, uint16_t* hi, uint16_t* lo) {
    int64_t bad = 0;
    for (int64_t e = 0; e < count; ++e) {
        int of = 0, of2 = 0;
        const float xs = X[e] * scale;
        hi[e] = ffo_float_to_half_bits(xs, &of);
        const float r = xs - ffo_half_bits_to_float(hi[e]);
        lo[e] = ffo_float_to_half_bits(r, &of2);
        bad += (of || of2);
    }
    return bad;
}

/* mixed_square emulation: Y = (hi hi + hi lo + lo hi) / scale^2 with binary32
 * accumulation over k in increasing order (X1 X1 dropped). */
void ffo_mixed_square_emul(const float* X, int64_t n, float scale, float* Y) {
    const size_t nn = (size_t)(n * n);
    uint16_t* hb = (uint16_t*)malloc(2 * nn);
    uint16_t* lb = (uint16_t*)malloc(2 * nn);
    float* h = (float*)malloc(4 * nn);
    float* l = (float*)malloc(4 * nn);
    ffo_split_half(X, (int64_t)nn, scale, hb, lb);
    for (size_t e = 0; e < nn; ++e) {
        h[e] = ffo_half_bits_to_float(hb[e]);
        l[e] = ffo_half_bits_to_float(lb[e]);
    }
    const float inv = 1.0f / (scale * scale);
    for (int64_t i = 0; i < n; ++i)
        for (int64_t j = i; j < n; ++j) {
            float acc = 0.0f;
            for (int64_t k = 0; k < n; ++k) {
                const float hik = h[i * n + k], lik = l[i * n + k];
                const float hkj = h[k * n + j], lkj = l[k * n + j];
                acc += hik * hkj;
                acc += hik * lkj;
                acc += lik * hkj;
            }
            Y[i * n + j] = acc * inv;
            Y[j * n + i] = acc * inv;
        }
    free(hb);
    free(lb);
    free(h);
    free(l);
}
