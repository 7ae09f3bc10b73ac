#pragma once

// fermiforge matrix engine on B200 -- header-only C++ drop-in over the C ABI (ffg.h).
//
// For a proj/core user: include this header next to the reference headers
// (fermiforge/scalar_models.hpp, symmetric_matrix.hpp, trainer.hpp), link
// libfermiforge_b200.so, and the SPEC matrix-engine / workflow entry points
// run on the tensor cores:
//
//   spectral_bounds(H)
//   in_region_of_validity(beta', mu', beta0, mu0)    SPEC.md:349-357 (mu' un-flipped, see ffg.h)
//   apply_model(H0, m, mode)
//   mixed_square(X)
//   density_statistics(D)
//   compute_density_matrix(H, mu, kT, m, mode, prov) SPEC.md:458-462 (model selected by the caller)
//   compute_density_matrices(Hs, mu, kT, m, mode)    batched
//   solve_chemical_potential(H, beta, n_occ, guess, m) SPEC.md:468-476 (Eqs. 42-45)
//   entropy_trace(H, mu, kT, entropy model)          SPEC.md:478-486 (Tr S, no extra GEMM)
//   thermodynamics(H, beta, mu, m, entropy model)
//   expectation(D, A)                                SPEC.md:488-495 (Eq. 9)
//
// Errors are rethrown as the reference's exception types: ValidationError
// (scalar_models.hpp:21-24), DivergedEvaluationError{layer} (trainer.hpp:20-25),
// HalfRangeError (half_precision.hpp:13-16), std::invalid_argument for dimension
// mismatch (symmetric_matrix.cpp:31), plus OutOfRegionError / DeviceError below.
// Results are returned by value as new matrices (symmetric_matrix.hpp:3-5).

#include <cstdint>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <variant>
#include <vector>

#include "fermiforge/ffg.h"
#include "fermiforge/half_precision.hpp"
#include "fermiforge/scalar_models.hpp"
#include "fermiforge/symmetric_matrix.hpp"
#include "fermiforge/trainer.hpp"

namespace fermiforge {

// friend of SymmetricMatrix, defined in symmetric_matrix.cpp:22-27 (zero-copy construction)
SymmetricMatrix unchecked_from_buffer(int n, std::vector<double>&& buf);

enum class PrecisionMode { Double = 0, Single = 1, MixedEmulated = 2, Bf16 = 3, Fp16 = 4 };

struct SpectralBounds {
    double eps_min = 0.0, eps_max = 0.0;
};
struct DensityStatistics {
    double trace = 0.0, trace_square = 0.0;
};
using Provenance = ffg_provenance;

/// rescale_to_model on (beta', mu') outside Eq. 41.
class OutOfRegionError : public std::runtime_error {
public:
    using std::runtime_error::runtime_error;
};
/// No usable sm_100 device or a CUDA failure (the B200 path has no CPU fallback).
class DeviceError : public std::runtime_error {
public:
    using std::runtime_error::runtime_error;
};

namespace detail {

inline void check(int rc, int layer = -1) {
    if (rc == FFG_OK) return;
    const std::string msg = ffg_last_error();
    switch (rc) {
        case FFG_ERR_VALIDATION: throw ValidationError(msg);
        case FFG_ERR_OUT_OF_REGION: throw OutOfRegionError(msg);
        case FFG_ERR_DIVERGED: throw DivergedEvaluationError(msg, layer);
        case FFG_ERR_HALF_RANGE: throw HalfRangeError(msg);
        case FFG_ERR_DIMENSION: throw std::invalid_argument(msg);
        case FFG_ERR_UNSUPPORTED: throw ValidationError(msg);
        default: throw DeviceError(msg);
    }
}

/// Flattens an MLSP2 ModelCoefficients into the ABI's [a,b,c,d] rows.
struct FlatModel {
    std::vector<double> abcd;
    ffg_model c{};
    explicit FlatModel(const ModelCoefficients& m) {
        m.validate();  // scalar_models.cpp:133-230
        if (m.architecture != Architecture::Mlsp2)
            throw ValidationError("B200 matrix engine: only the MLSP2 architecture is supported");
        const auto& layers = std::get<Mlsp2Coefficients>(m.payload).layers;
        abcd.reserve(layers.size() * 4);
        for (const auto& l : layers) {
            abcd.push_back(l.a);
            abcd.push_back(l.b);
            abcd.push_back(l.c);
            abcd.push_back(l.d);
        }
        c.abcd = abcd.data();
        c.n_layers = static_cast<int32_t>(layers.size());
        c.beta0 = m.trained_at.beta;
        c.mu0 = m.trained_at.mu;
    }
};

}  // namespace detail

inline bool in_region_of_validity(double beta_prime, double mu_prime, double beta0, double mu0) {
    return ffg_in_region_of_validity(beta_prime, mu_prime, beta0, mu0) != 0;
}

inline SpectralBounds spectral_bounds(const SymmetricMatrix& H) {
    SpectralBounds b;
    detail::check(ffg_spectral_bounds(H.data().data(), H.dim(), &b.eps_min, &b.eps_max));
    return b;
}

inline DensityStatistics density_statistics(const SymmetricMatrix& D) {
    double s[2];
    detail::check(ffg_density_statistics(D.data().data(), D.dim(), s));
    return {s[0], s[1]};
}

inline SymmetricMatrix mixed_square(const SymmetricMatrix& X) {
    const int n = X.dim();
    std::vector<float> xf(X.data().begin(), X.data().end()), yf(xf.size());
    detail::check(ffg_mixed_square(xf.data(), n, yf.data()));
    return unchecked_from_buffer(n, std::vector<double>(yf.begin(), yf.end()));
}

inline SymmetricMatrix apply_model(const SymmetricMatrix& H0, const ModelCoefficients& m,
                                   PrecisionMode mode = PrecisionMode::MixedEmulated) {
    detail::FlatModel fm(m);
    std::vector<double> D(static_cast<std::size_t>(H0.dim()) * H0.dim());
    ffg_provenance prov{};
    const int rc = ffg_apply_model(H0.data().data(), H0.dim(), &fm.c, static_cast<int32_t>(mode),
                                   D.data(), &prov);
    detail::check(rc, prov.diverged_layer);
    return unchecked_from_buffer(H0.dim(), std::move(D));
}

/// North-star entry: H, mu, kT and a trained MLSP2 set -> (D, {Tr D, Tr D^2}).
inline std::pair<SymmetricMatrix, DensityStatistics> compute_density_matrix(
    const SymmetricMatrix& H, double mu, double kT, const ModelCoefficients& m,
    PrecisionMode mode = PrecisionMode::MixedEmulated, Provenance* prov = nullptr) {
    detail::FlatModel fm(m);
    std::vector<double> D(static_cast<std::size_t>(H.dim()) * H.dim());
    double s[2];
    ffg_provenance p{};
    const int rc = ffg_density_matrix(H.data().data(), H.dim(), mu, kT, &fm.c,
                                      static_cast<int32_t>(mode), D.data(), s, &p);
    if (prov) *prov = p;
    detail::check(rc, p.diverged_layer);
    return {unchecked_from_buffer(H.dim(), std::move(D)), DensityStatistics{s[0], s[1]}};
}

/// Batched: independent H of equal size with per-matrix mu / kT.  D_out may be null.
inline std::vector<DensityStatistics> compute_density_matrices(
    std::span<const SymmetricMatrix> Hs, std::span<const double> mu, std::span<const double> kT,
    const ModelCoefficients& m, PrecisionMode mode = PrecisionMode::MixedEmulated,
    std::vector<SymmetricMatrix>* D_out = nullptr) {
    const std::size_t B = Hs.size();
    if (B == 0) return {};
    if (mu.size() != B || kT.size() != B)
        throw std::invalid_argument("compute_density_matrices: mu / kT size mismatch");
    const int n = Hs[0].dim();
    std::vector<const double*> hp(B);
    for (std::size_t k = 0; k < B; ++k) {
        if (Hs[k].dim() != n) throw std::invalid_argument("compute_density_matrices: dimension mismatch");
        hp[k] = Hs[k].data().data();
    }
    detail::FlatModel fm(m);
    std::vector<std::vector<double>> Dbuf;
    std::vector<double*> dp;
    if (D_out) {
        Dbuf.assign(B, std::vector<double>(static_cast<std::size_t>(n) * n));
        for (auto& d : Dbuf) dp.push_back(d.data());
    }
    std::vector<double> stats(2 * B);
    std::vector<ffg_provenance> prov(B);
    const int rc = ffg_density_matrices(static_cast<int32_t>(B), hp.data(), n, mu.data(), kT.data(),
                                        &fm.c, static_cast<int32_t>(mode),
                                        D_out ? dp.data() : nullptr, stats.data(), prov.data());
    int layer = -1;
    for (const auto& p : prov)
        if (p.diverged_layer >= 0) {
            layer = p.diverged_layer;
            break;
        }
    detail::check(rc, layer);
    std::vector<DensityStatistics> out(B);
    for (std::size_t k = 0; k < B; ++k) out[k] = {stats[2 * k], stats[2 * k + 1]};
    if (D_out) {
        D_out->clear();
        for (auto& d : Dbuf) D_out->push_back(unchecked_from_buffer(n, std::move(d)));
    }
    return out;
}

// ---------------------------------------------------------------- workflow

/// SPEC MuSolveReport.
struct MuSolveReport {
    double mu_final = 0.0;
    int iterations = 0;
    std::vector<std::pair<double, double>> residual_history;  // (mu, Tr D - n_occ)
    bool converged = false;
    int bisections = 0;
};

/// SPEC solve_chemical_potential: Newton on Tr D(mu) - n_occ with g'(mu) = beta (Tr D - Tr D^2)
/// from the fused statistics (Eq. 44), clamped steps, bisection fallback; returns the density
/// matrix at the converged mu.  Non-convergence throws DivergedEvaluationError.
inline std::pair<SymmetricMatrix, MuSolveReport> solve_chemical_potential(
    const SymmetricMatrix& H, double beta, double n_occ, double mu_guess, const ModelCoefficients& m,
    double tol = 1e-6, int max_iter = 30, PrecisionMode mode = PrecisionMode::MixedEmulated) {
    detail::FlatModel fm(m);
    std::vector<double> D(static_cast<std::size_t>(H.dim()) * H.dim());
    std::vector<double> hist(2 * static_cast<std::size_t>(max_iter));
    double s[2];
    ffg_mu_report r{};
    const int rc = ffg_solve_chemical_potential(H.data().data(), H.dim(), 1.0 / beta, n_occ, mu_guess, &fm.c,
                                                static_cast<int32_t>(mode), tol, max_iter, D.data(), s,
                                                hist.data(), &r);
    detail::check(rc);
    MuSolveReport rep;
    rep.mu_final = r.mu;
    rep.iterations = r.iterations;
    rep.converged = r.converged != 0;
    rep.bisections = r.bisections;
    for (int k = 0; k < r.iterations; ++k) rep.residual_history.emplace_back(hist[2 * k], hist[2 * k + 1]);
    return {unchecked_from_buffer(H.dim(), std::move(D)), std::move(rep)};
}

/// SPEC thermodynamics' entropy term: Tr s(H) at (mu, kT) through an entropy model
/// (EntropyModelCoefficients, scalar_models.hpp:150-156) trained at the Fermi model's (beta0, mu0).
inline double entropy_trace(const SymmetricMatrix& H, double mu, double kT, const ModelCoefficients& em,
                            PrecisionMode mode = PrecisionMode::MixedEmulated) {
    em.validate();
    if (em.architecture != Architecture::Entropy)
        throw ValidationError("entropy_trace: an Entropy-architecture model is required");
    const auto& e = std::get<EntropyModelCoefficients>(em.payload);
    ModelCoefficients inner;
    inner.architecture = Architecture::Mlsp2;
    inner.payload = e.inner;
    inner.trained_at = em.trained_at;
    detail::FlatModel fm(inner);
    ffg_entropy_model c{fm.c, e.alpha};
    double out = 0.0;
    ffg_provenance prov{};
    detail::check(ffg_entropy_trace(H.data().data(), H.dim(), mu, kT, &c, static_cast<int32_t>(mode), &out, &prov));
    return out;
}

/// SPEC expectation: Tr(D A) = sum_ij D_ij A_ij.
inline double expectation(const SymmetricMatrix& D, const SymmetricMatrix& A) {
    if (D.dim() != A.dim()) throw std::invalid_argument("expectation: dimension mismatch");
    double out = 0.0;
    detail::check(ffg_expectation(D.data().data(), A.data().data(), D.dim(), &out));
    return out;
}

/// SPEC ThermodynamicResult.
struct ThermodynamicResult {
    SymmetricMatrix density;
    double entropy_trace = 0.0, band_energy = 0.0, free_energy = 0.0;
};

/// SPEC thermodynamics with the models chosen by the caller (entropy model paired by exact
/// (beta0, mu0)).
inline ThermodynamicResult thermodynamics(const SymmetricMatrix& H, double beta, double mu,
                                          const ModelCoefficients& m, const ModelCoefficients& em,
                                          PrecisionMode mode = PrecisionMode::MixedEmulated) {
    if (m.trained_at.beta != em.trained_at.beta || m.trained_at.mu != em.trained_at.mu)
        throw ValidationError("thermodynamics: entropy model must share (beta0, mu0) with the Fermi model");
    auto [D, st] = compute_density_matrix(H, mu, 1.0 / beta, m, mode);
    const double ts = entropy_trace(H, mu, 1.0 / beta, em, mode);
    const double band = expectation(D, H) - mu * st.trace;
    return ThermodynamicResult{std::move(D), ts, band, band - ts / beta};
}

}  // namespace fermiforge
