// TEST INFRASTRUCTURE ONLY -- never linked into the product library.
//
// C wrapper over the reference's own compiled C++ (proj/core, namespace
// fermiforge).  oracle/Makefile compiles this file together with the read-only
// reference sources *where they lie* (/root/reference/proj/core/src/*.cpp) into
// oracle/_ref/libfermiforge_ref.so.  Nothing from the reference is copied into
// this repository; this file only calls the reference's public API:
//   evaluate_model        proj/core/src/scalar_models.cpp:330-351
//   fermi                 proj/core/src/scalar_models.cpp:36-43
//   layer_count_estimate  proj/core/src/scalar_models.cpp:353-360
//   sp2_sign_sequence     proj/core/src/scalar_models.cpp:63-88
//   embed (SP2->MLSP2)    proj/core/src/scalar_models.cpp:554-607
//   train_fermi           proj/core/src/trainer.cpp:1215-1272
//   pairwise_sum          proj/core/src/symmetric_matrix.cpp:12-20
//   SymmetricMatrix::{trace,frobenius_squared}  symmetric_matrix.cpp:57-67
// The tests use it to pin the CPU restatement in oracle/ffo_oracle.c and to
// regenerate the golden fixtures under tests/golden/.
#include "fermiforge/scalar_models.hpp"
#include "fermiforge/symmetric_matrix.hpp"
#include "fermiforge/trainer.hpp"

#include <cstdint>
#include <cstring>
#include <exception>
#include <span>
#include <vector>

using namespace fermiforge;

namespace {
thread_local char g_err[512];
int fail(const std::exception& e) {
    std::strncpy(g_err, e.what(), sizeof g_err - 1);
    return 1;
}
ModelCoefficients mlsp2_model(const double* abcd, int L, double beta0, double mu0) {
    Mlsp2Coefficients c;
    c.layers.resize(L);
    for (int i = 0; i < L; ++i) {
        c.layers[i].a = abcd[4 * i + 0];
        c.layers[i].b = abcd[4 * i + 1];
        c.layers[i].c = abcd[4 * i + 2];
        c.layers[i].d = abcd[4 * i + 3];
    }
    ModelCoefficients m;
    m.architecture = Architecture::Mlsp2;
    m.payload = std::move(c);
    m.trained_at = FermiParams{beta0, mu0};
    return m;
}
}  // namespace

extern "C" {

const char* ffr_last_error() { return g_err; }

// evaluate_model(m, x) for an MLSP2 coefficient table (rows [a,b,c,d]).
int ffr_evaluate_mlsp2_model(const double* abcd, int L, double beta0, double mu0,
                             const double* xs, int64_t n, double* out) {
    try {
        const ModelCoefficients m = mlsp2_model(abcd, L, beta0, mu0);
        for (int64_t i = 0; i < n; ++i) out[i] = evaluate_model(m, xs[i]);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

double ffr_fermi(double x, double beta, double mu) { return fermi(x, FermiParams{beta, mu}); }

int ffr_layer_count_estimate(double beta_prime) { return layer_count_estimate(beta_prime); }

// SP2 sign sequence at pivot mu_prime, embedded into MLSP2 rows.
int ffr_sp2_as_mlsp2(double mu_prime, int layers, double* abcd_out) {
    try {
        const auto seq = sp2_sign_sequence(mu_prime, layers, -1.0);
        ModelCoefficients m;
        m.architecture = Architecture::Sp2;
        m.payload = Sp2Coefficients{seq.signs};
        m.trained_at = FermiParams{1.0, mu_prime};
        const ModelCoefficients e = embed(m, Architecture::Mlsp2);
        const auto& c = std::get<Mlsp2Coefficients>(e.payload);
        for (std::size_t i = 0; i < c.layers.size(); ++i) {
            abcd_out[4 * i + 0] = c.layers[i].a;
            abcd_out[4 * i + 1] = c.layers[i].b;
            abcd_out[4 * i + 2] = c.layers[i].c;
            abcd_out[4 * i + 3] = c.layers[i].d;
        }
        return static_cast<int>(c.layers.size());
    } catch (const std::exception& e) {
        fail(e);
        return -1;
    }
}

// train_fermi with TrainingConfig{beta0, mu0, Mlsp2, layers, samples, seed,
// max_iter}; report = [final_max, final_rms, iterations, converged, initial_max].
int ffr_train_fermi_mlsp2(double beta0, double mu0, int layers, int samples, int max_iter,
                          uint64_t seed, double* abcd_out, double* report) {
    try {
        TrainingConfig cfg;
        cfg.beta0 = beta0;
        cfg.mu0 = mu0;
        cfg.architecture = Architecture::Mlsp2;
        cfg.layers = layers;
        cfg.sample_count = samples;
        cfg.max_iterations = max_iter;
        cfg.seed = seed;
        cfg.weighting = Weighting::Derivative;
        auto [m, rep] = train_fermi(cfg);
        const auto& c = std::get<Mlsp2Coefficients>(m.payload);
        for (std::size_t i = 0; i < c.layers.size(); ++i) {
            abcd_out[4 * i + 0] = c.layers[i].a;
            abcd_out[4 * i + 1] = c.layers[i].b;
            abcd_out[4 * i + 2] = c.layers[i].c;
            abcd_out[4 * i + 3] = c.layers[i].d;
        }
        report[0] = rep.final_max_error;
        report[1] = rep.final_rms_error;
        report[2] = rep.iterations;
        report[3] = rep.converged ? 1.0 : 0.0;
        report[4] = rep.initial_max_error;
        return static_cast<int>(c.layers.size());
    } catch (const std::exception& e) {
        fail(e);
        return -1;
    }
}


// train_entropy (trainer.cpp:1274) on an MLSP2 Fermi base; out: inner abcd rows, alpha;
// report = [final_max, final_rms, iterations, converged, initial_max].
int ffr_train_entropy_mlsp2(const double* base_abcd, int L, double beta0, double mu0, int samples,
                            int max_iter, uint64_t seed, double* abcd_out, double* alpha_out,
                            double* report) {
    try {
        const ModelCoefficients base = mlsp2_model(base_abcd, L, beta0, mu0);
        TrainingConfig cfg;
        cfg.beta0 = beta0;
        cfg.mu0 = mu0;
        cfg.architecture = Architecture::Mlsp2;
        cfg.layers = L;
        cfg.sample_count = samples;
        cfg.max_iterations = max_iter;
        cfg.seed = seed;
        cfg.weighting = Weighting::Derivative;
        auto [m, rep] = train_entropy(cfg, base);
        const auto& e = std::get<EntropyModelCoefficients>(m.payload);
        for (std::size_t i = 0; i < e.inner.layers.size(); ++i) {
            abcd_out[4 * i + 0] = e.inner.layers[i].a;
            abcd_out[4 * i + 1] = e.inner.layers[i].b;
            abcd_out[4 * i + 2] = e.inner.layers[i].c;
            abcd_out[4 * i + 3] = e.inner.layers[i].d;
        }
        *alpha_out = e.alpha;
        report[0] = rep.final_max_error;
        report[1] = rep.final_rms_error;
        report[2] = rep.iterations;
        report[3] = rep.converged ? 1.0 : 0.0;
        report[4] = rep.initial_max_error;
        return static_cast<int>(e.inner.layers.size());
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// evaluate_model (scalar_models.cpp:330, Architecture::Entropy) and the exact
// fermi_entropy (scalar_models.hpp:56) on a grid of model-frame x.
int ffr_evaluate_entropy_model(const double* abcd, int L, double alpha, double beta0, double mu0,
                               const double* xs, int64_t n, double* out, double* exact) {
    try {
        EntropyModelCoefficients e;
        e.inner = std::get<Mlsp2Coefficients>(mlsp2_model(abcd, L, beta0, mu0).payload);
        e.alpha = alpha;
        e.mu0 = mu0;
        ModelCoefficients m;
        m.architecture = Architecture::Entropy;
        m.payload = std::move(e);
        m.trained_at = FermiParams{beta0, mu0};
        for (int64_t i = 0; i < n; ++i) {
            out[i] = evaluate_model(m, xs[i]);
            if (exact) exact[i] = fermi_entropy(xs[i], FermiParams{beta0, mu0});
        }
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

double ffr_pairwise_sum(const double* v, int64_t n) {
    return pairwise_sum(std::span<const double>(v, static_cast<std::size_t>(n)));
}

// density_statistics through the reference SymmetricMatrix (from_dense
// symmetrises; trace/frobenius_squared use pairwise_sum).
int ffr_density_statistics(const double* rows, int n, double* stats) {
    try {
        const auto m = SymmetricMatrix::from_dense(
            n, std::span<const double>(rows, static_cast<std::size_t>(n) * n));
        stats[0] = m.trace();
        stats[1] = m.frobenius_squared();
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

}  // extern "C"
