// Drop-in test of include/fermiforge/matrix_engine.hpp: a proj/core program using the
// reference's own SymmetricMatrix / ModelCoefficients / Matrix Market I/O, with the
// density matrix computed on the B200 through the C ABI.
//   test_matrix_engine <coefficients.json> <H.mtx> <Dref.mtx> <mu> <kT>
// Exit 0 on success; prints one line of errors.
#include <cmath>
#include <cstdio>
#include <fstream>
#include <regex>
#include <sstream>
#include <string>

#include "fermiforge/matrix_engine.hpp"

using namespace fermiforge;

static ModelCoefficients load_mlsp2(const std::string& path) {
    std::ifstream f(path);
    std::stringstream ss;
    ss << f.rdbuf();
    const std::string s = ss.str();
    auto field = [&](const char* key) {
        std::smatch mm;
        std::regex re(std::string("\"") + key + "\"\\s*:\\s*\"([^\"]+)\"");
        if (!std::regex_search(s, mm, re)) throw std::runtime_error(std::string("missing ") + key);
        return std::stod(mm[1]);
    };
    Mlsp2Coefficients c;
    const auto pos = s.find("\"layers\"");
    std::regex num("\"(-?[0-9][^\"]*)\"");
    std::vector<double> v;
    for (auto it = std::sregex_iterator(s.begin() + pos, s.end(), num); it != std::sregex_iterator(); ++it)
        v.push_back(std::stod((*it)[1]));
    for (std::size_t i = 0; i + 3 < v.size(); i += 4) c.layers.push_back({v[i], v[i + 1], v[i + 2], v[i + 3]});
    ModelCoefficients m;
    m.architecture = Architecture::Mlsp2;
    m.payload = c;
    m.trained_at = FermiParams{field("beta0"), field("mu0")};
    return m;
}

int main(int argc, char** argv) {
    if (argc != 6) {
        std::fprintf(stderr, "usage: %s coeffs.json H.mtx Dref.mtx mu kT\n", argv[0]);
        return 64;
    }
    const ModelCoefficients m = load_mlsp2(argv[1]);
    const SymmetricMatrix H = read_matrix_market(argv[2]);
    const SymmetricMatrix Dref = read_matrix_market(argv[3]);
    const double mu = std::stod(argv[4]), kT = std::stod(argv[5]);
    int fails = 0;

    Provenance prov{};
    auto [D, st] = compute_density_matrix(H, mu, kT, m, PrecisionMode::MixedEmulated, &prov);
    double mx = 0.0;
    for (int i = 0; i < H.dim(); ++i)
        for (int j = 0; j < H.dim(); ++j) mx = std::max(mx, std::abs(D(i, j) - Dref(i, j)));
    const double tr_rel = std::abs(st.trace - Dref.trace()) / Dref.trace();
    const double tr_self = std::abs(st.trace - D.trace()) / D.trace();
    std::printf("n=%d max|dD|=%.3e |dTr|/Tr=%.3e stats-vs-pairwise=%.1e beta'=%.2f products=%lld\n",
                H.dim(), mx, tr_rel, tr_self, prov.beta_prime, (long long)prov.half_products);
    fails += !(mx <= 5e-6 && tr_rel <= 1e-6 && tr_self <= 1e-12);

    // H = diag(0,1), beta = 50, mu = 0.5 -> D ~ diag(f(0), f(1))
    const double d01[2] = {0.0, 1.0};
    auto [D2, st2] = compute_density_matrix(SymmetricMatrix::diagonal(d01), 0.5, 1.0 / 50.0, m);
    const double f0 = 1.0 / (1.0 + std::exp(-25.0)), f1 = 1.0 / (1.0 + std::exp(25.0));
    fails += !(std::abs(D2(0, 0) - f0) <= 1e-6 && std::abs(D2(1, 1) - f1) <= 1e-6);

    // batched entry with the reference container
    std::vector<SymmetricMatrix> Hs{H, H};
    std::vector<double> mus{mu, mu}, kTs{kT, kT};
    std::vector<SymmetricMatrix> Ds;
    auto stats = compute_density_matrices(Hs, mus, kTs, m, PrecisionMode::MixedEmulated, &Ds);
    fails += !(stats.size() == 2 && stats[1].trace == st.trace && Ds[1].data() == D.data());

    // error mapping: out of region -> OutOfRegionError; bad coefficients -> ValidationError
    try {
        compute_density_matrix(H, mu, kT / 20.0, m);
        fails += 1;
    } catch (const OutOfRegionError&) {
    }
    try {
        ModelCoefficients bad = m;
        bad.trained_at.mu = 1.5;
        compute_density_matrix(H, mu, kT, bad);
        fails += 1;
    } catch (const ValidationError&) {
    }
    const auto b = spectral_bounds(H);
    fails += !(b.eps_min < b.eps_max);

    // workflow: mu solve restores n_occ; entropy / thermodynamics with a reference-typed
    // EntropyModelCoefficients built from the Fermi set's own layers (structure test only)
    const double n_occ = st.trace;
    auto [Dm, rep] = solve_chemical_potential(H, 1.0 / kT, n_occ, mu + 0.03, m, 1e-3);
    fails += !(rep.converged && std::abs(rep.mu_final - mu) <= 1e-3 && std::abs(Dm.trace() - n_occ) <= 2e-3);
    std::printf("mu-solve: mu=%.6f (target %.6f) in %d evaluations\n", rep.mu_final, mu, rep.iterations);
    ModelCoefficients em;
    em.architecture = Architecture::Entropy;
    em.payload = EntropyModelCoefficients{std::get<Mlsp2Coefficients>(m.payload), 0.85, m.trained_at.mu};
    em.trained_at = m.trained_at;
    const auto th = thermodynamics(H, 1.0 / kT, mu, m, em);
    fails += !(std::isfinite(th.entropy_trace) &&
               std::abs(th.free_energy - (th.band_energy - th.entropy_trace * kT)) <= 1e-9 * (1 + std::abs(th.free_energy)));
    fails += !(std::abs(expectation(D, D) - st.trace_square) <= 1e-8 * st.trace_square);
    std::printf("%s\n", fails ? "FAIL" : "OK");
    return fails ? 1 : 0;
}
