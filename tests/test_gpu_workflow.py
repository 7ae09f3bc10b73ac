"""GPU tests of the workflow callers of the density-matrix path: chemical
potential Newton solve, the Eq. 44 derivative identity, entropy / thermodynamics and
expectation -- each against the CPU oracle on identical inputs."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2605_08523_b200 import engine as E
from paper_2605_08523_b200 import workflow as W
from paper_2605_08523_b200.hamiltonians import tight_binding

pytestmark = pytest.mark.gpu


def exact_mu(H, kT, n_occ):
    lam = np.linalg.eigvalsh(H)
    lo, hi = lam[0] - 1.0, lam[-1] + 1.0
    for _ in range(200):
        mid = 0.5 * (lo + hi)
        tr = np.sum(1.0 / (1.0 + np.exp(np.clip((lam - mid) / kT, -700, 700))))
        lo, hi = (mid, hi) if tr < n_occ else (lo, mid)
    return 0.5 * (lo + hi)


def test_mu_solve_spec_two_level():
    """H = diag(0,1), beta = 10, n_occ = 1, guess 0.4 -> mu = 0.5 (symmetry)."""
    H = np.diag([0.0, 1.0])
    D, st, rep = W.solve_chemical_potential(H, 10.0, 1.0, 0.4, tol=1e-6)
    assert rep.converged and rep.model.beta0 == 40.0
    assert abs(rep.mu_final - 0.5) <= 2e-5, rep
    assert rep.iterations <= 6
    assert abs(st.trace - 1.0) <= 1e-6


def test_mu_solve_matches_exact_mu_tight_binding():
    """N=256 TB, kT = 0.01: Newton from a guess 0.05 off converges to the exact mu of the
    eigenvalue bisection, in a few iterations; the converged D has Tr D = n_occ."""
    H = tight_binding(256, seed=1234)
    kT = 0.01
    n_occ = 100.0
    mu_star = exact_mu(H, kT, n_occ)
    model = E.load_model("M1500")
    D, st, rep = W.solve_chemical_potential(H, 1.0 / kT, n_occ, mu_star + 0.05, model, tol=1e-3)
    assert rep.converged and rep.iterations <= 8, rep
    assert abs(rep.mu_final - mu_star) <= 2e-4, (rep.mu_final, mu_star)
    assert abs(np.trace(D) - n_occ) <= 2e-3
    R = O.density_matrix_f64(H, rep.mu_final, kT, model.abcd, model.beta0, model.mu0)
    assert np.abs(D - R).max() <= 5e-6


def test_mu_solve_converged_start_takes_no_newton_step():
    """Tr D = n_occ at the guess -> one evaluation, no step."""
    H = tight_binding(256, seed=1234)
    model = E.load_model("M1500")
    _, st, _ = E.compute_density_matrix(H, 0.02, 0.01, model)
    _, _, rep = W.solve_chemical_potential(H, 100.0, st.trace, 0.02, model, tol=1e-3)
    assert rep.converged and rep.iterations == 1 and rep.mu_final == 0.02


def test_newton_derivative_identity():
    """g'(mu) = beta (Tr D - Tr D^2) (Eq. 44) matches central differences of Tr D."""
    H = tight_binding(256, seed=42)
    model = E.load_model("M1500")
    kT, mu, h = 0.01, 0.05, 2e-3
    _, st, _ = E.compute_density_matrix(H, mu, kT, model)
    _, sp, _ = E.compute_density_matrix(H, mu + h, kT, model)
    _, sm, _ = E.compute_density_matrix(H, mu - h, kT, model)
    fd = (sp.trace - sm.trace) / (2 * h)
    gp = (1.0 / kT) * (st.trace - st.trace_square)
    assert abs(fd - gp) <= 2e-2 * abs(gp), (fd, gp)


@pytest.mark.parametrize("name,kT,mu", [("E1500", 0.01, 0.1), ("E40", 0.5, 0.0)])
def test_entropy_trace_matches_oracle(name, kT, mu):
    """Tr S on the device (fused statistics, no extra GEMM) vs the fp64 recursion of the same
    entropy model, and vs the exact electronic entropy within N x model error."""
    em = W.load_entropy_model(name)
    H = tight_binding(256, seed=9)
    ts = W.entropy_trace(H, mu, kT, em)
    ref = O.entropy_trace_f64(H, mu, kT, em.inner.abcd, em.alpha, em.beta0, em.mu0)
    assert abs(ts - ref) <= 5e-5 * max(1.0, abs(ref)) + 256 * 2e-6, (ts, ref)
    assert abs(ts - O.entropy_trace_exact(H, mu, kT)) <= 256 * 3e-6 + 5e-5 * abs(ref)


def test_entropy_at_the_chemical_potential():
    """H = mu I -> every state at the chemical potential, Tr S = N ln 2."""
    em = W.load_entropy_model("E1500")
    n, mu = 128, 0.2
    ts = W.entropy_trace(mu * np.eye(n), mu, 0.01, em)
    assert abs(ts - n * np.log(2.0)) <= n * 2e-6


def test_thermodynamics_consistency():
    """free energy = band energy - Tr S / beta and equals the oracle
    sum_i [f(l_i)(l_i - mu) - s(l_i)/beta] within model tolerances."""
    H = tight_binding(256, seed=11)
    beta, mu = 100.0, 0.05
    r = W.thermodynamics(H, beta, mu)
    lam = np.linalg.eigvalsh(H)
    f = 1.0 / (1.0 + np.exp(np.clip((lam - mu) * beta, -700, 700)))
    band = float(np.sum(f * (lam - mu)))
    ts = O.entropy_trace_exact(H, mu, 1.0 / beta)
    assert r.entropy_trace >= 0.0
    assert abs(r.free_energy - (r.band_energy - r.entropy_trace / beta)) <= 1e-12 * max(1.0, abs(r.free_energy))
    assert abs(r.band_energy - band) <= 1e-3, (r.band_energy, band)
    assert abs(r.free_energy - (band - ts / beta)) <= 1e-3


def test_expectation():
    """A = I -> Tr D; D = 0 -> 0; A = H -> sum_ij D_ij H_ij."""
    H = tight_binding(128, seed=3)
    model = E.load_model("M1500")
    D, st, _ = E.compute_density_matrix(H, 0.0, 0.01, model)
    assert abs(W.expectation(D, np.eye(128)) - np.trace(D)) <= 1e-9
    assert W.expectation(np.zeros((128, 128)), H) == 0.0
    assert abs(W.expectation(D, H) - float(np.sum(D * H))) <= 1e-9
    with pytest.raises(E.DimensionError):
        W.expectation(D, np.eye(64))
