"""DOUBLE and SINGLE precision modes on the B200 (-m gpu): the recursion in fp64 / fp32
arithmetic (csrc/direct.cuh: library GEMM for the square, our fused layer update), checked against the
CPU oracle and SPEC.md's DOUBLE-mode acceptance properties:

  * fp64 recursion (oracle.mlsp2_recursion_f64, scalar_models.cpp:243-252): DOUBLE within 1e-12
  * spectral mapping: eigenvalues of apply_model(H0) = evaluate_model(lambda_i) to 1e-11
  * equivariance: ||apply(Q^T H0 Q) - Q^T apply(H0) Q||_2 <= 1e-10, N <= 64
  * matrix/scalar consistency: ||D - oracle D||_2 <= model error + 1e-12 N in DOUBLE
  * monotone degradation: err(MIXED) <= 50 err(SINGLE), both <= 1e-4 (2-norm vs DOUBLE)
  * multiplication accounting: exactly n squarings per application
"""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2605_08523_b200 import engine as E
from paper_2605_08523_b200.hamiltonians import tight_binding, goe, batch_params

pytestmark = pytest.mark.gpu
DOUBLE, SINGLE, MIXED = E.PrecisionMode.DOUBLE, E.PrecisionMode.SINGLE, E.PrecisionMode.MIXED_EMULATED


@pytest.fixture(scope="module", autouse=True)
def _need_device():
    if not E.device_available():
        pytest.fail("no sm_100 device: " + E.lib().ffg_last_error().decode())


@pytest.fixture(scope="module")
def model():
    return E.load_model("M1500")


def norm2(M):
    return float(np.linalg.norm(M, 2))


def random_frame_matrix(n, seed, lo=0.05, hi=0.95):
    """A symmetric H0 in the model frame: Q diag(lambda) Q^T, lambda in [lo, hi]."""
    rng = np.random.default_rng(seed)
    Q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    lam = rng.uniform(lo, hi, n)
    H0 = (Q * lam) @ Q.T
    return 0.5 * (H0 + H0.T), lam


@pytest.mark.parametrize("n", [1, 64, 256, 1000])
def test_double_matches_fp64_recursion(model, n):
    H = tight_binding(n, seed=n) if n >= 4 else np.diag(np.linspace(-0.3, 0.3, n))
    D, st, pv = E.compute_density_matrix(H, 0.0, 0.01, model, DOUBLE)
    Dref = O.density_matrix_f64(H, 0.0, 0.01, model.abcd, model.beta0, model.mu0)
    assert pv.status == 0 and np.array_equal(D, D.T)
    assert np.abs(D - Dref).max() <= 1e-12
    assert abs(st.trace - np.trace(Dref)) <= 1e-12 * max(1.0, abs(np.trace(Dref)))
    assert pv.half_products == model.layer_count            # n squarings


def test_single_close_to_fp64_recursion(model):
    H = tight_binding(512, seed=3)
    D, st, pv = E.compute_density_matrix(H, 0.0, 0.01, model, SINGLE)
    Dref = O.density_matrix_f64(H, 0.0, 0.01, model.abcd, model.beta0, model.mu0)
    assert pv.status == 0 and np.array_equal(D, D.T) and pv.half_products == model.layer_count
    err = np.abs(D - Dref).max()
    print(f"SINGLE N=512 max|dD| {err:.2e}")
    assert err <= 1e-3


def test_spectral_mapping_double(model):
    """the eigenvalues of apply_model(H0, m) equal evaluate_model(m, lambda_i) to 1e-11."""
    H0, lam = random_frame_matrix(48, seed=11)
    D = E.apply_model(H0, model, DOUBLE)
    ev = np.sort(np.linalg.eigvalsh(D))
    want = np.sort(O.evaluate_model_np(model.abcd, np.linalg.eigvalsh(H0)))
    assert np.abs(ev - want).max() <= 1e-11


def test_equivariance_double(model):
    """||apply(Q^T H0 Q) - Q^T apply(H0) Q||_2 <= 1e-10 for N <= 64."""
    H0, _ = random_frame_matrix(64, seed=12)
    rng = np.random.default_rng(13)
    Q, _ = np.linalg.qr(rng.standard_normal((64, 64)))
    Hq = Q.T @ H0 @ Q
    Hq = 0.5 * (Hq + Hq.T)
    lhs = E.apply_model(Hq, model, DOUBLE)
    rhs = Q.T @ E.apply_model(H0, model, DOUBLE) @ Q
    assert norm2(lhs - rhs) <= 1e-10


def test_matrix_scalar_consistency_double(model):
    """SPEC.md:704 (acceptance 4) in DOUBLE: ||D - oracle D||_2 <= model max error + 1e-12 N, with the
    oracle D = V evaluate_model(mu0 + s (lambda - mu)) V^T."""
    for seed in range(10):
        H = goe(64, seed=100 + seed)
        mu, kT = 0.0, 1.0  # beta' = W / kT inside the model's region for a unit-width GOE spectrum
        lo, hi = O.gershgorin(H)
        kT = (hi - lo) / 600.0
        D, st, pv = E.compute_density_matrix(H, mu, kT, model, DOUBLE)
        Dref = O.spectral_oracle(H, mu, kT, model.abcd, model.beta0, model.mu0)
        assert norm2(D - Dref) <= 1e-12 * 64 + 1e-11, seed


def test_monotone_degradation(model):
    """err(MIXED_EMULATED) <= 50 x err(SINGLE) and both <= 1e-4 in the 2-norm vs DOUBLE
    (random N=128 Hamiltonians)."""
    for seed in range(3):
        H = tight_binding(128, seed=500 + seed)
        Dd, _, _ = E.compute_density_matrix(H, 0.0, 0.01, model, DOUBLE)
        Ds, _, _ = E.compute_density_matrix(H, 0.0, 0.01, model, SINGLE)
        Dm, _, _ = E.compute_density_matrix(H, 0.0, 0.01, model, MIXED)
        es, em = norm2(Ds - Dd), norm2(Dm - Dd)
        print(f"seed {seed}: 2-norm err SINGLE {es:.2e} MIXED {em:.2e}")
        assert es <= 1e-4 and em <= 1e-4 and em <= 50 * es


def test_double_batch_device_entry_and_out_of_region(model):
    """The device entry point in DOUBLE mode: per-matrix status, an out-of-region member's D is NaN and
    reports no squarings, the others equal their single-matrix results bit for bit."""
    import torch
    B, n = 4, 256
    mu, kT = batch_params(B)
    kT = np.array(kT)
    kT[1] = 0.0005
    Hs = np.stack([tight_binding(n, seed=40 + k) for k in range(B)])
    H = torch.from_numpy(Hs).cuda()
    D = torch.empty_like(H)
    stats, status, _ = E.compute_density_matrices_device(H, mu, kT, model, DOUBLE, D_dev=D)
    torch.cuda.synchronize()
    assert status.cpu().tolist() == [0, E.OutOfRegionError.status, 0, 0]
    assert torch.isnan(D[1]).all()
    D0, _, _ = E.compute_density_matrix(Hs[0], float(mu[0]), float(kT[0]), model, DOUBLE)
    assert np.array_equal(D[0].cpu().numpy(), D0)


def test_double_rowblock_unsupported(model):
    import torch
    from paper_2605_08523_b200 import rowblock as RB
    H = torch.from_numpy(tight_binding(512, seed=1)).cuda()
    with pytest.raises(E.UnsupportedModeError, match="row-block"):
        RB.RowBlockRank(H, 0.0, 0.01, model, rank=0, world=2, mode=DOUBLE)


def test_double_workflow_callers():
    """The workflow callers run in DOUBLE mode too: the SPEC two-level mu-solve and the
    entropy trace against the fp64 recursion of the same entropy model (tighter than MIXED_EMULATED)."""
    from paper_2605_08523_b200 import workflow as W
    D, st, rep = W.solve_chemical_potential(np.diag([0.0, 1.0]), 10.0, 1.0, 0.4, tol=1e-9, mode=DOUBLE)
    # the electron count is met to the Newton tolerance; mu = 0.5 up to the model's own error
    assert rep.converged and abs(st.trace - 1.0) <= 1e-9 and abs(rep.mu_final - 0.5) <= 2e-5
    em = W.load_entropy_model("E1500")
    H = tight_binding(256, seed=9)
    ts = W.entropy_trace(H, 0.1, 0.01, em, mode=DOUBLE)
    ref = O.entropy_trace_f64(H, 0.1, 0.01, em.inner.abcd, em.alpha, em.beta0, em.mu0)
    assert abs(ts - ref) <= 1e-9 * max(1.0, abs(ref)), (ts, ref)
