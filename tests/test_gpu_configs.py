"""BASELINE configs 3-5 gated against the fp64 recursion on identical inputs (-m gpu).

North star: D within the per-mode max-abs / Frobenius tolerance and the electron count
within 1e-6 relative (FP32-emulated), against the CPU reference recursion
(scalar_models.cpp:243-252 lifted to matrices).  At these sizes the numpy oracle would take
minutes per matrix, so the reference is the same fp64 recursion evaluated with torch
float64 GEMMs on the device (oracle/device_ref.py), itself pinned against the numpy oracle
at N=512 below.  The gates are SURVEY.md 8(c) / BASELINE.md section 3, unchanged:

  MIXED_EMULATED: max|dD| <= 5e-6, ||dD||_F/||D||_F <= 1e-5, |dTr|/Tr <= 1e-6
  BF16:           max|dD| <= 1e-1,                           |dTr|/Tr <= 1e-2
  FP16:           max|dD| <= 1e-2,                           |dTr|/Tr <= 1e-3
"""
import numpy as np
import pytest

from oracle import device_ref as DR
from oracle import oracle as O
from paper_2605_08523_b200 import engine as E
from paper_2605_08523_b200.hamiltonians import tight_binding, batch_params

pytestmark = pytest.mark.gpu

MODES = (E.PrecisionMode.MIXED_EMULATED, E.PrecisionMode.BF16, E.PrecisionMode.FP16)
GATE = {
    E.PrecisionMode.MIXED_EMULATED: (5e-6, 1e-5, 1e-6),
    E.PrecisionMode.BF16: (1e-1, None, 1e-2),
    E.PrecisionMode.FP16: (1e-2, None, 1e-3),
}


@pytest.fixture(scope="module")
def torch():
    import torch as t
    if not E.device_available():
        pytest.fail("no sm_100 device: " + E.lib().ffg_last_error().decode())
    return t


@pytest.fixture(scope="module")
def model():
    return E.load_model("M1500")


def run_device(torch, H_dev, mu, kT, model, mode):
    """The product path on device-resident inputs (ffg_density_matrices_dev)."""
    D_dev = torch.empty_like(H_dev)
    stats, status, _ = E.compute_density_matrices_device(H_dev, mu, kT, model, mode, D_dev=D_dev)
    torch.cuda.synchronize()
    return D_dev, stats.cpu().numpy(), status.cpu().numpy()


def gate(mode, mx, fro, tr, what):
    gmx, gfro, gtr = GATE[mode]
    bad = [k for k in range(len(mx)) if not (mx[k] <= gmx and (gfro is None or fro[k] <= gfro) and tr[k] <= gtr)]
    print(f"{what} {mode.name}: worst max|dD| {mx.max():.2e}  ||dD||F/||D||F {fro.max():.2e}  "
          f"|dTr|/Tr {tr.max():.2e}")
    assert not bad, [(k, float(mx[k]), float(fro[k]), float(tr[k])) for k in bad[:8]]


def test_device_reference_pinned_to_numpy_oracle(torch, model):
    """The torch fp64 recursion equals the numpy oracle (oracle.density_matrix_f64) to fp64
    round-off, so it may stand in for it at the sizes below."""
    mu, kT = batch_params(3)
    Hs = [tight_binding(512, seed=10000 + k) for k in range(3)]
    R = DR.density_matrices_f64(torch.from_numpy(np.stack(Hs)).cuda(), mu, kT, model.abcd, model.beta0,
                                model.mu0).cpu().numpy()
    for k in range(3):
        ref = O.density_matrix_f64(Hs[k], mu[k], kT[k], model.abcd, model.beta0, model.mu0)
        assert np.abs(R[k] - ref).max() <= 1e-12, k


@pytest.mark.parametrize("n", [4096, 8192])
def test_config3_single_matrix_all_modes_vs_fp64_recursion(torch, model, n):
    """configs[2]: N=4096 and N=8192 single H (seed 1234, mu=0, kT=0.01), FP32-emulated, BF16
    and FP16, every element of D and the trace against the fp64 recursion."""
    H = torch.from_numpy(tight_binding(n, seed=1234)).cuda().unsqueeze(0)
    R = DR.density_matrices_f64(H, 0.0, 0.01, model.abcd, model.beta0, model.mu0)
    for mode in MODES:
        D, stats, status = run_device(torch, H, [0.0], [0.01], model, mode)
        assert status.tolist() == [0]
        assert torch.equal(D[0], D[0].T)
        mx, fro, tr = DR.errors(D, R)
        gate(mode, mx, fro, tr, f"N={n}")
        # the fused statistics are the trace of the D that was written
        assert abs(stats[0, 0] - float(torch.diagonal(D[0]).sum())) <= 1e-10 * abs(stats[0, 0])
        del D


@pytest.mark.parametrize("n,B", [(3000, 1), (2500, 2)])
def test_pair_kernel_between_2048_and_4096_vs_fp64_recursion(torch, model, n, B):
    """The selection band between the 16-worker pair kernel (np <= 2048) and the wide kernel (N >= 4096):
    ragged sizes on the 8+8-warp pair kernel (np = 3072 / 2560, more items per layer than CTA pairs),
    FP32-emulated, every element of D against the fp64 recursion; D exactly symmetric."""
    assert E.k2_kernel_name(n) == "mlsp2_pair_kernel"
    mu, kT = batch_params(B)
    H = torch.from_numpy(np.stack([tight_binding(n, seed=2500 + k) for k in range(B)])).cuda()
    R = DR.density_matrices_f64(H, mu, kT, model.abcd, model.beta0, model.mu0)
    D, stats, status = run_device(torch, H, mu, kT, model, E.PrecisionMode.MIXED_EMULATED)
    assert status.tolist() == [0] * B and torch.equal(D, D.transpose(1, 2))
    mx, fro, tr = DR.errors(D, R)
    gate(E.PrecisionMode.MIXED_EMULATED, mx, fro, tr, f"{B} x N={n}")


@pytest.mark.parametrize("mode", [E.PrecisionMode.MIXED_EMULATED, E.PrecisionMode.BF16])
def test_config4_all_512_members_vs_fp64_recursion(torch, model, mode):
    """configs[3]: the batch of 512 N=512 Hamiltonians (seeds 10000+k, mu_k ~ U(-0.5, 0.25),
    kT_k ~ U(0.010, 0.0125)) in one call: every member's whole D and trace gated."""
    B, n = 512, 512
    mu, kT = batch_params(B)
    H = torch.from_numpy(np.stack([tight_binding(n, seed=10000 + k) for k in range(B)])).cuda()
    D, stats, status = run_device(torch, H, mu, kT, model, mode)
    assert (status == 0).all()
    R = DR.density_matrices_f64(H, mu, kT, model.abcd, model.beta0, model.mu0)
    mx, fro, tr = DR.errors(D, R)
    gate(mode, mx, fro, tr, "512 x N=512")
    # statistics record of every member matches its own D
    trD = torch.diagonal(D, dim1=1, dim2=2).sum(-1).cpu().numpy()
    assert np.abs(stats[:, 0] - trD).max() <= 1e-10 * np.abs(trD).max()
    # a member computed alone is bit-identical to the same member inside the batch
    D1, s1, _ = run_device(torch, H[137:138].clone(), mu[137:138], kT[137:138], model, mode)
    assert torch.equal(D1[0], D[137]) and s1[0].tolist() == stats[137].tolist()


@pytest.mark.parametrize("wide", ["1", "0"])
def test_config5_n16384_single_gpu_vs_fp64_recursion(torch, model, wide, monkeypatch):
    """configs[4] on one GPU: N=16384 (seed 1234, mu=0, kT=0.01), FP32-emulated, whole D, with the
    wide kernel (the default at this size) and with the pair kernel (the row-block shards' kernel)."""
    n = 16384
    monkeypatch.setenv("FFG_WIDE", wide)
    H = torch.from_numpy(tight_binding(n, seed=1234)).cuda().unsqueeze(0)
    D, stats, status = run_device(torch, H, [0.0], [0.01], model, E.PrecisionMode.MIXED_EMULATED)
    assert status.tolist() == [0]
    assert torch.equal(D[0], D[0].T)
    R = DR.density_matrices_f64(H, 0.0, 0.01, model.abcd, model.beta0, model.mu0)
    del H
    mx, fro, tr = DR.errors(D, R)
    gate(E.PrecisionMode.MIXED_EMULATED, mx, fro, tr, f"N=16384 wide={wide}")


def test_config5_rowblock_8_ranks_bit_identical(torch, model, monkeypatch):
    """configs[4] as specified: N=16384 row-block sharded over 8 ranks (each its 2048 rows x all
    columns, operand rows exchanged every layer).  Emulated on one device (8 workspaces, exchange by
    device copies): the assembled D is bit-identical to the single-GPU D of the same (pair) kernel,
    so the fp64 gate of test_config5_n16384_single_gpu_vs_fp64_recursion[wide=0] carries over."""
    from paper_2605_08523_b200 import rowblock as RB
    n = 16384
    H = torch.from_numpy(tight_binding(n, seed=1234)).cuda()
    monkeypatch.setenv("FFG_WIDE", "0")
    D1, _, status = run_device(torch, H.unsqueeze(0), [0.0], [0.01], model, E.PrecisionMode.MIXED_EMULATED)
    assert status.tolist() == [0]
    D, stats, st = RB.rowblock_virtual(H, 0.0, 0.01, model, 8)
    torch.cuda.synchronize()
    assert st == 0
    assert torch.equal(D, D1[0])
