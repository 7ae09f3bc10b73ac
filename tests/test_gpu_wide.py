"""The wide K2 kernel (csrc/k2_wide.cuh: 256 x 256 super-block items, hi/lo blocks stored once and
read MN-major for the mirrored orientation) against the fp64 recursion (-m gpu).

The default for nb even and N >= 4096 (ffg_capi.cu use_wide); FFG_WIDE=1 forces it below that,
FFG_WIDE=0 selects the pair kernel.  Gates are SURVEY.md 8(c), unchanged:

  MIXED_EMULATED: max|dD| <= 5e-6, ||dD||_F/||D||_F <= 1e-5, |dTr|/Tr <= 1e-6
  BF16:           max|dD| <= 1e-1,                           |dTr|/Tr <= 1e-2
  FP16:           max|dD| <= 1e-2,                           |dTr|/Tr <= 1e-3

Reference: the fp64 recursion (scalar_models.cpp:243-252 lifted to matrices) evaluated with torch
float64 GEMMs (oracle/device_ref.py, pinned to the numpy oracle in test_gpu_configs.py).
"""
import numpy as np
import pytest

from oracle import device_ref as DR
from paper_2605_08523_b200 import engine as E
from paper_2605_08523_b200.hamiltonians import tight_binding, batch_params

pytestmark = pytest.mark.gpu

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


def run(torch, H, mu, kT, model, mode):
    D = torch.empty_like(H)
    stats, status, _ = E.compute_density_matrices_device(H, mu, kT, model, mode, D_dev=D)
    torch.cuda.synchronize()
    return D, stats.cpu().numpy(), status.cpu().numpy()


def gate(mode, D, R, what):
    mx, fro, tr = DR.errors(D, R)
    gmx, gfro, gtr = GATE[mode]
    print(f"{what} {mode.name}: max|dD| {mx.max():.2e} fro {fro.max():.2e} |dTr|/Tr {tr.max():.2e}")
    assert (mx <= gmx).all() and (gfro is None or (fro <= gfro).all()) and (tr <= gtr).all(), \
        (mx.max(), fro.max(), tr.max())


@pytest.mark.parametrize("n,B", [(1024, 6), (1000, 3), (1280, 2), (2048, 2)])
@pytest.mark.parametrize("mode", list(GATE))
def test_wide_vs_fp64_recursion(torch, model, n, B, mode, monkeypatch):
    """Forced at N >= 1000 (nb even; 1000 pads to 1024, 1280 has an odd number of super-rows; the
    default from N=4096): every member within the gates, D exactly symmetric, statistics consistent."""
    monkeypatch.setenv("FFG_WIDE", "1")
    mu, kT = batch_params(B)
    H = torch.from_numpy(np.stack([tight_binding(n, seed=300 + k) for k in range(B)])).cuda()
    D, stats, status = run(torch, H, mu, kT, model, mode)
    assert (status == 0).all()
    assert torch.equal(D, D.transpose(1, 2))
    R = DR.density_matrices_f64(H, mu, kT, model.abcd, model.beta0, model.mu0)
    gate(mode, D, R, f"wide {B}x N={n}")
    tr = torch.diagonal(D, dim1=1, dim2=2).sum(-1).cpu().numpy()
    assert np.allclose(stats[:, 0], tr, rtol=1e-12, atol=0)
    sq = (D * D).sum(dim=(1, 2)).cpu().numpy()
    assert np.allclose(stats[:, 1], sq, rtol=1e-11, atol=0)


@pytest.mark.parametrize("n", [256, 512, 768])
def test_wide_forced_small(torch, model, n, monkeypatch):
    """Forced below its default range: one super-block (N=256: the diagonal item only, its lower block
    discarded), three (N=512), six (N=768, odd super-row count); FP32-emulated gates hold."""
    monkeypatch.setenv("FFG_WIDE", "1")
    mu, kT = batch_params(3)
    H = torch.from_numpy(np.stack([tight_binding(n, seed=40 + k) for k in range(3)])).cuda()
    D, stats, status = run(torch, H, mu, kT, model, E.PrecisionMode.MIXED_EMULATED)
    assert (status == 0).all() and torch.equal(D, D.transpose(1, 2))
    R = DR.density_matrices_f64(H, mu, kT, model.abcd, model.beta0, model.mu0)
    gate(E.PrecisionMode.MIXED_EMULATED, D, R, f"wide forced N={n}")


def test_wide_and_pair_kernels_agree(torch, model, monkeypatch):
    """Both kernels evaluate the same recursion: at N=2048 their D differ only by rounding (both are
    within the gates of the fp64 recursion); the pair kernel is the default below N=4096."""
    assert E.k2_kernel_name(4096) == "mlsp2_wide_kernel" and E.k2_kernel_name(2048) == "mlsp2_pair_kernel"
    assert E.k2_kernel_name(4224) == "mlsp2_pair_kernel"  # nb = 33: no super-block tiling
    mu, kT = batch_params(2)
    H = torch.from_numpy(np.stack([tight_binding(2048, seed=70 + k) for k in range(2)])).cuda()
    Dd, _, _ = run(torch, H, mu, kT, model, E.PrecisionMode.MIXED_EMULATED)
    monkeypatch.setenv("FFG_WIDE", "1")
    Dw, _, _ = run(torch, H, mu, kT, model, E.PrecisionMode.MIXED_EMULATED)
    monkeypatch.setenv("FFG_WIDE", "0")
    Dp, _, _ = run(torch, H, mu, kT, model, E.PrecisionMode.MIXED_EMULATED)
    assert torch.equal(Dd, Dp)              # the default at N=2048 is the pair kernel
    assert (Dw - Dp).abs().max().item() < 5e-6
    assert not torch.equal(Dw, Dp)          # (different accumulation schedules: not the same bits)


def test_wide_schedule_invariance(torch, model, monkeypatch):
    """L2 group sizes reorder independent work only: D and the statistics are bit-identical; a
    member computed alone equals the same member inside the batch."""
    monkeypatch.setenv("FFG_WIDE", "1")
    mu, kT = batch_params(5)
    H = torch.from_numpy(np.stack([tight_binding(1024, seed=90 + k) for k in range(5)])).cuda()
    D0, s0, _ = run(torch, H, mu, kT, model, E.PrecisionMode.MIXED_EMULATED)
    for g in ("1", "2", "5"):
        monkeypatch.setenv("FFG_GROUP", g)
        D, s, _ = run(torch, H, mu, kT, model, E.PrecisionMode.MIXED_EMULATED)
        assert torch.equal(D, D0) and np.array_equal(s, s0), g
    monkeypatch.delenv("FFG_GROUP")
    D3, s3, _ = run(torch, H[3:4].clone(), mu[3:4], kT[3:4], model, E.PrecisionMode.MIXED_EMULATED)
    assert torch.equal(D3[0], D0[3]) and np.array_equal(s3[0], s0[3])


@pytest.mark.parametrize("mode", ["MIXED_EMULATED", "BF16"])
def test_wide_block_dependencies_bit_identical(torch, model, mode, monkeypatch):
    """Block-granular layer dependencies (single-matrix launches, FFG_BLOCKDEPS) only let an item's
    first K-blocks start before its whole super-rows are done: D and the statistics are bit-identical
    to the super-row-granular schedule."""
    monkeypatch.setenv("FFG_WIDE", "1")
    H = torch.from_numpy(tight_binding(2048, seed=77)[None]).cuda()
    mu, kT = batch_params(1)
    out = {}
    for bd in ("0", "1"):
        monkeypatch.setenv("FFG_BLOCKDEPS", bd)
        out[bd] = run(torch, H, mu, kT, model, E.PrecisionMode[mode])
    monkeypatch.delenv("FFG_BLOCKDEPS")
    assert torch.equal(out["0"][0], out["1"][0]) and np.array_equal(out["0"][1], out["1"][1])


def test_wide_out_of_region_member(torch, model, monkeypatch):
    """An out-of-region member of a wide batch issues no products and gets D = NaN; the other members
    are bit-identical to the batch without it."""
    monkeypatch.setenv("FFG_WIDE", "1")
    mu, kT = batch_params(4)
    kT = np.array(kT)
    H = torch.from_numpy(np.stack([tight_binding(1024, seed=120 + k) for k in range(4)])).cuda()
    kT_bad = kT.copy()
    kT_bad[2] = 0.0005  # beta' far beyond the model's region
    D, stats, status = run(torch, H, mu, kT_bad, model, E.PrecisionMode.MIXED_EMULATED)
    assert status.tolist() == [0, 0, E.OutOfRegionError.status, 0]
    assert torch.isnan(D[2]).all()
    keep = [0, 1, 3]
    D2, s2, _ = run(torch, H[keep].clone(), np.asarray(mu)[keep], kT[keep], model,
                    E.PrecisionMode.MIXED_EMULATED)
    assert torch.equal(D[keep], D2) and np.array_equal(stats[keep], s2)


def test_wide_provenance_products(model, monkeypatch):
    """Instrumented product count through the wide kernel: 4 products in the 10
    fixed-point layers, 3 in the others (FP32-emulated), 1 per layer in BF16."""
    monkeypatch.setenv("FFG_WIDE", "1")
    H = tight_binding(1024, seed=7)
    _, _, pv = E.compute_density_matrix(H, 0.0, 0.01, model, E.PrecisionMode.MIXED_EMULATED)
    assert pv.half_products == 10 * 4 + (model.layer_count - 10) * 3
    _, _, pv = E.compute_density_matrix(H, 0.0, 0.01, model, E.PrecisionMode.BF16)
    assert pv.half_products == model.layer_count


@pytest.mark.parametrize("mode", [E.PrecisionMode.MIXED_EMULATED, E.PrecisionMode.BF16])
def test_wide_default_padded_size(torch, model, mode):
    """The default selection at a padded size (n = 4300 -> np = 4352, 17 super-rows, 52 padded rows and
    columns): wide kernel, within the gates, exactly symmetric; n = 4200 (odd block count) and n = 2300
    stay on the pair kernel."""
    assert E.k2_kernel_name(4300) == "mlsp2_wide_kernel" and E.k2_kernel_name(4200) == "mlsp2_pair_kernel"
    assert E.k2_kernel_name(2300) == "mlsp2_pair_kernel"
    H = torch.from_numpy(tight_binding(4300, seed=23)).cuda().unsqueeze(0)
    D, stats, status = run(torch, H, [0.05], [0.011], model, mode)
    assert status.tolist() == [0] and torch.equal(D, D.transpose(1, 2))
    R = DR.density_matrices_f64(H, [0.05], [0.011], model.abcd, model.beta0, model.mu0)
    gate(mode, D, R, "wide default N=4300")
