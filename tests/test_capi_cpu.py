"""CPU tests of the C-ABI boundary: the library loads, exports every symbol the
header declares, validates inputs like the reference, and refuses to compute
without an sm_100 device (no CPU fallback)."""
import ctypes
import re
import subprocess

import numpy as np
import pytest

from paper_2605_08523_b200 import engine as E

HEADER = "include/fermiforge/ffg.h"


def declared_symbols():
    import os
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    txt = open(os.path.join(root, HEADER)).read()
    return sorted(set(re.findall(r"^\s*(?:int|int32_t|int64_t|void|const char\*)\s+(ffg_\w+)\(", txt, re.M)))


def test_library_exports_every_declared_symbol():
    syms = declared_symbols()
    assert len(syms) >= 12
    out = subprocess.run(["nm", "-D", "--defined-only", E.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (ffg_\w+)", out))
    missing = [s for s in syms if s not in exported]
    assert not missing, missing
    assert set(E.SYMBOLS) <= exported
    L = E.lib()
    for s in syms:
        assert hasattr(L, s)


def test_binary_contains_tcgen05_and_tma():
    sass = subprocess.run(["cuobjdump", "-sass", E.LIB_PATH], capture_output=True, text=True).stdout
    assert "UTCHMMA" in sass, "no tcgen05.mma in the product library"
    assert "UTMALDG" in sass, "no TMA loads in the product library"
    assert "LDTM" in sass, "no tcgen05.ld in the product library"
    assert "HMMA" not in re.sub(r"UTCHMMA", "", sass), "legacy mma.sync found"


def test_binary_has_both_k2_kernels_and_nvtx_ranges():
    """Both recursion kernels are in the product library (the wide one with MN-major operand reads:
    its instruction descriptors are built at run time, so only the kernel symbols are checked), and
    the entry points carry NVTX ranges (header-only NVTX3: no link dependency)."""
    syms = subprocess.run(["cuobjdump", "-symbols", E.LIB_PATH], capture_output=True, text=True).stdout
    assert "mlsp2_pair_kernel" in syms and "mlsp2_wide_kernel" in syms
    blob = open(E.LIB_PATH, "rb").read()
    for name in (b"ffg_density_matrices_dev", b"ffg K2 enqueue (recursion layers)", b"ffg_rowblock_layer"):
        assert name + b"\0" in blob, name
    deps = subprocess.run(["ldd", E.LIB_PATH], capture_output=True, text=True).stdout
    assert "nvToolsExt" not in deps


def test_validation_mirrors_reference():
    m = E.load_model("M1500")
    H = np.eye(8)
    with pytest.raises(E.ValidationError, match="kT"):
        E.compute_density_matrix(H, 0.0, 0.0, m)
    with pytest.raises(E.ValidationError, match="mu0 must lie in"):
        E.compute_density_matrix(H, 0.0, 0.01, E.Mlsp2Model(m.abcd, 1500.0, 1.0))
    with pytest.raises(E.ValidationError, match="beta must be positive"):
        E.compute_density_matrix(H, 0.0, 0.01, E.Mlsp2Model(m.abcd, -1.0, 0.3))
    bad = m.abcd.copy()
    bad[3, 1] = np.nan
    with pytest.raises(E.ValidationError, match="finite"):
        E.compute_density_matrix(H, 0.0, 0.01, E.Mlsp2Model(bad, 1500.0, 1 / 3))
    with pytest.raises(E.DimensionError):
        E.compute_density_matrix(np.zeros((3, 4)), 0.0, 0.01, m)
    with pytest.raises(E.DimensionError):
        E.compute_density_matrices([np.eye(4), np.eye(5)], 0.0, 0.01, m)


def test_kernel_selection(monkeypatch):
    """The recursion kernel depends only on n and the mode (ffg_k2_kernel, host logic): the pair kernel
    below N=4096 and for odd block counts, the wide kernel from N=4096 with an even block count;
    FFG_WIDE overrides where the wide tiling applies."""
    monkeypatch.delenv("FFG_WIDE", raising=False)
    for mode in (E.PrecisionMode.MIXED_EMULATED, E.PrecisionMode.BF16, E.PrecisionMode.FP16):
        for n in (1, 256, 1000, 1024, 2048, 3072, 3968, 4200):
            assert E.k2_kernel_name(n, mode) == "mlsp2_pair_kernel", (n, mode)
        for n in (4000, 4096, 4300, 8192, 16384):  # 4000 pads to 4096
            assert E.k2_kernel_name(n, mode) == "mlsp2_wide_kernel", (n, mode)
    monkeypatch.setenv("FFG_WIDE", "1")
    assert E.k2_kernel_name(1024) == "mlsp2_wide_kernel" and E.k2_kernel_name(4200) == "mlsp2_pair_kernel"
    monkeypatch.setenv("FFG_WIDE", "0")
    assert E.k2_kernel_name(8192) == "mlsp2_pair_kernel"


def test_modes():
    """Every PrecisionMode of SPEC.md:308-311 is accepted (DOUBLE / SINGLE run the library-GEMM path);
    an unknown mode id is a validation error before any device work."""
    m = E.load_model("M1500")
    m_c = m._c()
    assert E.k2_kernel_name(1024, E.PrecisionMode.DOUBLE) == "cublas_gemm+direct_layer"
    assert E.k2_kernel_name(1024, E.PrecisionMode.SINGLE) == "cublas_gemm+direct_layer"
    rc = E.lib().ffg_density_matrix(E._dp(np.eye(4)), 4, 0.0, 0.01, ctypes.byref(m_c), 7, None, None, None)
    with pytest.raises(E.ValidationError, match="PrecisionMode"):
        E._check(rc)


def test_no_cpu_fallback_without_device():
    if E.device_available():
        pytest.skip("device present")
    m = E.load_model("M1500")
    with pytest.raises(E.CudaError):
        E.compute_density_matrix(np.eye(8) * 0.1, 0.0, 0.01, m)
    with pytest.raises(E.CudaError):
        E.mixed_square(np.eye(8, dtype=np.float32))


def test_kernel_launch_accounting():
    m = E.load_model("M1500")
    # two launch-carried parameter uploads, reset, K1, K2 (all 30 layers), K3
    assert E.kernel_launches(1, 1024, m) == 6 and E.kernel_launches(16, 1024, m) == 6
    assert E.kernel_launches(8193, 512, m) == 7  # K2 once per 8192 matrices (validity bitmap)
    assert E.kernel_launches(4, 1024, m, E.PrecisionMode.DOUBLE) == 6 + 30
    assert E.algorithmic_flops(4096, 30, E.PrecisionMode.MIXED_EMULATED) == pytest.approx(6.19e12, rel=1e-3)
    assert E.algorithmic_flops(1024, 30, E.PrecisionMode.BF16) == pytest.approx(3.22e10, rel=1e-2)


@pytest.mark.parametrize("nb", list(range(1, 41)) + [64, 127, 128])
def test_pair_table_covers_upper_triangle_once(nb):
    """K2 decomposition (k2_pair.cuh): every block {R, C} exactly once, each pair shares its
    B panel, at most one dummy (only when the block count is odd)."""
    t = E.pair_table(nb)
    seen = {}
    for a0, a1, s, d in t.tolist():
        assert max(a0, a1, s) < nb
        for a in ([a0] if d else [a0, a1]):
            key = (min(a, s), max(a, s))
            seen[key] = seen.get(key, 0) + 1
        if not d:
            assert a0 != a1
    want = {(i, j) for i in range(nb) for j in range(i, nb)}
    assert set(seen) == want and set(seen.values()) == {1}
    assert int(t[:, 3].sum()) == (nb * (nb + 1) // 2) % 2
