"""CPU tests: the oracle pinned against the reference's golden vectors and its own
compiled code (oracle/_ref), plus the reference's scalar known answers that fix
the frame convention.  No GPU needed."""
import ctypes
import json
import os

import numpy as np
import pytest

from oracle import oracle as O
from paper_2605_08523_b200.hamiltonians import tight_binding, goe

G = O.GOLDEN


def _scalar(name):
    with open(os.path.join(G, f"scalar_{name}.json")) as f:
        d = json.load(f)
    return np.array([float(v) for v in d["x"]]), np.array([float(v) for v in d["evaluate_model"]])


# ----------------------------------------------------------------- fixtures themselves
def test_coefficients_match_survey_appendix_a(m1500, m40):
    # SURVEY.md Appendix A rows, %.17g, from train_fermi (trainer.cpp:1215)
    assert m1500["abcd"].shape == (30, 4) and m40["abcd"].shape == (14, 4)
    assert m1500["layers"][0] == ["0.99861406942339959", "-0.0010851153815639274",
                                  "-0.00084127984440128859", "5.9149661965328082e-07"]
    assert m1500["layers"][29][3] == "-0.036837212838032915"
    assert m40["layers"][13] == ["0.66872028737301248", "0.062662288047919984",
                                 "-0.24446097247130474", "0.062662288047919956"]
    assert m1500["report"]["final_max_error"] <= 1.01e-7
    assert m40["report"]["final_max_error"] <= 1e-6  # test_trainer.cpp:309


def test_package_coefficients_are_the_golden_ones():
    root = os.path.dirname(G.rstrip("/")).rsplit("/tests", 1)[0]
    for name in ("M1500", "M40"):
        with open(os.path.join(root, "paper_2605_08523_b200", "coefficients", f"{name}.json")) as f:
            a = json.load(f)
        with open(os.path.join(G, f"coefficients_{name}.json")) as f:
            b = json.load(f)
        assert a["layers"] == b["layers"] and a["beta0"] == b["beta0"] and a["mu0"] == b["mu0"]


# ----------------------------------------------------------------- scalar restatement
@pytest.mark.parametrize("name", ["M1500", "M40"])
def test_c_restatement_bit_exact_vs_golden_table(name):
    m = O.load_coefficients(name)
    xs, ys = _scalar(name)
    got = O.evaluate_model_c(m["abcd"], xs)
    assert np.array_equal(got, ys)          # same operation order -> bitwise
    got_np = O.evaluate_model_np(m["abcd"], xs)
    assert np.array_equal(got_np, ys)


@pytest.mark.parametrize("name", ["M1500", "M40"])
def test_c_restatement_bit_exact_vs_compiled_reference(name):
    if O.ref() is None:
        pytest.skip("oracle/_ref not built")
    m = O.load_coefficients(name)
    xs = np.random.default_rng(0).uniform(-0.1, 1.1, 5000)
    ref = O.evaluate_model_ref(m["abcd"], float(m["beta0"]), float(m["mu0"]), xs)
    assert np.array_equal(O.evaluate_model_c(m["abcd"], xs), ref)


@pytest.mark.parametrize("name,beta0,mu0,tol", [("M1500", 1500.0, 1 / 3, 1.01e-7), ("M40", 40.0, 0.3, 3e-7)])
def test_model_approximates_unflipped_fermi(name, beta0, mu0, tol):
    # frame pin: evaluate_model(m, x) ~ fermi(x; beta0, mu0), step DOWN at mu0
    m = O.load_coefficients(name)
    xs = np.linspace(0, 1, 20001)
    f = np.array([O.lib().ffo_fermi(x, beta0, mu0) for x in xs])
    assert np.abs(O.evaluate_model_np(m["abcd"], xs) - f).max() <= tol
    assert O.evaluate_model_np(m["abcd"], np.array([0.05]))[0] > 0.99  # test_trainer.cpp:274-278
    assert O.evaluate_model_np(m["abcd"], np.array([0.6]))[0] < 0.01


def test_recursion_range_envelope(m1500, m40):
    # test_scalar_models.cpp:225-238: intermediate x stays in [-0.5, 1.5]
    for m in (m1500, m40):
        x = 1.0 - np.linspace(0, 1, 2001)
        for a, b, c, d in m["abcd"]:
            x = a * x * x + b * x + c
            assert x.min() >= -0.5 and x.max() <= 1.5


def test_sp2_embedding_golden():
    # SP2 -> MLSP2 coefficient map (test_scalar_models.cpp:163-177): a=+1,b=0 or a=-1,b=2
    with open(os.path.join(G, "sp2_mlsp2.json")) as f:
        d = json.load(f)
    for rows in d.values():
        for a, b, c, dd in rows:
            assert (float(a), float(b)) in ((1.0, 0.0), (-1.0, 2.0))
            assert float(c) == 0.0 and float(dd) == 0.0


# ----------------------------------------------------------------- reductions
def test_pairwise_sum_matches_reference():
    v = np.random.default_rng(1).standard_normal(10007)
    got = O.lib().ffo_pairwise_sum(O._dp(v), v.size)
    if O.ref() is not None:
        assert got == O.ref().ffr_pairwise_sum(O._dp(v), v.size)
    assert abs(got - v.sum()) <= 1e-12 * np.abs(v).sum()


def test_density_statistics_known_answers():
    assert O.density_statistics(np.eye(4)) == (4.0, 4.0)
    assert O.density_statistics(np.diag([0.5, 0.5])) == (1.0, 0.5)
    if O.ref() is not None:
        A = np.random.default_rng(2).standard_normal((50, 50))
        D = np.ascontiguousarray((A + A.T) / 2)
        st = np.zeros(2)
        O.ref().ffr_density_statistics(O._dp(D), 50, O._dp(st))
        assert O.density_statistics(D) == (st[0], st[1])


# ----------------------------------------------------------------- bounds / rescale
def test_gershgorin_c_vs_numpy():
    for H in (tight_binding(256, seed=1234), goe(64, seed=3)):
        lo = ctypes.c_double()
        hi = ctypes.c_double()
        Hc = np.ascontiguousarray(H)
        O.lib().ffo_gershgorin(O._dp(Hc), H.shape[0], ctypes.byref(lo), ctypes.byref(hi))
        nlo, nhi = O.gershgorin(H)
        assert abs(lo.value - nlo) <= 1e-14 * abs(nlo) and abs(hi.value - nhi) <= 1e-14 * abs(nhi)
    # SPEC.md:325-326 known answers
    lo, hi = O.gershgorin(np.array([[0.0, 1.0], [1.0, 0.0]]))
    assert lo < -1.0 and hi > 1.0 and abs(lo + 1) < 1e-11
    lo, hi = O.gershgorin(np.diag([1.0, 2.0]))
    assert abs(lo - (1 - 1e-12)) < 1e-15 and abs(hi - (2 + 1e-12)) < 1e-15


def test_tb_bounds_inside_4p5():
    for n in (256, 512, 1024):
        lo, hi = O.gershgorin(tight_binding(n, seed=1234))
        assert -4.5 <= lo and hi <= 4.5


def test_spec_rescale_example_in_reference_frame():
    # H'=diag(0,1), beta'=20, mu'=0.5, beta0=40, mu0=0.3 -> H0 = diag(0.05, 0.55)
    # in the SPEC (flipped) frame; our closed form works in the UN-flipped frame where the
    # same physics maps x = mu0 + (beta/beta0)(lambda - mu).  With H=diag(1,0) (un-flipped
    # H' of the example, W=1, beta=20, mu=0.5): x = 0.3 + 0.5 (lambda - 0.5)
    X0 = O.rescale(np.diag([1.0, 0.0]), 0.5, 1 / 20.0, 40.0, 0.3)
    x = 1.0 - np.diag(X0)
    assert np.allclose(x, [0.55, 0.05], atol=1e-15)


def test_spec_two_level_frame_trap(m1500):
    # SPEC.md:464 with the reference model: D ~ diag(f(0), f(1)) (NOT reversed)
    D = O.density_matrix_f64(np.diag([0.0, 1.0]), 0.5, 1 / 50.0, m1500["abcd"], 1500.0, 1 / 3)
    f0, f1 = 1 / (1 + np.exp(-25.0)), 1 / (1 + np.exp(25.0))
    assert abs(D[0, 0] - f0) < 1e-6 and abs(D[1, 1] - f1) < 1e-6


def test_region_of_validity_truth_table():
    # Eq. 41 with un-flipped mu' (SPEC.md:355-357 examples)
    from paper_2605_08523_b200.engine import in_region_of_validity
    assert in_region_of_validity(20, 0.3, 40, 0.3)
    assert not in_region_of_validity(40, 0.5, 40, 0.3)
    assert in_region_of_validity(900, 0.5, 1500, 1 / 3)
    assert not in_region_of_validity(2000, 0.5, 1500, 1 / 3)


# ----------------------------------------------------------------- matrix recursion
@pytest.mark.parametrize("tag", ["tb16", "tb64", "tb64_m40", "goe64"])
def test_recursion_restatements_agree_with_spectral_fixture(tag):
    f = np.load(os.path.join(G, f"matrix_{tag}.npz"))
    m = O.load_coefficients(str(f["model"]))
    H, mu, kT = f["H"], float(f["mu"]), float(f["kT"])
    b0, m0 = float(m["beta0"]), float(m["mu0"])
    Dnp = O.density_matrix_f64(H, mu, kT, m["abcd"], b0, m0)
    assert np.abs(Dnp - f["D_spectral"]).max() <= 5e-14
    assert np.array_equal(Dnp, f["D_recursion"])
    # plain-C restatement (unblocked loops)
    n = H.shape[0]
    Dc = np.zeros((n, n))
    st = np.zeros(2)
    bd = np.zeros(2)
    abcd = np.ascontiguousarray(m["abcd"])
    rc = O.lib().ffo_density_matrix_f64(O._dp(np.ascontiguousarray(H)), n, mu, kT, O._dp(abcd),
                                        abcd.shape[0], b0, m0, O._dp(Dc), O._dp(st), O._dp(bd))
    assert rc == 1
    assert np.abs(Dc - f["D_spectral"]).max() <= 5e-14
    assert abs(st[0] - f["stats_ref"][0]) <= 1e-13 * abs(st[0])


def test_emulation_meets_survey_gates(m1500):
    # the CPU emulation of FP32-emulated mode meets the parity gates it is used to set
    H = tight_binding(256, seed=1234)
    X0 = O.rescale(H, 0.0, 0.01, 1500.0, 1 / 3)
    Dref = O.mlsp2_recursion_f64(X0, m1500["abcd"])
    De = O.mlsp2_recursion_emulated(X0, m1500["abcd"], "fp32emul")
    assert np.abs(De - Dref).max() <= 5e-6
    assert abs(np.trace(De) - np.trace(Dref)) / np.trace(Dref) <= 1e-6


# ----------------------------------------------------------------- binary16 restatement
def test_half_conversion_matches_numpy_rne():
    rng = np.random.default_rng(4)
    xs = np.concatenate([rng.standard_normal(20000).astype(np.float32) * 10.0 ** rng.integers(-9, 5, 20000),
                         np.array([0.0, -0.0, 65504.0, 65519.0, 5.96e-8, 2.98e-8, 1e-30], dtype=np.float32)])
    xs = xs.astype(np.float32)
    L = O.lib()
    of = ctypes.c_int()
    for x in xs:
        h = L.ffo_float_to_half_bits(float(x), ctypes.byref(of))
        ref = np.array([x], dtype=np.float32).astype(np.float16).view(np.uint16)[0]
        assert h == ref, (x, h, ref)
        assert L.ffo_half_bits_to_float(h) == np.float32(np.uint16(h).view(np.float16))
    L.ffo_float_to_half_bits(70000.0, ctypes.byref(of))
    assert of.value == 1  # HalfRangeError condition (half_precision.hpp:13-16)
