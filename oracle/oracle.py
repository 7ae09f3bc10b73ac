"""TEST INFRASTRUCTURE ONLY -- the CPU oracle for the MLSP2 density-matrix path.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU legs
(``cpu_baseline`` and ``--impl reference``) may import this module, and only as
the checker / the timed CPU baseline.  The product path
(``paper_2605_08523_b200``) never imports it and fails loudly without its CUDA
library.

Three layers, strongest pinning first:

* ``ref()``      -- ctypes handle on ``oracle/_ref/libfermiforge_ref.so``: the
  reference's own ``scalar_models.cpp``/``trainer.cpp``/``symmetric_matrix.cpp``
  compiled from /root/reference by ``oracle/Makefile`` (absent on a box that
  did not build it; callers skip).
* ``lib()``      -- ctypes handle on ``oracle/libffo_oracle.so``: the plain-C
  restatement (``oracle/ffo_oracle.c``), each function citing its reference
  file:line.
* numpy functions below -- the same arithmetic with BLAS matmuls so the fp64
  recursion finishes in seconds at N >= 1024, plus the spectral-mapping oracle
  D = V diag(evaluate_model(m, lambda0)) V^T.

Frame convention: the reference model approximates
fermi(x; beta0, mu0) in the UN-flipped frame and flips internally
(scalar_models.cpp:333), so the rescale is
    X0 = (1 - mu0) I - (beta/beta0) (H - mu I),   x = mu0 + (beta/beta0)(lambda - mu).
"""
from __future__ import annotations

import ctypes
import json
import os
from functools import lru_cache

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_D = ctypes.POINTER(ctypes.c_double)
_F = ctypes.POINTER(ctypes.c_float)
_U16 = ctypes.POINTER(ctypes.c_uint16)


def _dp(a: np.ndarray):
    return a.ctypes.data_as(_D)


@lru_cache(maxsize=None)
def lib() -> ctypes.CDLL:
    path = os.path.join(HERE, "libffo_oracle.so")
    if not os.path.exists(path):
        import subprocess

        subprocess.run(["make", "-s", "-C", HERE, "liboracle"], check=True)
    L = ctypes.CDLL(path)
    L.ffo_evaluate_mlsp2.restype = ctypes.c_double
    L.ffo_evaluate_mlsp2.argtypes = [_D, ctypes.c_int, ctypes.c_double]
    L.ffo_evaluate_model.restype = ctypes.c_double
    L.ffo_evaluate_model.argtypes = [_D, ctypes.c_int, ctypes.c_double]
    L.ffo_fermi.restype = ctypes.c_double
    L.ffo_fermi.argtypes = [ctypes.c_double] * 3
    L.ffo_pairwise_sum.restype = ctypes.c_double
    L.ffo_pairwise_sum.argtypes = [_D, ctypes.c_int64]
    L.ffo_density_statistics.argtypes = [_D, ctypes.c_int64, _D]
    L.ffo_gershgorin.argtypes = [_D, ctypes.c_int64, _D, _D]
    L.ffo_region_check.restype = ctypes.c_int
    L.ffo_region_check.argtypes = [ctypes.c_double] * 6
    L.ffo_rescale.argtypes = [_D, ctypes.c_int64] + [ctypes.c_double] * 4 + [_D]
    L.ffo_mlsp2_from_x0.argtypes = [_D, ctypes.c_int64, _D, ctypes.c_int, _D]
    L.ffo_density_matrix_f64.restype = ctypes.c_int
    L.ffo_density_matrix_f64.argtypes = [_D, ctypes.c_int64, ctypes.c_double, ctypes.c_double,
                                         _D, ctypes.c_int, ctypes.c_double, ctypes.c_double,
                                         _D, _D, _D]
    L.ffo_float_to_half_bits.restype = ctypes.c_uint16
    L.ffo_float_to_half_bits.argtypes = [ctypes.c_float, ctypes.POINTER(ctypes.c_int)]
    L.ffo_half_bits_to_float.restype = ctypes.c_float
    L.ffo_half_bits_to_float.argtypes = [ctypes.c_uint16]
    L.ffo_split_half.restype = ctypes.c_int64
    L.ffo_split_half.argtypes = [_F, ctypes.c_int64, ctypes.c_float, _U16, _U16]
    L.ffo_mixed_square_emul.argtypes = [_F, ctypes.c_int64, ctypes.c_float, _F]
    return L


@lru_cache(maxsize=None)
def ref() -> ctypes.CDLL | None:
    """The compiled reference (oracle/_ref), or None when it was not built."""
    path = os.path.join(HERE, "_ref", "libfermiforge_ref.so")
    if not os.path.exists(path):
        return None
    R = ctypes.CDLL(path)
    R.ffr_last_error.restype = ctypes.c_char_p
    R.ffr_evaluate_mlsp2_model.restype = ctypes.c_int
    R.ffr_evaluate_mlsp2_model.argtypes = [_D, ctypes.c_int, ctypes.c_double, ctypes.c_double,
                                           _D, ctypes.c_int64, _D]
    R.ffr_fermi.restype = ctypes.c_double
    R.ffr_fermi.argtypes = [ctypes.c_double] * 3
    R.ffr_layer_count_estimate.restype = ctypes.c_int
    R.ffr_layer_count_estimate.argtypes = [ctypes.c_double]
    R.ffr_sp2_as_mlsp2.restype = ctypes.c_int
    R.ffr_sp2_as_mlsp2.argtypes = [ctypes.c_double, ctypes.c_int, _D]
    R.ffr_train_fermi_mlsp2.restype = ctypes.c_int
    R.ffr_train_fermi_mlsp2.argtypes = [ctypes.c_double, ctypes.c_double, ctypes.c_int,
                                        ctypes.c_int, ctypes.c_int, ctypes.c_uint64, _D, _D]
    R.ffr_pairwise_sum.restype = ctypes.c_double
    R.ffr_pairwise_sum.argtypes = [_D, ctypes.c_int64]
    R.ffr_density_statistics.restype = ctypes.c_int
    R.ffr_density_statistics.argtypes = [_D, ctypes.c_int, _D]
    return R


# ----------------------------------------------------------------------------- fixtures

GOLDEN = os.path.join(os.path.dirname(HERE), "tests", "golden")


def load_coefficients(name: str) -> dict:
    """tests/golden/coefficients_<name>.json -> {'abcd': (L,4) f64, 'beta0', 'mu0', ...}."""
    with open(os.path.join(GOLDEN, f"coefficients_{name}.json")) as f:
        d = json.load(f)
    d["abcd"] = np.array([[float(v) for v in row] for row in d["layers"]], dtype=np.float64)
    return d


def load_entropy_coefficients(name: str) -> dict:
    """tests/golden/coefficients_<E...>.json -> {'abcd', 'alpha', 'beta0', 'mu0', ...}."""
    d = load_coefficients(name)
    d["alpha"] = float(d["alpha"])
    return d


def evaluate_entropy_ref(abcd: np.ndarray, alpha: float, beta0: float, mu0: float, x: np.ndarray):
    """Reference evaluate_model for an Entropy model and fermi_entropy(x; beta0, mu0)."""
    R = ref()
    if R is None:
        raise RuntimeError("oracle/_ref not built")
    R.ffr_evaluate_entropy_model.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_double, ctypes.c_double,
                                             ctypes.c_double, ctypes.c_void_p, ctypes.c_int64,
                                             ctypes.c_void_p, ctypes.c_void_p]
    abcd = np.ascontiguousarray(abcd, dtype=np.float64)
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.zeros_like(x)
    ex = np.zeros_like(x)
    rc = R.ffr_evaluate_entropy_model(abcd.ctypes.data, abcd.shape[0], float(alpha), float(beta0), float(mu0),
                                      x.ctypes.data, x.size, y.ctypes.data, ex.ctypes.data)
    if rc != 0:
        raise RuntimeError(R.ffr_last_error().decode())
    return y, ex


def entropy_scalar(abcd: np.ndarray, alpha: float, mu0: float, x: np.ndarray) -> np.ndarray:
    """evaluate_entropy (scalar_models.cpp:320-326) restated: x0 = alpha (x - mu0) + mu0 (no flip),
    y = evaluate_mlsp2(x0) (acc += d x before the square; acc + x at the end), (4 ln 2) y (1 - y)."""
    x0 = alpha * (np.asarray(x, dtype=np.float64) - mu0) + mu0
    acc = np.zeros_like(x0)
    xx = x0.copy()
    for a, b, c, d in abcd:
        acc = acc + d * xx
        xx = a * xx * xx + b * xx + c
    y = acc + xx
    return 4.0 * np.log(2.0) * y * (1.0 - y)


def entropy_trace_f64(H: np.ndarray, mu: float, kT: float, abcd: np.ndarray, alpha: float, beta0: float,
                      mu0: float) -> float:
    """Tr s(H) by the fp64 matrix recursion: X0 = alpha (beta/beta0)(H - mu I) + mu0 I, Y = MLSP2(X0),
    Tr S = (4 ln 2)(Tr Y - Tr Y^2) (S = (4 ln 2) Y (I - Y), Y symmetric)."""
    n = H.shape[0]
    s = (1.0 / kT) / beta0
    X = alpha * s * (H - mu * np.eye(n)) + mu0 * np.eye(n)
    A = np.zeros_like(X)
    for a, b, c, d in abcd:
        A = A + d * X
        X = a * (X @ X) + b * X + c * np.eye(n)
    Y = A + X
    return float(4.0 * np.log(2.0) * (np.trace(Y) - np.sum(Y * Y)))


def entropy_trace_exact(H: np.ndarray, mu: float, kT: float) -> float:
    """sum_i s(f(lambda_i)) with s(y) = -y ln y - (1-y) ln(1-y) (exact electronic entropy)."""
    lam = np.linalg.eigvalsh(H)
    z = (lam - mu) / kT
    f = 1.0 / (1.0 + np.exp(np.clip(z, -700, 700)))
    with np.errstate(divide="ignore", invalid="ignore"):
        s = -np.where(f > 0, f * np.log(f), 0.0) - np.where(f < 1, (1 - f) * np.log1p(-f), 0.0)
    return float(np.sum(s))


# ----------------------------------------------------------------------------- scalar

def evaluate_model_c(abcd: np.ndarray, x: np.ndarray) -> np.ndarray:
    """ffo_evaluate_model elementwise (the C restatement)."""
    abcd = np.ascontiguousarray(abcd, dtype=np.float64)
    L = lib()
    return np.array([L.ffo_evaluate_model(_dp(abcd), abcd.shape[0], float(v)) for v in np.ravel(x)])


def evaluate_model_ref(abcd: np.ndarray, beta0: float, mu0: float, x: np.ndarray) -> np.ndarray:
    """The reference's compiled evaluate_model (scalar_models.cpp:330)."""
    R = ref()
    if R is None:
        raise RuntimeError("oracle/_ref not built")
    abcd = np.ascontiguousarray(abcd, dtype=np.float64)
    xs = np.ascontiguousarray(np.ravel(x), dtype=np.float64)
    out = np.empty_like(xs)
    rc = R.ffr_evaluate_mlsp2_model(_dp(abcd), abcd.shape[0], beta0, mu0, _dp(xs), xs.size, _dp(out))
    if rc:
        raise RuntimeError(R.ffr_last_error().decode())
    return out


def evaluate_model_np(abcd: np.ndarray, x: np.ndarray) -> np.ndarray:
    """Vectorised evaluate_mlsp2(1 - x), same operation order as scalar_models.cpp:243-252."""
    xv = 1.0 - np.asarray(x, dtype=np.float64)
    acc = np.zeros_like(xv)
    for a, b, c, d in abcd:
        acc = acc + d * xv
        x2 = xv * xv
        xv = a * x2 + b * xv + c
    return acc + xv


# ----------------------------------------------------------------------------- matrix

def gershgorin(H: np.ndarray) -> tuple[float, float]:
    """SPEC.md:319-327 (vectorised; same discs as ffo_gershgorin)."""
    d = np.diag(H)
    off = np.abs(H)
    off[np.diag_indices_from(off)] = 0.0  # sum over j != i only
    r = off.sum(axis=1)
    lo, hi = float((d - r).min()), float((d + r).max())
    w = 1e-12 * (hi - lo)
    return lo - w, hi + w


def region_ok(eps_min, eps_max, mu, kT, beta0, mu0) -> int:
    """1 valid, 0 lower inequality violated, -1 upper violated (see ffo_region_check)."""
    s = (1.0 / kT) / beta0
    if not (mu0 + s * (eps_min - mu) >= 0.0):
        return 0
    if not (mu0 + s * (eps_max - mu) <= 1.0):
        return -1
    return 1


def rescale(H: np.ndarray, mu: float, kT: float, beta0: float, mu0: float) -> np.ndarray:
    """X0 = (1 - mu0) I - (beta/beta0)(H - mu I)  (SPEC.md:329-347 + scalar_models.cpp:333)."""
    s = (1.0 / kT) / beta0
    X0 = -s * H
    X0[np.diag_indices_from(X0)] += (1.0 - mu0) + s * mu
    return X0


def mlsp2_recursion_f64(X0: np.ndarray, abcd: np.ndarray) -> np.ndarray:
    """fp64 matrix lift of evaluate_mlsp2 (scalar_models.cpp:243-252) with BLAS squares."""
    X = np.array(X0, dtype=np.float64, copy=True)
    A = np.zeros_like(X)
    idx = np.diag_indices_from(X)
    for a, b, c, d in abcd:
        A += d * X
        Y = X @ X
        Y = np.triu(Y) + np.triu(Y, 1).T  # exact symmetry, as SymmetricMatrix keeps it
        X = a * Y + b * X
        X[idx] += c
    return A + X


def density_matrix_f64(H, mu, kT, abcd, beta0, mu0):
    """compute_density_matrix in DOUBLE mode (numpy/BLAS); raises on out-of-region."""
    lo, hi = gershgorin(H)
    ok = region_ok(lo, hi, mu, kT, beta0, mu0)
    if ok != 1:
        raise ValueError(f"out of region ({'lower' if ok == 0 else 'upper'} inequality)")
    return mlsp2_recursion_f64(rescale(H, mu, kT, beta0, mu0), abcd)


def density_statistics(D: np.ndarray) -> tuple[float, float]:
    """(Tr D, sum D_ij^2) via the C pairwise tree (symmetric_matrix.cpp:57-67)."""
    D = np.ascontiguousarray(D, dtype=np.float64)
    out = np.zeros(2)
    lib().ffo_density_statistics(_dp(D), D.shape[0], _dp(out))
    return float(out[0]), float(out[1])


def spectral_oracle(H, mu, kT, abcd, beta0, mu0, evaluate=None) -> np.ndarray:
    """D = V diag(evaluate_model(m, mu0 + s (lambda - mu))) V^T with fp64 LAPACK eigh.

    ``evaluate`` defaults to the compiled reference evaluate_model when oracle/_ref
    exists, else to the C restatement (which the tests pin bit-for-bit to it).
    """
    lam, V = np.linalg.eigh(np.asarray(H, dtype=np.float64))
    s = (1.0 / kT) / beta0
    x = mu0 + s * (lam - mu)
    if evaluate is None:
        evaluate = (lambda xx: evaluate_model_ref(abcd, beta0, mu0, xx)) if ref() is not None \
            else (lambda xx: evaluate_model_np(abcd, xx))
    f = evaluate(x)
    return (V * f) @ V.T


def exact_fermi_density(H, mu, kT) -> np.ndarray:
    lam, V = np.linalg.eigh(np.asarray(H, dtype=np.float64))
    t = (lam - mu) / kT
    f = np.where(t > 0, np.exp(-np.abs(t)) / (1 + np.exp(-np.abs(t))), 1 / (1 + np.exp(-np.abs(t))))
    return (V * f) @ V.T


# ----------------------------------------------------------------------------- mixed precision emulation

HALF_SCALE = 16384.0  # global 2^14 pre-scale of X before the binary16 split


def split_half(X: np.ndarray, scale: float = HALF_SCALE):
    """hi = fp16(X*scale), lo = fp16(X*scale - hi), RNE (numpy float16 casts are RNE)."""
    xs = np.asarray(X, dtype=np.float32) * np.float32(scale)
    hi = xs.astype(np.float16)
    lo = (xs - hi.astype(np.float32)).astype(np.float16)
    return hi, lo


def mlsp2_recursion_emulated(X0: np.ndarray, abcd: np.ndarray, mode: str = "fp32emul") -> np.ndarray:
    """CPU emulation of the tensor-core recursion (SURVEY.md Appendix B recipe).

    fp32emul: Y = (hi@hi + hi@lo + lo@hi) / scale^2 with fp32 matmuls of
    fp16-valued operands; bf16 / fp16: one single-product square.  X and A are
    kept in fp32 between layers.  Products are exact in fp32; the summation
    order differs from the tensor core, so this is a statistical reference.
    """
    import torch

    X = torch.from_numpy(np.asarray(X0, dtype=np.float32).copy())
    A = torch.zeros_like(X)
    n = X.shape[0]
    eye = torch.eye(n, dtype=torch.float32)
    for a, b, c, d in abcd:
        A += np.float32(d) * X
        if mode == "fp32emul":
            xs = X * HALF_SCALE
            hi = xs.to(torch.float16).to(torch.float32)
            lo = (xs - hi).to(torch.float16).to(torch.float32)
            Y = (hi @ hi + (hi @ lo + lo @ hi)) / (HALF_SCALE * HALF_SCALE)
        elif mode == "fp16":
            hi = (X * HALF_SCALE).to(torch.float16).to(torch.float32)
            Y = (hi @ hi) / (HALF_SCALE * HALF_SCALE)
        elif mode == "bf16":
            hi = X.to(torch.bfloat16).to(torch.float32)
            Y = hi @ hi
        else:
            raise ValueError(mode)
        Y = torch.triu(Y) + torch.triu(Y, 1).T
        X = (float(a) * Y.double() + float(b) * X.double() + float(c) * eye.double()).float()
    return (A.double() + X.double()).numpy()
