"""Python mirror of the reference matrix-engine / workflow interface, bound to the
B200 C ABI (include/fermiforge/ffg.h) through ctypes.

Names, argument meaning and error behaviour follow the reference specification
(SPEC.md module matrix_engine :288-425 and workflow :427-524, over the proj/core
types of scalar_models.hpp / symmetric_matrix.hpp):

    spectral_bounds(H)
    in_region_of_validity(beta', mu', b0, m0)  SPEC.md:349-357 (Eq. 41)
    apply_model(H0, model, mode)
    mixed_square(X)
    density_statistics(D)
    compute_density_matrix(H, mu, kT, model)   SPEC.md:458-462 (model already selected)
    compute_density_matrices(Hs, mu, kT, ...)  batched
    compute_density_matrices_device(...)       device-resident, async on a stream

There is no CPU fallback: every call goes through libfermiforge_b200.so, and
importing this module raises if the library was not built.
"""
from __future__ import annotations

import ctypes
import json
import os
from dataclasses import dataclass, field
from enum import IntEnum
from functools import lru_cache
from typing import Sequence

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FFG_LIB_PATH") or os.path.join(_PKG, "lib", "libfermiforge_b200.so")

_D = ctypes.POINTER(ctypes.c_double)
_F = ctypes.POINTER(ctypes.c_float)
MODEL_SCHEMA_VERSION = 1  # ModelFile schema


class PrecisionMode(IntEnum):
    """SPEC.md:308-311 PrecisionMode plus the B200 single-product modes."""
    DOUBLE = 0
    SINGLE = 1
    MIXED_EMULATED = 2  # FP32-emulated: binary16 hi/lo, 3 tensor-core products / square
    BF16 = 3
    FP16 = 4


# ------------------------------------------------------------------ errors (ffg_status)
class FermiforgeError(RuntimeError):
    status = -1


class ValidationError(FermiforgeError):      # scalar_models.hpp:21-24
    status = 1


class OutOfRegionError(FermiforgeError):
    status = 2


class DivergedEvaluationError(FermiforgeError):  # trainer.hpp:20-25 (carries the layer)
    status = 3

    def __init__(self, msg, layer=None):
        super().__init__(msg)
        self.layer = layer


class HalfRangeError(FermiforgeError):       # half_precision.hpp:13-16
    status = 4


class UnsupportedModeError(FermiforgeError):
    status = 5


class DimensionError(FermiforgeError, ValueError):  # std::invalid_argument
    status = 6


class CudaError(FermiforgeError):
    status = 7


class NcclError(FermiforgeError):
    status = 8


_ERRORS = {c.status: c for c in (ValidationError, OutOfRegionError, DivergedEvaluationError,
                                 HalfRangeError, UnsupportedModeError, DimensionError, CudaError,
                                 NcclError)}


class _Model(ctypes.Structure):
    _fields_ = [("abcd", _D), ("n_layers", ctypes.c_int32), ("beta0", ctypes.c_double),
                ("mu0", ctypes.c_double)]


class _EntropyModel(ctypes.Structure):
    _fields_ = [("inner", _Model), ("alpha", ctypes.c_double)]


class _MuReport(ctypes.Structure):
    _fields_ = [("mu", ctypes.c_double), ("residual", ctypes.c_double), ("iterations", ctypes.c_int32),
                ("converged", ctypes.c_int32), ("bisections", ctypes.c_int32)]


class _Prov(ctypes.Structure):
    _fields_ = [("eps_min", ctypes.c_double), ("eps_max", ctypes.c_double),
                ("beta_prime", ctypes.c_double), ("mu_prime", ctypes.c_double),
                ("x_min", ctypes.c_double), ("x_max", ctypes.c_double),
                ("mode", ctypes.c_int32), ("n_layers", ctypes.c_int32),
                ("half_products", ctypes.c_int64), ("diverged_layer", ctypes.c_int32),
                ("half_range_layer", ctypes.c_int32), ("status", ctypes.c_int32),
                ("n", ctypes.c_int32), ("device_ms", ctypes.c_double)]


SYMBOLS = ("ffg_abi_version", "ffg_last_error", "ffg_device_available", "ffg_in_region_of_validity",
           "ffg_spectral_bounds", "ffg_apply_model", "ffg_mixed_square", "ffg_density_statistics",
           "ffg_density_matrix", "ffg_density_matrices", "ffg_density_matrices_dev",
           "ffg_kernel_launches", "ffg_profile_layers", "ffg_profile_read",
           "ffg_profile_read_ex", "ffg_pair_table", "ffg_release_workspaces",
           "ffg_entropy_trace", "ffg_expectation", "ffg_solve_chemical_potential",
           "ffg_density_matrices_async", "ffg_wait", "ffg_k2_kernel")


@lru_cache(maxsize=None)
def lib() -> ctypes.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with `make lib` "
                          "(or __graft_entry__.build()); there is no CPU fallback")
    L = ctypes.CDLL(LIB_PATH)
    L.ffg_abi_version.restype = ctypes.c_int
    L.ffg_last_error.restype = ctypes.c_char_p
    L.ffg_device_available.restype = ctypes.c_int
    L.ffg_in_region_of_validity.restype = ctypes.c_int
    L.ffg_in_region_of_validity.argtypes = [ctypes.c_double] * 4
    L.ffg_spectral_bounds.argtypes = [_D, ctypes.c_int64, _D, _D]
    L.ffg_apply_model.argtypes = [_D, ctypes.c_int64, ctypes.POINTER(_Model), ctypes.c_int32, _D,
                                  ctypes.POINTER(_Prov)]
    L.ffg_mixed_square.argtypes = [_F, ctypes.c_int64, _F]
    L.ffg_density_statistics.argtypes = [_D, ctypes.c_int64, _D]
    L.ffg_density_matrix.argtypes = [_D, ctypes.c_int64, ctypes.c_double, ctypes.c_double,
                                     ctypes.POINTER(_Model), ctypes.c_int32, _D, _D,
                                     ctypes.POINTER(_Prov)]
    L.ffg_density_matrices.argtypes = [ctypes.c_int32, ctypes.POINTER(_D), ctypes.c_int64, _D, _D,
                                       ctypes.POINTER(_Model), ctypes.c_int32, ctypes.POINTER(_D),
                                       _D, ctypes.POINTER(_Prov)]
    L.ffg_density_matrices_dev.argtypes = [ctypes.c_int32, ctypes.c_void_p, ctypes.c_int64, _D, _D,
                                           ctypes.POINTER(_Model), ctypes.c_int32, ctypes.c_void_p,
                                           ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                           ctypes.c_void_p]
    L.ffg_k2_kernel.restype = ctypes.c_int32
    L.ffg_k2_kernel.argtypes = [ctypes.c_int64, ctypes.c_int32]
    L.ffg_kernel_launches.restype = ctypes.c_int64
    L.ffg_kernel_launches.argtypes = [ctypes.c_int32, ctypes.c_int64, ctypes.POINTER(_Model),
                                      ctypes.c_int32]
    L.ffg_profile_layers.argtypes = [ctypes.c_int]
    L.ffg_profile_read.argtypes = [_D, ctypes.POINTER(ctypes.c_int64)]
    L.ffg_profile_read_ex.argtypes = [_D, ctypes.POINTER(ctypes.c_int64), _D]
    L.ffg_entropy_trace.argtypes = [_D, ctypes.c_int64, ctypes.c_double, ctypes.c_double,
                                    ctypes.POINTER(_EntropyModel), ctypes.c_int32, _D, ctypes.POINTER(_Prov)]
    L.ffg_expectation.argtypes = [_D, _D, ctypes.c_int64, _D]
    L.ffg_solve_chemical_potential.argtypes = [_D, ctypes.c_int64, ctypes.c_double, ctypes.c_double,
                                               ctypes.c_double, ctypes.POINTER(_Model), ctypes.c_int32,
                                               ctypes.c_double, ctypes.c_int32, _D, _D, _D,
                                               ctypes.POINTER(_MuReport)]
    L.ffg_density_matrices_async.argtypes = [ctypes.c_int32, ctypes.POINTER(_D), ctypes.c_int64, _D, _D,
                                             ctypes.POINTER(_Model), ctypes.c_int32, ctypes.POINTER(_D),
                                             ctypes.POINTER(ctypes.c_int64)]
    L.ffg_wait.argtypes = [ctypes.c_int64, _D, ctypes.POINTER(_Prov)]
    L.ffg_pair_table.restype = ctypes.c_int32
    L.ffg_pair_table.argtypes = [ctypes.c_int32, ctypes.c_void_p, ctypes.c_int32]
    L.ffg_release_workspaces.restype = None
    assert L.ffg_abi_version() == 1
    return L


def _check(rc: int):
    if rc == 0:
        return
    msg = lib().ffg_last_error().decode()
    cls = _ERRORS.get(rc, FermiforgeError)
    raise cls(msg)


def _dp(a: np.ndarray):
    return a.ctypes.data_as(_D)


def device_available() -> bool:
    return bool(lib().ffg_device_available())


# ------------------------------------------------------------------ types
@dataclass
class Mlsp2Model:
    """ModelCoefficients with architecture MLSP2 (scalar_models.hpp:80-88, :173-183)."""
    abcd: np.ndarray           # (L, 4) rows a, b, c, d
    beta0: float
    mu0: float
    name: str = ""
    meta: dict = field(default_factory=dict)

    def __post_init__(self):
        self.abcd = np.ascontiguousarray(np.asarray(self.abcd, dtype=np.float64).reshape(-1, 4))

    @property
    def layer_count(self) -> int:
        return int(self.abcd.shape[0])

    def _c(self) -> _Model:
        # keep abcd alive through self
        return _Model(_dp(self.abcd), self.layer_count, float(self.beta0), float(self.mu0))

    @staticmethod
    def from_json(path: str) -> "Mlsp2Model":
        """Load a ModelFile: schema_version is checked on load, coefficients are
        decimal strings with 17 significant digits (bit-exact binary64 round trip)."""
        with open(path) as f:
            d = json.load(f)
        ver = d.get("schema_version")
        if ver != MODEL_SCHEMA_VERSION:
            raise ValidationError(f"{path}: ModelFile schema_version {ver!r} is not supported "
                                  f"(expected {MODEL_SCHEMA_VERSION})")
        if str(d.get("architecture", "")).lower() != "mlsp2":
            raise ValidationError(f"{path}: architecture {d.get('architecture')!r} is not MLSP2")
        abcd = np.array([[float(v) for v in row] for row in d["layers"]], dtype=np.float64)
        return Mlsp2Model(abcd, float(d["beta0"]), float(d["mu0"]), d.get("name", ""), d)

    def to_json(self, path: str, **extra) -> None:
        """Write a ModelFile: schema_version, created timestamp, 17-significant-digit decimals."""
        import datetime
        d = {k: v for k, v in self.meta.items() if k not in ("layers", "beta0", "mu0")}
        d.update(extra)
        d.update({"schema_version": MODEL_SCHEMA_VERSION, "name": self.name or d.get("name", ""),
                  "architecture": "mlsp2", "beta0": "%.17g" % self.beta0, "mu0": "%.17g" % self.mu0,
                  "layers": [["%.17g" % v for v in row] for row in self.abcd]})
        d.setdefault("created", datetime.datetime.now(datetime.timezone.utc).strftime("%Y-%m-%dT%H:%M:%SZ"))
        with open(path, "w") as f:
            json.dump(d, f, indent=1)
            f.write("\n")


def load_model(name: str = "M1500") -> Mlsp2Model:
    """Coefficient sets produced by the reference trainer."""
    path = name if os.path.exists(name) else os.path.join(_PKG, "coefficients", f"{name}.json")
    return Mlsp2Model.from_json(path)


@dataclass
class SpectralBounds:
    eps_min: float
    eps_max: float


@dataclass
class DensityStatistics:
    trace: float
    trace_square: float


@dataclass
class Provenance:
    eps_min: float
    eps_max: float
    beta_prime: float
    mu_prime: float
    x_min: float
    x_max: float
    mode: int
    n_layers: int
    half_products: int
    diverged_layer: int
    half_range_layer: int
    status: int
    n: int
    device_ms: float

    @staticmethod
    def _from(p: _Prov) -> "Provenance":
        return Provenance(*[getattr(p, f) for f, _ in _Prov._fields_])


def _sym(H) -> np.ndarray:
    H = np.ascontiguousarray(np.asarray(H, dtype=np.float64))
    if H.ndim != 2 or H.shape[0] != H.shape[1]:
        raise DimensionError(f"expected a square matrix, got shape {H.shape}")
    return H


# ------------------------------------------------------------------ API
def in_region_of_validity(beta_prime: float, mu_prime: float, beta0: float, mu0: float) -> bool:
    """Eq. 41 with mu' in the model's un-flipped frame."""
    return bool(lib().ffg_in_region_of_validity(beta_prime, mu_prime, beta0, mu0))


def spectral_bounds(H) -> SpectralBounds:
    H = _sym(H)
    lo, hi = ctypes.c_double(), ctypes.c_double()
    _check(lib().ffg_spectral_bounds(_dp(H), H.shape[0], ctypes.byref(lo), ctypes.byref(hi)))
    return SpectralBounds(lo.value, hi.value)


def apply_model(H0, model: Mlsp2Model, mode: PrecisionMode = PrecisionMode.MIXED_EMULATED):
    """D = p(H0), H0 already in the model frame (spectrum in [0,1])."""
    H0 = _sym(H0)
    D = np.empty_like(H0)
    pv = _Prov()
    m = model._c()
    _check(lib().ffg_apply_model(_dp(H0), H0.shape[0], ctypes.byref(m), int(mode), _dp(D),
                                 ctypes.byref(pv)))
    return D


def mixed_square(X) -> np.ndarray:
    X = np.ascontiguousarray(np.asarray(X, dtype=np.float32))
    if X.ndim != 2 or X.shape[0] != X.shape[1]:
        raise DimensionError(f"expected a square matrix, got shape {X.shape}")
    Y = np.empty_like(X)
    _check(lib().ffg_mixed_square(X.ctypes.data_as(_F), X.shape[0], Y.ctypes.data_as(_F)))
    return Y


def density_statistics(D) -> DensityStatistics:
    D = _sym(D)
    out = np.zeros(2)
    _check(lib().ffg_density_statistics(_dp(D), D.shape[0], _dp(out)))
    return DensityStatistics(float(out[0]), float(out[1]))


def compute_density_matrix(H, mu: float, kT: float | None = None, model: Mlsp2Model | None = None,
                           mode: PrecisionMode = PrecisionMode.MIXED_EMULATED, *,
                           beta: float | None = None, want_D: bool = True):
    """North-star entry: (H, mu, kT, coefficients) -> (D, DensityStatistics, Provenance).

    Pass either kT or beta (SPEC.md:458 uses beta; the B200 boundary takes kT = 1/beta).
    """
    if model is None:
        model = load_model()
    if kT is None:
        if beta is None:
            raise ValidationError("pass kT or beta")
        kT = 1.0 / beta
    H = _sym(H)
    n = H.shape[0]
    D = np.empty_like(H) if want_D else None
    stats = np.zeros(2)
    pv = _Prov()
    m = model._c()
    rc = lib().ffg_density_matrix(_dp(H), n, float(mu), float(kT), ctypes.byref(m), int(mode),
                                  _dp(D) if want_D else None, _dp(stats), ctypes.byref(pv))
    if rc == DivergedEvaluationError.status:
        raise DivergedEvaluationError(lib().ffg_last_error().decode(), pv.diverged_layer)
    _check(rc)
    return D, DensityStatistics(float(stats[0]), float(stats[1])), Provenance._from(pv)


def compute_density_matrices(Hs: Sequence[np.ndarray], mu, kT, model: Mlsp2Model | None = None,
                             mode: PrecisionMode = PrecisionMode.MIXED_EMULATED,
                             want_D: bool = True):
    """Batched compute_density_matrix over independent H with per-matrix mu / kT."""
    if model is None:
        model = load_model()
    Hs = [_sym(H) for H in Hs]
    B = len(Hs)
    n = Hs[0].shape[0]
    if any(H.shape[0] != n for H in Hs):
        raise DimensionError("all matrices of a batch must share N")
    mu = np.ascontiguousarray(np.broadcast_to(np.asarray(mu, dtype=np.float64), (B,)))
    kT = np.ascontiguousarray(np.broadcast_to(np.asarray(kT, dtype=np.float64), (B,)))
    Ds = [np.empty_like(H) for H in Hs] if want_D else []
    Hp = (_D * B)(*[_dp(H) for H in Hs])
    Dp = (_D * B)(*[_dp(D) for D in Ds]) if want_D else None
    stats = np.zeros((B, 2))
    pv = (_Prov * B)()
    m = model._c()
    _check(lib().ffg_density_matrices(B, Hp, n, _dp(mu), _dp(kT), ctypes.byref(m), int(mode), Dp,
                                      _dp(stats), pv))
    return Ds, [DensityStatistics(*map(float, s)) for s in stats], [Provenance._from(p) for p in pv]


class AsyncBatch:
    """Handle of ffg_density_matrices_async: results land in the caller's D buffers; wait()
    returns (stats, provenance) and raises the batch's first error."""

    def __init__(self, ticket, B, keep):
        self.ticket, self.B, self._keep = ticket, B, keep

    def wait(self):
        stats = np.zeros((self.B, 2))
        pv = (_Prov * self.B)()
        _check(lib().ffg_wait(self.ticket, _dp(stats), pv))
        return [DensityStatistics(*map(float, st)) for st in stats], [Provenance._from(p) for p in pv]


def compute_density_matrices_async(Hs, mu, kT, model: Mlsp2Model, Ds,
                                   mode: PrecisionMode = PrecisionMode.MIXED_EMULATED) -> AsyncBatch:
    """Asynchronous host-buffer batch (at most three in flight): Hs / Ds are lists of C-contiguous
    float64 arrays (page-locked for transfer overlap) that must stay alive until wait()."""
    B = len(Hs)
    n = Hs[0].shape[0]
    mu = np.ascontiguousarray(np.broadcast_to(np.asarray(mu, dtype=np.float64), (B,)))
    kT = np.ascontiguousarray(np.broadcast_to(np.asarray(kT, dtype=np.float64), (B,)))
    Hp = (_D * B)(*[_dp(H) for H in Hs])
    Dp = (_D * B)(*[_dp(D) for D in Ds])
    m = model._c()
    t = ctypes.c_int64()
    _check(lib().ffg_density_matrices_async(B, Hp, n, _dp(mu), _dp(kT), ctypes.byref(m), int(mode), Dp,
                                            ctypes.byref(t)))
    return AsyncBatch(t.value, B, (Hs, Ds, mu, kT, Hp, Dp, m, model))


def compute_density_matrices_device(H_dev, mu, kT, model: Mlsp2Model,
                                    mode: PrecisionMode = PrecisionMode.MIXED_EMULATED,
                                    D_dev=None, stats_dev=None, status_dev=None, bounds_dev=None,
                                    stream=None):
    """Asynchronous device-resident batch.  H_dev: torch.float64 CUDA tensor [B, n, n].

    Returns (stats_dev [B,2] f64, status_dev [B] i32, bounds_dev [B,4] f64) torch tensors,
    valid once `stream` (a torch.cuda.Stream, default: current) reaches this point.
    """
    import torch

    if H_dev.dtype != torch.float64 or not H_dev.is_cuda or H_dev.dim() != 3 or H_dev.shape[1] != H_dev.shape[2]:
        raise ValidationError("H_dev must be a CUDA float64 tensor [B, n, n]")
    B, n, _ = H_dev.shape
    dev = H_dev.device
    st = stream if stream is not None else torch.cuda.current_stream(dev)

    def _out(t, shape, dtype, name):
        # caller-supplied outputs receive raw device writes: check them exactly
        if t is None:
            return torch.empty(shape, dtype=dtype, device=dev)
        if t.dtype != dtype or tuple(t.shape) != shape or t.device != dev or not t.is_contiguous():
            raise ValidationError(f"{name} must be a contiguous {dtype} tensor {list(shape)} on {dev} "
                                  f"(got {t.dtype} {list(t.shape)} on {t.device})")
        return t

    if D_dev is not None:
        _out(D_dev, (B, n, n), torch.float64, "D_dev")
    stats_dev = _out(stats_dev, (B, 2), torch.float64, "stats_dev")
    status_dev = _out(status_dev, (B,), torch.int32, "status_dev")
    bounds_dev = _out(bounds_dev, (B, 4), torch.float64, "bounds_dev")
    if not H_dev.is_contiguous():
        H_dev = H_dev.contiguous()
        H_dev.record_stream(st)  # the temporary must outlive the kernels queued on `st`
    mu = np.ascontiguousarray(np.broadcast_to(np.asarray(mu, dtype=np.float64), (B,)))
    kT = np.ascontiguousarray(np.broadcast_to(np.asarray(kT, dtype=np.float64), (B,)))
    m = model._c()
    _check(lib().ffg_density_matrices_dev(B, H_dev.data_ptr(), n, _dp(mu), _dp(kT), ctypes.byref(m),
                                          int(mode), D_dev.data_ptr() if D_dev is not None else None,
                                          stats_dev.data_ptr(), status_dev.data_ptr(),
                                          bounds_dev.data_ptr(), st.cuda_stream))
    return stats_dev, status_dev, bounds_dev


def kernel_launches(batch: int, n: int, model: Mlsp2Model, mode=PrecisionMode.MIXED_EMULATED) -> int:
    m = model._c()
    return int(lib().ffg_kernel_launches(batch, n, ctypes.byref(m), int(mode)))


def k2_kernel_name(n: int, mode: PrecisionMode = PrecisionMode.MIXED_EMULATED) -> str:
    """The recursion kernel that computes order-n matrices in `mode` (depends only on n and mode)."""
    k = int(lib().ffg_k2_kernel(int(n), int(mode)))
    if k < 0:
        raise ValidationError(f"no recursion kernel for n={n}, mode={mode}")
    return ("mlsp2_pair_kernel", "mlsp2_wide_kernel", "cublas_gemm+direct_layer")[k]


def profile_layers(enable: bool) -> None:
    """Bracket every layer-kernel launch with CUDA events (measurement only)."""
    _check(lib().ffg_profile_layers(1 if enable else 0))


def profile_read() -> tuple[float, int]:
    """(summed K2 device ms, K2 launches) since the last read (CUDA events on the stream)."""
    t, n, _ = profile_read_ex()
    return t, n


def profile_read_ex() -> tuple[float, int, float]:
    """(summed K2 device ms, K2 launches, algorithmic flops of those launches)."""
    t = ctypes.c_double()
    n = ctypes.c_int64()
    f = ctypes.c_double()
    _check(lib().ffg_profile_read_ex(ctypes.byref(t), ctypes.byref(n), ctypes.byref(f)))
    return t.value, n.value, f.value


def pair_table(nb: int) -> np.ndarray:
    """K2 work decomposition for an nb x nb grid of 128-blocks: rows (A0, A1, S, dummy);
    the CTA pair computes blocks (A0, S) and (A1, S) sharing B panel S."""
    cnt = lib().ffg_pair_table(nb, None, 0)
    if cnt < 0:
        raise DimensionError(f"bad block count {nb}")
    buf = np.zeros(cnt, dtype=np.uint32)
    lib().ffg_pair_table(nb, buf.ctypes.data, cnt)
    return np.stack([buf & 1023, (buf >> 10) & 1023, (buf >> 20) & 1023, (buf >> 30) & 1], axis=1)


def algorithmic_flops(n: int, layers: int, mode: PrecisionMode) -> float:
    """F = L * c * N^2 (N + 1): c = 3 FP32-emulated, 1 BF16/FP16."""
    c = 3 if mode == PrecisionMode.MIXED_EMULATED else 1
    return float(layers) * c * n * n * (n + 1)
