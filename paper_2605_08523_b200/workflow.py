"""Python mirror of the reference workflow module over the B200 C ABI.

    ModelLibrary / select_model(lib, beta', mu')
    compute_density_matrix(H, beta, mu, lib, mode)        SPEC.md:458-466 (library form)
    solve_chemical_potential(H, beta, n_occ, mu_guess, ...) SPEC.md:468-476 (Eqs. 42-45)
    thermodynamics(H, beta, mu, lib, mode)                SPEC.md:478-486 (Eq. 25)
    expectation(D, A)                                     SPEC.md:488-495 (Eq. 9)

Every density-matrix evaluation is the K1 -> K2 -> K3 pipeline of libfermiforge_b200.so; the
Newton derivative g'(mu) = beta (Tr D - Tr D^2) and the entropy trace (4 ln 2)(Tr Y - Tr Y^2)
come from the fused statistics, so none of these callers adds a matrix multiply.

Frame convention: validity uses the model's UN-flipped frame,
x = mu0 + (beta/beta0)(lambda - mu) in [0, 1]; with SPEC's normalized (beta', mu'_u =
(mu - eps_min)/W) this is Eq. 41.
"""
from __future__ import annotations

import ctypes
import json
import math
import os
from dataclasses import dataclass, field

import numpy as np

from . import engine as E

_PKG = os.path.dirname(os.path.abspath(__file__))


# ------------------------------------------------------------------ entropy models
@dataclass
class EntropyModel:
    """EntropyModelCoefficients (scalar_models.hpp:150-156): inner MLSP2 rows at
    x0 = alpha (x - mu0) + mu0 (no flip), s = (4 ln 2) y (1 - y)."""
    inner: E.Mlsp2Model
    alpha: float
    name: str = ""
    meta: dict = field(default_factory=dict)

    @property
    def beta0(self) -> float:
        return self.inner.beta0

    @property
    def mu0(self) -> float:
        return self.inner.mu0

    def _c(self) -> E._EntropyModel:
        return E._EntropyModel(self.inner._c(), float(self.alpha))

    @staticmethod
    def from_json(path: str) -> "EntropyModel":
        with open(path) as f:
            d = json.load(f)
        if d.get("schema_version") != E.MODEL_SCHEMA_VERSION:
            raise E.ValidationError(f"{path}: ModelFile schema_version {d.get('schema_version')!r} is not "
                                    f"supported (expected {E.MODEL_SCHEMA_VERSION})")
        abcd = np.array([[float(v) for v in row] for row in d["layers"]], dtype=np.float64)
        inner = E.Mlsp2Model(abcd, float(d["beta0"]), float(d["mu0"]), d.get("name", ""), d)
        return EntropyModel(inner, float(d["alpha"]), d.get("name", ""), d)


def load_entropy_model(name: str = "E1500") -> EntropyModel:
    path = name if os.path.exists(name) else os.path.join(_PKG, "coefficients", f"{name}.json")
    return EntropyModel.from_json(path)


# ------------------------------------------------------------------ model library
class NoValidModelError(E.OutOfRegionError):
    """select_model: no library model contains (beta', mu')."""


@dataclass
class ModelLibrary:
    """SPEC ModelLibrary: Fermi models with metadata, entropy models paired by
    exact (beta0, mu0)."""
    models: list = field(default_factory=list)          # Mlsp2Model
    entropy_models: list = field(default_factory=list)  # EntropyModel

    def add(self, m):
        (self.entropy_models if isinstance(m, EntropyModel) else self.models).append(m)
        return self

    @staticmethod
    def default() -> "ModelLibrary":
        lib = ModelLibrary()
        for name in ("M40", "M1500"):
            lib.add(E.load_model(name))
        for name in ("E40", "E1500"):
            if os.path.exists(os.path.join(_PKG, "coefficients", f"{name}.json")):
                lib.add(load_entropy_model(name))
        return lib

    def entropy_for(self, model: E.Mlsp2Model) -> EntropyModel:
        for e in self.entropy_models:
            if e.beta0 == model.beta0 and e.mu0 == model.mu0:
                return e
        raise E.ValidationError(f"no entropy model for (beta0={model.beta0:.17g}, mu0={model.mu0:.17g})")


def final_max_error(m: E.Mlsp2Model) -> float:
    rep = m.meta.get("report", {}) if isinstance(m.meta, dict) else {}
    return float(rep.get("final_max_error", math.inf))


def select_model(lib: ModelLibrary, beta_prime: float, mu_prime: float) -> E.Mlsp2Model:
    """SPEC select_model: among models whose region of validity (Eq. 41)
    contains (beta', mu') -- mu' in the un-flipped normalized frame (mu - eps_min)/W -- the one
    with the fewest layers; ties by smaller final_max_error, then insertion order."""
    if not lib.models:
        raise E.ValidationError("select_model: empty library")
    valid = [(m.layer_count, final_max_error(m), i, m) for i, m in enumerate(lib.models)
             if E.in_region_of_validity(beta_prime, mu_prime, m.beta0, m.mu0)]
    if not valid:
        # Eq. 41 solved for beta0 at each library mu0; report the least demanding
        need = min(max(beta_prime * mu_prime / m.mu0, beta_prime * (1.0 - mu_prime) / (1.0 - m.mu0))
                   for m in lib.models)
        raise NoValidModelError(f"select_model: no model contains beta'={beta_prime:.6g}, mu'={mu_prime:.6g}; "
                                f"a model with beta0 >= {need:.6g} is needed")
    return min(valid, key=lambda t: t[:3])[3]


def normalized_problem(H, mu: float, beta: float):
    """(beta', mu'_u, bounds) with mu'_u = (mu - eps_min)/W in the un-flipped frame."""
    b = E.spectral_bounds(H)
    W = b.eps_max - b.eps_min
    return beta * W, (mu - b.eps_min) / W, b


def compute_density_matrix(H, beta: float, mu: float, lib: ModelLibrary | None = None,
                           mode: E.PrecisionMode = E.PrecisionMode.MIXED_EMULATED):
    """SPEC compute_density_matrix with a model library: spectral_bounds -> select_model ->
    the device pipeline.  Returns (D, DensityStatistics, Provenance, model)."""
    lib = lib or ModelLibrary.default()
    bp, mp, _ = normalized_problem(H, mu, beta)
    model = select_model(lib, bp, mp)
    D, st, pv = E.compute_density_matrix(H, mu, 1.0 / beta, model, mode)
    return D, st, pv, model


# ------------------------------------------------------------------ chemical potential
@dataclass
class MuSolveReport:
    """SPEC MuSolveReport."""
    mu_final: float
    iterations: int
    residual_history: list
    converged: bool
    bisections: int
    model: E.Mlsp2Model | None = None


def solve_chemical_potential(H, beta: float, n_occ: float, mu_guess: float,
                             model: E.Mlsp2Model | ModelLibrary | None = None, tol: float = 1e-6,
                             max_iter: int = 30, mode: E.PrecisionMode = E.PrecisionMode.MIXED_EMULATED):
    """SPEC solve_chemical_potential: Newton on Tr D(mu) - n_occ with
    g'(mu) = beta (Tr D - Tr D^2) (Eq. 44), clamped steps, bisection fallback -- native loop
    in ffg_solve_chemical_potential.  A library selects the model at mu_guess."""
    H = E._sym(H)
    n = H.shape[0]
    if model is None or isinstance(model, ModelLibrary):
        lib = model or ModelLibrary.default()
        bp, mp, _ = normalized_problem(H, mu_guess, beta)
        model = select_model(lib, bp, mp)
    D = np.empty_like(H)
    stats = np.zeros(2)
    hist = np.zeros(2 * max_iter)
    rep = E._MuReport()
    m = model._c()
    rc = E.lib().ffg_solve_chemical_potential(E._dp(H), n, 1.0 / beta, float(n_occ), float(mu_guess),
                                              ctypes.byref(m), int(mode), float(tol), int(max_iter),
                                              E._dp(D), E._dp(stats), E._dp(hist), ctypes.byref(rep))
    E._check(rc)
    it = int(rep.iterations)
    report = MuSolveReport(float(rep.mu), it, [(float(hist[2 * k]), float(hist[2 * k + 1])) for k in range(it)],
                           bool(rep.converged), int(rep.bisections), model)
    return D, E.DensityStatistics(float(stats[0]), float(stats[1])), report


# ------------------------------------------------------------------ thermodynamics
@dataclass
class ThermodynamicResult:
    """SPEC ThermodynamicResult."""
    density: np.ndarray
    entropy_trace: float
    band_energy: float
    free_energy: float


def expectation(D, A) -> float:
    """SPEC expectation: Tr(D A) = sum_ij D_ij A_ij (device reduction)."""
    D = E._sym(D)
    A = E._sym(A)
    if D.shape != A.shape:
        raise E.DimensionError("expectation: dimension mismatch")
    out = np.zeros(1)
    E._check(E.lib().ffg_expectation(E._dp(D), E._dp(A), D.shape[0], E._dp(out)))
    return float(out[0])


def entropy_trace(H, mu: float, kT: float, em: EntropyModel,
                  mode: E.PrecisionMode = E.PrecisionMode.MIXED_EMULATED) -> float:
    H = E._sym(H)
    out = np.zeros(1)
    pv = E._Prov()
    c = em._c()
    E._check(E.lib().ffg_entropy_trace(E._dp(H), H.shape[0], float(mu), float(kT), ctypes.byref(c), int(mode),
                                       E._dp(out), ctypes.byref(pv)))
    return float(out[0])


def thermodynamics(H, beta: float, mu: float, lib: ModelLibrary | None = None,
                   mode: E.PrecisionMode = E.PrecisionMode.MIXED_EMULATED) -> ThermodynamicResult:
    """SPEC thermodynamics: D from the selected Fermi model, Tr S from the
    paired entropy model, band energy Tr[D(H - mu I)], free energy = band - Tr S / beta."""
    lib = lib or ModelLibrary.default()
    H = E._sym(H)
    D, st, pv, model = compute_density_matrix(H, beta, mu, lib, mode)
    em = lib.entropy_for(model)
    ts = entropy_trace(H, mu, 1.0 / beta, em, mode)
    band = expectation(D, H) - mu * st.trace
    return ThermodynamicResult(D, ts, band, band - ts / beta)
