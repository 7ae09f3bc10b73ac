"""Command-line surface over the B200 path (SPEC.md:598-696 cli, the matrix-path commands):

    python -m paper_2605_08523_b200 apply    --model M1500 --hamiltonian H.mtx --kT 0.01 --mu 0 --out D.mtx
    python -m paper_2605_08523_b200 solve-mu --model M1500 --hamiltonian H.mtx --kT 0.01 --nocc 100 --mu 0
    python -m paper_2605_08523_b200 thermo   --hamiltonian H.mtx --beta 100 --mu 0
    python -m paper_2605_08523_b200 bench    --sizes 256,1024 --precision mixed,bf16
    python -m paper_2605_08523_b200 info     --model M40

Exit codes follow the SPEC: 0 ok, 3 out of region of validity (the violated Eq. 41
inequality is printed), 64 usage, 74 I/O.  `--model` takes a name of the packaged
reference-trained sets (M40, M1500) or a model JSON path; omitted, the library selects.
train / validate / convert stay with the reference (trainer and scalar tooling are out of
scope for the B200 path).
"""
from __future__ import annotations

import argparse
import json
import sys
import time

import numpy as np

from . import engine as E
from . import workflow as W
from .mm import IoError, read_matrix_market, write_matrix_market

PRECISION = {"mixed": E.PrecisionMode.MIXED_EMULATED, "bf16": E.PrecisionMode.BF16,
             "fp16": E.PrecisionMode.FP16, "double": E.PrecisionMode.DOUBLE, "single": E.PrecisionMode.SINGLE}
EX_USAGE, EX_IOERR, EX_REGION = 64, 74, 3


def _beta(a) -> float:
    if a.beta is not None:
        return float(a.beta)
    if a.kT is not None:
        return 1.0 / float(a.kT)
    raise SystemExit(EX_USAGE)


def _model(name):
    try:
        return E.load_model(name)
    except OSError as e:
        raise IoError(f"cannot open model: {name}") from e


def cmd_apply(a) -> int:
    H = read_matrix_market(a.hamiltonian)
    beta = _beta(a)
    mode = PRECISION[a.precision]
    if a.model:
        model = _model(a.model)
        D, st, pv = E.compute_density_matrix(H, a.mu, 1.0 / beta, model, mode)
    else:
        D, st, pv, model = W.compute_density_matrix(H, beta, a.mu, W.ModelLibrary.default(), mode)
    if a.out:
        write_matrix_market(D, a.out)
    prov = {"n": pv.n, "beta_prime": pv.beta_prime, "mu_prime": pv.mu_prime, "eps_min": pv.eps_min,
            "eps_max": pv.eps_max, "model": {"name": model.name, "beta0": model.beta0, "mu0": model.mu0,
                                             "layers": model.layer_count},
            "precision": a.precision, "half_products": pv.half_products, "trace": st.trace,
            "trace_square": st.trace_square, "device_ms": pv.device_ms}
    print(json.dumps(prov))
    return 0


def cmd_solve_mu(a) -> int:
    H = read_matrix_market(a.hamiltonian)
    n = H.shape[0]
    if not (0.0 < a.nocc < n):
        print(f"--nocc must lie in (0, {n})", file=sys.stderr)
        return EX_USAGE
    beta = _beta(a)
    model = _model(a.model) if a.model else None
    D, st, rep = W.solve_chemical_potential(H, beta, a.nocc, a.mu, model, tol=a.tol, max_iter=a.max_iter,
                                            mode=PRECISION[a.precision])
    print(f"{'iter':>4} {'mu':>22} {'Tr D - n_occ':>14} {'dmu':>12}")
    prev = None
    for k, (mu, g) in enumerate(rep.residual_history):
        print(f"{k:4d} {mu:22.15f} {g:14.6e} {'' if prev is None else '%12.4e' % (mu - prev):>12}")
        prev = mu
    print(json.dumps({"mu": rep.mu_final, "iterations": rep.iterations, "converged": rep.converged,
                      "bisections": rep.bisections, "model": rep.model.name, "trace": st.trace}))
    if a.out:
        write_matrix_market(D, a.out)
    return 0


def cmd_thermo(a) -> int:
    H = read_matrix_market(a.hamiltonian)
    r = W.thermodynamics(H, _beta(a), a.mu, W.ModelLibrary.default(), PRECISION[a.precision])
    print(json.dumps({"entropy_trace": r.entropy_trace, "band_energy": r.band_energy,
                      "free_energy": r.free_energy, "trace": float(np.trace(r.density))}))
    if a.out:
        write_matrix_market(r.density, a.out)
    return 0


def cmd_bench(a) -> int:
    """SPEC cmd_bench analogue on the B200: per N and precision, device time (K1..K3, CUDA
    events), wall time of the host call, tensor-core half-products per matrix, and the error
    against a LAPACK eigendecomposition Fermi matrix."""
    from .hamiltonians import tight_binding
    model = _model(a.model)
    print(f"{'N':>6} {'precision':>10} {'device ms':>10} {'wall ms':>9} {'half-products':>14} {'max|D-D_eigh|':>14}")
    for n in (int(x) for x in a.sizes.split(",")):
        H = tight_binding(n, seed=1234)
        lam, V = np.linalg.eigh(H)
        Dx = (V / (1.0 + np.exp(np.clip(lam / a.kT, -700, 700)))) @ V.T
        for p in a.precision.split(","):
            D, st, pv = E.compute_density_matrix(H, 0.0, a.kT, model, PRECISION[p])
            dev, wall = [], []
            for _ in range(a.reps):
                t0 = time.perf_counter()
                _, _, q = E.compute_density_matrix(H, 0.0, a.kT, model, PRECISION[p], want_D=False)
                wall.append((time.perf_counter() - t0) * 1e3)
                dev.append(q.device_ms)
            print(f"{n:6d} {p:>10} {min(dev):10.3f} {min(wall):9.3f} {pv.half_products:14d} "
                  f"{np.abs(D - Dx).max():14.3e}")
    return 0


def cmd_info(a) -> int:
    m = _model(a.model)
    rep = m.meta.get("report", {}) if isinstance(m.meta, dict) else {}
    print(json.dumps({"name": m.name, "architecture": "mlsp2", "beta0": m.beta0, "mu0": m.mu0,
                      "layers": m.layer_count, "final_max_error": rep.get("final_max_error"),
                      "provenance": m.meta.get("provenance") if isinstance(m.meta, dict) else None}))
    return 0


def parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="python -m paper_2605_08523_b200")
    sub = ap.add_subparsers(dest="cmd", required=True)

    def common(p, ham=True):
        if ham:
            p.add_argument("--hamiltonian", required=True)
        p.add_argument("--model")
        p.add_argument("--beta", type=float)
        p.add_argument("--kT", type=float)
        p.add_argument("--mu", type=float, default=0.0)
        p.add_argument("--precision", default="mixed", choices=sorted(PRECISION))
        p.add_argument("--out")

    p = sub.add_parser("apply")
    common(p)
    p.set_defaults(fn=cmd_apply)
    p = sub.add_parser("solve-mu")
    common(p)
    p.add_argument("--nocc", type=float, required=True)
    p.add_argument("--tol", type=float, default=1e-6)
    p.add_argument("--max-iter", type=int, default=30)
    p.set_defaults(fn=cmd_solve_mu)
    p = sub.add_parser("thermo")
    common(p)
    p.set_defaults(fn=cmd_thermo)
    p = sub.add_parser("bench")
    p.add_argument("--sizes", default="256,1024")
    p.add_argument("--model", default="M1500")
    p.add_argument("--kT", type=float, default=0.01)
    p.add_argument("--precision", default="mixed,bf16")
    p.add_argument("--reps", type=int, default=5)
    p.set_defaults(fn=cmd_bench)
    p = sub.add_parser("info")
    p.add_argument("--model", required=True)
    p.set_defaults(fn=cmd_info)
    return ap


def main(argv=None) -> int:
    try:
        a = parser().parse_args(argv)
    except SystemExit as e:
        return EX_USAGE if e.code not in (0, None) else 0
    try:
        return a.fn(a)
    except IoError as e:
        print(str(e), file=sys.stderr)
        return EX_IOERR
    except E.OutOfRegionError as e:
        print(str(e), file=sys.stderr)
        return EX_REGION
    except (E.ValidationError, E.DimensionError) as e:
        print(str(e), file=sys.stderr)
        return EX_USAGE


if __name__ == "__main__":
    sys.exit(main())
