"""TEST INFRASTRUCTURE -- regenerates tests/golden/* from the compiled reference.

Run here (where /root/reference exists):  python oracle/gen_fixtures.py [--skip-train]

* coefficients_{M1500,M40}.json : train_fermi (trainer.cpp:1215) through
  oracle/_ref with the configs of SURVEY.md Appendix A (seed 42, Derivative
  weighting).  The trainer is deterministic; the script checks the result is
  bit-identical to the committed file when one exists.
* scalar_{M1500,M40}.json : evaluate_model (scalar_models.cpp:330) of the
  compiled reference on a fixed x grid, %.17g.
* sp2_mlsp2.json : sp2_sign_sequence + embed(SP2->MLSP2) coefficient tables.
* matrix_*.npz : small H, the spectral-mapping D from the reference
  evaluate_model, the fp64 recursion D, and the reference pairwise stats.
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
from oracle import oracle as O  # noqa: E402
from paper_2605_08523_b200.hamiltonians import tight_binding, goe  # noqa: E402

# entropy models (train_entropy, trainer.cpp:1274) on the Fermi fixtures above
ENTROPY = {"E40": dict(base="M40", samples=6000, max_iter=1000, seed=42),
           "E1500": dict(base="M1500", samples=20000, max_iter=400, seed=42)}

CONFIGS = {
    "M1500": dict(beta0=1500.0, mu0=1.0 / 3.0, layers=30, samples=20000, max_iter=400, seed=42),
    "M40": dict(beta0=40.0, mu0=0.3, layers=14, samples=6000, max_iter=1000, seed=42),
}


def g17(v: float) -> str:
    return "%.17g" % float(v)


def now_utc() -> str:
    import datetime
    return datetime.datetime.now(datetime.timezone.utc).strftime("%Y-%m-%dT%H:%M:%SZ")


def train(name: str) -> dict:
    c = CONFIGS[name]
    R = O.ref()
    abcd = np.zeros((c["layers"], 4))
    rep = np.zeros(5)
    L = R.ffr_train_fermi_mlsp2(c["beta0"], c["mu0"], c["layers"], c["samples"], c["max_iter"],
                                c["seed"], O._dp(abcd), O._dp(rep))
    if L < 0:
        raise RuntimeError(R.ffr_last_error().decode())
    return {
        "schema_version": 1, "created": now_utc(),
        "name": name, "architecture": "mlsp2", "beta0": g17(c["beta0"]), "mu0": g17(c["mu0"]),
        "training": {k: c[k] for k in ("layers", "samples", "max_iter", "seed")} | {"weighting": "derivative"},
        "report": {"final_max_error": rep[0], "final_rms_error": rep[1], "iterations": int(rep[2]),
                   "converged": bool(rep[3]), "initial_max_error": rep[4]},
        "provenance": "train_fermi (proj/core/src/trainer.cpp:1215) compiled from /root/reference via oracle/Makefile",
        "layers": [[g17(v) for v in row] for row in abcd],
    }


def train_entropy(name: str) -> dict:
    c = ENTROPY[name]
    R = O.ref()
    m = O.load_coefficients(c["base"])
    L = m["abcd"].shape[0]
    abcd = np.zeros((L, 4))
    alpha = ctypes.c_double()
    rep = np.zeros(5)
    rc = R.ffr_train_entropy_mlsp2(O._dp(np.ascontiguousarray(m["abcd"])), L, float(m["beta0"]),
                                   float(m["mu0"]), c["samples"], c["max_iter"], c["seed"], O._dp(abcd),
                                   ctypes.byref(alpha), O._dp(rep))
    if rc < 0:
        raise RuntimeError(R.ffr_last_error().decode())
    return {
        "schema_version": 1, "created": now_utc(),
        "name": name, "architecture": "entropy", "base": c["base"], "beta0": g17(m["beta0"]),
        "mu0": g17(m["mu0"]), "alpha": g17(alpha.value),
        "training": {k: c[k] for k in ("samples", "max_iter", "seed")} | {"weighting": "derivative"},
        "report": {"final_max_error": rep[0], "final_rms_error": rep[1], "iterations": int(rep[2]),
                   "converged": bool(rep[3]), "initial_max_error": rep[4]},
        "provenance": "train_entropy (proj/core/src/trainer.cpp:1274) compiled from /root/reference via oracle/Makefile",
        "layers": [[g17(v) for v in row] for row in abcd],
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--skip-train", action="store_true")
    ap.add_argument("--only-fermi", action="store_true", help="skip the entropy models")
    args = ap.parse_args()
    R = O.ref()
    assert R is not None, "build oracle/_ref first (make -C oracle)"
    os.makedirs(O.GOLDEN, exist_ok=True)
    for name in CONFIGS:
        path = os.path.join(O.GOLDEN, f"coefficients_{name}.json")
        if args.skip_train and os.path.exists(path):
            continue
        d = train(name)
        if os.path.exists(path):
            with open(path) as f:
                old = json.load(f)
            assert old["layers"] == d["layers"], f"{name}: trainer no longer bit-identical"
            d["created"] = old.get("created", d["created"])
        with open(path, "w") as f:
            json.dump(d, f, indent=1)
        print(name, d["report"])

    # scalar golden tables: x in [-0.05, 1.05] (out-of-[0,1] points are evaluated as-is)
    xs = np.concatenate([np.linspace(0.0, 1.0, 1001), np.linspace(-0.05, 1.05, 23),
                         np.array([1.0 / 3.0, 0.3, 0.5, 1e-9, 1 - 1e-9])])
    for name in CONFIGS:
        m = O.load_coefficients(name)
        ys = O.evaluate_model_ref(m["abcd"], float(m["beta0"]), float(m["mu0"]), xs)
        with open(os.path.join(O.GOLDEN, f"scalar_{name}.json"), "w") as f:
            json.dump({"x": [g17(v) for v in xs], "evaluate_model": [g17(v) for v in ys],
                       "provenance": "reference evaluate_model (scalar_models.cpp:330) via oracle/_ref"}, f)

    # entropy models + scalar golden tables (reference evaluate_model, Architecture::Entropy,
    # and the exact fermi_entropy) on the same x grid
    for name in ENTROPY if not args.only_fermi else ():
        path = os.path.join(O.GOLDEN, f"coefficients_{name}.json")
        if not (args.skip_train and os.path.exists(path)):
            d = train_entropy(name)
            if os.path.exists(path):
                with open(path) as f:
                    old = json.load(f)
                assert old["layers"] == d["layers"] and old["alpha"] == d["alpha"], \
                    f"{name}: trainer no longer bit-identical"
                d["created"] = old.get("created", d["created"])
            with open(path, "w") as f:
                json.dump(d, f, indent=1)
            print(name, d["report"])
        e = O.load_entropy_coefficients(name)
        ys, ex = O.evaluate_entropy_ref(e["abcd"], e["alpha"], float(e["beta0"]), float(e["mu0"]), xs)
        with open(os.path.join(O.GOLDEN, f"scalar_{name}.json"), "w") as f:
            json.dump({"x": [g17(v) for v in xs], "evaluate_model": [g17(v) for v in ys],
                       "fermi_entropy": [g17(v) for v in ex],
                       "provenance": "reference evaluate_model (Entropy, scalar_models.cpp:320-347) and "
                                     "fermi_entropy via oracle/_ref"}, f)

    # SP2 sign sequences embedded into MLSP2 (scalar_models.cpp:63-88, :554-607)
    sp2 = {}
    for mu_p, n in ((0.35, 18), (0.5, 12), (2.0 / 3.0, 20)):
        abcd = np.zeros((n, 4))
        L = R.ffr_sp2_as_mlsp2(mu_p, n, O._dp(abcd))
        sp2[g17(mu_p)] = [[g17(v) for v in row] for row in abcd[:L]]
    with open(os.path.join(O.GOLDEN, "sp2_mlsp2.json"), "w") as f:
        json.dump(sp2, f, indent=1)

    # small matrix fixtures
    cases = [("tb16", tight_binding(16, seed=7), 0.0, 0.01, "M1500"),
             ("tb64", tight_binding(64, seed=1234), 0.0, 0.01, "M1500"),
             ("tb64_m40", tight_binding(64, seed=99), 0.0, 0.5, "M40"),
             ("goe64", goe(64, seed=3), 0.1, 0.05, "M1500")]
    for tag, H, mu, kT, name in cases:
        m = O.load_coefficients(name)
        b0, m0 = float(m["beta0"]), float(m["mu0"])
        lo, hi = O.gershgorin(H)
        assert O.region_ok(lo, hi, mu, kT, b0, m0) == 1, tag
        Dspec = O.spectral_oracle(H, mu, kT, m["abcd"], b0, m0)
        Drec = O.density_matrix_f64(H, mu, kT, m["abcd"], b0, m0)
        st = np.zeros(2)
        R.ffr_density_statistics(O._dp(np.ascontiguousarray(Drec)), H.shape[0], O._dp(st))
        np.savez_compressed(os.path.join(O.GOLDEN, f"matrix_{tag}.npz"), H=H, mu=mu, kT=kT,
                            model=name, D_spectral=Dspec, D_recursion=Drec, stats_ref=st,
                            bounds=np.array([lo, hi]))
        print(tag, "max|Drec-Dspec| =", np.abs(Drec - Dspec).max())


if __name__ == "__main__":
    main()
