"""Accuracy of the GPU modes vs the fp64 recursion oracle on the parity cases."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle import oracle as O
from paper_2605_08523_b200 import engine as E
from paper_2605_08523_b200.hamiltonians import tight_binding, batch_params

def err(D, R):
    d = D - R
    return np.abs(d).max(), np.linalg.norm(d) / np.linalg.norm(R), abs(np.trace(D) - np.trace(R)) / abs(np.trace(R))

modes = [E.PrecisionMode[m] for m in (sys.argv[1:] or ["MIXED_EMULATED"])]
cases = []
for tag in ("tb16", "tb64", "tb64_m40"):
    f = np.load(f"{O.GOLDEN}/matrix_{tag}.npz")
    cases.append((tag, f["H"], float(f["mu"]), float(f["kT"]), str(f["model"]), f["D_recursion"]))
mu, kT = batch_params(512)
for n, seed, m_, k_ in [(256, 1234, 0.0, 0.01), (1024, 1234, 0.0, 0.01)] + [(512, 10000 + k, mu[k], kT[k]) for k in (0, 5, 11, 23, 100, 200, 300, 400)]:
    cases.append((f"tb{n}_s{seed}", tight_binding(n, seed=seed), m_, k_, "M1500", None))
worst = {}
worst_big = {}
for tag, H, mu_, kT_, mname, Dref in cases:
    model = E.load_model(mname)
    if Dref is None:
        Dref = O.density_matrix_f64(H, mu_, kT_, model.abcd, model.beta0, model.mu0)
    for mode in modes:
        D, st, pv = E.compute_density_matrix(H, mu_, kT_, model, mode)
        e = err(D, Dref)
        for dct in ([worst, worst_big] if H.shape[0] >= 256 else [worst]):
            w = dct.setdefault(mode.name, [0, 0, 0])
            for i in range(3):
                w[i] = max(w[i], e[i])
        print(f"{tag:16s} {mode.name:15s} max {e[0]:.2e} fro {e[1]:.2e} tr {e[2]:.2e}", flush=True)
tag = " ".join(f"{k}={v}" for k, v in os.environ.items() if k.startswith("FFG_"))
for k, w in worst.items():
    print(f"WORST     {k:15s} max {w[0]:.2e} fro {w[1]:.2e} tr {w[2]:.2e}  [{tag}]")
for k, w in worst_big.items():
    print(f"WORST_BIG {k:15s} max {w[0]:.2e} fro {w[1]:.2e} tr {w[2]:.2e}  [{tag}]")
