"""Small-size GPU smoke of every mode against the CPU oracle (development aid)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2605_08523_b200 import engine as E
from paper_2605_08523_b200.hamiltonians import tight_binding, batch_params
from oracle import oracle as O
print("dev", E.device_available(), flush=True)
Y = E.mixed_square(np.eye(256, dtype=np.float32)); print("I ok", np.array_equal(Y, np.eye(256)), flush=True)
m = E.load_model("M1500")
for n in (100, 128, 256, 384, 512, 1024):
    H = tight_binding(n, seed=1234) if n not in (100, 384) else tight_binding(n, seed=1234)
    R = O.density_matrix_f64(H, 0.0, 0.01, m.abcd, m.beta0, m.mu0)
    for mode in (E.PrecisionMode.MIXED_EMULATED, E.PrecisionMode.BF16):
        D, st, pv = E.compute_density_matrix(H, 0.0, 0.01, m, mode)
        print(n, mode.name, "max %.2e" % np.abs(D - R).max(),
              "tr %.2e" % (abs(st.trace - np.trace(R)) / np.trace(R)), "sym", np.array_equal(D, D.T), flush=True)
mu, kT = batch_params(6)
Hs = [tight_binding(512, seed=10000 + k) for k in range(6)]
Ds, sts, pvs = E.compute_density_matrices(Hs, mu, kT, m)
for k in range(6):
    R = O.density_matrix_f64(Hs[k], mu[k], kT[k], m.abcd, m.beta0, m.mu0)
    print("batch", k, "max %.2e" % np.abs(Ds[k] - R).max(), "tr %.2e" % (abs(sts[k].trace - np.trace(R)) / np.trace(R)), flush=True)
