import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2605_08523_b200 import engine as E
from paper_2605_08523_b200.hamiltonians import tight_binding
print("dev", E.device_available(), flush=True)
Y = E.mixed_square(np.eye(256, dtype=np.float32)); print("I ok", np.array_equal(Y, np.eye(256)), flush=True)
m = E.load_model("M1500")
from oracle import oracle as O
for n in (128, 256, 512):
    H = tight_binding(n, seed=1234)
    D, st, pv = E.compute_density_matrix(H, 0.0, 0.01, m)
    R = O.density_matrix_f64(H, 0.0, 0.01, m.abcd, m.beta0, m.mu0)
    print(n, "max", np.abs(D - R).max(), "tr", abs(st.trace - np.trace(R)) / np.trace(R), flush=True)
