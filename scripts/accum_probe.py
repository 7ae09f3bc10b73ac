"""Probe tcgen05 FP32 accumulation behaviour through ffg_mixed_square."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2605_08523_b200 import engine as E
from paper_2605_08523_b200.hamiltonians import tight_binding
from oracle import oracle as O
S = 16384.0
m = O.load_coefficients("M1500")

def parts(X):
    xs = X.astype(np.float32) * np.float32(S)
    hi = xs.astype(np.float16).astype(np.float64)
    lo = (xs - hi.astype(np.float32)).astype(np.float16).astype(np.float64)
    return hi, lo

def x_at_layer(H, L, mu=0.0, kT=0.01):
    X = O.rescale(H, mu, kT, 1500.0, 1 / 3)
    for a, b, c, d in m["abcd"][:L]:
        X = a * (X @ X) + b * X + c * np.eye(X.shape[0])
    return X.astype(np.float32)

cases = {}
for n in (16, 64, 256, 1024):
    H = tight_binding(n, seed=1234)
    for L in (0, 5, 15, 25):
        cases[(n, L)] = x_at_layer(H, L)
rng = np.random.default_rng(0)
cases[("rand", 0)] = np.triu(rng.uniform(-1, 1, (128, 128))).astype(np.float32); cases[("rand", 0)] += np.triu(cases[("rand", 0)], 1).T
# one large + many small
X = np.zeros((128, 128), np.float32); X[0, 0] = 1.0; X[0, 1:] = X[1:, 0] = 2.0 ** -9; cases[("spike", 0)] = X
for key, X in cases.items():
    hi, lo = parts(X)
    Yx = (hi @ hi + hi @ lo + lo @ hi) / S / S          # exact value of the kernel's products
    Yg = E.mixed_square(X).astype(np.float64)
    ulp = np.spacing(np.abs(Yx).astype(np.float32)).astype(np.float64)
    err = (Yg - Yx) / np.maximum(ulp, 1e-45)
    sgn = np.sign(Yx)
    print(f"{str(key):12s} err/ulp: mean {np.mean(err):+7.3f}  mean*sign {np.mean(err*sgn):+7.3f}  "
          f"rms {np.sqrt(np.mean(err**2)):7.3f}  max {np.abs(err).max():8.2f}", flush=True)
