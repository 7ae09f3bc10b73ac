"""K2 device time at a given config for the library FFG_LIB_PATH points to (measurement script).

    FFG_LIB_PATH=... python scripts/k2_time.py [n] [batch] [mode] [reps]  -> one JSON line
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_08523_b200 import engine as E  # noqa: E402
from paper_2605_08523_b200.hamiltonians import tight_binding, batch_params  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
B = int(sys.argv[2]) if len(sys.argv) > 2 else 16
mode = E.PrecisionMode[sys.argv[3]] if len(sys.argv) > 3 else E.PrecisionMode.MIXED_EMULATED
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 10
m = E.load_model("M1500")
mu, kT = batch_params(B)
H = torch.from_numpy(np.stack([tight_binding(n, seed=10000 + k) for k in range(B)])).cuda()
D = torch.empty_like(H)
for _ in range(3):
    E.compute_density_matrices_device(H, mu, kT, m, mode, D_dev=D)
torch.cuda.synchronize()
E.profile_layers(True)
E.profile_read_ex()
t = []
for _ in range(reps):
    E.compute_density_matrices_device(H, mu, kT, m, mode, D_dev=D)
    torch.cuda.synchronize()
    ms, k, f = E.profile_read_ex()
    t.append(ms)
E.profile_layers(False)
flops = f
print(json.dumps({"lib": os.environ.get("FFG_LIB_PATH", "default"), "n": n, "B": B, "mode": mode.name,
                  "k2_ms_median": float(np.median(t)), "k2_ms_min": float(min(t)),
                  "tflops_median": flops / (np.median(t) / 1e3) / 1e12}))
