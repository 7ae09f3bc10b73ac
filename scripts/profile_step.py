"""A few steps of the bench workload, for ncu (launch list / full capture)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2605_08523_b200 import engine as E
from paper_2605_08523_b200.hamiltonians import tight_binding, batch_params
n = int(os.environ.get("N", 1024)); B = int(os.environ.get("B", 16)); steps = int(os.environ.get("STEPS", 2))
mode = E.PrecisionMode[os.environ.get("MODE", "MIXED_EMULATED")]
m = E.load_model("M1500")
mu, kT = batch_params(B)
H = torch.from_numpy(np.stack([tight_binding(n, seed=10000 + k) for k in range(B)])).cuda()
D = torch.empty_like(H)
for _ in range(steps):
    E.compute_density_matrices_device(H, mu, kT, m, mode, D_dev=D)
torch.cuda.synchronize()
print("done")
