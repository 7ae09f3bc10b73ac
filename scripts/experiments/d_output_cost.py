import sys, os, numpy as np, torch
sys.path.insert(0, ".")
from paper_2605_08523_b200 import engine as E
from paper_2605_08523_b200.hamiltonians import tight_binding, batch_params
m = E.load_model("M1500")
mu, kT = batch_params(16)
H = torch.from_numpy(np.stack([tight_binding(1024, seed=10000 + k) for k in range(16)])).cuda()
D = torch.empty_like(H)
for withD in (True, False, True, False):
    for _ in range(2):
        E.compute_density_matrices_device(H, mu, kT, m, E.PrecisionMode.MIXED_EMULATED, D_dev=D if withD else None)
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10):
        E.compute_density_matrices_device(H, mu, kT, m, E.PrecisionMode.MIXED_EMULATED, D_dev=D if withD else None)
    b.record(); torch.cuda.synchronize()
    print("D output" if withD else "no D   ", "%.3f ms/step" % (a.elapsed_time(b) / 10))
