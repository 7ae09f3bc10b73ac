"""K2 average launch time for the current FFG_DEBUG_K2 / FFG_DRAIN_K16 settings."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2605_08523_b200 import engine as E
from paper_2605_08523_b200.hamiltonians import tight_binding, batch_params
m = E.load_model("M1500")
for n, B in [(1024, 16), (4096, 1), (512, 64)]:
    for mode in (E.PrecisionMode.MIXED_EMULATED, E.PrecisionMode.BF16):
        mu, kT = batch_params(B)
        H = torch.from_numpy(np.stack([tight_binding(n, seed=10000 + k) for k in range(B)])).cuda()
        D = torch.empty_like(H)
        E.compute_density_matrices_device(H, mu, kT, m, mode, D_dev=D); torch.cuda.synchronize()
        E.profile_layers(True); E.profile_read()
        for _ in range(3):
            E.compute_density_matrices_device(H, mu, kT, m, mode, D_dev=D)
        torch.cuda.synchronize()
        ms, k = E.profile_read(); E.profile_layers(False)
        F = B * E.algorithmic_flops(n, 1, mode)
        print(f"dbg={os.environ.get('FFG_DEBUG_K2','0')} dr={os.environ.get('FFG_DRAIN_K16','1')} n={n} B={B} {mode.name:15s} "
              f"K2 {ms/k*1e3:8.1f} us  {F/(ms/k/1e3)/1e12:7.1f} TF/s", flush=True)
