"""K2 device time per layer (CUDA events) and algorithmic TF/s for the current FFG_* settings."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2605_08523_b200 import engine as E
from paper_2605_08523_b200.hamiltonians import tight_binding, batch_params
m = E.load_model("M1500")
cases = [(1024, 16), (4096, 1), (512, 64), (8192, 1), (1024, 64), (512, 512)]
if len(sys.argv) > 1:
    cases = [tuple(int(x) for x in c.split("x")) for c in sys.argv[1:]]
tag = " ".join(f"{k}={v}" for k, v in os.environ.items() if k.startswith("FFG_"))
for n, B in cases:
    for mode in (E.PrecisionMode.MIXED_EMULATED, E.PrecisionMode.BF16):
        mu, kT = batch_params(B)
        H = torch.from_numpy(np.stack([tight_binding(n, seed=10000 + k) for k in range(B)])).cuda()
        D = torch.empty_like(H)
        E.compute_density_matrices_device(H, mu, kT, m, mode, D_dev=D); torch.cuda.synchronize()
        E.profile_layers(True); E.profile_read_ex()
        for _ in range(3):
            E.compute_density_matrices_device(H, mu, kT, m, mode, D_dev=D)
        torch.cuda.synchronize()
        ms, k, F = E.profile_read_ex(); E.profile_layers(False)
        per_layer_us = ms / 3 / m.layer_count * 1e3
        print(f"[{tag}] n={n} B={B} {mode.name:15s} K2 {per_layer_us:8.1f} us/layer  "
              f"{F / (ms / 1e3) / 1e12:7.1f} TF/s", flush=True)
        del H, D
        torch.cuda.empty_cache()
