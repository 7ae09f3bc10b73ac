"""Quick device-time survey of the pipeline (dev variant, inputs resident)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2605_08523_b200 import engine as E
from paper_2605_08523_b200.hamiltonians import tight_binding, batch_params

m = E.load_model("M1500")
peak = 1630.1e12

def run(n, B, mode, reps=5):
    mu, kT = batch_params(B)
    H = torch.from_numpy(np.stack([tight_binding(n, seed=10000 + k) for k in range(B)])).cuda()
    D = torch.empty_like(H)
    for _ in range(2):
        E.compute_density_matrices_device(H, mu, kT, m, mode, D_dev=D)
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); st, status, _ = E.compute_density_matrices_device(H, mu, kT, m, mode, D_dev=D); b.record()
        torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    t = min(ts) / 1e3
    F = B * E.algorithmic_flops(n, m.layer_count, mode)
    print(f"n={n:5d} B={B:4d} mode={mode.name:15s} t={t*1e3:8.3f} ms  mats/s={B/t:9.1f}  "
          f"TF/s={F/t/1e12:7.1f}  frac={F/t/peak:.3f}  status={set(status.cpu().tolist())}", flush=True)

for n, B in [(1024, 1), (1024, 8), (512, 64), (4096, 1), (8192, 1)]:
    for mode in (E.PrecisionMode.MIXED_EMULATED, E.PrecisionMode.BF16):
        run(n, B, mode)
