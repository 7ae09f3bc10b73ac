"""GPU timeline of a few bench steps (torch.profiler / CUPTI): kernels and copies with start offsets,
to locate the gaps between the launches of a step (measurement only)."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from torch.profiler import profile, ProfilerActivity
from paper_2605_08523_b200 import engine as E
from paper_2605_08523_b200.hamiltonians import tight_binding, batch_params
n, B = int(os.environ.get("N", 1024)), int(os.environ.get("B", 16))
m = E.load_model("M1500")
mu, kT = batch_params(B)
H = torch.from_numpy(np.stack([tight_binding(n, seed=10000 + k) for k in range(B)])).cuda()
D = torch.empty_like(H)
for _ in range(3):
    E.compute_density_matrices_device(H, mu, kT, m, E.PrecisionMode.MIXED_EMULATED, D_dev=D)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(3):
        E.compute_density_matrices_device(H, mu, kT, m, E.PrecisionMode.MIXED_EMULATED, D_dev=D)
    torch.cuda.synchronize()
prof.export_chrome_trace("/tmp/trace.json")
ev = [e for e in json.load(open("/tmp/trace.json"))["traceEvents"] if e.get("ph") == "X" and e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")]
ev.sort(key=lambda e: e["ts"])
t0 = ev[0]["ts"]; prev_end = t0
for e in ev:
    print(f"{e['ts'] - t0:9.1f} us  dur {e['dur']:8.1f}  gap {e['ts'] - prev_end:7.1f}  {e['cat']:10s} {e['name'][:60]}")
    prev_end = e["ts"] + e["dur"]
