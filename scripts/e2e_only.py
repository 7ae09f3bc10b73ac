"""Host-path (e2e) throughput only: the bench's async two-in-flight loop, N=1024 B=16 FP32E."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2605_08523_b200 import engine as E
from paper_2605_08523_b200.hamiltonians import tight_binding, batch_params
n, B = 1024, 16
m = E.load_model("M1500")
mu, kT = batch_params(B)
H = torch.from_numpy(np.stack([tight_binding(n, seed=10000 + k) for k in range(B)])).pin_memory()
Ds = [torch.empty_like(H).pin_memory() for _ in range(2)]
Hp = [H[k].numpy() for k in range(B)]
Dp = [[D[k].numpy() for k in range(B)] for D in Ds]
def run(steps):
    infl = []
    for s in range(steps):
        infl.append(E.compute_density_matrices_async(Hp, mu, kT, m, Dp[s % 2], E.PrecisionMode.MIXED_EMULATED))
        if len(infl) == 2:
            infl.pop(0).wait()
    for h in infl:
        h.wait()
run(3)
t = time.perf_counter(); run(30); dt = time.perf_counter() - t
print(os.environ.get("FFG_LIB_PATH", "head"), "e2e %.0f matrices/s" % (B * 30 / dt), flush=True)
