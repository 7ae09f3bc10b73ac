"""GPU timeline of the async host path (DEPTH calls in flight, default 3), kernels and copies (measurement only)."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from torch.profiler import profile, ProfilerActivity
from paper_2605_08523_b200 import engine as E
from paper_2605_08523_b200.hamiltonians import tight_binding, batch_params
n, B = 1024, 16
m = E.load_model("M1500")
mu, kT = batch_params(B)
H = torch.from_numpy(np.stack([tight_binding(n, seed=10000 + k) for k in range(B)])).pin_memory()
DEPTH = int(os.environ.get("DEPTH", 3))
Ds = [torch.empty_like(H).pin_memory() for _ in range(DEPTH)]
Hp = [H[k].numpy() for k in range(B)]
Dp = [[D[k].numpy() for k in range(B)] for D in Ds]
def run(steps):
    infl = []
    for s in range(steps):
        infl.append(E.compute_density_matrices_async(Hp, mu, kT, m, Dp[s % DEPTH], E.PrecisionMode.MIXED_EMULATED))
        if len(infl) == DEPTH:
            infl.pop(0).wait()
    for h in infl:
        h.wait()
run(3)
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    run(4)
prof.export_chrome_trace("/tmp/trace.json")
ev = [e for e in json.load(open("/tmp/trace.json"))["traceEvents"] if e.get("ph") == "X" and e.get("cat") in ("kernel", "gpu_memcpy")]
ev.sort(key=lambda e: e["ts"])
t0 = ev[0]["ts"]
agg = {}
for e in ev:
    k = ("K2" if "pair" in e["name"] else "K1" if "rescale" in e["name"] else "memcpy " + e["name"].split("(")[0].strip()[-4:] if e["cat"] == "gpu_memcpy" else e["name"][:20])
    agg.setdefault(k, []).append(e["dur"])
for k, v in agg.items():
    print(f"{k:22s} n={len(v):3d} mean {np.mean(v):9.1f} us  total {np.sum(v):9.1f} us")
print("span", (ev[-1]["ts"] + ev[-1]["dur"] - t0), "us for 4 calls")
if os.environ.get("TL_DUMP"):
    for e in ev:
        print(f"{e['ts'] - t0:9.1f} {e['dur']:8.1f} s{e.get('args', {}).get('stream', '?')} {e['name'][:50]}")
# copy-engine utilisation over the captured span
span = ev[-1]["ts"] + ev[-1]["dur"] - t0
for tag in ("HtoD", "DtoH"):
    busy = sum(e["dur"] for e in ev if e["cat"] == "gpu_memcpy" and tag in e["name"])
    print(f"{tag} engine busy {busy / span:.2f} of the span")
kb = sum(e["dur"] for e in ev if e["cat"] == "kernel")
print(f"kernels busy {kb / span:.2f} of the span")
