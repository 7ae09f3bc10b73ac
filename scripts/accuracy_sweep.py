"""FP32-emulated accuracy vs the fp64 recursion under the precision knobs (measurement script).

For each environment setting (read once per process, so each runs in a subprocess): worst
errors over all 512 members of configs[3] (512 x N=512, mu/kT per matrix), the N=4096 and
N=8192 single matrices of configs[2], and the bench step's K2 time (16 x N=1024).

    python scripts/accuracy_sweep.py [ENV=V,ENV=V ...]  -> one JSON line per setting
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import json, sys, time
import numpy as np, torch
sys.path.insert(0, %r)
from paper_2605_08523_b200 import engine as E
from paper_2605_08523_b200.hamiltonians import tight_binding, batch_params
from oracle import device_ref as DR
m = E.load_model("M1500")
mode = E.PrecisionMode[%r]
out = {}
def run(H, mu, kT):
    D = torch.empty_like(H)
    s, st, _ = E.compute_density_matrices_device(H, mu, kT, m, mode, D_dev=D)
    torch.cuda.synchronize()
    assert (st.cpu().numpy() == 0).all()
    return D
mu, kT = batch_params(512)
H = torch.from_numpy(np.stack([tight_binding(512, seed=10000 + k) for k in range(512)])).cuda()
R = DR.density_matrices_f64(H, mu, kT, m.abcd, m.beta0, m.mu0)
mx, fro, tr = DR.errors(run(H, mu, kT), R)
out["b512"] = dict(max=float(mx.max()), fro=float(fro.max()), tr=float(tr.max()),
                   tr_over_1e6=int((tr > 1e-6).sum()), tr_p99=float(np.quantile(tr, 0.99)))
del H, R
for n in (4096, 8192):
    H = torch.from_numpy(tight_binding(n, seed=1234)).cuda().unsqueeze(0)
    R = DR.density_matrices_f64(H, 0.0, 0.01, m.abcd, m.beta0, m.mu0)
    mx, fro, tr = DR.errors(run(H, [0.0], [0.01]), R)
    out[f"n{n}"] = dict(max=float(mx[0]), fro=float(fro[0]), tr=float(tr[0]))
    del H, R
mu, kT = batch_params(16)
H = torch.from_numpy(np.stack([tight_binding(1024, seed=10000 + k) for k in range(16)])).cuda()
for _ in range(3):
    run(H, mu, kT)
E.profile_layers(True); E.profile_read_ex()
for _ in range(10):
    run(H, mu, kT)
ms, launches, flops = E.profile_read_ex()
out["k2_ms_bench"] = ms / max(launches, 1)
print("RESULT " + json.dumps(out))
"""


def main():
    mode = os.environ.get("SWEEP_MODE", "MIXED_EMULATED")
    settings = sys.argv[1:] or [""]
    for s in settings:
        env = dict(os.environ)
        kv = dict(x.split("=", 1) for x in s.split(",") if x)
        env.update(kv)
        r = subprocess.run([sys.executable, "-c", CHILD % (ROOT, mode)], capture_output=True, text=True, env=env,
                           timeout=900)
        line = [l for l in r.stdout.splitlines() if l.startswith("RESULT ")]
        rec = {"env": kv, "mode": mode}
        if line:
            rec.update(json.loads(line[0][7:]))
        else:
            rec["error"] = (r.stdout + r.stderr)[-1500:]
        print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()
