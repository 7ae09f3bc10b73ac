#!/bin/bash
# fixed-point exact layers: accuracy (incl. a large-N Frobenius check) and K2 time vs their count
for e in ${FIX_E:-6 10 15 30}; do
  export FFG_EXACT_DRAIN_LAYERS=$e
  timeout 300 python scripts/accuracy_report.py MIXED_EMULATED 2>&1 | grep WORST | sed "s/^/E=$e /"
  timeout 300 python - <<'PY'
import os, numpy as np, torch
from paper_2605_08523_b200 import engine as E
from paper_2605_08523_b200.hamiltonians import tight_binding
import sys; sys.path.insert(0, "scripts")
from config_sweep import recursion_f64, errors
m = E.load_model("M1500")
for n in (2048, 4096):
    H = torch.from_numpy(tight_binding(n, seed=1234)[None]).cuda()
    D = torch.empty_like(H)
    E.compute_density_matrices_device(H, [0.0], [0.01], m, E.PrecisionMode.MIXED_EMULATED, D_dev=D)
    torch.cuda.synchronize()
    R = recursion_f64(H[0], 0.0, 0.01, m)
    print("E=%s n=%d" % (os.environ["FFG_EXACT_DRAIN_LAYERS"], n), {k: "%.2e" % v for k, v in errors(D[0], R).items()}, flush=True)
PY
  timeout 120 python scripts/k2_variants.py 1024x16 4096x1 2>&1 | grep MIXED | sed "s/^.*\] //" | sed "s/^/E=$e /"
done
