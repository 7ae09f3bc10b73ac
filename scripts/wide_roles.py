"""Per-role wait/work cycles of the wide K2 kernel (build with -DFFG_ROLE_PROF=1; FFG_DEBUG_K2=8).

    FFG_LIB_PATH=paper_2605_08523_b200/lib/var/prof.so python scripts/wide_roles.py 1024x16 512x64 ...
"""
import ctypes
import os
import sys

os.environ["FFG_DEBUG_K2"] = str(int(os.environ.get("FFG_DEBUG_K2", "0")) | 8)
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2605_08523_b200 import engine as E
from paper_2605_08523_b200.hamiltonians import tight_binding, batch_params

m = E.load_model("M1500")
names = ["total", "prod_dep", "prod_empty", "mma_full", "mma_slot", "mma_slot2",
         "w0_chunk", "w0_drainwork", "w0_dep", "w0_epi", "w0_pub", "w0_setup",
         "w5_chunk", "w5_drainwork", "w5_dep", "w5_epi"]
modes = [E.PrecisionMode[x] for x in os.environ.get("MODES", "MIXED_EMULATED").split(",")]
for spec in (sys.argv[1:] or ["1024x16", "512x64", "4096x1"]):
    n, B = (int(x) for x in spec.split("x"))
    for mode in modes:
        mu, kT = batch_params(B)
        H = torch.from_numpy(np.stack([tight_binding(n, seed=10000 + k) for k in range(B)])).cuda()
        D = torch.empty_like(H)
        for _ in range(2):
            E.compute_density_matrices_device(H, mu, kT, m, mode, D_dev=D)
        torch.cuda.synchronize()
        buf = (ctypes.c_uint64 * (16 * 148))()
        E._check(E.lib().ffg_debug_role_cycles(buf, 148))
        a = np.frombuffer(buf, dtype=np.uint64).reshape(148, 16).astype(float)
        tot = a[:, 0].mean()
        lead = a[0::2]
        row = {k: a[:, i].mean() / tot for i, k in enumerate(names)}
        for i, k in enumerate(names[3:6], start=3):
            row[k] = lead[:, i].mean() / tot
        print(f"n={n} B={B} {mode.name:15s} total {tot / 1e6:7.2f} Mcyc  " +
              "  ".join(f"{k}={v:.2f}" for k, v in row.items() if k != "total"), flush=True)
        del H, D
        torch.cuda.empty_cache()
