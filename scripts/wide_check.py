"""Wide (256x256) vs pair kernel: errors vs the fp64 recursion, symmetry, status and K2 time.

    FFG_WIDE=0|1 python scripts/wide_check.py [n x B ...]   -> one line per (config, mode)
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from oracle import device_ref as DR
from paper_2605_08523_b200 import engine as E
from paper_2605_08523_b200.hamiltonians import tight_binding, batch_params

m = E.load_model("M1500")
cases = [tuple(int(x) for x in c.split("x")) for c in sys.argv[1:]] or [(256, 1), (512, 8), (1024, 4), (1024, 16),
                                                                        (2048, 2), (4096, 1)]
modes = [E.PrecisionMode[x] for x in os.environ.get("MODES", "MIXED_EMULATED,BF16").split(",")]
tag = "wide" if os.environ.get("FFG_WIDE", "1") != "0" else "pair"
for n, B in cases:
    mu, kT = batch_params(B)
    H = torch.from_numpy(np.stack([tight_binding(n, seed=10000 + k) for k in range(B)])).cuda()
    R = DR.density_matrices_f64(H, mu, kT, m.abcd, m.beta0, m.mu0)
    for mode in modes:
        D = torch.empty_like(H)
        st, status, _ = E.compute_density_matrices_device(H, mu, kT, m, mode, D_dev=D)
        torch.cuda.synchronize()
        mx, fro, tr = DR.errors(D, R)
        sym = bool(torch.equal(D, D.transpose(1, 2)))
        trk = torch.diagonal(D, dim1=1, dim2=2).sum(-1)
        strel = float(((st[:, 0] - trk).abs() / trk.abs()).max())
        E.profile_layers(True)
        E.profile_read_ex()
        reps = 5
        for _ in range(reps):
            E.compute_density_matrices_device(H, mu, kT, m, mode, D_dev=D)
        torch.cuda.synchronize()
        ms, k, F = E.profile_read_ex()
        E.profile_layers(False)
        print(f"{tag} n={n:5d} B={B:4d} {mode.name:15s} status={sorted(set(status.cpu().tolist()))} sym={sym} "
              f"max={mx.max():.2e} fro={fro.max():.2e} tr={tr.max():.2e} stats-vs-D={strel:.1e} "
              f"K2={ms / reps:8.3f} ms {F / (ms / 1e3) / 1e12:7.1f} TF/s", flush=True)
        del D
    del H, R
    torch.cuda.empty_cache()
