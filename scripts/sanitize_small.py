"""Workload for compute-sanitizer (memcheck / racecheck / synccheck): K1 -> K2 -> K3 at N=256 in
FP32-emulated and BF16 mode, a 3-matrix batch (8-warp and 16-worker epilogues), one row-block rank,
the wide kernel (forced, FFG_WIDE=1) on a 2-matrix N=512 batch in both modes, and DOUBLE / SINGLE at N=256.

    compute-sanitizer --tool racecheck python scripts/sanitize_small.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2605_08523_b200 import engine as E  # noqa: E402
from paper_2605_08523_b200 import rowblock as RB  # noqa: E402
from paper_2605_08523_b200.hamiltonians import tight_binding, batch_params  # noqa: E402

m = E.load_model("M1500")
H = tight_binding(256, seed=1234)
for mode in (E.PrecisionMode.MIXED_EMULATED, E.PrecisionMode.BF16):
    D, st, pv = E.compute_density_matrix(H, 0.0, 0.01, m, mode)
    print(mode.name, "trace", st.trace, "status", pv.status, flush=True)
mu, kT = batch_params(3)
Hd = torch.from_numpy(np.stack([tight_binding(384, seed=7 + k) for k in range(3)])).cuda()
Dd = torch.empty_like(Hd)
for s16 in ("0", "1"):
    os.environ["FFG_S16"] = s16  # read per call
    s, status, _ = E.compute_density_matrices_device(Hd, mu, kT, m, D_dev=Dd)
    torch.cuda.synchronize()
    print("batch S16", s16, status.tolist(), flush=True)
D, stats, status = RB.rowblock_virtual(torch.from_numpy(H).cuda(), 0.0, 0.01, m, 2)
torch.cuda.synchronize()
print("rowblock", status, stats.trace, flush=True)
os.environ["FFG_WIDE"] = "1"
Hw = torch.from_numpy(np.stack([tight_binding(512, seed=11 + k) for k in range(2)])).cuda()
Dw = torch.empty_like(Hw)
for mode in (E.PrecisionMode.MIXED_EMULATED, E.PrecisionMode.BF16):
    s, status, _ = E.compute_density_matrices_device(Hw, mu[:2], kT[:2], m, mode, D_dev=Dw)
    torch.cuda.synchronize()
    print("wide", mode.name, status.tolist(), s[:, 0].tolist(), flush=True)
os.environ.pop("FFG_WIDE")
for mode in (E.PrecisionMode.DOUBLE, E.PrecisionMode.SINGLE):
    D, st, pv = E.compute_density_matrix(H, 0.0, 0.01, m, mode)
    print(mode.name, "trace", st.trace, "status", pv.status, flush=True)
