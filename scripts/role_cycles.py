"""Per-role wait cycles of the K2 pair kernel (FFG_DEBUG_K2=8), averaged over CTAs."""
import sys, os, ctypes
os.environ["FFG_DEBUG_K2"] = str(int(os.environ.get("FFG_DEBUG_K2", "0")) | 8)
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2605_08523_b200 import engine as E
from paper_2605_08523_b200.hamiltonians import tight_binding, batch_params
m = E.load_model("M1500")
names = ["total", "prod_dep", "prod_empty", "mma_full", "mma_slot", "drain_slotfull", "epi_y", "epi_publish",
         "epi_stwait", "epi_compute", "epi_pieces", "epi_tail", "epi_item"]
for spec in (sys.argv[1:] or ["1024x16", "4096x1", "512x64"]):
    n, B = (int(x) for x in spec.split("x"))
    for mode in (E.PrecisionMode.MIXED_EMULATED, E.PrecisionMode.BF16):
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
        row["mma_full"] = lead[:, 3].mean() / tot
        row["mma_slot"] = lead[:, 4].mean() / tot
        items = (p_items := None)
        print(f"n={n} B={B} {mode.name:15s} total {tot/1e6:8.2f} Mcyc  " +
              "  ".join(f"{k}={v:.2f}" for k, v in row.items() if k != "total"), flush=True)
