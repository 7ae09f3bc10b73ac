"""Per-item event times of the pair kernel (FFG_ROLE_PROF build, FFG_DEBUG_K2=8|4096): producer start,
first operand load issued, last chunk drained, block published -- per layer, the critical path of a
single-matrix launch.

    FFG_LIB_PATH=paper_2605_08523_b200/lib/var/prof.so python scripts/item_timeline.py 1024 [MODE] [B]

B > 1 (a batch): the per-layer table is skipped; the per-item MMA phase and in-loop operand waits are summarised.
"""
import ctypes
import os
import sys

os.environ["FFG_DEBUG_K2"] = str(int(os.environ.get("FFG_DEBUG_K2", "0")) | 8 | 4096)
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2605_08523_b200 import engine as E  # noqa: E402
from paper_2605_08523_b200.hamiltonians import tight_binding, batch_params  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
mode = E.PrecisionMode[sys.argv[2]] if len(sys.argv) > 2 else E.PrecisionMode.MIXED_EMULATED
m = E.load_model("M1500")
B = int(sys.argv[3]) if len(sys.argv) > 3 else 1
mu, kT = batch_params(B)
H = torch.from_numpy(np.stack([tight_binding(n, seed=1234 + k) for k in range(B)])).cuda()
D = torch.empty_like(H)
for _ in range(3):
    E.compute_density_matrices_device(H, mu, kT, m, mode, D_dev=D)
torch.cuda.synchronize()
nb = (n + 127) // 128
PT = (nb * (nb + 1) // 2 + 1) // 2
L = m.layer_count
items = L * PT * B
ctas = 1024 + (12 * items + 15) // 16
buf = (ctas * 16 * ctypes.c_uint64)()
E._check(E.lib().ffg_debug_role_cycles(buf, ctas))
raw = np.frombuffer(buf, dtype=np.uint64)[16 * 1024:16 * 1024 + 12 * items].reshape(items, 12).astype(np.int64)
w = raw[:, 8:12].astype(float)  # cumulative wait cycles per CTA at each item's end
t = raw[:, :8]
prof = np.frombuffer(buf, dtype=np.uint64)[:16 * 148].reshape(148, 16).astype(float)
t0 = t[t > 0].min()
t = np.where(t > 0, t - t0, -1) / 1000.0  # us
print(f"n={n} {mode.name}: {PT} items per layer, {L} layers, K2 {t.max():.1f} us; SM clock ~"
      f"{prof[0, 0] / (t.max() * 1e3):.2f} GHz (CTA 0 producer cycles / K2 span)")
names = ["start", "load0", "drained", "published", "landed0", "mma_last", "computed", "stored"]
inloop = (w[:, 0] - w[:, 1]) / 1000  # MMA waits for operand stages inside the K loop, kcycles per item
mma = t[:, 5] - t[:, 4]                # first stage landed -> last MMA issued, us per item
if B == 1:
    order = [0, 1, 4, 5, 2, 6, 7, 3]
    print("layer  " + "  ".join(f"{names[e]:>15s}" for e in order) + "   [us, first..last item]")
    for l in range(L):
        r = t[l * PT:(l + 1) * PT]
        cols = []
        for e in order:
            v = r[:, e][r[:, e] >= 0]
            cols.append(f"{v.min():7.1f}..{v.max():7.1f}" if v.size else "      -..      -")
        print(f"{l:4d}   " + "  ".join(cols))
    print("MMA full-stage waits inside the K loop (x1000 cycles per item): mean %.1f" % inloop[PT * 5:].mean())
    for l in (1, 15):
        print(f"layer {l}: {inloop[l * PT:(l + 1) * PT].mean():.1f}")
else:
    ok = (t[:, 4] >= 0) & (t[:, 5] >= 0)
    print(f"B={B}: {items} items; per item: MMA phase (landed0 -> last MMA issued) mean {mma[ok].mean():.2f} us, "
          f"in-loop operand waits mean {inloop[ok].mean():.2f} kcycles")
    # exact (first 10 layers) vs normal layers: item index order is group -> layer -> matrix -> pair
