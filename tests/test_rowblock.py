"""Row-block sharding of one large H: host logic on CPU, arithmetic on the GPU.

CPU: the row-block pair tables cover every block of every rank's rows exactly once and carry the
cross-order bit of the symmetric table's orientation; the per-layer in-place all-gather of the
operand rows (world size 2 over gloo).  GPU: `world` ranks emulated on one device (own workspaces,
exchange by device copies) give a D bit-identical to the single-GPU path."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2605_08523_b200 import engine as E
from paper_2605_08523_b200 import rowblock as RB
from paper_2605_08523_b200.hamiltonians import tight_binding


@pytest.mark.parametrize("nb,world", [(8, 1), (8, 2), (8, 4), (16, 4), (128, 8), (9, 3)])
def test_rowblock_tables_cover_rows_once_with_symmetric_orientation(nb, world):
    sym = E.pair_table(nb)
    orient = {}
    for a0, a1, s, d in sym:
        orient[(min(a0, s), max(a0, s))] = a0
        if not d:
            orient[(min(a1, s), max(a1, s))] = a1
    seen = {}
    for r in range(world):
        t = RB.rowblock_table(nb, r, world)
        rows = range(nb // world * r, nb // world * (r + 1))
        for a0, a1, s, d, sw in t:
            blocks = [(a0, s)] + ([] if d else [(a1, s)])
            assert a0 in rows and a1 in rows
            for R, C in blocks:
                assert (R, C) not in seen
                seen[(R, C)] = r
                want = 0 if R == C else int(orient[(min(R, C), max(R, C))] != R)
                assert sw == want, (R, C, sw, want)
            if not d:
                assert a1 == a0 + 1
    assert len(seen) == nb * nb


def test_rowblock_table_rejects_uneven_rows():
    with pytest.raises(E.DimensionError):
        RB.rowblock_table(10, 0, 4)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _exchange_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        npad, rows = 8, 4
        bufs = [torch.full((npad, 6), -1, dtype=torch.uint8) for _ in range(2)]
        for k, b in enumerate(bufs):  # this rank writes its rows only (as a layer does)
            b[rank * rows:(rank + 1) * rows] = 10 * k + rank
        RB.exchange_rows(bufs, rank * rows, rows, world)
        q.put((rank, [b.clone() for b in bufs]))
    finally:
        dist.destroy_process_group()


def test_exchange_rows_world2_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_exchange_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    for r in range(2):
        for k, b in enumerate(out[r]):
            assert (b[:4] == 10 * k + 0).all() and (b[4:] == 10 * k + 1).all()


# ----------------------------------------------------------------------------------------- GPU
@pytest.mark.gpu
@pytest.mark.parametrize("n,world,mode", [(2048, 2, "MIXED_EMULATED"), (2048, 4, "MIXED_EMULATED"),
                                          (1000, 2, "MIXED_EMULATED"), (1024, 1, "MIXED_EMULATED"),
                                          (1024, 2, "BF16"), (1024, 4, "FP16")])
def test_rowblock_virtual_bit_identical_to_single_gpu(n, world, mode, monkeypatch):
    """Each rank computes its block rows against all columns (the blocks below the diagonal with
    the swapped cross-term order), exchanging the operand rows every layer: the assembled D equals
    the single-GPU D of the same (pair) kernel bit for bit; the rank-order statistics agree to fp64
    summation order.  (Row-block shards run the pair kernel; the single-GPU default for nb even and
    N >= 1024 is the wide kernel, gated separately in tests/test_gpu_wide.py.)"""
    if not E.device_available():
        pytest.fail("no sm_100 device")
    m = E.load_model("M1500")
    md = E.PrecisionMode[mode]
    H = torch.from_numpy(tight_binding(n, seed=2024)).cuda()
    D1 = torch.empty((1, n, n), dtype=torch.float64, device="cuda")
    monkeypatch.setenv("FFG_WIDE", "0")
    s1, st1, _ = E.compute_density_matrices_device(H.unsqueeze(0), [0.02], [0.011], m, md, D_dev=D1)
    D, stats, status = RB.rowblock_virtual(H, 0.02, 0.011, m, world, md)
    torch.cuda.synchronize()
    assert status == 0 and st1.item() == 0
    bad = (D != D1[0]).nonzero()
    assert bad.shape[0] == 0, (bad.shape[0], bad[:5].tolist())
    ref = s1[0].cpu().numpy()
    assert abs(stats.trace - ref[0]) <= 1e-12 * abs(ref[0])
    assert abs(stats.trace_square - ref[1]) <= 1e-12 * abs(ref[1])


@pytest.mark.gpu
def test_rowblock_out_of_region_and_order_checks():
    m = E.load_model("M1500")
    H = torch.from_numpy(tight_binding(512, seed=1)).cuda()
    r = RB.RowBlockRank(H, 0.0, 0.001, m, rank=0, world=2)  # beta' ~ 9000: out of region
    D = torch.zeros((r.d_rows, 512), dtype=torch.float64, device="cuda")
    with pytest.raises(E.ValidationError, match="out of order"):
        r.layer(3)
    for l in range(m.layer_count):
        r.layer(l, D if l == m.layer_count - 1 else None)
    stats, status, pv = r.end()
    assert status == E.OutOfRegionError.status and pv.half_products == 0
    assert torch.isnan(D).all()
    with pytest.raises(E.DimensionError, match="divide evenly"):
        RB.RowBlockRank(H, 0.0, 0.01, m, rank=0, world=3)


@pytest.mark.gpu
def test_rowblock_nccl_driver_single_rank():
    """The torch.distributed driver (per-layer in-place NCCL all-gather of the operand rows, rank-order
    statistics) with one rank on the one GPU of this box: D equals the single-GPU D bit for bit."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = r"""
import os, sys, torch, numpy as np, torch.distributed as dist
sys.path.insert(0, %r)
from paper_2605_08523_b200 import engine as E, rowblock as RB
from paper_2605_08523_b200.hamiltonians import tight_binding
os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=%r)
torch.cuda.set_device(0)
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
m = E.load_model("M1500")
H = torch.from_numpy(tight_binding(1024, seed=5)).cuda()
D1 = torch.empty((1, 1024, 1024), dtype=torch.float64, device="cuda")
s1, st1, _ = E.compute_density_matrices_device(H.unsqueeze(0), [0.0], [0.01], m, D_dev=D1)
D, row0, stats, status = RB.rowblock_density_matrix(H, 0.0, 0.01, m)
torch.cuda.synchronize()
assert status == 0 and row0 == 0 and torch.equal(D, D1[0])
assert abs(stats.trace - s1[0, 0].item()) <= 1e-12 * stats.trace
dist.destroy_process_group()
print("NCCL_ROWBLOCK_OK")
""" % (root, str(_free_port()))
    env = dict(os.environ, FFG_WIDE="0")  # the single-GPU reference on the row-block shards' kernel
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300, env=env)
    assert r.returncode == 0 and "NCCL_ROWBLOCK_OK" in r.stdout, r.stdout[-2000:] + r.stderr[-3000:]
