"""world_size-2 gloo tests of the batch-sharding host logic (no GPU)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2605_08523_b200.distributed import shard_range, max_shard, ResultGather, sharded_density_matrices
from paper_2605_08523_b200.hamiltonians import tight_binding


def test_shard_range_covers_exactly():
    for total in (0, 1, 7, 512, 513):
        for world in (1, 2, 3, 8):
            ranges = [shard_range(total, world, r) for r in range(world)]
            assert ranges[0][0] == 0 and ranges[-1][1] == total
            for (a, b), (c, d) in zip(ranges, ranges[1:]):
                assert b == c
            sizes = [b - a for a, b in ranges]
            assert max(sizes) - min(sizes) <= 1 and max(sizes) <= max_shard(total, world)


def _fake_compute(Hd, mu, kT):
    # stand-in for the device pipeline: (Tr H, sum H^2) and a status derived from kT
    st = torch.stack([Hd.diagonal(dim1=1, dim2=2).sum(-1), (Hd * Hd).sum((1, 2))], dim=1)
    status = torch.tensor([0 if k > 0 else 1 for k in kT], dtype=torch.int32)
    return st, status


def _worker(rank, world, port, G, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        Hs = [tight_binding(16, seed=k) for k in range(G)]
        mu = np.linspace(-0.1, 0.1, G)
        kT = np.full(G, 0.01)
        kT[3] = -1.0
        stats, status = sharded_density_matrices(Hs, mu, kT, compute=_fake_compute,
                                                 device=torch.device("cpu"))
        q.put((rank, stats, status))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("G", [5, 8])
def test_sharded_gather_world2_gloo(G):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, G, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    Hs = [tight_binding(16, seed=k) for k in range(G)]
    want = np.array([[np.trace(H), (H * H).sum()] for H in Hs])
    for rank, stats, status in out:
        assert np.allclose(stats, want, rtol=0, atol=1e-12)
        assert status.tolist() == [0 if k != 3 else 1 for k in range(G)]


def test_result_gather_single_process():
    g = ResultGather(1, 0, 3, torch.device("cpu"))
    rec = g.gather(torch.ones((3, 2), dtype=torch.float64), torch.zeros(3, dtype=torch.int32))
    stats, status = ResultGather.unpack(rec, 3)
    assert stats.shape == (3, 2) and status.tolist() == [0, 0, 0]


def test_bench_gpus_2_self_launches_two_ranks():
    """`python bench.py --gpus 2` (no torchrun in the environment) re-launches itself as two
    ranks under torch.distributed.run; with --fake-compute they run over gloo on CPU, gather
    every matrix's record and rank 0 prints exactly one JSON line for n_gpus=2."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--fake-compute",
                        "--n", "64", "--batch", "3", "--steps", "2", "--warmup", "3"],
                       capture_output=True, text=True, env=env, timeout=240, cwd=root)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["fake"] and d["gathered"] == 6 and d["gather_ok"]
    assert d["config"]["global_batch"] == 6 and d["value"] > 0
