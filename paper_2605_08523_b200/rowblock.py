"""Row-block sharding of one large Hamiltonian over GPUs.

Rank r of `world` owns block rows [r nb/world, (r+1) nb/world) (128-row blocks) of X, A and D
and computes those rows against all columns every layer (ffg_rowblock_*, include/fermiforge/ffg.h).
Between layers every rank needs the binary16 operands of X_{l+1} for ALL rows: one in-place
all-gather of the hi and lo arrays (NCCL over NVLink, one process per GPU).  D stays distributed
as row slabs; Tr D and Tr D^2 are the rank partials summed in rank order (deterministic).

The arithmetic of every block is that of the single-GPU pair kernel (the pair table's cross-order
bit), so the assembled D equals the single-GPU pair-kernel D (FFG_WIDE=0) bit for bit -- the
row-block path changes where the work runs, never the result.  (The single-GPU default for N >= 2048
is the wide kernel, k2_wide.cuh: the same recursion with another accumulation schedule, gated
against the fp64 recursion on its own.)

Drivers:
  rowblock_density_matrix(...)   one rank per process under torch.distributed (NCCL)
  rowblock_virtual(...)          `world` ranks emulated in one process on one device, the exchange
                                 done by device copies (tests, and the single-GPU check of the
                                 sharded arithmetic)
  exchange_rows(...)             the per-layer all-gather, shared by both (gloo-testable on CPU)
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import engine as E

_VP = ctypes.c_void_p


def _bind(L):
    if getattr(L, "_rowblock_bound", False):
        return L
    L.ffg_rowblock_begin.argtypes = [_VP, ctypes.c_int64, ctypes.c_double, ctypes.c_double,
                                     ctypes.POINTER(E._Model), ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, _VP,
                                     ctypes.POINTER(_VP)]
    L.ffg_rowblock_rows.argtypes = [_VP, ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int64),
                                    ctypes.POINTER(ctypes.c_int64)]
    L.ffg_rowblock_operands.argtypes = [_VP, ctypes.c_int32, ctypes.POINTER(_VP), ctypes.POINTER(_VP)]
    L.ffg_rowblock_layer.argtypes = [_VP, ctypes.c_int32, _VP, _VP]
    L.ffg_rowblock_end.argtypes = [_VP, E._D, ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(E._Prov), _VP]
    L.ffg_rowblock_table.restype = ctypes.c_int32
    L.ffg_rowblock_table.argtypes = [ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, _VP, ctypes.c_int32]
    L._rowblock_bound = True
    return L


def rowblock_table(nb: int, rank: int, world: int) -> np.ndarray:
    """Rows (A0, A1, S, dummy, swap) of rank `rank`'s row-block pair table."""
    L = _bind(E.lib())
    cnt = L.ffg_rowblock_table(nb, rank, world, None, 0)
    if cnt < 0:
        raise E.DimensionError(f"bad row-block table ({nb} blocks, rank {rank} of {world})")
    buf = np.zeros(cnt, dtype=np.uint32)
    L.ffg_rowblock_table(nb, rank, world, buf.ctypes.data, cnt)
    return np.stack([buf & 1023, (buf >> 10) & 1023, (buf >> 20) & 1023, (buf >> 30) & 1, buf >> 31], axis=1)


class _DevArray:
    """__cuda_array_interface__ view of a library-owned device buffer (no ownership)."""

    def __init__(self, ptr: int, shape, typestr: str):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr, "data": (int(ptr), False),
                                         "version": 3, "strides": None}


class RowBlockRank:
    """One rank's row-block session on the current device (ffg_rowblock_begin .. end)."""

    def __init__(self, H_dev, mu: float, kT: float, model: E.Mlsp2Model,
                 mode: E.PrecisionMode = E.PrecisionMode.MIXED_EMULATED, rank: int = 0, world: int = 1,
                 stream=None):
        import torch

        if H_dev.dtype != torch.float64 or not H_dev.is_cuda or H_dev.dim() != 2 or not H_dev.is_contiguous():
            raise E.ValidationError("H_dev must be a contiguous CUDA float64 tensor [n, n]")
        self.L = _bind(E.lib())
        self.H = H_dev  # kept alive: K1 reads it asynchronously
        self.n = H_dev.shape[0]
        self.model, self.mode, self.rank, self.world = model, mode, rank, world
        self.stream = stream if stream is not None else torch.cuda.current_stream(H_dev.device)
        self._m = model._c()
        h = _VP()
        E._check(self.L.ffg_rowblock_begin(H_dev.data_ptr(), self.n, float(mu), float(kT), ctypes.byref(self._m),
                                           int(mode), rank, world, self.stream.cuda_stream, ctypes.byref(h)))
        self.h = h
        r0, rows, np_ = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        E._check(self.L.ffg_rowblock_rows(h, ctypes.byref(r0), ctypes.byref(rows), ctypes.byref(np_)))
        self.row0, self.rows, self.np = r0.value, rows.value, np_.value
        self.d_rows = max(0, min(self.row0 + self.rows, self.n) - self.row0)
        self.layer_next = 0

    def operands(self, parity: int):
        """[np, np] uint8-pair views (bytes) of the hi / lo arrays of operand parity `parity`."""
        import torch

        hi, lo = _VP(), _VP()
        E._check(self.L.ffg_rowblock_operands(self.h, parity, ctypes.byref(hi), ctypes.byref(lo)))
        out = []
        for p in (hi, lo):
            if p.value:
                out.append(torch.as_tensor(_DevArray(p.value, (self.np, 2 * self.np), "|u1"), device=self.H.device))
        return out

    def my_rows(self, buf):
        return buf[self.row0:self.row0 + self.rows]

    def layer(self, l: int, D_rows=None):
        ptr = D_rows.data_ptr() if D_rows is not None else None
        E._check(self.L.ffg_rowblock_layer(self.h, l, ptr, self.stream.cuda_stream))
        self.layer_next = l + 1

    def end(self):
        """-> ({sum of D_ii, sum of D_ij^2} over this rank's rows, status, Provenance)."""
        stats = np.zeros(2)
        st = ctypes.c_int32()
        pv = E._Prov()
        rc = self.L.ffg_rowblock_end(self.h, E._dp(stats), ctypes.byref(st), ctypes.byref(pv),
                                     self.stream.cuda_stream)
        self.h = None
        if rc not in (0, E.OutOfRegionError.status, E.DivergedEvaluationError.status, E.HalfRangeError.status):
            E._check(rc)
        return stats, int(st.value), E.Provenance._from(pv)

    def __del__(self):
        if getattr(self, "h", None):
            try:
                self.L.ffg_rowblock_end(self.h, None, None, None, self.stream.cuda_stream)
            except Exception:
                pass


def exchange_rows(bufs, row0: int, rows: int, world: int, group=None):
    """In-place all-gather of every rank's rows of each [np, X] buffer (rank r's rows are
    [r rows, (r+1) rows); equal counts on every rank)."""
    import torch.distributed as dist

    for b in bufs:
        flat = b.view(-1)
        chunk = rows * b.shape[1]
        dist.all_gather_into_tensor(flat, flat[row0 * b.shape[1]:row0 * b.shape[1] + chunk], group=group)


def _combine_stats(partials):
    """Rank-order sum of per-rank (Tr, Tr^2) partials (deterministic)."""
    tr = sq = 0.0
    for t, s in partials:
        tr += float(t)
        sq += float(s)
    return tr, sq


def rowblock_density_matrix(H_dev, mu: float, kT: float, model: E.Mlsp2Model,
                            mode: E.PrecisionMode = E.PrecisionMode.MIXED_EMULATED, group=None):
    """One rank of the row-block path under torch.distributed (one process per GPU, NCCL).

    H_dev: the whole H on this rank's device (replicated input).  Returns (D_rows [rows, n] of this
    rank's rows, starting at row0), row0, DensityStatistics of the whole D (rank-order sum), status."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    r = RowBlockRank(H_dev, mu, kT, model, mode, rank, world)
    D_rows = torch.empty((r.d_rows, r.n), dtype=torch.float64, device=H_dev.device)
    with torch.cuda.stream(r.stream):
        for l in range(model.layer_count):
            r.layer(l, D_rows if l == model.layer_count - 1 else None)
            if l + 1 < model.layer_count:
                exchange_rows(r.operands((l + 1) & 1), r.row0, r.rows, world, group)
    stats, status, pv = r.end()
    allp = torch.zeros((world, 2), dtype=torch.float64, device=H_dev.device)
    dist.all_gather_into_tensor(allp.view(-1), torch.tensor(stats, device=H_dev.device), group=group)
    tr, sq = _combine_stats(allp.cpu().numpy())
    return D_rows, r.row0, E.DensityStatistics(tr, sq), status


def rowblock_virtual(H_dev, mu: float, kT: float, model: E.Mlsp2Model, world: int,
                     mode: E.PrecisionMode = E.PrecisionMode.MIXED_EMULATED):
    """`world` row-block ranks emulated on ONE device: every rank has its own workspace and operand
    buffers, runs its layer, and the exchange copies each rank's rows into every other rank's
    buffers (what the all-gather does across GPUs).  Returns (D, DensityStatistics, status)."""
    import torch

    ranks = [RowBlockRank(H_dev, mu, kT, model, mode, r, world) for r in range(world)]
    n = ranks[0].n
    D = torch.empty((n, n), dtype=torch.float64, device=H_dev.device)
    for l in range(model.layer_count):
        last = l == model.layer_count - 1
        for r in ranks:
            r.layer(l, D[r.row0:r.row0 + r.d_rows] if last else None)
        if not last:
            par = (l + 1) & 1
            views = [r.operands(par) for r in ranks]
            torch.cuda.current_stream().synchronize()
            for src, r in enumerate(ranks):
                for dst in range(world):
                    if dst != src:
                        for a, b in zip(views[dst], views[src]):
                            r.my_rows(a).copy_(r.my_rows(b))
            torch.cuda.current_stream().synchronize()
    res = [r.end() for r in ranks]
    tr, sq = _combine_stats([s for s, _, _ in res])
    status = max(st for _, st, _ in res)
    return D, E.DensityStatistics(tr, sq), status
