"""TEST INFRASTRUCTURE ONLY -- the fp64 MLSP2 recursion restated with torch float64 GEMMs.

The checker for the BASELINE configs whose sizes the numpy oracle cannot finish in seconds
(N = 4096 .. 16384, and the 512-member N=512 batch).  Only ``tests/`` may use it.  It is
the same arithmetic as ``oracle.density_matrix_f64`` (scalar_models.cpp:243-252 lifted to
matrices: ``A += d X; X = a X^2 + b X + c I``; ``D = A + X``) with the frame of
SURVEY.md 0.4 (``X0 = (1 - mu0) I - (beta/beta0)(H - mu I)``), evaluated by cuBLAS DGEMM
on whatever device the inputs live on; ``tests/test_gpu_configs.py`` pins it against the
numpy oracle at N=512 before trusting it at the large sizes.
"""
from __future__ import annotations

import numpy as np


def density_matrices_f64(H, mu, kT, abcd, beta0: float, mu0: float):
    """H: torch float64 [B, n, n] (or [n, n]); mu, kT: scalars or length-B arrays.
    Returns D (same shape as H), float64, computed in fp64 throughout."""
    import torch

    squeeze = H.dim() == 2
    if squeeze:
        H = H.unsqueeze(0)
    B, n, _ = H.shape
    mu = torch.as_tensor(np.broadcast_to(np.asarray(mu, dtype=np.float64), (B,)).copy(), device=H.device)
    kT = torch.as_tensor(np.broadcast_to(np.asarray(kT, dtype=np.float64), (B,)).copy(), device=H.device)
    s = (1.0 / kT) / beta0                                     # beta / beta0 per matrix
    X = -s.view(B, 1, 1) * H
    diag = torch.diagonal(X, dim1=1, dim2=2)
    diag += ((1.0 - mu0) + s * mu).view(B, 1)                  # (1 - mu0) I + (beta/beta0) mu I
    A = torch.zeros_like(X)
    Y = torch.empty_like(X)
    for a, b, c, d in np.asarray(abcd, dtype=np.float64).reshape(-1, 4):
        A.add_(X, alpha=float(d))                              # acc += d * x
        torch.bmm(X, X, out=Y)                                 # x2 = x * x
        X.mul_(float(b)).add_(Y, alpha=float(a))               # x = a * x2 + b * x + c
        torch.diagonal(X, dim1=1, dim2=2).add_(float(c))
    A.add_(X)                                                  # return acc + x
    del X, Y
    return A[0] if squeeze else A


def errors(D, R):
    """Per-matrix (max|dD|, ||dD||_F / ||R||_F, |dTr| / |Tr R|) of torch tensors [B, n, n]."""
    import torch

    if D.dim() == 2:
        D, R = D.unsqueeze(0), R.unsqueeze(0)
    dD = D - R
    mx = dD.abs().amax(dim=(1, 2))
    fro = torch.linalg.matrix_norm(dD) / torch.linalg.matrix_norm(R)
    trR = torch.diagonal(R, dim1=1, dim2=2).sum(-1)
    trD = torch.diagonal(D, dim1=1, dim2=2).sum(-1)
    tr = (trD - trR).abs() / trR.abs()
    return mx.cpu().numpy(), fro.cpu().numpy(), tr.cpu().numpy()
