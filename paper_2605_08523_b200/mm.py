"""Matrix Market array I/O in the reference's exact format (symmetric_matrix.cpp:120-189):
write `%%MatrixMarket matrix array real symmetric`, `N N`, then the lower triangle in
column-major order with %.17g; read `array real` files, `symmetric` or `general` (the latter
symmetrised (M + M^T)/2 like SymmetricMatrix::from_dense, symmetric_matrix.cpp:29-43)."""
from __future__ import annotations

import numpy as np


class IoError(RuntimeError):
    """The reference's IoError (symmetric_matrix.hpp)."""


def write_matrix_market(M: np.ndarray, path: str) -> None:
    M = np.asarray(M, dtype=np.float64)
    n = M.shape[0]
    if M.shape != (n, n):
        raise ValueError("write_matrix_market: square matrix required")
    try:
        with open(path, "w") as f:
            f.write("%%MatrixMarket matrix array real symmetric\n")
            f.write(f"{n} {n}\n")
            lower = M.T[np.triu_indices(n)]  # column j, rows i >= j  ==  (M^T)[j, i] for i >= j
            f.write("\n".join("%.17g" % v for v in lower))
            f.write("\n")
    except OSError as e:
        raise IoError(f"cannot open for writing: {path}") from e


def read_matrix_market(path: str) -> np.ndarray:
    try:
        with open(path) as f:
            header = f.readline()
            if not header:
                raise IoError(f"empty file: {path}")
            tok = header.split()
            if len(tok) < 5 or tok[0] != "%%MatrixMarket" or tok[1].lower() != "matrix" or \
                    tok[2].lower() != "array" or tok[3].lower() != "real":
                raise IoError(f"unsupported Matrix Market header: {header.rstrip()}")
            sym = tok[4].lower()
            if sym not in ("symmetric", "general"):
                raise IoError(f"unsupported Matrix Market symmetry: {tok[4]}")
            line = f.readline()
            while line and line.startswith("%"):
                line = f.readline()
            dims = line.split()
            if len(dims) < 2 or int(dims[0]) <= 0 or int(dims[0]) != int(dims[1]):
                raise IoError(f"Matrix Market size line must be a square N N: {path}")
            n = int(dims[0])
            vals = np.array(f.read().split(), dtype=np.float64)
    except OSError as e:
        raise IoError(f"cannot open: {path}") from e
    if sym == "symmetric":
        if vals.size < n * (n + 1) // 2:
            raise IoError(f"truncated Matrix Market data: {path}")
        M = np.zeros((n, n))
        iu = np.triu_indices(n)
        M.T[iu] = vals[: n * (n + 1) // 2]   # lower triangle, column-major
        M = M + np.tril(M, -1).T
        return M
    if vals.size < n * n:
        raise IoError(f"truncated Matrix Market data: {path}")
    full = vals[: n * n].reshape(n, n).T     # column-major
    return 0.5 * (full + full.T)
