"""Matrix Market I/O in the reference's format and the CLI surface."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

from paper_2605_08523_b200 import cli
from paper_2605_08523_b200.hamiltonians import tight_binding
from paper_2605_08523_b200.mm import IoError, read_matrix_market, write_matrix_market

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_matrix_market_format_and_round_trip(tmp_path):
    """write: banner, `N N`, lower triangle column-major, %.17g (symmetric_matrix.cpp:120-138);
    read returns the exact matrix."""
    M = np.array([[1.0, 0.1, 1 / 3], [0.1, 2.0, -0.5], [1 / 3, -0.5, 3.0]])
    p = tmp_path / "m.mtx"
    write_matrix_market(M, str(p))
    lines = p.read_text().splitlines()
    assert lines[0] == "%%MatrixMarket matrix array real symmetric" and lines[1] == "3 3"
    assert lines[2:] == ["%.17g" % v for v in (1.0, 0.1, 1 / 3, 2.0, -0.5, 3.0)]
    assert np.array_equal(read_matrix_market(str(p)), M)
    H = tight_binding(64, seed=2)
    write_matrix_market(H, str(p))
    assert np.array_equal(read_matrix_market(str(p)), H)


def test_matrix_market_general_and_errors(tmp_path):
    """`general` arrays are symmetrised like SymmetricMatrix::from_dense; bad headers, sizes
    and truncation raise IoError (symmetric_matrix.cpp:140-189)."""
    p = tmp_path / "g.mtx"
    p.write_text("%%MatrixMarket matrix array real general\n% comment\n2 2\n1\n2\n4\n3\n")
    assert np.array_equal(read_matrix_market(str(p)), np.array([[1.0, 3.0], [3.0, 3.0]]))
    for body in ("%%MatrixMarket matrix coordinate real symmetric\n2 2\n",
                 "%%MatrixMarket matrix array complex symmetric\n2 2\n",
                 "%%MatrixMarket matrix array real symmetric\n2 3\n1\n2\n3\n",
                 "%%MatrixMarket matrix array real symmetric\n3 3\n1\n2\n"):
        p.write_text(body)
        with pytest.raises(IoError):
            read_matrix_market(str(p))
    with pytest.raises(IoError):
        read_matrix_market(str(tmp_path / "missing.mtx"))


def test_cli_info_and_exit_codes(capsys):
    assert cli.main(["info", "--model", "M40"]) == 0
    info = json.loads(capsys.readouterr().out)
    assert info["beta0"] == 40.0 and info["mu0"] == 0.3 and info["layers"] == 14
    assert cli.main(["info", "--model", "no-such-model"]) == cli.EX_IOERR
    assert cli.main(["frobnicate"]) == cli.EX_USAGE
    assert cli.main(["apply", "--hamiltonian", "/nonexistent.mtx", "--kT", "0.01"]) == cli.EX_IOERR


@pytest.mark.gpu
def test_cli_apply_and_solve_mu(tmp_path):
    """apply writes D (bitwise the engine's result) and provenance; out of region -> exit 3;
    solve-mu on the two-level system converges to mu = 0.5."""
    from paper_2605_08523_b200 import engine as E
    H = tight_binding(256, seed=1234)
    hp, dp = tmp_path / "H.mtx", tmp_path / "D.mtx"
    write_matrix_market(H, str(hp))
    r = subprocess.run([sys.executable, "-m", "paper_2605_08523_b200", "apply", "--model", "M1500",
                        "--hamiltonian", str(hp), "--kT", "0.01", "--mu", "0", "--out", str(dp)],
                       capture_output=True, text=True, cwd=ROOT, timeout=300)
    assert r.returncode == 0, r.stderr
    prov = json.loads(r.stdout.splitlines()[-1])
    assert prov["model"]["beta0"] == 1500.0 and prov["half_products"] == 100
    D, _, _ = E.compute_density_matrix(read_matrix_market(str(hp)), 0.0, 0.01, E.load_model("M1500"))
    assert np.array_equal(read_matrix_market(str(dp)), D)
    r = subprocess.run([sys.executable, "-m", "paper_2605_08523_b200", "apply", "--model", "M1500",
                        "--hamiltonian", str(hp), "--kT", "0.0005"], capture_output=True, text=True,
                       cwd=ROOT, timeout=300)
    assert r.returncode == 3 and "violated" in r.stderr
    two = tmp_path / "two.mtx"
    write_matrix_market(np.diag([0.0, 1.0]), str(two))
    r = subprocess.run([sys.executable, "-m", "paper_2605_08523_b200", "solve-mu", "--hamiltonian", str(two),
                        "--beta", "10", "--nocc", "1", "--mu", "0.4"], capture_output=True, text=True,
                       cwd=ROOT, timeout=300)
    assert r.returncode == 0, r.stderr
    res = json.loads(r.stdout.splitlines()[-1])
    assert res["converged"] and abs(res["mu"] - 0.5) <= 2e-5
    r = subprocess.run([sys.executable, "-m", "paper_2605_08523_b200", "solve-mu", "--hamiltonian", str(two),
                        "--beta", "10", "--nocc", "2"], capture_output=True, text=True, cwd=ROOT, timeout=300)
    assert r.returncode == 64


@pytest.mark.gpu
def test_cli_double_precision(tmp_path):
    """SPEC.md:630 / :660: `apply --precision double` writes the DOUBLE-mode D (bitwise the engine's)
    with n squarings in the provenance; `bench --precision double` reports matmul count = layers."""
    from paper_2605_08523_b200 import engine as E
    H = tight_binding(128, seed=77)
    hp, dp = tmp_path / "H.mtx", tmp_path / "D.mtx"
    write_matrix_market(H, str(hp))
    r = subprocess.run([sys.executable, "-m", "paper_2605_08523_b200", "apply", "--model", "M1500",
                        "--hamiltonian", str(hp), "--kT", "0.01", "--mu", "0", "--precision", "double",
                        "--out", str(dp)], capture_output=True, text=True, cwd=ROOT, timeout=300)
    assert r.returncode == 0, r.stderr
    prov = json.loads(r.stdout.splitlines()[-1])
    assert prov["precision"] == "double" and prov["half_products"] == 30
    D, _, _ = E.compute_density_matrix(read_matrix_market(str(hp)), 0.0, 0.01, E.load_model("M1500"),
                                       E.PrecisionMode.DOUBLE)
    assert np.array_equal(read_matrix_market(str(dp)), D)
    r = subprocess.run([sys.executable, "-m", "paper_2605_08523_b200", "bench", "--sizes", "128,256",
                        "--precision", "double"], capture_output=True, text=True, cwd=ROOT, timeout=300)
    assert r.returncode == 0, r.stderr
    rows = [l.split() for l in r.stdout.splitlines() if l.strip() and l.split()[0] in ("128", "256")]
    assert len(rows) == 2 and all(row[1] == "double" and int(row[4]) == 30 for row in rows), r.stdout
