"""CPU tests of the workflow layer: the entropy oracle pinned to the compiled
reference, and the host-side model selection (SPEC select_model examples)."""
import json
import os

import numpy as np
import pytest

from oracle import oracle as O
from paper_2605_08523_b200 import engine as E
from paper_2605_08523_b200 import workflow as W
from paper_2605_08523_b200.hamiltonians import tight_binding


@pytest.mark.parametrize("name", ["E40", "E1500"])
def test_entropy_oracle_matches_reference_scalar(name):
    """oracle.entropy_scalar (evaluate_entropy restated, scalar_models.cpp:320-326) equals the
    reference's own evaluate_model on the golden grid, and the trained model meets its
    reported max error against the exact fermi_entropy on [0, 1]."""
    e = O.load_entropy_coefficients(name)
    with open(os.path.join(O.GOLDEN, f"scalar_{name}.json")) as f:
        g = json.load(f)
    x = np.array([float(v) for v in g["x"]])
    ref = np.array([float(v) for v in g["evaluate_model"]])
    ex = np.array([float(v) for v in g["fermi_entropy"]])
    mine = O.entropy_scalar(e["abcd"], e["alpha"], float(e["mu0"]), x)
    assert np.abs(mine - ref).max() <= 1e-14
    inside = (x >= 0) & (x <= 1)
    assert np.abs(ref[inside] - ex[inside]).max() <= 1.05 * e["report"]["final_max_error"] + 1e-12


def test_entropy_trace_recursion_equals_spectral_mapping():
    """Tr S by the fp64 matrix recursion equals sum_i s_model(x_i) over the eigenvalues
    (SPEC.md:365-366 spectral property lifted to the entropy model)."""
    e = O.load_entropy_coefficients("E1500")
    H = tight_binding(64, seed=5)
    mu, kT = 0.1, 0.01
    tr = O.entropy_trace_f64(H, mu, kT, e["abcd"], e["alpha"], float(e["beta0"]), float(e["mu0"]))
    lam = np.linalg.eigvalsh(H)
    x = float(e["mu0"]) + (1.0 / kT) / float(e["beta0"]) * (lam - mu)
    spec = float(np.sum(O.entropy_scalar(e["abcd"], e["alpha"], float(e["mu0"]), x)))
    assert abs(tr - spec) <= 1e-10
    assert abs(tr - O.entropy_trace_exact(H, mu, kT)) <= 64 * 2e-6


def test_select_model_spec_examples():
    """fewest layers among valid models; the 1500 model alone at (900, 0.5);
    no valid model at (2000, 0.5), naming the beta0 needed."""
    lib = W.ModelLibrary.default()
    assert W.select_model(lib, 20.0, 0.3).beta0 == 40.0
    assert W.select_model(lib, 900.0, 0.5).beta0 == 1500.0
    with pytest.raises(W.NoValidModelError, match="beta0 >= 3000"):
        W.select_model(lib, 2000.0, 0.5)
    with pytest.raises(E.ValidationError):
        W.select_model(W.ModelLibrary(), 1.0, 0.5)


def test_library_pairs_entropy_models_by_trained_at():
    lib = W.ModelLibrary.default()
    for m in lib.models:
        em = lib.entropy_for(m)
        assert (em.beta0, em.mu0) == (m.beta0, m.mu0)
        assert 0.5 <= em.alpha <= 0.98


def test_model_file_schema_version_checked_and_round_trips(tmp_path):
    """schema_version checked on load; 17-significant-digit decimals round-trip
    the coefficients bit-exactly; a created timestamp is written."""
    import json
    from paper_2605_08523_b200 import engine as E
    m = E.load_model("M40")
    assert m.meta["schema_version"] == E.MODEL_SCHEMA_VERSION and "created" in m.meta
    p = tmp_path / "m.json"
    m.to_json(str(p))
    m2 = E.Mlsp2Model.from_json(str(p))
    assert np.array_equal(m2.abcd, m.abcd) and m2.beta0 == m.beta0 and m2.mu0 == m.mu0
    d = json.loads(p.read_text())
    for bad in (None, 2):
        d2 = dict(d)
        if bad is None:
            d2.pop("schema_version")
        else:
            d2["schema_version"] = bad
        q = tmp_path / f"bad{bad}.json"
        q.write_text(json.dumps(d2))
        with pytest.raises(E.ValidationError, match="schema_version"):
            E.Mlsp2Model.from_json(str(q))
