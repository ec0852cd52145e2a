"""Pin the CPU oracle against the reference's own outputs (golden fixtures).

These run on CPU (no GPU marker): before the oracle is trusted as the
checker for the CUDA path, it must reproduce the reference bit-for-bit on
every golden case.
"""
import math

import numpy as np
import pytest

import oracle as O
from golden_io import (case, case_names, cascade_doc, model_docs, solves,
                       spmv_keys)


def coo_of(c):
    return O.OCoo(int(c["nrows"]), int(c["ncols"]), c["coo_rows"].astype(np.int64),
                  c["coo_cols"].astype(np.int64), c["coo_vals"])


@pytest.mark.parametrize("name", case_names())
def test_conversions_bit_exact(name):
    c = case(name)
    coo = coo_of(c)
    csr = O.coo_to_csr(coo)
    assert np.array_equal(csr.ptr, c["csr_ptr"])
    ell = O.coo_to_ell(coo)
    assert ell.width == int(c["ell_width"])
    assert np.array_equal(ell.cols.T, c["ell_cols"])
    assert np.array_equal(ell.vals.T, c["ell_vals"])
    if int(c["dia_ok"]):
        dia = O.coo_to_dia(coo)
        assert np.array_equal(dia.offsets, c["dia_offsets"])
        assert np.array_equal(dia.data, c["dia_data"])
    else:
        with pytest.raises(O.OracleInapplicable):
            O.coo_to_dia(coo)
    hyb = O.coo_to_hyb(coo)
    assert hyb.width == int(c["hyb_width"])
    assert np.array_equal(hyb.ell.cols.T, c["hyb_ell_cols"])
    assert np.array_equal(hyb.ell.vals.T, c["hyb_ell_vals"])
    assert np.array_equal(hyb.spill.rows, c["hyb_spill_rows"])
    assert np.array_equal(hyb.spill.cols, c["hyb_spill_cols"])
    assert np.array_equal(hyb.spill.vals, c["hyb_spill_vals"])
    # round trips through the COO hub (formats.py:281-299)
    for m in (csr, ell, hyb) + ((O.coo_to_dia(coo),) if int(c["dia_ok"]) else ()):
        back = O.to_coo(m)
        if isinstance(m, O.ODia):   # DIA drops stored zeros only
            keep = coo.vals != 0.0
            assert np.array_equal(back.rows, coo.rows[keep])
            continue
        assert np.array_equal(back.rows, coo.rows)
        assert np.array_equal(back.cols, coo.cols)
        assert np.array_equal(back.vals, coo.vals)


@pytest.mark.parametrize("name", case_names())
def test_spmv_bit_exact(name):
    c = case(name)
    coo = coo_of(c)
    reps = {"COO": coo, "CSR": O.coo_to_csr(coo), "ELL": O.coo_to_ell(coo),
            "HYB": O.coo_to_hyb(coo)}
    if int(c["dia_ok"]):
        reps["DIA"] = O.coo_to_dia(coo)
    assert np.array_equal(O.spmv_sequential(reps["CSR"], c["x"]), c["y_reference"])
    for tok, w in spmv_keys(c):
        got = O.spmv(tok, reps[tok.split("/")[0]], c["x"], workers=w)
        assert np.array_equal(got, c[f"y|{tok}|{w}"]), (tok, w)
    # the nondeterministic atomic kernel: the reference's 1e-8 bar
    got = O.spmv("COO/LibB", coo, c["x"])
    ref = c["y_reference"]
    scale = np.linalg.norm(ref) or 1.0
    assert np.linalg.norm(got - ref) / scale <= 1e-8


@pytest.mark.parametrize("name", case_names())
def test_features_bit_exact(name):
    c = case(name)
    csr = O.coo_to_csr(coo_of(c))
    got = O.features(csr)
    want = c["features"]
    assert [float(v) for v in got] == [float(v) for v in want]


def test_pairwise_restatement_matches_numpy():
    rng = np.random.default_rng(9)
    for n in list(range(1, 260)) + [513, 1031, 4099]:
        a = rng.standard_normal(n) * 10.0 ** rng.uniform(-3, 3)
        assert O.segment_sum(a, 0, n) == np.add.reduceat(a, [0])[0], n


def test_model_file_parity():
    """Replaces the reference's missing heldout_predictions.json check
    (test_acceptance.py:199-210): >= 5000 rows, 100 % agreement."""
    doc = cascade_doc()
    docs = model_docs()
    total = 0
    for name, data in doc["models"].items():
        for row, lab, sc in zip(data["rows"], data["labels"], data["scores"]):
            got, scores = O.tree_predict(docs[name], row)
            assert got == lab
            assert scores == sc
            total += 1
    assert total >= 5000


def test_cascade_decisions():
    doc = cascade_doc()
    docs = model_docs()
    for entry in doc["cascade"]:
        assert O.cascade(docs, entry["row"]) == entry["decisions"]
        assert entry["decisions"][-1] == entry["final"]


@pytest.mark.parametrize("name", sorted(solves()))
def test_gmres_matches_reference(name):
    s = solves()[name]
    c = case(s["matrix"])
    csr = O.coo_to_csr(coo_of(c))
    n = csr.nrows
    if s["rhs"] == "ones":
        b = O.spmv_sequential(csr, np.ones(n))
    else:
        b = np.random.default_rng(s["seed"]).standard_normal(n)
    res = O.gmres(lambda v: O.spmv("CSR/LibB", csr, v), b, restart=s["restart"],
                  tol=s["tol"], max_iters=s["max_iters"])
    assert res["iterations"] == s["iterations"]
    assert res["converged"] == s["converged"]
    # same BLAS thread count as the generator -> identical arithmetic
    assert res["history"] == s["history"]
    assert np.array_equal(res["x"], np.asarray(s["solution"]))


def test_cg_against_scipy_iteration_count():
    """The CG oracle is new (no reference CG): cross-check its iteration
    count with scipy's independent implementation on config-1 structure."""
    scipy_sparse = pytest.importorskip("scipy.sparse")
    from scipy.sparse.linalg import cg as scipy_cg
    from paper_2411_10143_b200 import generators as G
    n, _, ptr, cols, vals = G.poisson2d(40)
    csr = O.OCsr(n, n, ptr, cols, vals)
    b = O.spmv_sequential(csr, np.ones(n))
    res = O.cg(lambda v: O.spmv("CSR/LibB", csr, v), b, tol=1e-8, max_iters=5000)
    assert res["converged"]
    A = scipy_sparse.csr_matrix((vals, cols, ptr), shape=(n, n))
    it = [0]
    scipy_cg(A, b, rtol=1e-8, maxiter=5000, callback=lambda xk: it.__setitem__(0, it[0] + 1))
    assert abs(res["iterations"] - it[0]) <= 1
    assert np.linalg.norm(res["x"] - 1.0) / math.sqrt(n) < 1e-6
