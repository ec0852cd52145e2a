"""Edge cases through the C ABI on the GPU: rectangular matrices, empty and
very long rows, a single row/column, odd sizes for the paired/bulk-copied
vector kernels, and solves too small to give every SM a slice — each against
the oracle (bit-exact SpMV/conversions/features, +-1 iteration solves)."""
import numpy as np
import pytest

import oracle as O
import paper_2411_10143_b200 as P

pytestmark = pytest.mark.gpu
ATOMIC = P.SpmvConfig.from_token("COO/LibB")


def _csr_from_dense(d):
    r, c = np.nonzero(d)
    n, m = d.shape
    ptr = np.zeros(n + 1, np.int64)
    np.cumsum(np.bincount(r, minlength=n), out=ptr[1:])
    return n, m, ptr, c.astype(np.int64), d[r, c].astype(np.float64)


def _check_all_configs(n, m, ptr, cols, vals, seed=0):
    A = P.CsrMatrix(n, m, ptr, cols, vals)
    oc = O.OCsr(n, m, ptr, cols, vals)
    x = np.random.default_rng(seed).uniform(-1, 1, m)
    assert P.extract_features(A).to_array().tolist() == O.features(oc)
    for cfg in P.enumerate_configs():
        try:
            want_rep = O.convert(oc, cfg.format.value) if cfg.format.value != "CSR" else oc
        except O.OracleInapplicable:
            with pytest.raises(P.FormatInapplicableError):
                P.convert(A, cfg.format)
            continue
        rep = A if cfg.format is P.FormatTag.CSR else P.convert(A, cfg.format)
        got = P.execute_spmv(cfg, rep, x, workers=4)
        if cfg == ATOMIC:
            want = O.spmv_sequential(oc, x)
            assert np.linalg.norm(got - want) <= 1e-12 * max(1.0, np.linalg.norm(want))
        else:
            assert np.array_equal(got, O.spmv(cfg.token(), want_rep, x, workers=4)), cfg.token()


@pytest.mark.parametrize("shape", [(1, 1), (1, 7), (7, 1), (5, 300), (300, 5), (1001, 999)])
def test_rectangular_and_degenerate_shapes(shape):
    rng = np.random.default_rng(sum(shape))
    d = (rng.random(shape) < 0.3) * rng.uniform(-1, 1, shape)
    d[0, 0] = 2.0                               # at least one entry
    _check_all_configs(*_csr_from_dense(d))


def test_empty_rows_and_one_very_long_row():
    n = 4000
    rng = np.random.default_rng(3)
    d = np.zeros((n, n))
    d[np.arange(0, n, 3), np.arange(0, n, 3)] = 1.0          # two of three rows empty... diagonal only
    d[17, :] = rng.uniform(-1, 1, n)                         # one row with n entries
    d[n - 1, rng.choice(n, 300, replace=False)] = 1.5
    _check_all_configs(*_csr_from_dense(d))


@pytest.mark.parametrize("n", [1, 2, 3, 37, 1001])
def test_tiny_and_odd_solves(n):
    """GMRES and CG on SPD tridiagonal systems of sizes below the SM count
    and odd sizes (paired vector loads, bulk-copy tails)."""
    main, off = 4.0 * np.ones(n), -1.0 * np.ones(n - 1)
    d = np.diag(main) + np.diag(off, 1) + np.diag(off, -1)
    n_, m, ptr, cols, vals = _csr_from_dense(d)
    A = P.CsrMatrix(n_, m, ptr, cols, vals)
    oc = O.OCsr(n_, m, ptr, cols, vals)
    b = O.spmv_sequential(oc, np.ones(n))
    mv = lambda v: O.spmv("CSR/LibB", oc, v)   # noqa: E731
    params = P.GmresParams(restart_m=30, tol=1e-10, max_iters=500)
    for cfg in ("CSR/LibA/32", "DIA/LibA"):
        g = P.gmres_solve(A, None, params, initial_config=P.SpmvConfig.from_token(cfg))
        c = P.cg_solve(A, None, params, initial_config=P.SpmvConfig.from_token(cfg))
        rg = O.gmres(mv, b, restart=30, tol=1e-10, max_iters=500)
        rc = O.cg(mv, b, tol=1e-10, max_iters=500)
        assert g.converged and abs(g.iterations - rg["iterations"]) <= 1, (cfg, g.iterations, rg["iterations"])
        assert c.converged and abs(c.iterations - rc["iterations"]) <= 1, (cfg, c.iterations, rc["iterations"])
        assert np.allclose(g.solution, np.ones(n), atol=1e-8)
        assert np.allclose(c.solution, np.ones(n), atol=1e-8)
