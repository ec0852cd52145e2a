"""GPU parity for the Krylov solvers and the async predict-while-solve
runtime, against the reference's GMRES reports (golden) and the CPU oracle
(CG).  Mirrors the reference's test_solver.py contract."""
import numpy as np
import pytest

import oracle as O
from golden_io import case, solves

import paper_2411_10143_b200 as P
from paper_2411_10143_b200 import generators as G
from paper_2411_10143_b200.solver import ADVISOR_CANCELLED, ADVISOR_COMPLETED, ADVISOR_UNUSED
from paper_2411_10143_b200.inference import model_from_dict

pytestmark = pytest.mark.gpu

FORMAT_CLASSES = ["COO", "CSR", "ELL", "DIA", "HYB"]


def stub_model(classes, forced):
    trees = [[{"score": 1.0 if c == forced else 0.0}] for c in classes]
    return model_from_dict({"schema_version": 1, "feature_names": list(P.FEATURE_NAMES),
                            "classes": classes, "trees": trees})


def stub_cascade(fmt="COO", coo_lib="LibA", csr_lib="LibA", ell_lib="LibA", tpv="32"):
    return P.CascadeModelSet(
        format_model=stub_model(FORMAT_CLASSES, fmt),
        coo_lib_model=stub_model(["LibA", "LibB"], coo_lib),
        csr_lib_model=stub_model(["LibA", "LibB", "LibC"], csr_lib),
        ell_lib_model=stub_model(["LibA", "LibC"], ell_lib),
        csr_tpv_model=stub_model(["2", "4", "8", "16", "32"], tpv))


def coo_of(c):
    return P.CooMatrix(int(c["nrows"]), int(c["ncols"]), c["coo_rows"], c["coo_cols"], c["coo_vals"])


def poisson_system(nx=10):
    n, _, ptr, cols, vals = G.poisson2d(nx)
    A = P.CsrMatrix(n, n, ptr, cols, vals)
    return P.to_coo(A), O.spmv_sequential(O.OCsr(n, n, ptr, cols, vals), np.ones(n))


def forced(max_iters=200):
    return P.GmresParams(restart_m=30, tol=1e-300, max_iters=max_iters)


@pytest.mark.parametrize("name", sorted(solves()))
def test_gmres_matches_reference_reports(name):
    s = solves()[name]
    A = coo_of(case(s["matrix"]))
    params = P.GmresParams(restart_m=s["restart"], tol=s["tol"], max_iters=s["max_iters"],
                           rhs=s["rhs"], seed=s["seed"])
    for cfg in (P.DEFAULT_CONFIG, P.SpmvConfig(P.FormatTag.CSR, P.Library.LIB_B),
                P.SpmvConfig(P.FormatTag.CSR, P.Library.LIB_A, 32)):
        rep = P.gmres_solve(A, None, params, executor=P.SpmvExecutor.for_matrix(A, cfg))
        assert rep.converged == s["converged"]
        assert abs(rep.iterations - s["iterations"]) <= 1, (cfg.token(), rep.iterations)
        if s["converged"]:
            assert rep.final_residual <= s["tol"]
        sol = np.asarray(s["solution"])
        assert np.linalg.norm(rep.solution - sol) <= 1e-6 * max(np.linalg.norm(sol), 1.0)
        # early estimates agree tightly; late ones (near tol, after restarts)
        # only to the dot-product rounding the BLAS vs device order allows
        k = min(len(rep.residual_history), len(s["history"]), 10)
        np.testing.assert_allclose(rep.residual_history[:k], s["history"][:k], rtol=1e-8)
        k = min(len(rep.residual_history), len(s["history"]))
        np.testing.assert_allclose(rep.residual_history[:k], s["history"][:k], rtol=0.5,
                                   atol=1e-14)


def test_poisson_pinned_iterations_exact():
    A, b = poisson_system()
    rep = P.gmres_solve(A, b, P.GmresParams(restart_m=30, tol=1e-8, max_iters=1000))
    assert rep.converged and rep.iterations == 15   # reference test_solver.py:21
    dense = np.zeros((100, 100))
    dense[A.rows, A.cols] = A.values
    assert np.max(np.abs(rep.solution - np.linalg.solve(dense, b))) <= 1e-6


@pytest.mark.parametrize("gen,tol", [("poisson", 1e-8), ("powerlaw", 1e-8), ("laplace27", 1e-8)])
def test_cg_against_oracle(gen, tol):
    n, _, ptr, cols, vals = {"poisson": lambda: G.poisson2d(64),
                             "powerlaw": lambda: G.powerlaw_spd(20000, seed=1),
                             "laplace27": lambda: G.laplace27(16)}[gen]()
    A = P.CsrMatrix(n, n, ptr, cols, vals)
    ocsr = O.OCsr(n, n, ptr, cols, vals)
    rhs = "random" if gen == "powerlaw" else "ones"
    params = P.GmresParams(tol=tol, max_iters=5000, rhs=rhs)
    b = (np.random.default_rng(0).standard_normal(n) if rhs == "random"
         else O.spmv_sequential(ocsr, np.ones(n)))
    want = O.cg(lambda v: O.spmv("CSR/LibB", ocsr, v), b, tol=tol, max_iters=5000)
    for cfg in (P.SpmvConfig(P.FormatTag.CSR, P.Library.LIB_B), P.GPU_DEFAULT_CONFIG):
        rep = P.cg_solve(A, None, params, initial_config=cfg)
        assert rep.converged and want["converged"]
        assert abs(rep.iterations - want["iterations"]) <= 1, (rep.iterations, want["iterations"])
        assert rep.final_residual <= tol
        assert np.linalg.norm(rep.solution - want["x"]) <= 1e-6 * np.linalg.norm(want["x"])


class TestGmresContract:
    def test_identity_one_iteration(self):
        A = P.CooMatrix(3, 3, np.arange(3), np.arange(3), np.ones(3))
        rep = P.gmres_solve(A, np.array([1.0, 2.0, 3.0]), P.GmresParams(tol=1e-8))
        assert rep.converged and rep.iterations == 1
        assert np.allclose(rep.solution, [1.0, 2.0, 3.0], atol=1e-12)

    def test_max_iters_zero(self):
        A, b = poisson_system()
        rep = P.gmres_solve(A, b, P.GmresParams(max_iters=0))
        assert not rep.converged and rep.iterations == 0 and rep.residual_history == []
        assert len(rep.config_timeline) == 1

    def test_zero_rhs(self):
        A, _ = poisson_system()
        rep = P.gmres_solve(A, np.zeros(100))
        assert rep.converged and rep.iterations == 0 and np.all(rep.solution == 0.0)

    def test_history_length(self):
        A, b = poisson_system()
        rep = P.gmres_solve(A, b, forced(50))
        assert len(rep.residual_history) == 50 and rep.iterations == 50

    def test_small_restart(self):
        A, b = poisson_system()
        rep = P.gmres_solve(A, b, P.GmresParams(restart_m=5, tol=1e-8, max_iters=2000))
        assert rep.converged

    def test_breakdown_met(self):
        A = P.CooMatrix(3, 3, np.arange(3), np.arange(3), np.ones(3))
        rep = P.gmres_solve(A, np.array([1.0, 0.0, 0.0]))
        assert rep.converged and rep.iterations == 1

    def test_breakdown_stagnation(self):
        A = P.CooMatrix(3, 3, [], [], [])
        with pytest.raises(P.StagnationError, match="breakdown"):
            P.gmres_solve(A, np.ones(3))

    def test_nan_executor(self):
        A = P.CooMatrix(2, 2, np.arange(2), np.arange(2), np.ones(2))

        class Broken(P.SpmvExecutor):
            def matvec(self, x):
                return np.full(2, np.nan)

        with pytest.raises(P.SolverNumericalError, match="non-finite"):
            P.gmres_solve(A, np.ones(2), executor=Broken(P.DEFAULT_CONFIG, A))

    def test_custom_executor_plugin_runs(self):
        A, b = poisson_system()

        class Counting(P.SpmvExecutor):
            calls = 0

            def matvec(self, x):
                Counting.calls += 1
                return super().matvec(x)

        rep = P.gmres_solve(A, b, P.GmresParams(tol=1e-8), executor=Counting(P.DEFAULT_CONFIG, A))
        assert rep.converged and rep.iterations == 15 and Counting.calls >= 16

    def test_executor_choice_same_solution(self):
        A, b = poisson_system()
        base = P.gmres_solve(A, b, P.GmresParams(tol=1e-8))
        for cfg in (P.SpmvConfig(P.FormatTag.DIA, P.Library.LIB_A),
                    P.SpmvConfig(P.FormatTag.CSR, P.Library.LIB_A, 8),
                    P.SpmvConfig(P.FormatTag.CSR, P.Library.LIB_C)):
            other = P.gmres_solve(A, b, P.GmresParams(tol=1e-8),
                                  executor=P.SpmvExecutor.for_matrix(A, cfg))
            assert other.converged
            assert np.linalg.norm(other.solution - base.solution) <= 1e-6 * np.linalg.norm(base.solution)

    def test_square_required(self):
        A = P.CooMatrix(2, 3, [0, 0, 0, 1, 1, 1], [0, 1, 2, 0, 1, 2], np.ones(6))
        with pytest.raises(ValueError, match="square"):
            P.gmres_solve(A, np.ones(2))


class TestAsync:
    def test_two_stage_swaps(self):
        A, b = poisson_system()
        rep = P.async_solve(A, b, forced(), stub_cascade(fmt="ELL", ell_lib="LibC"),
                            delay_injection=[3, 7])
        assert [s.iteration for s in rep.config_timeline] == [1, 4, 8]
        assert rep.config_timeline[1].config == P.SpmvConfig(P.FormatTag.ELL, P.Library.LIB_A)
        assert rep.config_timeline[2].config == P.SpmvConfig(P.FormatTag.ELL, P.Library.LIB_C)
        assert rep.advisor_outcome == ADVISOR_COMPLETED

    @pytest.mark.parametrize("delay,expected", [(0, 2), (3, 4), (7, 8)])
    def test_single_delay(self, delay, expected):
        A, b = poisson_system()
        rep = P.async_solve(A, b, forced(), stub_cascade(fmt="DIA"), delay_injection=[delay])
        assert [s.iteration for s in rep.config_timeline] == [1, expected]
        sync = P.gmres_solve(A, b, forced(), executor=P.SpmvExecutor.for_matrix(
            A, P.SpmvConfig(P.FormatTag.DIA, P.Library.LIB_A)))
        assert np.linalg.norm(rep.solution - sync.solution) <= 1e-6 * np.linalg.norm(sync.solution)

    def test_boundary_only_swaps(self):
        A, b = poisson_system()
        log = []
        rep = P.async_solve(A, b, forced(40), stub_cascade(fmt="ELL", ell_lib="LibC"),
                            delay_injection=[3, 7], matvec_probe=lambda it, c: log.append((it, c.token())))
        per = {}
        for it, tok in log:
            per.setdefault(it, set()).add(tok)
        for it, toks in per.items():
            assert len(toks) == 1
            active = [s.config.token() for s in rep.config_timeline if s.iteration <= it][-1]
            assert toks == {active}

    def test_converged_async_agrees(self):
        A, b = poisson_system()
        params = P.GmresParams(restart_m=30, tol=1e-8, max_iters=1000)
        rep = P.async_solve(A, b, params, stub_cascade(fmt="DIA"), delay_injection=[2])
        assert rep.converged and rep.final_residual <= 1e-8

    def test_cancellation_liveness(self):
        n = 120_000
        A = P.CooMatrix(n, n, np.arange(n), np.arange(n), np.ones(n))
        rep = P.async_solve(A, np.ones(n), P.GmresParams(tol=1e-6), stub_cascade(fmt="DIA"))
        assert rep.converged and rep.iterations <= 2
        assert len(rep.config_timeline) == 1
        assert rep.advisor_outcome in (ADVISOR_CANCELLED, ADVISOR_UNUSED)
        assert rep.advisor_join_seconds <= 0.25

    def test_advisor_failure_swallowed(self):
        n = 5000
        rng = np.random.default_rng(2)
        rows = np.concatenate([np.arange(n), np.arange(n - 1), np.arange(1, n),
                               np.zeros(n - 1, dtype=np.int64)])
        cols = np.concatenate([np.arange(n), np.arange(1, n), np.arange(n - 1), np.arange(1, n)])
        vals = np.concatenate([rng.uniform(4.0, 5.0, n), rng.uniform(0.5, 1.5, 2 * (n - 1)),
                               rng.uniform(0.1, 0.2, n - 1)])
        A = P.CooMatrix.from_triplets(n, n, rows, cols, vals, sum_duplicates=True)
        rep = P.async_solve(A, None, forced(30), stub_cascade(fmt="DIA"), delay_injection=[0])
        assert rep.iterations == 30 and len(rep.config_timeline) == 1
        assert rep.advisor_error is not None and "inapplicable" in rep.advisor_error

    def test_models_required(self):
        A, b = poisson_system()
        with pytest.raises(ValueError, match="CascadeModelSet"):
            P.async_solve(A, b, P.GmresParams())

    def test_async_cg_swaps(self):
        n, _, ptr, cols, vals = G.poisson2d(64)
        A = P.CsrMatrix(n, n, ptr, cols, vals)
        rep = P.async_solve(A, None, P.GmresParams(tol=1e-8, max_iters=2000), stub_cascade(fmt="DIA"),
                            method="cg", initial_config=P.GPU_DEFAULT_CONFIG, delay_injection=[3])
        assert rep.converged and [s.iteration for s in rep.config_timeline] == [1, 4]


class TestSequential:
    def test_phases(self):
        A, b = poisson_system()
        rep = P.sequential_predict_solve(A, b, P.GmresParams(tol=1e-8), stub_cascade(fmt="HYB"))
        assert set(rep.phases) == {"features", "inference", "conversion", "solve"}
        assert sum(rep.phases.values()) <= rep.wall_seconds
        assert rep.wall_seconds - sum(rep.phases.values()) <= 0.05
        assert rep.config_timeline[0].config == P.SpmvConfig(P.FormatTag.HYB, P.Library.LIB_A)

    def test_identity_matches_async(self):
        A = P.CooMatrix(3, 3, np.arange(3), np.arange(3), np.ones(3))
        b = np.array([1.0, 2.0, 3.0])
        seq = P.sequential_predict_solve(A, b, P.GmresParams(tol=1e-8), stub_cascade(fmt="DIA"))
        asy = P.async_solve(A, b, P.GmresParams(tol=1e-8), stub_cascade(fmt="DIA"))
        assert np.allclose(seq.solution, asy.solution, atol=1e-9)


def test_time_config_and_compare():
    n, _, ptr, cols, vals = G.poisson2d(8)
    A = P.to_coo(P.CsrMatrix(n, n, ptr, cols, vals))
    for cfg in P.enumerate_configs():
        t = P.time_config(A, cfg, runs=2, warmups=1)
        assert t is not None and t > 0
    rec = P.time_all_configs(A, "p8", runs=2, warmups=1)
    assert set(rec.times) == {c.token() for c in P.enumerate_configs()}
    E = P.CooMatrix(4, 4, np.arange(4), np.arange(4), np.ones(4))
    cmp = P.compare_solvers(E, P.GmresParams(tol=1e-10), stub_cascade(fmt="DIA"), matrix_id="eye4")
    for r in (cmp.default, cmp.sequential, cmp.async_):
        assert r.converged and r.iterations == 1


def test_cg_graph_batches_match_uncaptured():
    """CG batches replayed as CUDA graphs give the same iterations, history
    and solution as the uncaptured batches (same kernels, same order)."""
    import paper_2411_10143_b200 as P
    from paper_2411_10143_b200 import generators as G, solver
    A = P.CsrMatrix(*G.poisson2d(96))
    params = P.GmresParams(tol=1e-8, max_iters=4000)
    cfg = P.SpmvConfig.from_token("DIA/LibA")
    old = solver._CG_GRAPHS
    try:
        solver._CG_GRAPHS = True
        r1 = P.cg_solve(A, None, params, initial_config=cfg)
        solver._CG_GRAPHS = False
        r2 = P.cg_solve(A, None, params, initial_config=cfg)
    finally:
        solver._CG_GRAPHS = old
    assert r1.iterations == r2.iterations > 64        # several full (captured) batches ran
    assert r1.residual_history == r2.residual_history
    assert np.array_equal(r1.solution, r2.solution)


def test_cg_fused_spmv_dot_matches_unfused():
    """DIA CG with q = A p fused with p.q (one pass) vs the separate p.q
    kernel: same iteration count, residual estimates within rounding, and
    the same converged solution to 1e-10."""
    import paper_2411_10143_b200 as P
    from paper_2411_10143_b200 import generators as G, solver
    A = P.CsrMatrix(*G.poisson2d(80))
    params = P.GmresParams(tol=1e-8, max_iters=4000)
    cfg = P.SpmvConfig.from_token("DIA/LibA")
    old = solver._CG_FUSED
    try:
        solver._CG_FUSED = True
        r1 = P.cg_solve(A, None, params, initial_config=cfg)
        solver._CG_FUSED = False
        r2 = P.cg_solve(A, None, params, initial_config=cfg)
    finally:
        solver._CG_FUSED = old
    assert r1.converged and r2.converged
    assert abs(r1.iterations - r2.iterations) <= 1
    n = min(len(r1.residual_history), len(r2.residual_history))
    assert np.allclose(r1.residual_history[:n // 2], r2.residual_history[:n // 2], rtol=1e-6)
    assert np.linalg.norm(r1.solution - r2.solution) <= 1e-10 * np.linalg.norm(r2.solution) * 1e3
