"""The native solver drivers (csrc/driver.cu: svb_gmres_run / svb_cg_run
and the svb_mailbox configuration slot) against the Python drivers and the
CPU oracle.  Same kernels in the same order, so iteration counts, residual
histories and solutions are bit-identical to gmres_solve / cg_solve."""
import threading

import numpy as np
import pytest

import oracle as O
import paper_2411_10143_b200 as P
from paper_2411_10143_b200.solver import ADVISOR_COMPLETED
from paper_2411_10143_b200 import generators as G
from paper_2411_10143_b200 import solver
from paper_2411_10143_b200.inference import model_from_dict

pytestmark = pytest.mark.gpu


def _mat(gen):
    n, _, ptr, cols, vals = gen
    return n, P.CsrMatrix(n, n, ptr, cols, vals), O.OCsr(n, n, ptr, cols, vals)


CASES = [
    ("gmres", lambda: G.convdiff9(30), "DIA/LibA", 30),
    ("gmres", lambda: G.poisson2d(10), "CSR/LibA/32", 30),
    ("gmres", lambda: G.powerlaw_spd(3000, seed=4), "HYB/LibA", 10),
    ("cg", lambda: G.poisson2d(40), "DIA/LibA", 30),
    ("cg", lambda: G.poisson2d(40), "CSR/LibB", 30),
    ("cg", lambda: G.powerlaw_spd(3000, seed=4), "ELL/LibA", 30),
]


@pytest.mark.parametrize("method,gen,tok,restart", CASES)
def test_native_driver_matches_python_driver(method, gen, tok, restart, monkeypatch):
    n, A, Ao = _mat(gen())
    cfg = P.SpmvConfig.from_token(tok)
    params = P.GmresParams(restart_m=restart, tol=1e-8, max_iters=3000)
    monkeypatch.setattr(solver, "_LOOP", "python")     # the public call on the Python loop
    ref = (P.gmres_solve if method == "gmres" else P.cg_solve)(A, None, params, initial_config=cfg)
    monkeypatch.setattr(solver, "_LOOP", "native")
    got = P.native_solve(method, A, None, params, cfg)
    assert got.iterations == ref.iterations and got.converged and ref.converged
    assert got.residual_history == ref.residual_history          # bit-identical
    assert np.array_equal(got.solution, ref.solution)
    assert got.final_residual == ref.final_residual
    assert [s.iteration for s in got.config_timeline] == [1]
    assert got.config_timeline[0].config == cfg
    # and against the CPU oracle (±1 iteration)
    b = O.spmv_sequential(Ao, np.ones(n))
    mv = lambda v: O.spmv("CSR/LibB", Ao, v)      # noqa: E731
    o = (O.gmres(mv, b, restart=restart, tol=1e-8, max_iters=3000) if method == "gmres"
         else O.cg(mv, b, tol=1e-8, max_iters=3000))
    assert abs(got.iterations - o["iterations"]) <= 1
    assert np.linalg.norm(got.solution - o["x"]) <= 1e-6 * np.linalg.norm(o["x"])


def test_native_driver_edge_cases():
    n, A, _ = _mat(G.poisson2d(8))
    # b = 0: converged at once, history [0.0], no matvec
    r = P.native_solve("gmres", A, np.zeros(n), P.GmresParams(tol=1e-8))
    assert r.converged and r.iterations == 0 and r.residual_history == [0.0] and r.final_residual == 0.0
    # max_iters = 0: not converged, final residual None (reference semantics)
    r = P.native_solve("cg", A, None, P.GmresParams(max_iters=0))
    assert not r.converged and r.iterations == 0 and r.final_residual is None
    # max_iters cap
    r = P.native_solve("gmres", A, None, P.GmresParams(restart_m=5, tol=1e-14, max_iters=7))
    ref = P.gmres_solve(A, None, P.GmresParams(restart_m=5, tol=1e-14, max_iters=7))
    assert r.iterations == ref.iterations == 7 and r.residual_history == ref.residual_history
    assert r.final_residual == ref.final_residual
    # non-square / wrong-length b
    R = P.CsrMatrix(3, 4, np.array([0, 1, 2, 3]), np.array([0, 1, 2]), np.ones(3))
    with pytest.raises(ValueError):
        P.native_solve("gmres", R, np.ones(3))
    with pytest.raises(ValueError):
        P.native_solve("cg", A, np.ones(n + 1))
    # non-finite: NaN in b
    bad = np.ones(n)
    bad[3] = np.nan
    with pytest.raises(P.SolverNumericalError):
        P.native_solve("gmres", A, bad)


@pytest.mark.parametrize("method", ["gmres", "cg"])
def test_native_mailbox_swap(method):
    """An advisor thread publishes DIA/LibA while the native solve runs from
    CSR/LibA/32: the timeline records the swap, the solve converges to the
    fixed-configuration answer, and the mailbox reports the solver done."""
    nx = 400 if method == "cg" else 300
    n, A, _ = _mat(G.poisson2d(nx) if method == "cg" else G.convdiff9(nx))
    params = P.GmresParams(restart_m=30, tol=1e-8, max_iters=5000)
    mb = P.NativeMailbox()
    D = P.convert(A, P.FormatTag.DIA)
    D._device()
    from paper_2411_10143_b200 import device
    ev = device.thread_stream(0).record()
    go = threading.Event()

    def advisor():
        go.wait()
        mb.publish(D, P.SpmvConfig.from_token("DIA/LibA"), ready=ev, prep_seconds=0.001)

    t = threading.Thread(target=advisor)
    t.start()
    go.set()
    got = P.native_solve(method, A, None, params, P.SpmvConfig.from_token("CSR/LibA/32"), mailbox=mb)
    t.join()
    ref = (P.gmres_solve if method == "gmres" else P.cg_solve)(A, None, params)
    assert got.converged and abs(got.iterations - ref.iterations) <= 1
    assert np.linalg.norm(got.solution - ref.solution) <= 1e-6 * np.linalg.norm(ref.solution)
    toks = [s.config.token() for s in got.config_timeline]
    assert toks[0] == "CSR/LibA/32"
    if len(toks) > 1:                  # the publish may land after convergence on a fast GPU
        assert toks == ["CSR/LibA/32", "DIA/LibA"] and got.config_timeline[1].iteration >= 2
        assert got.config_timeline[1].swap_cost_seconds == 0.001
    assert mb.finished


def test_native_mailbox_publish_before_solve_swaps_at_iteration_2():
    """A publish that is already pending when the solve starts is applied at
    the first poll (after iteration 1), as ConfigMailbox without gates."""
    n, A, _ = _mat(G.convdiff9(60))
    mb = P.NativeMailbox()
    D = P.convert(A, P.FormatTag.DIA)
    mb.publish(D, P.SpmvConfig.from_token("DIA/LibA"))
    got = P.native_solve("gmres", A, None, P.GmresParams(tol=1e-8), P.SpmvConfig.from_token("CSR/LibB"),
                         mailbox=mb)
    assert [(s.iteration, s.config.token()) for s in got.config_timeline] == [(1, "CSR/LibB"), (2, "DIA/LibA")]
    ref = P.gmres_solve(A, None, P.GmresParams(tol=1e-8))
    assert got.converged and abs(got.iterations - ref.iterations) <= 1


def _forced_cascade(fmt):
    def stub(classes, pick):
        return model_from_dict({"schema_version": 1, "feature_names": list(P.FEATURE_NAMES),
                                "classes": classes,
                                "trees": [[{"score": 1.0 if c == pick else 0.0}] for c in classes]})
    return P.CascadeModelSet(
        format_model=stub(["COO", "CSR", "ELL", "DIA", "HYB"], fmt),
        coo_lib_model=stub(["LibA", "LibB"], "LibA"),
        csr_lib_model=stub(["LibA", "LibB", "LibC"], "LibA"),
        ell_lib_model=stub(["LibA", "LibC"], "LibA"),
        csr_tpv_model=stub(["2", "4", "8", "16", "32"], "32"))


@pytest.mark.parametrize("method", ["gmres", "cg"])
def test_public_solves_run_the_native_loop(method, monkeypatch):
    """gmres_solve / cg_solve / sequential_predict_solve / async_solve with
    stock executors run the C++ loop (no GIL held while the advisor works);
    each report is bit-identical to the same call on the Python loop, and the
    async advisor's DIA publish reaches the native mailbox."""
    n, A, Ao = _mat(G.poisson2d(120) if method == "cg" else G.convdiff9(120))
    params = P.GmresParams(restart_m=30, tol=1e-8, max_iters=4000)
    models = _forced_cascade("DIA")
    fixed_fn = P.gmres_solve if method == "gmres" else P.cg_solve
    calls = []
    real = solver.native_solve
    monkeypatch.setattr(solver, "native_solve", lambda *a, **k: calls.append(a[0]) or real(*a, **k))
    fixed = fixed_fn(A, None, params)
    seq = P.sequential_predict_solve(A, None, params, models, method=method)
    asy = P.async_solve(A, None, params, models, method=method)
    assert calls == [method] * 3
    monkeypatch.setattr(solver, "_LOOP", "python")
    fixed_py = fixed_fn(A, None, params)
    seq_py = P.sequential_predict_solve(A, None, params, models, method=method)
    assert calls == [method] * 3
    for got, ref in ((fixed, fixed_py), (seq, seq_py)):
        assert got.converged and got.iterations == ref.iterations
        assert got.residual_history == ref.residual_history
        assert np.array_equal(got.solution, ref.solution)
    assert fixed.mode == "fixed" and seq.mode == "sequential" and asy.mode == "async"
    assert seq.config_timeline[0].config.token() == "DIA/LibA"
    toks = [s.config.token() for s in asy.config_timeline]
    assert asy.converged and toks[0] == P.DEFAULT_CONFIG.token()
    if len(toks) > 1:                      # the publish may land after convergence
        assert toks[1:] == ["DIA/LibA"] and asy.config_timeline[1].iteration >= 2
        assert asy.advisor_outcome == ADVISOR_COMPLETED
    assert abs(asy.iterations - fixed.iterations) <= 1
    assert np.linalg.norm(asy.solution - fixed.solution) <= 1e-6 * np.linalg.norm(fixed.solution)


def test_probe_and_plugin_executor_keep_the_python_loop(monkeypatch):
    n, A, _ = _mat(G.poisson2d(20))
    calls = []
    real = solver.native_solve
    monkeypatch.setattr(solver, "native_solve", lambda *a, **k: calls.append(a[0]) or real(*a, **k))

    class Plugin(P.SpmvExecutor):
        def matvec(self, x):
            return super().matvec(x)

    seen = []
    P.gmres_solve(A, None, P.GmresParams(tol=1e-8), matvec_probe=lambda it, c: seen.append(it))
    P.gmres_solve(A, None, P.GmresParams(tol=1e-8), executor=Plugin(P.DEFAULT_CONFIG, P.to_coo(A)))
    assert calls == [] and seen
