"""BASELINE configs[2]: CG on the synthetic power-law SPD matrix (8 M rows,
~120 M nnz), b = rhs "random" seed 0 (solver.py:190-191), tol 1e-8.
Default CSR-vector solve vs cascade predict-then-solve vs async
predict-while-solve from CSR/LibA/32, plus the per-configuration SpMV times
the cascade chooses between.  Prints one JSON line.

    python profiles/run_config3.py [n_rows]
"""
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import paper_2411_10143_b200 as P  # noqa: E402
from paper_2411_10143_b200 import generators as G  # noqa: E402
from paper_2411_10143_b200.solver import DeviceOptions  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8_000_000
t0 = time.perf_counter()
nr, nc, ptr, cols, vals = G.powerlaw_spd(n, seed=0)
gen_s = time.perf_counter() - t0
A = P.CsrMatrix(nr, nc, ptr, cols, vals)
A._device()
import os  # noqa: E402
models = P.CascadeModelSet.load_dir(P.B200_MODELS_DIR if os.environ.get("MODELS") == "b200"
                                    else ROOT / "tests" / "golden" / "models")
params = P.GmresParams(tol=1e-8, max_iters=20000, rhs="random", seed=0)
start = P.GPU_DEFAULT_CONFIG
out = {"models": os.environ.get("MODELS", "shipped"), "workload": f"config3: CG fp64 power-law SPD n={nr:,} nnz={A.nnz:,}, b random seed 0, tol 1e-8",
       "host_generation_s": gen_s}
fv = P.extract_features(A)
out["features"] = {k: getattr(fv, k) for k in ("mean", "sd", "cov", "max", "ndiag", "diagfill")}
out["cascade"] = P.cascade_predict(models, fv).token()
# b computed once, outside every clock (the reference times solves with b
# given: solver.py:355-358, 470-471, 508-510)
from paper_2411_10143_b200.solver import default_rhs  # noqa: E402
bvec = default_rhs(A, params)
with DeviceOptions(keep_solution_on_device=True):
    P.async_solve(A, bvec, params, models, method="cg", initial_config=start)      # warm-up
    runs = []
    for _ in range(3):
        t = time.perf_counter()
        r = P.async_solve(A, bvec, params, models, method="cg", initial_config=start)
        runs.append(time.perf_counter() - t)
    out["async_s"] = sorted(runs)[1]
    out["async_iterations"] = r.iterations
    out["async_timeline"] = [(s.iteration, s.config.token()) for s in r.config_timeline]
    out["converged"], out["final_residual"] = r.converged, r.final_residual
    # medians of 3 (single runs see occasional first-use / pool-growth stalls)
    dts, sts = [], []
    for _ in range(3):
        t = time.perf_counter()
        d = P.cg_solve(A, bvec, params, initial_config=start)
        dts.append(time.perf_counter() - t)
    out["default_csr_vector_s"] = sorted(dts)[1]
    out["default_iterations"] = d.iterations
    for _ in range(3):
        t = time.perf_counter()
        s = P.sequential_predict_solve(A, bvec, params, models, method="cg")
        sts.append((time.perf_counter() - t, s.phases))
    sts.sort(key=lambda e: e[0])
    out["sequential_s"], out["sequential_phases"] = sts[1]
times = {}
for tok in ("CSR/LibA/32", "CSR/LibA/8", "CSR/LibB", "CSR/LibC", "COO/LibA", "HYB/LibA", "ELL/LibA"):
    cfg = P.SpmvConfig.from_token(tok)
    try:
        rep = A if cfg.format is P.FormatTag.CSR else P.convert(A, cfg.format)
        times[tok] = P.time_config(rep, cfg, runs=50, warmups=5) * 1e6
    except P.SpmvTuneError as exc:
        times[tok] = f"inapplicable: {exc}"[:80]
out["spmv_us"] = times
print(json.dumps(out), flush=True)
