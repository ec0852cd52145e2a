"""Config-1 CG timing (Poisson 1024^2, tol 1e-8): default CSR-vector solve and
async solve, median of 5, with and without CUDA-graph batches."""
import os
import statistics
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import paper_2411_10143_b200 as P  # noqa: E402
from paper_2411_10143_b200 import solver  # noqa: E402
from paper_2411_10143_b200.solver import DeviceOptions  # noqa: E402

A = P.CsrMatrix.stencil((1024, 1024), [(0, 0), (0, -1), (0, 1), (-1, 0), (1, 0)], [4.0, -1, -1, -1, -1])
models = P.CascadeModelSet.load_dir(ROOT / "tests" / "golden" / "models")
params = P.GmresParams(tol=1e-8, max_iters=5000)
for graphs in (True, False):
    solver._CG_GRAPHS = graphs
    with DeviceOptions(keep_solution_on_device=True):
        for mode in ("default", "async", "dia"):
            ts = []
            for _ in range(6):
                t = time.perf_counter()
                if mode == "default":
                    r = P.cg_solve(A, None, params, initial_config=P.GPU_DEFAULT_CONFIG)
                elif mode == "dia":
                    r = P.cg_solve(A, None, params, initial_config=P.SpmvConfig.from_token("DIA/LibA"))
                else:
                    r = P.async_solve(A, None, params, models, method="cg", initial_config=P.GPU_DEFAULT_CONFIG)
                ts.append(time.perf_counter() - t)
            print(f"graphs={graphs} {mode:8s} {statistics.median(ts[1:]) * 1e3:8.2f} ms  it={r.iterations} "
                  f"res={r.final_residual:.2e} swaps={[(s.iteration, s.config.token()) for s in r.config_timeline]}",
                  flush=True)
