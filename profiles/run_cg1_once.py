"""Profiling driver: two config-1 CG solves on DIA (fused k_dia_dot path)."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import paper_2411_10143_b200 as P  # noqa: E402

A = P.CsrMatrix.stencil((1024, 1024), [(0, 0), (0, -1), (0, 1), (-1, 0), (1, 0)], [4.0, -1, -1, -1, -1])
for _ in range(2):
    r = P.cg_solve(A, None, P.GmresParams(tol=1e-8, max_iters=5000),
                   initial_config=P.SpmvConfig.from_token("DIA/LibA"))
print(r.iterations, r.converged)
