"""GMRES(30) on conv-diff 512^2 (n = 262 K, DIA/LibA): the reduced-grid TMA
Arnoldi kernel (64 CTAs) for ncu captures; SPMVTUNE_MGS_GRID=148 for the
all-SM grid."""
import sys
sys.path.insert(0, ".")
import paper_2411_10143_b200 as P
from paper_2411_10143_b200 import generators as G

n, m, ptr, cols, vals = G.convdiff9(512)
A = P.convert(P.CsrMatrix(n, m, ptr, cols, vals), P.FormatTag.DIA)
cfg = P.SpmvConfig(P.FormatTag.DIA, P.Library.LIB_A)
for _ in range(2):
    r = P.gmres_solve(A, None, P.GmresParams(restart_m=30, tol=1e-8, max_iters=1000), initial_config=cfg)
print(r.iterations, r.final_residual)
