"""A/B of the TMA Arnoldi kernel's grid size (SPMVTUNE_MGS_GRID) on small
GMRES(30) systems: per-iteration time of gmres_solve (DIA/LibA, forced
300 iterations) and the converged iteration count at tol 1e-8.  One process
per grid size (the variable is read when the workspace is created)."""
import json
import os
import subprocess
import sys

CHILD = r'''
import json, sys, time
import numpy as np
sys.path.insert(0, ".")
import paper_2411_10143_b200 as P
from paper_2411_10143_b200 import generators as G
out = {}
for name, gen in [("poisson2d_256", lambda: G.poisson2d(256)), ("convdiff9_362", lambda: G.convdiff9(362)),
                  ("convdiff9_512", lambda: G.convdiff9(512)), ("convdiff9_1024", lambda: G.convdiff9(1024))]:
    n, _, ptr, cols, vals = gen()
    A = P.CsrMatrix(n, n, ptr, cols, vals)
    cfg = P.SpmvConfig(P.FormatTag.DIA, P.Library.LIB_A)
    D = P.convert(A, P.FormatTag.DIA)
    forced = P.GmresParams(restart_m=30, tol=1e-300, max_iters=300)
    ts = []
    for r in range(6):
        t = time.perf_counter()
        P.gmres_solve(D, None, forced, initial_config=cfg)
        ts.append(time.perf_counter() - t)
    conv = P.gmres_solve(D, None, P.GmresParams(restart_m=30, tol=1e-8, max_iters=5000), initial_config=cfg)
    out[name] = {"n": n, "us_per_iter": 1e6 * float(np.median(ts[1:])) / 300,
                 "iterations": conv.iterations, "final": conv.final_residual}
print(json.dumps(out))
'''
res = {}
for g in [int(a) for a in (sys.argv[1:] or ["148", "96", "64", "32", "16", "8"])]:
    env = dict(os.environ, SPMVTUNE_MGS_GRID=str(g))
    p = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True, timeout=600)
    if p.returncode != 0:
        res[g] = {"error": p.stderr[-800:]}
    else:
        res[g] = json.loads(p.stdout.strip().splitlines()[-1])
    print(g, json.dumps(res[g]), flush=True)
print(json.dumps(res))
