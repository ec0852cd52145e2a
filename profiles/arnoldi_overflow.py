"""GMRES(30) on conv-diff nx^2 (default 2830: 8.0 M rows, above the 4.85 M
on-chip Arnoldi capacity): solve time and per-launch Arnoldi time with the
partially resident TMA kernel, or with SPMVTUNE_MGS=stream set by the caller.
    python profiles/arnoldi_overflow.py [nx]"""
import itertools
import json
import statistics
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

import paper_2411_10143_b200 as P  # noqa: E402
from paper_2411_10143_b200.solver import DeviceOptions  # noqa: E402
sys.path.insert(0, str(ROOT))
from bench import EventTimer  # noqa: E402

nx = int(sys.argv[1]) if len(sys.argv) > 1 else 2830
offs, w = [], []
for o in itertools.product((-1, 0, 1), repeat=2):
    offs.append(o)
    w.append(8.5 if not any(o) else -1.0 - 0.25 * (o[1] + o[0]))
A = P.CsrMatrix.stencil((nx, nx), offs, w)
params = P.GmresParams(restart_m=30, tol=1e-8, max_iters=1000)
cfg = P.SpmvConfig(P.FormatTag.DIA, P.Library.LIB_A)
D = P.convert(A, P.FormatTag.DIA)
for _ in range(2):
    r = P.gmres_solve(D, None, params, initial_config=cfg)
ts = []
for _ in range(5):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = P.gmres_solve(D, None, params, initial_config=cfg)
    torch.cuda.synchronize()
    ts.append(time.perf_counter() - t0)
timer = EventTimer()
with DeviceOptions(timer=timer):
    P.gmres_solve(D, None, params, initial_config=cfg)
k = timer.summary()
print(json.dumps({"n": A.nrows, "iterations": r.iterations, "final": r.final_residual,
                  "solve_ms": statistics.median(ts) * 1e3,
                  "per_tag_ms_avg": {t: sum(v) / len(v) for t, v in k.items()},
                  "per_tag_launches": {t: len(v) for t, v in k.items()}}))
