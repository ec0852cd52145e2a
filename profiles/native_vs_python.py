"""Config 2 (GMRES(30), conv-diff 2000^2, DIA/LibA fixed) and config 1 (CG,
Poisson 1024^2, DIA/LibA): the Python driver loop (gmres_solve / cg_solve)
against the native C++ driver (native_solve) on the same device matrix.
Median of 5 wall-clock solves after 2 warm-ups; prints one JSON line.

    python profiles/native_vs_python.py
"""
import json
import statistics
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2411_10143_b200 as P  # noqa: E402
from paper_2411_10143_b200 import device  # noqa: E402
from paper_2411_10143_b200.solver import DeviceOptions  # noqa: E402


def problem(kind):
    if kind == "config2":
        offs = [(dy, dx) for dy in (-1, 0, 1) for dx in (-1, 0, 1)]
        w = [8.5 if o == (0, 0) else -1.0 - 0.25 * (o[1] + o[0]) for o in offs]
        return "gmres", P.CsrMatrix.stencil((2000, 2000), offs, w)
    offs = [(0, 0), (-1, 0), (1, 0), (0, -1), (0, 1)]
    w = [4.0, -1.0, -1.0, -1.0, -1.0]
    return "cg", P.CsrMatrix.stencil((1024, 1024), offs, w)


out = {}
for kind in ("config2", "config1"):
    method, A = problem(kind)
    D = P.convert(A, P.FormatTag.DIA)
    cfg = P.SpmvConfig.from_token("DIA/LibA")
    params = P.GmresParams(restart_m=30, tol=1e-8, max_iters=20000)
    n = A.nrows
    ones = device.DeviceVector(n)
    import numpy as np
    ones_h = np.ones(n)
    device.copy(ones.ptr, ones_h.ctypes.data, 8 * n, device.thread_stream(0))
    device.thread_stream(0).sync()
    b = device.DeviceVector(n)
    P.execute_spmv(P.SpmvConfig.from_token("CSR/LibB"), A, ones, out=b)
    device.thread_stream(0).sync()
    bh = b.to_numpy(device.thread_stream(0))
    py = (P.gmres_solve if method == "gmres" else P.cg_solve)
    res = {}
    for name, fn in (("python", lambda: py(D, bh, params, initial_config=cfg)),
                     ("native", lambda: P.native_solve(method, D, bh, params, cfg))):
        ts, its = [], None
        with DeviceOptions(keep_solution_on_device=False):
            for r in range(7):
                t0 = time.perf_counter()
                rep = fn()
                dt = time.perf_counter() - t0
                if r >= 2:
                    ts.append(dt)
                its = rep.iterations
        res[name] = {"median_s": statistics.median(ts), "min_s": min(ts), "iterations": its}
    out[kind] = res
print(json.dumps(out))
