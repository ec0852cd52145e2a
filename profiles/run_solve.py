"""Profiling driver: one warm-up + one measured async GMRES solve of the bench
workload (config 2), for ncu launch lists / full captures.

    ncu --metrics gpu__time_duration.sum --clock-control none --csv \
        --log-file gpurun_out/launches.csv python profiles/run_solve.py
"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

import paper_2411_10143_b200 as P  # noqa: E402
from paper_2411_10143_b200 import _lib, device  # noqa: E402
from paper_2411_10143_b200.solver import DeviceOptions  # noqa: E402

NX = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
MODE = sys.argv[2] if len(sys.argv) > 2 else "async"
offs, w = [], []
for dy in (-1, 0, 1):
    for dx in (-1, 0, 1):
        offs.append((dy, dx))
        w.append(8.5 if (dx, dy) == (0, 0) else -1.0 - 0.25 * (dx + dy))
A = P.CsrMatrix.stencil((NX, NX), offs, w)
models = P.CascadeModelSet.load_dir(ROOT / "tests" / "golden" / "models")
params = P.GmresParams(restart_m=30, tol=1e-8)
s = device.thread_stream()
ones = device.DeviceVector.from_numpy(np.ones(A.nrows), s)
b = device.DeviceVector(A.nrows)
_lib.check(_lib.lib().svb_spmv_sequential(A._device().handle, ones.ptr, b.ptr, s.handle))
s.sync()
for k in range(2):
    with DeviceOptions(keep_solution_on_device=True):
        if MODE == "async":
            r = P.async_solve(A, b, params, models, initial_config=P.GPU_DEFAULT_CONFIG)
        else:
            r = P.gmres_solve(A, b, params, initial_config=P.SpmvConfig.from_token(MODE))
    print(k, r.iterations, r.converged, [x.to_dict() for x in r.config_timeline], flush=True)
