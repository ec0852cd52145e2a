"""Config-2 async predict-while-solve A/B (profiling aid): the stock advisor,
the advisor with its feature pass blocking in native code instead of
polling the cancel event from Python (GIL hand-offs with the solver
thread), and predict-then-solve; median of 9 after 3 warm-ups, with the
swap iterations and advisor stage times of the last run."""
import statistics
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2411_10143_b200 as P  # noqa: E402
from paper_2411_10143_b200 import _lib, device, solver  # noqa: E402
from paper_2411_10143_b200.solver import DeviceOptions  # noqa: E402

offs, w = [], []
for dy in (-1, 0, 1):
    for dx in (-1, 0, 1):
        offs.append((dy, dx))
        w.append(8.5 if (dx, dy) == (0, 0) else -1.0 - 0.25 * (dx + dy))
A = P.CsrMatrix.stencil((2000, 2000), offs, w)
models = P.CascadeModelSet.load_dir(ROOT / "tests" / "golden" / "models")
params = P.GmresParams(restart_m=30, tol=1e-8, max_iters=1000)
s = device.thread_stream()
ones = device.DeviceVector.from_numpy(np.ones(A.nrows), s)
b = device.DeviceVector(A.nrows)
_lib.check(_lib.lib().svb_spmv_sequential(A._device().handle, ones.ptr, b.ptr, s.handle))
s.sync()
stages = {}
orig_pipeline = solver._Advisor._pipeline


def traced(self, cancel):
    try:
        return orig_pipeline(self, cancel)
    finally:
        stages.update(self.stage_times)


solver._Advisor._pipeline = traced


def run(fn, reps=9):
    with DeviceOptions(keep_solution_on_device=True):
        for _ in range(3):
            fn()
        ts = []
        for _ in range(reps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            r = fn()
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t0)
    return statistics.median(ts), min(ts), r


def async_():
    return P.async_solve(A, b, params, models, initial_config=P.GPU_DEFAULT_CONFIG)


out = {}
for name, fn in (("async", async_),
                 ("sequential", lambda: P.sequential_predict_solve(A, b, params, models)),
                 ("default", lambda: P.gmres_solve(A, b, params, initial_config=P.GPU_DEFAULT_CONFIG)),
                 ("dia_fixed", lambda: P.gmres_solve(A, b, params,
                                                     initial_config=P.SpmvConfig(P.FormatTag.DIA, P.Library.LIB_A)))):
    stages.clear()
    med, best, r = run(fn)
    tl = [(x.iteration, x.config.token()) for x in getattr(r, "config_timeline", [])]
    print(f"{name:12s} median {med * 1e3:7.3f} ms  best {best * 1e3:7.3f} ms  it {r.iterations}  "
          f"timeline {tl}  stages {({k: round(v * 1e3, 3) for k, v in stages.items()})}  "
          f"phases {getattr(r, 'phases', None)}", flush=True)
