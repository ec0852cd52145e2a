"""Diagnose async-solve step variance: per-iteration host timestamps (via the
matvec probe) and advisor stage times for repeated solves of the bench
workload.  Profiling aid only."""
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

if "torch" in sys.argv:
    import torch  # noqa: E402,F401
    torch.cuda.set_device(0)
import paper_2411_10143_b200 as P  # noqa: E402
from paper_2411_10143_b200 import _lib, device, solver  # noqa: E402
from paper_2411_10143_b200.solver import DeviceOptions  # noqa: E402

NX = 2000
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

orig_pipeline = solver._Advisor._pipeline


def timed_pipeline(self, cancel):
    self.t_start = time.perf_counter()
    try:
        return orig_pipeline(self, cancel)
    finally:
        self.t_end = time.perf_counter()


solver._Advisor._pipeline = timed_pipeline
if len(sys.argv) > 2 and sys.argv[2] == "nvml":
    import threading
    import pynvml
    pynvml.nvmlInit()
    hdl = pynvml.nvmlDeviceGetHandleByIndex(0)
    what = sys.argv[3] if len(sys.argv) > 3 else "all"

    def sampler():
        while True:
            pynvml.nvmlDeviceGetClockInfo(hdl, pynvml.NVML_CLOCK_SM)
            if what == "all":
                pynvml.nvmlDeviceGetCurrentClocksEventReasons(hdl)
                pynvml.nvmlDeviceGetUtilizationRates(hdl)
            time.sleep(0.05)
    threading.Thread(target=sampler, daemon=True).start()
if "nogc" in sys.argv:
    import gc
    gc.collect()
    gc.disable()
out = []
for rep in range(int(sys.argv[1]) if len(sys.argv) > 1 else 8):
    stamps = []
    t0 = time.perf_counter()
    with DeviceOptions(keep_solution_on_device=True):
        r = P.async_solve(A, b, params, models, initial_config=P.GPU_DEFAULT_CONFIG,
                          matvec_probe=lambda it, cfg: stamps.append((it, time.perf_counter() - t0)))
    wall = time.perf_counter() - t0
    first = {}
    for it, t in stamps:
        first.setdefault(it, t)
    its = sorted(first)
    gaps = [round((first[its[k]] - first[its[k - 1]]) * 1e3, 2) for k in range(1, min(len(its), 12))]
    allg = [(first[its[k]] - first[its[k - 1]], its[k]) for k in range(1, len(its))]
    worst = max(allg) if allg else (0.0, 0)
    out.append({"wall_ms": round(wall * 1e3, 1), "swaps": [(x.iteration, x.config.token(),
                round(x.swap_cost_seconds * 1e3, 2)) for x in r.config_timeline],
                "first_iter_gaps_ms": gaps, "iters": r.iterations,
                "worst_gap": (round(worst[0] * 1e3, 2), worst[1]),
                "free_gb": round(device.device_info()["free_bytes"] / 1e9, 2),
                "pool_gb": [round(device.device_info()[k] / 1e9, 2)
                            for k in ("pool_reserved_bytes", "pool_used_bytes")]})
    print(json.dumps(out[-1]), flush=True)
