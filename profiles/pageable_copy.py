"""Host<->device copies of solve-sized vectors (2-32 MB) through the
package's device.copy (plain cudaMemcpyAsync) and device.copy_host (the
staged path gmres_solve's b upload and x download use): pageable numpy vs
pinned host memory; wall time, median of 9."""
import json
import statistics
import sys
import time
sys.path.insert(0, ".")
import numpy as np
from paper_2411_10143_b200 import device
import torch

out = {}
s = device.thread_stream(0)
for mb in (2, 8, 16, 32):
    n = mb * 1024 * 1024 // 8
    a = np.random.default_rng(0).random(n)
    p = torch.empty(n, dtype=torch.float64, pin_memory=True).numpy()
    p[:] = a
    d = device.DeviceVector(n)
    res = {}
    for name, src in (("pageable", a), ("pinned", p)):
        for direction in ("h2d", "d2h"):
            ts = []
            for _ in range(10):
                t0 = time.perf_counter()
                if direction == "h2d":
                    device.copy(d.ptr, src.ctypes.data, src.nbytes, s)
                else:
                    device.copy(src.ctypes.data, d.ptr, src.nbytes, s)
                s.sync()
                ts.append(time.perf_counter() - t0)
            res[f"{name}_{direction}_ms"] = round(statistics.median(ts[1:]) * 1e3, 3)
        for direction in ("h2d", "d2h"):      # the library's staged path (svb_copy_host)
            ts = []
            for _ in range(10):
                t0 = time.perf_counter()
                if direction == "h2d":
                    device.copy_host(d.ptr, src.ctypes.data, src.nbytes, True, s)
                else:
                    device.copy_host(src.ctypes.data, d.ptr, src.nbytes, False, s)
                ts.append(time.perf_counter() - t0)
            res[f"{name}_copy_host_{direction}_ms"] = round(statistics.median(ts[1:]) * 1e3, 3)
    out[f"{mb}MB"] = res
    print(mb, res, flush=True)
print(json.dumps(out))
