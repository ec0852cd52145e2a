"""DIA SpMV timing on the 27-point Laplacian n3^3 (config 5 at 600): CUDA
events over `reps` launches on one stream, algorithmic bytes 8*ndiag*n +
16*n.  SPMVTUNE_DIA=0 selects the thread-per-row k_dia, 1 (default) the
TMA-staged k_dia_tma; SPMVTUNE_DIA_NS its ring depth.

    python profiles/bench_dia.py [n3] [reps]
"""
import json
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2411_10143_b200 as P  # noqa: E402
from paper_2411_10143_b200 import _lib, device  # noqa: E402
from paper_2411_10143_b200.kernels import launch  # noqa: E402

n3 = int(sys.argv[1]) if len(sys.argv) > 1 else 600
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
offs, w = [], []
for dz in (-1, 0, 1):
    for dy in (-1, 0, 1):
        for dx in (-1, 0, 1):
            offs.append((dz, dy, dx))
            w.append(26.0 if (dx, dy, dz) == (0, 0, 0) else -1.0)
A = P.CsrMatrix.stencil((n3, n3, n3), offs, w)
D = P.convert(A, P.FormatTag.DIA)
del A
n = D.nrows
s = device.thread_stream()
x = device.DeviceVector(n)
_lib.check(_lib.lib().svb_fill(x.ptr, n, 1.0, s.handle))
y = device.DeviceVector(n)
cfg = P.SpmvConfig(P.FormatTag.DIA, P.Library.LIB_A)
ext = torch.cuda.ExternalStream(s.handle)
for _ in range(3):
    launch(cfg, D, x.ptr, y.ptr, workers=4, stream=s)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(ext)
for _ in range(reps):
    launch(cfg, D, x.ptr, y.ptr, workers=4, stream=s)
e1.record(ext)
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
byts = 8 * 27 * n + 16 * n
ysum = float(np.sum(y.to_numpy(s)))
print(json.dumps({"n3": n3, "variant": os.environ.get("SPMVTUNE_DIA", "1"), "ns": os.environ.get("SPMVTUNE_DIA_NS"),
                  "ms": ms, "gbs": byts / ms / 1e6, "frac_of_6457": byts / ms / 1e6 / 6457.4, "ysum": ysum}))
