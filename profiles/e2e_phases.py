"""Phases of the e2e path on config 2: CsrMatrix upload from pinned int64/f64
host arrays (svb_csr_create), b upload, async solve, solution download.
Median of 5 after 2 warm-ups; SPMVTUNE_LIB_VARIANT selects a library build."""
import json
import statistics
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2411_10143_b200 as P  # noqa: E402
from paper_2411_10143_b200 import device  # noqa: E402

offs = [(dy, dx) for dy in (-1, 0, 1) for dx in (-1, 0, 1)]
w = [8.5 if o == (0, 0) else -1.0 - 0.25 * (o[1] + o[0]) for o in offs]
A0 = P.CsrMatrix.stencil((2000, 2000), offs, w)
n = A0.nrows
pin = {}
for k, arr in (("rp", np.asarray(A0.row_ptr)), ("ci", np.asarray(A0.col_idx)), ("vv", np.asarray(A0.values))):
    t = torch.empty(arr.size, dtype=torch.from_numpy(arr[:1]).dtype, pin_memory=True)
    t.numpy()[:] = arr
    pin[k] = t
A = P.CsrMatrix(n, n, pin["rp"].numpy(), pin["ci"].numpy(), pin["vv"].numpy())
ts = []
for r in range(7):
    A._dev = None
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    A._device()
    ts.append(time.perf_counter() - t0)
up = statistics.median(ts[2:])
print(json.dumps({"upload_ms": up * 1e3, "bytes": int(sum(t.numel() * t.element_size() for t in pin.values())),
                  "gbs": sum(t.numel() * t.element_size() for t in pin.values()) / up / 1e9}))
