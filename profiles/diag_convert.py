"""Time the advisor's device stages (features, CSR->DIA conversion) on the
bench matrix, host wall clock around each synchronous call.  Profiling aid."""
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import paper_2411_10143_b200 as P  # noqa: E402
from paper_2411_10143_b200 import device  # noqa: E402

NX = 2000
offs, w = [], []
for dy in (-1, 0, 1):
    for dx in (-1, 0, 1):
        offs.append((dy, dx))
        w.append(8.5 if (dx, dy) == (0, 0) else -1.0 - 0.25 * (dx + dy))
A = P.CsrMatrix.stencil((NX, NX), offs, w)
s = device.thread_stream()
for k in range(6):
    t0 = time.perf_counter()
    fv = P.extract_features(A)
    t1 = time.perf_counter()
    D = P.convert(A, P.FormatTag.DIA)
    s.sync()
    t2 = time.perf_counter()
    del D
    print(f"features {1e3 * (t1 - t0):7.2f} ms  convert DIA {1e3 * (t2 - t1):7.2f} ms", flush=True)
