"""Conversion times (CSR -> HYB / ELL / COO / DIA) on a power-law matrix and
config 2, median of 5 wall-clock (device-synchronised) conversions."""
import statistics
import sys
import time
sys.path.insert(0, ".")
import paper_2411_10143_b200 as P  # noqa: E402
from paper_2411_10143_b200 import generators as G  # noqa: E402
n = int(sys.argv[1]) if len(sys.argv) > 1 else 4_000_000
mats = {f"powerlaw_{n}": P.CsrMatrix(*G.powerlaw_spd(n, seed=0))}
offs = [(dy, dx) for dy in (-1, 0, 1) for dx in (-1, 0, 1)]
w = [8.5 if o == (0, 0) else -1.0 - 0.25 * (o[1] + o[0]) for o in offs]
mats["convdiff2000"] = P.CsrMatrix.stencil((2000, 2000), offs, w)
for name, A in mats.items():
    A._device()
    out = []
    for fmt in (P.FormatTag.HYB, P.FormatTag.COO, P.FormatTag.ELL, P.FormatTag.DIA):
        ts = []
        try:
            for _ in range(5):
                t0 = time.perf_counter()
                r = P.convert(A, fmt)
                r._device()
                from paper_2411_10143_b200 import device
                device.thread_stream(0).sync()
                ts.append(time.perf_counter() - t0)
                del r
            out.append(f"{fmt.value} {statistics.median(ts) * 1e3:.2f} ms")
        except Exception as e:
            out.append(f"{fmt.value} n/a ({type(e).__name__})")
    print(name, " | ".join(out), flush=True)
