"""extract_features on power-law matrices (rows of thousands of entries) and
config 2: device time of the feature pass, median of 7 after warm-up."""
import statistics
import sys
import time
sys.path.insert(0, ".")
import paper_2411_10143_b200 as P  # noqa: E402
from paper_2411_10143_b200 import generators as G  # noqa: E402
mats = {"powerlaw_1M_seed1": P.CsrMatrix(*G.powerlaw_spd(1 << 20, seed=1)),
        "powerlaw_4M": P.CsrMatrix(*G.powerlaw_spd(4_000_000, seed=0))}
offs = [(dy, dx) for dy in (-1, 0, 1) for dx in (-1, 0, 1)]
w = [8.5 if o == (0, 0) else -1.0 - 0.25 * (o[1] + o[0]) for o in offs]
mats["convdiff2000"] = P.CsrMatrix.stencil((2000, 2000), offs, w)
for name, A in mats.items():
    A._device()
    P.extract_features(A)
    ts = []
    for _ in range(7):
        t0 = time.perf_counter()
        P.extract_features(A)
        ts.append(time.perf_counter() - t0)
    print(f"{name}: {statistics.median(ts) * 1e3:.3f} ms", flush=True)
