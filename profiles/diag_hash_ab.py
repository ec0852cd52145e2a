"""Feature pass and CSR->DIA conversion on stencils whose grid pitch is a
power of two (the diagonal cache's slot collisions), on neighbours that
are not, and on power-law matrices (every entry a new diagonal); device-synchronised wall time, median of 7 after warm-up.  Run
with SPMVTUNE_LIB_VARIANT=old for the low-bits slot build."""
import json
import statistics
import sys
import time
sys.path.insert(0, ".")
import paper_2411_10143_b200 as P  # noqa: E402
from paper_2411_10143_b200 import generators as G  # noqa: E402

mats = {"poisson2d_1024 (config 1)": G.poisson2d(1024), "poisson2d_1000": G.poisson2d(1000),
        "convdiff9_2048": G.convdiff9(2048), "convdiff9_2000 (config 2)": G.convdiff9(2000),
        "convdiff9_512": G.convdiff9(512), "laplace27_128": G.laplace27(128), "laplace27_120": G.laplace27(120),
        "powerlaw_1M": G.powerlaw_spd(1 << 20, seed=1), "powerlaw_4M": G.powerlaw_spd(4_000_000, seed=0)}
out = {}
for name, gen in mats.items():
    A = P.CsrMatrix(*gen)
    A._device()
    fv = P.extract_features(A)
    res = {}
    for what, fn in (("features_ms", lambda: P.extract_features(A)),
                     ("to_dia_ms", lambda: P.convert(A, P.FormatTag.DIA))):
        try:
            fn()
        except P.FormatInapplicableError:      # power-law: more diagonals than DIA allows
            res[what] = None
            continue
        ts = []
        for _ in range(7):
            t0 = time.perf_counter()
            fn()
            ts.append(time.perf_counter() - t0)
        res[what] = round(statistics.median(ts) * 1e3, 3)
    res["features"] = fv.to_array().tolist()
    out[name] = res
    print(name, res["features_ms"], res["to_dia_ms"], flush=True)
print(json.dumps(out))
