"""A/B timing of ELL/HYB SpMV on the config-3 power-law matrix (2 M rows) and
the config-2 stencil (profiling aid)."""
import sys
sys.path.insert(0, ".")
import paper_2411_10143_b200 as P  # noqa: E402
from paper_2411_10143_b200 import generators as G  # noqa: E402

offs = [(dy, dx) for dy in (-1, 0, 1) for dx in (-1, 0, 1)]
w = [8.5 if o == (0, 0) else -1.0 - 0.25 * (o[1] + o[0]) for o in offs]
mats = {"convdiff2000": P.CsrMatrix.stencil((2000, 2000), offs, w),
        "powerlaw4M": P.CsrMatrix(*G.powerlaw_spd(4_000_000, seed=0))}
for name, A in mats.items():
    out = []
    for tok in ("ELL/LibA", "HYB/LibA"):
        cfg = P.SpmvConfig.from_token(tok)
        try:
            rep = P.convert(A, cfg.format)
            out.append(f"{tok} {P.time_config(rep, cfg, runs=100, warmups=10) * 1e6:8.1f}us")
        except P.SpmvTuneError as e:
            out.append(f"{tok} n/a")
    print(name, " | ".join(out), flush=True)
