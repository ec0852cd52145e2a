import sys, time
sys.path.insert(0, ".")
import numpy as np
import paper_2411_10143_b200 as P
from paper_2411_10143_b200 import generators as G
mats = {"convdiff2000": None, "powerlaw2M": P.CsrMatrix(*G.powerlaw_spd(2_000_000, seed=0)),
        "random1M": None}
offs = [(dy, dx) for dy in (-1, 0, 1) for dx in (-1, 0, 1)]
w = [8.5 if o == (0, 0) else -1.0 - 0.25 * (o[1] + o[0]) for o in offs]
mats["convdiff2000"] = P.CsrMatrix.stencil((2000, 2000), offs, w)
from paper_2411_10143_b200.cli import _random_dd
mats["random1M"] = P.CsrMatrix(*_random_dd(1_000_000, 12, 1))
for name, A in mats.items():
    out = []
    for tok in ("CSR/LibA/32", "CSR/LibA/8", "CSR/LibA/2"):
        t = P.time_config(A, P.SpmvConfig.from_token(tok), runs=100, warmups=10)
        out.append(f"{tok} {t*1e6:8.1f}us")
    print(name, " | ".join(out), flush=True)
