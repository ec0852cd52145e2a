"""Row-kernel variant sensitivity (SPMVTUNE_ROWCFG=1..3 pins the tile
capacity / ring depth) on a power-law matrix."""
import sys
sys.path.insert(0, ".")
import paper_2411_10143_b200 as P  # noqa: E402
from paper_2411_10143_b200 import generators as G  # noqa: E402
n = int(sys.argv[1]) if len(sys.argv) > 1 else 4_000_000
A = P.CsrMatrix(*G.powerlaw_spd(n, seed=0))
out = []
for tok in ("CSR/LibA/32", "CSR/LibA/8", "CSR/LibB", "COO/LibA", "HYB/LibA", "COO/LibB"):
    cfg = P.SpmvConfig.from_token(tok)
    rep = A if cfg.format is P.FormatTag.CSR else P.convert(A, cfg.format)
    t = P.time_config(rep, cfg, runs=30, warmups=5)
    out.append(f"{tok} {t*1e6:7.1f}us")
print(" | ".join(out), flush=True)
