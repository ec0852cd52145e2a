import sys
sys.path.insert(0, ".")
import paper_2411_10143_b200 as P
offs = [(dy, dx) for dy in (-1, 0, 1) for dx in (-1, 0, 1)]
w = [8.5 if o == (0, 0) else -1.0 - 0.25 * (o[1] + o[0]) for o in offs]
A = P.CsrMatrix.stencil((2000, 2000), offs, w)
B = P.CsrMatrix.stencil((1024, 1024), [(0, 0), (-1, 0), (1, 0), (0, -1), (0, 1)], [4.0, -1, -1, -1, -1])
out = []
for name, M in (("c2", A), ("c1", B)):
    for tok in ("CSR/LibA/32", "CSR/LibB", "COO/LibA"):
        cfg = P.SpmvConfig.from_token(tok)
        rep = M if cfg.format is P.FormatTag.CSR else P.convert(M, cfg.format)
        out.append(f"{name} {tok} {P.time_config(rep, cfg, runs=50, warmups=10) * 1e6:6.1f}")
print(" | ".join(out), flush=True)
