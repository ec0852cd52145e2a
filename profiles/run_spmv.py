"""Profiling driver: a few launches of one SpMV configuration on one of the
sweep matrices (for ncu).  python profiles/run_spmv.py <matrix> <token[,token...]> [reps]
matrix: poisson1024 | convdiff2000 | powerlaw2M | powerlaw8M"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

import paper_2411_10143_b200 as P  # noqa: E402
from paper_2411_10143_b200 import device, generators as G  # noqa: E402
from paper_2411_10143_b200.kernels import launch  # noqa: E402

name, toks = sys.argv[1], sys.argv[2].split(",")
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
if name == "poisson1024":
    A = P.CsrMatrix.stencil((1024, 1024), [(0, 0), (0, -1), (0, 1), (-1, 0), (1, 0)], [4.0, -1, -1, -1, -1])
elif name == "convdiff2000":
    offs, w = [], []
    for dy in (-1, 0, 1):
        for dx in (-1, 0, 1):
            offs.append((dy, dx))
            w.append(8.5 if (dx, dy) == (0, 0) else -1.0 - 0.25 * (dx + dy))
    A = P.CsrMatrix.stencil((2000, 2000), offs, w)
elif name == "powerlaw8M":
    A = G.powerlaw_spd_device(8_000_000, seed=0)     # config 3, built on the device
else:
    A = P.CsrMatrix(*G.powerlaw_spd(2_000_000, seed=0))
s = device.thread_stream()
x = device.DeviceVector.from_numpy(np.random.default_rng(0).uniform(0.5, 1.5, A.nrows), s)
y = device.DeviceVector(A.nrows)
for tok in toks:       # comma-separated tokens: one matrix, several configurations
    cfg = P.SpmvConfig.from_token(tok)
    rep = A if cfg.format is P.FormatTag.CSR else P.convert(A, cfg.format)
    for _ in range(reps):
        launch(cfg, rep, x.ptr, y.ptr, workers=4, stream=s)
    s.sync()
    print("ok", name, tok)
