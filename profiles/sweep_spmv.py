"""SpMV roofline sweep: every configuration on the BASELINE stencil matrices
(and a power-law matrix), device time per launch from CUDA events on the
launching stream, achieved GB/s from the algorithmic bytes of SURVEY.md §8(d)
against the measured HBM copy peak.

    python profiles/sweep_spmv.py [runs] [poisson1024,convdiff2000,powerlaw2M,powerlaw8M] > out.json
"""
import json
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2411_10143_b200 as P  # noqa: E402
from paper_2411_10143_b200 import device, generators as G  # noqa: E402
from paper_2411_10143_b200.kernels import launch  # noqa: E402

RUNS = int(sys.argv[1]) if len(sys.argv) > 1 else 50
PEAK = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"] \
    if (ROOT / "MEASURED_PEAKS.json").exists() else 6650.0


F32 = os.environ.get("SWEEP_DTYPE", "f64") == "f32"   # fp32 values, x and y (north star: fp64/fp32)


def alg_bytes(fmt, rep, n, ncols, lib=""):
    inf = rep._device().info
    v = 4 if F32 else 8                 # value / vector element bytes
    if fmt == "CSR":
        return (4 + v) * inf.nnz + 4 * (n + 1) + v * ncols + v * n
    if fmt == "COO" and lib == "LibA":
        return (4 + v) * inf.nnz + 8 * (n + 1) + v * ncols + v * n
    if fmt == "COO":
        return (8 + v) * inf.nnz + v * ncols + v * n
    if fmt == "ELL":
        return (4 + v) * n * inf.width + v * ncols + v * n
    if fmt == "DIA":
        return v * inf.ndiag * n + v * ncols + v * n
    return (4 + v) * n * inf.width + (8 + v) * inf.spill_nnz + v * ncols + 2 * v * n


def stencil(kind):
    if kind == "poisson1024":
        return P.CsrMatrix.stencil((1024, 1024), [(0, 0), (0, -1), (0, 1), (-1, 0), (1, 0)],
                                   [4.0, -1, -1, -1, -1])
    offs, w = [], []
    for dy in (-1, 0, 1):
        for dx in (-1, 0, 1):
            offs.append((dy, dx))
            w.append(8.5 if (dx, dy) == (0, 0) else -1.0 - 0.25 * (dx + dy))
    return P.CsrMatrix.stencil((2000, 2000), offs, w)


def main():
    which = sys.argv[2].split(",") if len(sys.argv) > 2 else ["poisson1024", "convdiff2000", "powerlaw2M"]
    build = {"poisson1024": ("config1_poisson1024", lambda: stencil("poisson1024")),
             "convdiff2000": ("config2_convdiff2000", lambda: stencil("cd")),
             "powerlaw2M": ("powerlaw_2M", lambda: P.CsrMatrix(*G.powerlaw_spd(2_000_000, seed=0))),
             "powerlaw8M": ("config3_powerlaw_8M", lambda: G.powerlaw_spd_device(8_000_000, seed=0))}
    mats = {build[w][0]: build[w][1]() for w in which}
    s = device.thread_stream()
    ext = torch.cuda.ExternalStream(s.handle)
    out = {"peak_gbs": PEAK, "runs": RUNS, "dtype": "f32" if F32 else "f64", "results": {}}
    for name, A in mats.items():
        n = A.nrows
        xh = np.random.default_rng(0).uniform(0.5, 1.5, n)
        x = device.DeviceVector.from_numpy(xh.astype(np.float32) if F32 else xh, s)
        y = device.DeviceVector(n, np.float32) if F32 else device.DeviceVector(n)
        res = {}
        reps = {}
        only = os.environ.get("SWEEP_TOKENS")
        for cfg in P.enumerate_configs():
            if only and cfg.token() not in only.split(","):
                continue
            f = cfg.format
            if f not in reps:
                try:
                    reps[f] = A if f is P.FormatTag.CSR else P.convert(A, f)
                except (P.FormatInapplicableError, MemoryError) as exc:
                    reps[f] = None
                    res[f.value] = f"inapplicable: {exc}"[:120]
            rep = reps[f]
            if rep is None:
                continue
            for _ in range(3):
                launch(cfg, rep, x.ptr, y.ptr, workers=4, f32=F32, stream=s)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(ext)
            for _ in range(RUNS):
                launch(cfg, rep, x.ptr, y.ptr, workers=4, f32=F32, stream=s)
            e1.record(ext)
            e1.synchronize()
            us = e0.elapsed_time(e1) / RUNS * 1e3
            b = alg_bytes(f.value, rep, n, n, cfg.library.value if hasattr(cfg.library, "value") else str(cfg.library))
            res[cfg.token()] = {"us": round(us, 2), "alg_MB": round(b / 1e6, 1),
                                "gbs": round(b / us / 1e3, 1), "frac": round(b / us / 1e3 / PEAK, 3)}
        out["results"][name] = {"n": n, "nnz": A.nnz, "configs": res}
        print(name, json.dumps(res), file=sys.stderr, flush=True)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
