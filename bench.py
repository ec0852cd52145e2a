"""Benchmark: CG time-to-solution including preprocessing, row-partitioned, on B200.

Workload (every N): BASELINE.json configs[4], the largest configuration that
fits one GPU and the north star's scaling target — CG fp64, tol 1e-8,
b = A*1, on the 3-D 27-point Laplacian 600^3 (n = 216,000,000,
nnz = 5,812,581,592), rows split into z-slabs across N ranks (N = 1: one
slab).  One step = the reference's predict-then-solve flow (solver.py:
496-540) on the row-partitioned operator: exact global features -> cascade
(the reference's shipped models) -> conversion of each rank's slab to the
predicted format -> CG with NCCL halo exchange + scalar all-reduces.  The
same code path runs at N = 1, 2, 4, 8 (strong scaling: the problem is fixed).

  value   — seconds per solve, slabs generated in HBM before the clock
  e2e     — the same solve through distributed_solve_slab from each rank's
            PINNED HOST slab (row_ptr int64, global col_idx int32, values f64,
            b): upload + device validation inside the clock, x back to host
  roofline — the dominant kernel (the local SpMV in the predicted format),
            algorithmic bytes per SURVEY §8(d) / its average launch time
            from CUDA events on the solver stream over one instrumented solve
  cpu_baseline — the reference algorithm (oracle port) on the host cores,
            bounded 120^3 sample scaled per nnz (the 600^3 matrix does not fit
            the host), with a 150^3 / 300^3 linearity check in the reference arm
  detail  — (N = 1) config 2 (GMRES(30) async predict-while-solve, 4 M rows,
            e2e, default CSR-vector and sequential), config 1 (CG Poisson
            1024^2) and config 3 (CG power-law 8 M rows) on one B200

`python bench.py --gpus N` without torchrun re-launches itself under
torch.distributed.run with N ranks; under torchrun WORLD_SIZE must equal N.
`--impl reference` prints the reference arm (CPU oracle port) instead.
"""
from __future__ import annotations

import argparse
import gc
import json
import os
import socket
import statistics
import subprocess
import sys
import tempfile
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))
# load every kernel at context creation: a lazily loaded kernel's first
# launch must not land inside a timed step
os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")

TOL = 1e-8
N3 = int(os.environ.get("SPMVTUNE_CONFIG5_N", "600"))
NX2 = 2000
RESTART = 30
METRIC = "CG time-to-solution incl. preprocessing (features+cascade+conversion)"
METRIC2 = "GMRES(30) time-to-solution incl. preprocessing (features+cascade+conversion)"


def workload5(n3: int = N3) -> str:
    return (f"config5: CG fp64, tol {TOL:g}, b=A*1, 3-D 27-point Laplacian {n3}^3 "
            f"(n={n3 ** 3:,}, nnz={(3 * n3 - 2) ** 3:,}); row-partitioned z-slabs, predict-then-solve "
            "(exact global features -> shipped cascade models -> per-rank conversion), NCCL halo + "
            "all-reduce; the same code path at every N")


WORKLOAD2 = (f"config2: GMRES({RESTART}) fp64, tol {TOL:g}, b=A*1, nonsymmetric 9-point "
             f"convection-diffusion {NX2}x{NX2} (n={NX2 * NX2:,}, nnz={(3 * NX2 - 2) ** 2:,}); async "
             "predict-while-solve starting on CSR/LibA/32 with the reference's shipped cascade models")


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy bandwidth)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def self_launch(args) -> int:
    """`--gpus N` without torchrun: run this script under torch.distributed.run
    with N ranks (one per GPU) and pass its output and exit code through."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={free_port()}", str(Path(__file__).resolve())]
    cmd += sys.argv[1:]
    return subprocess.call(cmd, cwd=ROOT)


# ---------------------------------------------------------------------------
# reference arm: the CPU oracle port on the host cores
# ---------------------------------------------------------------------------
def _oracle_env():
    env = dict(os.environ)
    env["OPENBLAS_NUM_THREADS"] = str(os.cpu_count() or 1)
    env.pop("CUDA_VISIBLE_DEVICES", None)
    return env


def run_oracle(args_list, timeout=1800) -> dict:
    o = subprocess.run([sys.executable, "-m", "oracle.bench_cpu", *args_list], cwd=ROOT, env=_oracle_env(),
                       capture_output=True, text=True, timeout=timeout)
    if o.returncode != 0:
        raise RuntimeError(o.stderr[-2000:])
    return json.loads(o.stdout.strip().splitlines()[-1])


def cpu_config5_sample(total_iters: int, n3: int = 120, iters: int = 4) -> dict:
    return run_oracle(["--laplace27", str(n3), "--iters", str(iters), "--total-iters", str(total_iters),
                       "--target", str(N3)])


def reference_arm(args):
    """The reference's CPU path (oracle port, bit-exact to /root/reference)
    on the host cores, same workload, metric and unit as the B200 arm.  The
    600^3 matrix (94.7 GB as int64 CSR) does not fit the host's RAM next to
    its conversions, so each step is a bounded 120^3 sample of the
    predict-then-solve flow, scaled per nnz (EXTRAPOLATED — labelled); a
    150^3 and a 300^3 sample check that per-nnz scaling is linear; config 2
    runs in full (async flow, measured, not extrapolated) in `detail`."""
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    t0 = time.perf_counter()
    total_iters = args.total_iters
    vals, last = [], None
    for k in range(args.warmup + args.steps):
        last = cpu_config5_sample(total_iters)
        if k >= args.warmup:
            vals.append(last["value"])
    value = statistics.median(vals)
    detail = {"per_step_values": vals, "phases": last["phases"], "config": last["config"],
              "per_iteration_s_extrapolated": last["per_iteration_s"], "total_iterations": total_iters}
    if not args.no_extra:
        lin = {}
        for n3 in (150, 300):
            try:
                r = cpu_config5_sample(total_iters, n3=n3, iters=2)
                lin[f"{n3}^3"] = {"extrapolated_s": r["value"], "per_iteration_s": r["per_iteration_s"],
                                  "sampled_nnz": r.get("sampled_nnz")}
            except Exception as exc:
                lin[f"{n3}^3"] = f"failed: {exc}"[:300]
        if all(isinstance(v, dict) for v in lin.values()):
            a, b = lin["150^3"]["extrapolated_s"], lin["300^3"]["extrapolated_s"]
            lin["ratio_300_over_150"] = b / a     # 1.0 = per-nnz scaling is linear
        detail["linearity_check"] = lin
        try:
            detail["config2_cpu_async_measured"] = run_oracle(["--nx", str(NX2), "--async-full"], timeout=1200)
        except Exception as exc:
            detail["config2_cpu_async_measured"] = f"failed: {exc}"[:300]
    detail["wall_seconds"] = time.perf_counter() - t0
    line = {"metric": METRIC, "value": value, "unit": "s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": value * 1e3,
            "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "impl": "reference",
            "config": {"workload": workload5(), "mode": "predict-then-solve (CPU, reference algorithm)"},
            "cpu_baseline": {"value": value, "unit": "s", "cores": last["cores"], "kind": last["kind"],
                             "sample": last["sample"], "cpu_model": last.get("cpu_model")},
            "e2e": {"value": value, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "extrapolated": True,
            "detail": detail}
    emit(line)


# ---------------------------------------------------------------------------
# measurement helpers
# ---------------------------------------------------------------------------
class EventTimer:
    """CUDA-event pairs around solver launches, recorded on the launching
    stream (the solver's own stream, not torch's current one)."""

    def __init__(self):
        import torch
        self.torch = torch
        self.streams = {}
        self.open = {}
        self.done = []

    def _stream(self, h):
        s = self.streams.get(h)
        if s is None:
            s = self.streams[h] = self.torch.cuda.ExternalStream(h)
        return s

    def begin(self, tag, h):
        ev = self.torch.cuda.Event(enable_timing=True)
        ev.record(self._stream(h))
        self.open[tag] = ev

    def end(self, tag, h):
        ev = self.torch.cuda.Event(enable_timing=True)
        ev.record(self._stream(h))
        self.done.append((tag, self.open.pop(tag), ev))

    def summary(self):
        self.torch.cuda.synchronize()
        out = {}
        for tag, a, b in self.done:
            out.setdefault(tag, []).append(a.elapsed_time(b))
        return out


class NvmlClockSampler:
    """In-process NVML sampling of SM clock and throttle reasons during the
    timed region.  (An `nvidia-smi -lms` child process holds driver locks
    long enough to stall CUDA API calls by tens of ms; NVML reads are cheap.)"""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "sw_power_cap": 0x4}

    def __init__(self, index: int, period: float = 0.02):
        import pynvml
        self.nv = pynvml
        pynvml.nvmlInit()
        self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
        self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        self.samples = []
        self.stop_ev = threading.Event()
        self.period = period
        self.t = threading.Thread(target=self._run, daemon=True)
        self.t.start()

    def _sample(self):
        nv = self.nv
        sm = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
        reasons = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
        util = nv.nvmlDeviceGetUtilizationRates(self.h).gpu
        self.samples.append((sm, reasons, util))

    def _run(self):
        while not self.stop_ev.is_set():
            try:
                self._sample()
            except Exception:
                pass
            self.stop_ev.wait(self.period)

    def stop(self) -> dict:
        self.stop_ev.set()
        self.t.join()
        try:
            self._sample()
        except Exception:
            pass
        loaded = [s for s in self.samples if s[2] > 0] or self.samples
        reasons = sorted({name for s in loaded for name, bit in self.REASONS.items() if s[1] & bit})
        sm = [s[0] for s in loaded]
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": self.max_mhz,
                "reasons": reasons, "samples": len(self.samples), "samples_under_load": len(loaded),
                "source": "nvml"}


class ClockSampler:
    """nvidia-smi fallback when NVML is unavailable."""

    def __init__(self, index: int):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap,utilization.gpu")
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--query-gpu={q}", "--format=csv,noheader,nounits",
                                       "-i", str(index), "-lms", "200"], stdout=self.f,
                                      stderr=subprocess.DEVNULL)
        except FileNotFoundError:
            self.p = None

    def stop(self) -> dict:
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        self.p.wait()
        self.f.flush()
        rows = [[x.strip() for x in line.split(",")] for line in Path(self.f.name).read_text().splitlines()]
        rows = [r for r in rows if len(r) >= 8]
        os.unlink(self.f.name)
        loaded = [r for r in rows if r[7].isdigit() and int(r[7]) > 0] or rows
        sm = [float(r[0]) for r in loaded if r[0].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = {name for r in loaded for k, name in enumerate(names) if r[3 + k].lower() == "active"}
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": float(loaded[0][1]) if loaded else None,
                "reasons": sorted(reasons), "samples": len(rows), "samples_under_load": len(loaded)}


def clock_sampler(index: int):
    try:
        return NvmlClockSampler(index)
    except Exception:
        return ClockSampler(index)


def algorithmic_bytes(tok: str, info, n: int, ncols: int | None = None) -> float:
    """Bytes per SpMV launch per SURVEY.md §8(d) (device layout: fp64 values,
    int32 column indices; x read once, y written once)."""
    fmt = tok.split("/")[0]
    nnz = info["nnz"]
    ncols = n if ncols is None else ncols
    ptrb = 8 if info.get("ptr64") else 4
    if fmt == "CSR":
        return 12 * nnz + ptrb * (n + 1) + 8 * ncols + 8 * n
    if fmt == "DIA":
        return 8 * info["ndiag"] * n + 8 * ncols + 8 * n
    if fmt == "ELL":
        return 12 * n * info["width"] + 8 * ncols + 8 * n
    if fmt == "HYB":
        return 12 * n * info["width"] + 16 * info["spill"] + 8 * ncols + 16 * n
    if tok.startswith("COO/LibA"):               # row kernel over cached run starts
        return 12 * nnz + 8 * (n + 1) + 8 * ncols + 8 * n
    return 16 * nnz + 8 * ncols + 8 * n          # COO (rows + cols + vals)


def mgs_bytes(n: int, j: int, resident: bool = True) -> float:
    """Algorithmic bytes of one Arnoldi orthogonalisation at column j: the
    resident kernel reads w and V_0..V_j once and writes V_{j+1} once ->
    8n(j+3); the streaming fallback re-reads w every pass."""
    if resident:
        return 8 * n * (j + 3)
    return 16 * n + 32 * n * j + 24 * n + 16 * n


def info_of(mat) -> dict:
    inf = mat._device().info
    return {"nnz": int(inf.nnz), "ndiag": int(inf.ndiag), "width": int(inf.width),
            "spill": int(inf.spill_nnz), "ptr64": bool(inf.ptr64)}


def load_traffic(tag: str):
    """ncu dram bytes per launch of `tag` (profiles/ncu_traffic.json, written
    from one `ncu --set full` capture), or None."""
    prof = ROOT / "profiles" / "ncu_traffic.json"
    if prof.exists():
        return json.loads(prof.read_text()).get(tag)
    return None


# ---------------------------------------------------------------------------
# the B200 arm: config 5, row-partitioned, every N
# ---------------------------------------------------------------------------
def stencil27():
    offs, wts = [], []
    for dz in (-1, 0, 1):
        for dy in (-1, 0, 1):
            for dx in (-1, 0, 1):
                offs.append((dz, dy, dx))
                wts.append(26.0 if (dx, dy, dz) == (0, 0, 0) else -1.0)
    return offs, wts


def b200_arm(args):
    ws, rank, local = dist_env()
    # SPMVTUNE_DIST_BACKEND=gloo: every rank on GPU 0, collectives staged
    # through the host (HostStagedComm) — exercises the N > 1 path of this
    # script on a one-GPU box; not a performance mode
    host_staged = os.environ.get("SPMVTUNE_DIST_BACKEND") == "gloo"
    if host_staged:
        local = 0
    os.environ.setdefault("SPMVTUNE_DEVICE", str(local))
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2411_10143_b200 as P
    from paper_2411_10143_b200 import _lib, device
    from paper_2411_10143_b200.distributed import (HostStagedComm, distributed_solve_slab,
                                                    distributed_stencil_solve, stencil_block,
                                                    stencil_partition)
    from paper_2411_10143_b200.solver import DeviceOptions

    torch.cuda.set_device(local)
    if not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", str(29517))
        if host_staged:
            dist.init_process_group("gloo", rank=rank, world_size=ws)
        else:
            dist.init_process_group("nccl", rank=rank, world_size=ws, device_id=torch.device("cuda", local))
    comm_class = HostStagedComm if host_staged else None
    L = _lib.lib()

    dims = (N3, N3, N3)
    offs, wts = stencil27()
    models = P.CascadeModelSet.load_dir(ROOT / "tests" / "golden" / "models")
    params = P.GmresParams(tol=TOL, max_iters=20000)
    bounds = stencil_partition(dims, ws)
    r0, r1 = int(bounds[rank]), int(bounds[rank + 1])
    s = device.thread_stream(0)
    ext = torch.cuda.ExternalStream(s.handle)
    t0 = time.perf_counter()
    blk = stencil_block(dims, offs, wts, r0, r1, s)          # this rank's slab, generated in HBM
    gen_s = time.perf_counter() - t0

    def step(timer=None):
        t = {}
        with DeviceOptions(timer=timer):
            res, _ = distributed_stencil_solve("cg", dims, offs, wts, params, models=models, blk=blk,
                                               comm_class=comm_class, timings=t)
        return res, t

    for _ in range(args.warmup):
        step()

    # --- timed region (slabs resident in HBM) -------------------------------
    clocks = clock_sampler(local)
    launches0 = _lib.launch_count()
    dist.barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    gc.collect()
    gc.disable()        # no cyclic-GC pauses inside the timed steps
    ev0.record(ext)
    wall0 = time.perf_counter()
    steps, results = [], []
    for _ in range(args.steps):
        res, t = step()
        steps.append(t)
        results.append({k: res[k] for k in ("converged", "iterations", "final", "config")})
    ev1.record(ext)
    torch.cuda.synchronize()
    wall = time.perf_counter() - wall0
    gc.enable()
    dist.barrier()
    clk = clocks.stop()
    launches = _lib.launch_count() - launches0
    dev_s = ev0.elapsed_time(ev1) / 1e3
    region = torch.tensor([max(dev_s, wall)], device="cpu" if host_staged else "cuda")
    dist.all_reduce(region, op=dist.ReduceOp.MAX)
    value = float(region.item()) / args.steps
    its = results[-1]["iterations"]

    # --- dominant kernel: events around every local SpMV of one instrumented
    # solve on the solver stream (kept out of `value`: per-launch event
    # records add host work)
    timer = EventTimer()
    res_i, t_i = step(timer)
    kern = timer.summary()
    cfg = P.SpmvConfig.from_token(results[-1]["config"])
    tag = "spmv:" + cfg.token()
    mat = blk._dev_csr if cfg.format is P.FormatTag.CSR else P.convert(blk._dev_csr, cfg.format)
    inf = info_of(mat)
    del mat
    hbm, peak_kind = peaks()
    ms = kern.get(tag, [])
    spmv_bytes = algorithmic_bytes(cfg.token(), inf, blk.nloc, blk.window)
    parts = 1 if (ws == 1) else max(1, round(len(ms) / max(1, res_i["iterations"] + 1)))
    spmv_total_ms = sum(ms)
    applies = len(ms) / parts
    avg_ms = spmv_total_ms / max(1.0, applies)           # one local SpMV (all its row parts)
    gbs = spmv_bytes / (avg_ms / 1e3) / 1e9 if ms else 0.0
    roofline = {"kernel": tag + (" (k_dia)" if cfg.format is P.FormatTag.DIA else ""), "bound": "hbm",
                "achieved": round(gbs, 1), "peak": hbm, "unit": "GB/s", "frac": round(gbs / hbm, 4),
                "traffic": load_traffic(f"config5:{tag}") if ws == 1 else None, "peak_kind": peak_kind,
                "bytes_per_launch": spmv_bytes, "avg_launch_ms": avg_ms, "launches": len(ms),
                "share_of_step": spmv_total_ms / 1e3 / max(1e-9, t_i["total_s"]),
                "bytes_formula": "8*ndiag*n + 8*window + 8*n (DIA; SURVEY §8d)"}

    # --- e2e: the same solve from this rank's pinned host slab ----------------
    e2e = None
    if not args.no_e2e:
        e2e = e2e_slab(args, blk, r0, r1, params, models, comm_class, ws)
    gathered = [None] * ws
    dist.all_gather_object(gathered, {"rank": rank, "rows": [r0, r1], "gen_s": gen_s,
                                      "last_step": steps[-1], "spmv_ms": avg_ms, "gbs": gbs})
    del blk
    gc.collect()

    cpu, detail = None, {}
    if rank == 0 and ws == 1:
        if not args.no_cpu:
            try:
                r = cpu_config5_sample(its)
                cpu = {k: r[k] for k in ("value", "unit", "cores", "kind", "sample", "cpu_model")}
                cpu["extrapolated"] = True
            except Exception as exc:  # measurement must not kill the bench line
                cpu = {"value": None, "unit": "s", "cores": os.cpu_count(), "kind": "port",
                       "sample": f"failed: {exc}"[:300]}
        if not args.no_extra:
            for name, fn in (("config2_gmres_async", config2_detail), ("config1_cg", config1_detail),
                             ("config3_cg_powerlaw", config3_detail)):
                try:
                    detail[name] = fn(args, P, device, _lib, models)
                except Exception as exc:
                    detail[name] = f"failed: {type(exc).__name__}: {exc}"[:400]
    dist.barrier()
    if rank == 0:
        detail.update({"results": results[-1], "per_step": steps, "per_rank": gathered,
                       "per_iteration_solve_s": steps[-1]["solve_s"] / max(1, its),
                       "device_region_s": dev_s, "wall_region_s": wall,
                       "slab_generation_s_rank0": gen_s})
        line = {"metric": METRIC, "value": value, "unit": "s", "n_gpus": ws, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": value * 1e3, "higher_is_better": False,
                "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {"workload": workload5(), "parallelism": f"row-partitioned x{ws}",
                           "comm": ("gloo, host-staged (path validation, not a performance number)"
                                    if host_staged else "nccl") + (
                               "; per-iteration all-reduces and halo by peer-memory kernels (PeerComm)"
                               if ws > 1 and os.environ.get("SPMVTUNE_P2P", "1") != "0" else ""),
                           "l2": "inputs larger than L2 (47 GB DIA + 71.5 GB CSR per GPU at N=1, 126 MB L2)"},
                "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches),
                "clocks": clk, "detail": detail}
        emit(line)
    dist.destroy_process_group()


def e2e_slab(args, blk, r0, r1, params, models, comm_class, ws):
    """Every rank copies its slab to pinned host memory once (outside the
    clock), drops the device copy, then times solves through the public
    per-rank entry point distributed_solve_slab: H2D of row_ptr/col_idx/
    values/b + device validation + global features + cascade + conversion +
    CG + D2H of x, all inside the clock."""
    import ctypes

    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2411_10143_b200 import _lib, device
    from paper_2411_10143_b200.distributed import distributed_solve_slab
    L = _lib.lib()
    s = device.thread_stream(0)
    csr = blk._dev_csr
    n = blk.ncols_global
    nloc, nnz = blk.nloc, (csr.nnz if csr is not None else 0)
    handles = []

    def pinned(count, dtype):
        if count == 0:
            return np.zeros(0, dtype)
        h = ctypes.c_void_p()
        nbytes = int(count) * np.dtype(dtype).itemsize
        _lib.check(L.svb_host_alloc(nbytes, ctypes.byref(h)))
        handles.append(h.value)
        return np.frombuffer((ctypes.c_char * nbytes).from_address(h.value), dtype=dtype, count=int(count))

    t0 = time.perf_counter()
    hp, hc, hv, hb = pinned(nloc + 1, np.int64), pinned(nnz, np.int32), pinned(nnz, np.float64), \
        pinned(nloc, np.float64)
    if csr is not None:
        _lib.check(L.svb_csr_export(csr._device().handle, blk.cmin, hp.ctypes.data, hc.ctypes.data,
                                    hv.ctypes.data, s.handle))
        # b = A*1 on this rank's rows, as the device-resident arm computes it
        ones = device.DeviceVector(blk.window)
        _lib.check(L.svb_fill(ones.ptr, blk.window, 1.0, s.handle))
        bd = device.DeviceVector(nloc)
        _lib.check(L.svb_spmv_sequential(csr._device().handle, ones.ptr, bd.ptr, s.handle))
        device.copy(hb.ctypes.data, bd.ptr, bd.nbytes, s)
        s.sync()
        del ones, bd
    else:
        hp[:] = 0
    prep_s = time.perf_counter() - t0
    blk._dev_csr = None                      # the slab now lives on the host only
    del csr
    gc.collect()

    def one():
        t = {}
        res = distributed_solve_slab("cg", r0, r1, n, hp, hc, hv, hb, params, models=models, timings=t,
                                     comm_class=comm_class)
        return res, t

    one()                                     # warm (pool growth, first use of the slab path)
    k = max(1, min(args.steps, args.e2e_steps))
    dist.barrier()
    torch.cuda.synchronize()
    w0 = time.perf_counter()
    phases = []
    for _ in range(k):
        res, t = one()
        phases.append(t)
    torch.cuda.synchronize()
    wall = time.perf_counter() - w0
    dist.barrier()
    dev = "cpu" if comm_class else "cuda"
    tt = torch.tensor([wall], device=dev)
    dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    byts = torch.tensor([hp.nbytes + hc.nbytes + hv.nbytes + hb.nbytes, 8 * nloc], dtype=torch.float64,
                        device=dev)
    dist.all_reduce(byts)
    del hp, hc, hv, hb
    for h in handles:
        L.svb_host_free(h)
    return {"value": float(tt.item()) / k, "unit": "s", "h2d_bytes_per_step": int(byts[0].item()),
            "d2h_bytes_per_step": int(byts[1].item()), "steps": k, "iterations": res["iterations"],
            "converged": res["converged"], "final_residual": res["final"], "phases_last": phases[-1],
            "phases": phases,
            "host_slab_prep_s": prep_s,
            "note": "each rank: pinned host slab (row_ptr int64, GLOBAL col_idx int32, values f64, b f64) -> "
                    "distributed_solve_slab (H2D + device validation + features + cascade + conversion + "
                    "CG) -> x slice to host; max over ranks; totals over ranks"}


# ---------------------------------------------------------------------------
# single-GPU detail workloads (N = 1, rank 0)
# ---------------------------------------------------------------------------
def _timed(fn, reps=3):
    import torch
    ts, rep = [], None
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        rep = fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
        if hasattr(rep, "solution"):
            rep.solution = None
    _timed.last = [round(t, 6) for t in ts]       # every rep, so slow outliers stay visible
    return statistics.median(ts), rep


def config2_detail(args, P, device, _lib, models) -> dict:
    """BASELINE configs[1]: GMRES(30) async predict-while-solve (the paper's
    AsyGMRES) on one B200, device-resident and end to end from pinned host
    CSR, against the default CSR-vector solve and predict-then-solve, with
    the Arnoldi kernel's roofline from per-launch events."""
    import numpy as np
    import torch
    from paper_2411_10143_b200.solver import DeviceOptions
    offs, wts = [], []
    for dy in (-1, 0, 1):
        for dx in (-1, 0, 1):
            offs.append((dy, dx))
            wts.append(8.5 if (dx, dy) == (0, 0) else -1.0 - 0.25 * (dx + dy))
    A = P.CsrMatrix.stencil((NX2, NX2), offs, wts)
    n = A.nrows
    params = P.GmresParams(restart_m=RESTART, tol=TOL, max_iters=1000)
    start = P.GPU_DEFAULT_CONFIG
    s = device.thread_stream()
    ones = device.DeviceVector.from_numpy(np.ones(n), s)
    b_dev = device.DeviceVector(n)
    _lib.check(_lib.lib().svb_spmv_sequential(A._device().handle, ones.ptr, b_dev.ptr, s.handle))
    s.sync()
    out = {"workload": WORKLOAD2, "metric": METRIC2}
    with DeviceOptions(keep_solution_on_device=True):
        for _ in range(3):
            P.async_solve(A, b_dev, params, models, initial_config=start).solution = None
        reps = max(5, min(args.steps, 20))
        ts, swaps = [], []
        for _ in range(reps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            r = P.async_solve(A, b_dev, params, models, initial_config=start)
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t0)
            swaps.append([(x.iteration, x.config.token()) for x in r.config_timeline])
            r.solution = None
        out.update({"async_s": statistics.median(ts), "async_runs_s": ts, "iterations": r.iterations,
                    "converged": r.converged, "final_residual": r.final_residual, "swaps": swaps[-1]})
        out["default_csr_vector_s"], d = _timed(lambda: P.gmres_solve(A, b_dev, params, initial_config=start))
        out["default_iterations"] = d.iterations
        out["sequential_s"], sq = _timed(lambda: P.sequential_predict_solve(A, b_dev, params, models))
        out["sequential_phases"] = sq.phases
        timer = EventTimer()
        with DeviceOptions(timer=timer, keep_solution_on_device=True):
            ri = P.async_solve(A, b_dev, params, models, initial_config=start)
        kern = timer.summary()
    hbm, _ = peaks()
    groups = {}
    for tag, ms in kern.items():
        tot = sum(ms)
        if tag.startswith("spmv:"):
            tok = tag.split(":", 1)[1]
            mat = A if tok.startswith("CSR") else P.convert(A, P.SpmvConfig.from_token(tok).format)
            byts = algorithmic_bytes(tok, info_of(mat), n) * len(ms)
        elif tag == "mgs":
            js = [it % RESTART for it in range(ri.iterations)]
            byts = sum(mgs_bytes(n, j) for j in js[:len(ms)])
        else:
            continue
        groups[tag] = {"launches": len(ms), "ms_avg": tot / len(ms), "gbs": byts / (tot / 1e3) / 1e9,
                       "frac": byts / (tot / 1e3) / 1e9 / hbm, "share_of_solve": tot / 1e3 / out["async_s"]}
    out["kernels"] = groups
    # e2e from pinned host CSR (int64 indices, the reference layout)
    rp, ci, vv = np.asarray(A.row_ptr), np.asarray(A.col_idx), np.asarray(A.values)
    bh = b_dev.to_numpy(s)
    pin = {}
    for k, arr in (("rp", rp), ("ci", ci), ("vv", vv), ("b", bh)):
        t = torch.empty(arr.size, dtype=torch.from_numpy(arr[:1].copy()).dtype, pin_memory=True)
        t.numpy()[:] = arr
        pin[k] = t
    Ah = P.CsrMatrix(n, n, pin["rp"].numpy(), pin["ci"].numpy(), pin["vv"].numpy())
    b_host = pin["b"].numpy()

    def e2e_step():
        Ah._dev = None                      # drop the device copy: upload inside the clock
        return P.async_solve(Ah, b_host, params, models, initial_config=start)
    e2e_step()
    k = max(5, min(args.steps, 20))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(k):
        re = e2e_step()
    torch.cuda.synchronize()
    out["e2e"] = {"value": (time.perf_counter() - t0) / k, "unit": "s", "steps": k,
                  "h2d_bytes_per_step": int(rp.nbytes + ci.nbytes + vv.nbytes + bh.nbytes),
                  "d2h_bytes_per_step": int(re.solution.nbytes + 48 * (re.iterations + 4)),
                  "note": "CsrMatrix from pinned host int64/f64 arrays -> async_solve -> solution to host"}
    return out


def config1_detail(args, P, device, _lib, models) -> dict:
    """BASELINE configs[0]: CG fp64 on the 2-D 5-point Poisson 1024^2
    (n = 1,048,576, nnz = 5,238,784), tol 1e-8, b = A*1; async
    predict-while-solve from CSR/LibA/32 vs the fixed default CSR-vector solve."""
    import numpy as np
    from paper_2411_10143_b200.solver import DeviceOptions
    A = P.CsrMatrix.stencil((1024, 1024), [(0, 0), (0, -1), (0, 1), (-1, 0), (1, 0)],
                            [4.0, -1.0, -1.0, -1.0, -1.0])
    s = device.thread_stream()
    ones = device.DeviceVector.from_numpy(np.ones(A.nrows), s)
    b = device.DeviceVector(A.nrows)
    _lib.check(_lib.lib().svb_spmv_sequential(A._device().handle, ones.ptr, b.ptr, s.handle))
    s.sync()
    params = P.GmresParams(tol=TOL, max_iters=5000)
    start = P.GPU_DEFAULT_CONFIG
    out = {"workload": "config1: CG fp64 Poisson 1024^2, tol 1e-8, b=A*1"}
    with DeviceOptions(keep_solution_on_device=True):
        P.async_solve(A, b, params, models, method="cg", initial_config=start).solution = None
        out["async_s"], r = _timed(lambda: P.async_solve(A, b, params, models, method="cg",
                                                         initial_config=start), reps=5)
        out["async_reps_s"] = _timed.last
        out.update({"iterations": r.iterations, "converged": r.converged, "final_residual": r.final_residual,
                    "swaps": [(x.iteration, x.config.token()) for x in r.config_timeline]})
        out["default_csr_vector_s"], d = _timed(lambda: P.cg_solve(A, b, params, initial_config=start), reps=3)
        out["default_reps_s"] = _timed.last
        out["default_iterations"] = d.iterations
    return out


def config3_detail(args, P, device, _lib, models) -> dict:
    """BASELINE configs[2]: CG on the power-law SPD matrix (8 M rows, ~112 M
    nnz; device-built, bit-identical to generators.powerlaw_spd), b random
    seed 0 (solver.py:190-191), tol 1e-8: async from CSR/LibA/32 with the
    shipped and the B200-trained cascade, vs the default CSR-vector solve."""
    from paper_2411_10143_b200 import generators as G
    from paper_2411_10143_b200.solver import DeviceOptions, default_rhs
    t0 = time.perf_counter()
    A = G.powerlaw_spd_device(8_000_000, seed=0)
    gen_s = time.perf_counter() - t0
    params = P.GmresParams(tol=TOL, max_iters=20000, rhs="random", seed=0)
    start = P.GPU_DEFAULT_CONFIG
    b = default_rhs(A, params)
    out = {"workload": f"config3: CG fp64 power-law SPD n={A.nrows:,} nnz={A.nnz:,}, b random seed 0",
           "generation_s": gen_s}
    b200 = P.CascadeModelSet.load_dir(P.B200_MODELS_DIR)
    with DeviceOptions(keep_solution_on_device=True):
        for name, ms in (("shipped", models), ("b200", b200)):
            P.async_solve(A, b, params, ms, method="cg", initial_config=start).solution = None
            t, r = _timed(lambda: P.async_solve(A, b, params, ms, method="cg", initial_config=start))
            out[f"async_{name}_models_s"] = t
            out[f"async_{name}_models"] = {"iterations": r.iterations, "converged": r.converged,
                                           "swaps": [(x.iteration, x.config.token()) for x in r.config_timeline]}
        out["default_csr_vector_s"], d = _timed(lambda: P.cg_solve(A, b, params, initial_config=start))
        out["default_iterations"] = d.iterations
    return out


_RESULT_OUT = None


def _claim_stdout() -> None:
    """Keep stdout for the one JSON line: whatever native libraries write to
    fd 1 (NCCL prints its version banner there when NCCL_DEBUG is set) goes
    to stderr.  Called in the process that measures, never before
    self_launch (the ranks inherit fd 1)."""
    global _RESULT_OUT
    if _RESULT_OUT is None:
        sys.stdout.flush()
        _RESULT_OUT = os.fdopen(os.dup(1), "w")
        os.dup2(2, 1)


def emit(line: dict) -> None:
    out = _RESULT_OUT or sys.stdout
    out.write(json.dumps(line) + "\n")
    out.flush()


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--total-iters", type=int, default=763,
                    help="reference arm: CG iterations the 600^3 solve takes (763, measured on B200)")
    ap.add_argument("--e2e-steps", type=int, default=3, help="timed e2e solves (each re-uploads the slab)")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-e2e", action="store_true", help="skip the e2e leg")
    ap.add_argument("--no-extra", action="store_true", help="skip the config 1/2/3 detail workloads")
    args = ap.parse_args(argv)
    if args.warmup < 0 or args.steps < 1 or args.gpus < 1:
        raise SystemExit("--steps >= 1, --warmup >= 0, --gpus >= 1")
    if args.impl == "reference":
        _claim_stdout()
        reference_arm(args)
        return 0
    ws_env = os.environ.get("WORLD_SIZE")
    if ws_env is None and args.gpus > 1:
        return self_launch(args)
    if ws_env is not None and int(ws_env) != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={ws_env}: launch one rank per GPU")
    _claim_stdout()
    b200_arm(args)
    return 0


if __name__ == "__main__":
    sys.exit(main())
