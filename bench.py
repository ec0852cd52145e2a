"""Benchmark: GMRES(30) time-to-solution including preprocessing on B200.

Workload (BASELINE.json configs[1], the metric's single-GPU configuration):
GMRES(30), fp64, tol 1e-8, b = A*1, on the nonsymmetric 9-point
convection-diffusion matrix 2000x2000 (n = 4,000,000, nnz = 35,976,004).
One step = one full async predict-while-solve (the paper's AsyGMRES): the
solve starts at once on the default CSR-vector kernel (CSR/LibA/32) while
the advisor stream extracts features, runs the shipped cascade models and
converts to the predicted format; the solver swaps mid-solve.  Time to
solution therefore includes all preprocessing.

  value  — seconds per solve with the matrix and b resident in HBM
  e2e    — the same solve through the public API from pinned HOST buffers:
           CSR upload (H2D) inside the clock, solution download (D2H)
  roofline — the dominant kernel group of the step, bytes per §8(d),
           timed with CUDA events on the solver stream inside the timed steps
  cpu_baseline — the reference algorithm (oracle port, bit-exact to the
           reference) on the host cores, bounded sample (oracle/bench_cpu.py)

`--impl reference` prints the reference arm (CPU oracle port) instead.
Multi-GPU (torchrun, N > 1): the row-partitioned solver (distributed.py) on
the same config-2 problem — each rank generates its slab on its GPU, the
cascade runs on exact global features, SpMV halos and dot products go over
NCCL (strong scaling, value = max over ranks).  `--workload config5` runs
BASELINE configs[4] (row-partitioned CG, 27-point Laplacian 600^3) the same
way at any N, including N = 1.
"""
from __future__ import annotations

import argparse
import gc
import json
import os
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

NX = 2000
TOL = 1e-8
RESTART = 30
METRIC = "GMRES(30) time-to-solution incl. preprocessing (features+cascade+conversion)"
METRIC5 = "CG time-to-solution incl. preprocessing (features+cascade+conversion)"
WORKLOAD = (f"config2: GMRES({RESTART}) fp64, tol {TOL:g}, b=A*1, nonsymmetric 9-point "
            f"convection-diffusion {NX}x{NX} (n={NX * NX:,}, nnz={(3 * NX - 2) ** 2:,}); async "
            "predict-while-solve starting on CSR/LibA/32 with the reference's shipped cascade "
            "models")


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


# ---------------------------------------------------------------------------
# reference arm: the CPU oracle port on the host cores
# ---------------------------------------------------------------------------
def run_cpu_sample(steps: int, warmup: int, total_iters: int, iters: int = 8) -> dict:
    env = dict(os.environ)
    env["OPENBLAS_NUM_THREADS"] = str(os.cpu_count() or 1)
    env.pop("CUDA_VISIBLE_DEVICES", None)
    cmd = [sys.executable, "-m", "oracle.bench_cpu", "--nx", str(NX), "--iters", str(iters),
           "--total-iters", str(total_iters), "--repeat", str(steps), "--warmup", str(warmup)]
    out = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=1800)
    if out.returncode != 0:
        raise RuntimeError(out.stderr[-2000:])
    return json.loads(out.stdout.strip().splitlines()[-1])


def reference_arm(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    t0 = time.perf_counter()
    if args.workload == "config5":
        # the 600^3 matrix does not fit the host: a 120^3 sample, extrapolated
        env = dict(os.environ)
        env["OPENBLAS_NUM_THREADS"] = str(os.cpu_count() or 1)
        env.pop("CUDA_VISIBLE_DEVICES", None)
        vals = []
        for _ in range(args.warmup + args.steps):
            o = subprocess.run([sys.executable, "-m", "oracle.bench_cpu", "--laplace27", "120", "--iters", "4",
                                "--total-iters", "763", "--target", "600"], cwd=ROOT, env=env,
                               capture_output=True, text=True, timeout=1800)
            vals.append(json.loads(o.stdout.strip().splitlines()[-1]))
        r = vals[-1]
        r["values"] = [v["value"] for v in vals[args.warmup:]]
        r["value"] = statistics.median(r["values"])
        metric, workload = METRIC5, stencil_problem("config5")[4]
    else:
        r = run_cpu_sample(args.steps, args.warmup, args.total_iters)
        metric, workload = METRIC, WORKLOAD
    line = {"metric": metric, "value": r["value"], "unit": "s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": r["value"] * 1e3,
            "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "impl": "reference",
            "config": {"workload": workload, "mode": "sequential predict-then-solve (CPU)"},
            "cpu_baseline": {"value": r["value"], "unit": "s", "cores": r["cores"],
                             "kind": r["kind"], "sample": r["sample"]},
            "e2e": {"value": r["value"], "unit": "s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0},
            "detail": {"phases": r["phases"], "values": r.get("values"), "config": r["config"],
                       "wall_seconds": time.perf_counter() - t0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# measurement helpers
# ---------------------------------------------------------------------------
class EventTimer:
    """CUDA-event pairs around solver launches, recorded on the solver stream."""

    def __init__(self):
        import torch
        self.torch = torch
        self.streams = {}
        self.open = {}
        self.done = []
        self.active = False

    def _stream(self, h):
        s = self.streams.get(h)
        if s is None:
            s = self.streams[h] = self.torch.cuda.ExternalStream(h)
        return s

    def begin(self, tag, h):
        if not self.active:
            return
        ev = self.torch.cuda.Event(enable_timing=True)
        ev.record(self._stream(h))
        self.open[tag] = ev

    def end(self, tag, h):
        if not self.active:
            return
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
        rows = []
        for line in Path(self.f.name).read_text().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 8:
                rows.append(parts)
        os.unlink(self.f.name)
        loaded = [r for r in rows if r[7].isdigit() and int(r[7]) > 0] or rows
        sm = [float(r[0]) for r in loaded if r[0].replace(".", "").isdigit()]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in loaded:
            for k, name in enumerate(names):
                if r[3 + k].lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": float(loaded[0][1]) if loaded else None,
                "reasons": sorted(reasons), "samples": len(rows), "samples_under_load": len(loaded)}


def algorithmic_bytes(tag: str, info, n: int) -> float:
    """Bytes per launch per SURVEY.md §8(d) (device layout: fp64 values,
    int32 indices)."""
    tok = tag.split(":", 1)[1]
    fmt = tok.split("/")[0]
    nnz, ncols = info["nnz"], n
    if fmt == "CSR":
        return 12 * nnz + 4 * (n + 1) + 8 * ncols + 8 * n
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
    """Algorithmic bytes of one Arnoldi orthogonalisation at column j.

    Resident kernel (w kept on chip): read w once, each basis row V[0..j]
    once, write the normalised w once -> 8n(j+3).  Streaming fallback: dot0
    reads V0,w (16n); pass i reads w,V[i-1],V[i] and writes w (32n); final
    reads w,V[j] and writes w (24n); normalise reads+writes w (16n)."""
    if resident:
        return 8 * n * (j + 3)
    return 16 * n + 32 * n * j + 24 * n + 16 * n


def config1_cg(P, device, _lib, models, start_cfg, reps: int = 3) -> dict:
    """Side measurement (not `value`): BASELINE configs[0], CG fp64 on the 2-D
    5-point Poisson 1024^2 (n = 1,048,576, nnz = 5,238,784), tol 1e-8,
    b = A*1; async predict-while-solve from CSR/LibA/32 vs the fixed
    default CSR-vector solve."""
    import numpy as np
    import torch
    from paper_2411_10143_b200.solver import DeviceOptions
    A = P.CsrMatrix.stencil((1024, 1024), [(0, 0), (0, -1), (0, 1), (-1, 0), (1, 0)],
                            [4.0, -1.0, -1.0, -1.0, -1.0])
    s = device.thread_stream()
    ones = device.DeviceVector.from_numpy(np.ones(A.nrows), s)
    b = device.DeviceVector(A.nrows)
    _lib.check(_lib.lib().svb_spmv_sequential(A._device().handle, ones.ptr, b.ptr, s.handle))
    s.sync()
    params = P.GmresParams(tol=1e-8, max_iters=5000)
    out = {"workload": "config1: CG fp64 Poisson 1024^2, tol 1e-8, b=A*1"}
    with DeviceOptions(keep_solution_on_device=True):
        P.async_solve(A, b, params, models, method="cg", initial_config=start_cfg)   # warm
        ts, its, swaps = [], None, None
        for _ in range(reps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            r = P.async_solve(A, b, params, models, method="cg", initial_config=start_cfg)
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t0)
            its, swaps = r.iterations, [(x.iteration, x.config.token()) for x in r.config_timeline]
        out.update({"async_s": statistics.median(ts), "iterations": its, "swaps": swaps,
                    "converged": r.converged, "final_residual": r.final_residual})
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        d = P.cg_solve(A, b, params, initial_config=start_cfg)
        torch.cuda.synchronize()
        out.update({"default_csr_vector_s": time.perf_counter() - t0, "default_iterations": d.iterations})
    return out


# ---------------------------------------------------------------------------
# the B200 arm
# ---------------------------------------------------------------------------
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

    import paper_2411_10143_b200 as P
    from paper_2411_10143_b200 import _lib, device
    from paper_2411_10143_b200.solver import DeviceOptions

    torch.cuda.set_device(local)
    if ws > 1 or args.workload == "config5":
        import torch.distributed as dist
        if not dist.is_initialized():
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29517")
            if host_staged:
                dist.init_process_group("gloo", rank=rank, world_size=ws)
            else:
                dist.init_process_group("nccl", rank=rank, world_size=ws,
                                        device_id=torch.device("cuda", local))
        return dist_arm(args, ws, rank, local)
    L = _lib.lib()

    def barrier():
        if ws > 1:
            torch.distributed.barrier()

    # --- inputs ------------------------------------------------------------
    offs, wts = [], []
    for dy in (-1, 0, 1):
        for dx in (-1, 0, 1):
            offs.append((dy, dx))
            wts.append(8.5 if (dx, dy) == (0, 0) else -1.0 - 0.25 * (dx + dy))
    A = P.CsrMatrix.stencil((NX, NX), offs, wts)              # generated in HBM
    n = A.nrows
    models = P.CascadeModelSet.load_dir(ROOT / "tests" / "golden" / "models")
    params = P.GmresParams(restart_m=RESTART, tol=TOL, max_iters=1000)
    start_cfg = P.GPU_DEFAULT_CONFIG
    s = device.thread_stream()
    ones = device.DeviceVector.from_numpy(np.ones(n), s)
    b_dev = device.DeviceVector(n)
    _lib.check(L.svb_spmv_sequential(A._device().handle, ones.ptr, b_dev.ptr, s.handle))  # b = A*1
    s.sync()

    def step(timer=None):
        with DeviceOptions(timer=timer, keep_solution_on_device=True):
            return P.async_solve(A, b_dev, params, models, initial_config=start_cfg)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    # --- timed region (device-resident inputs) -----------------------------
    try:
        clocks = NvmlClockSampler(local)
    except Exception:
        clocks = ClockSampler(local)
    launches0 = _lib.launch_count()
    barrier()
    torch.cuda.synchronize()
    t_ev0 = torch.cuda.Event(enable_timing=True)
    t_ev1 = torch.cuda.Event(enable_timing=True)
    per_step, reports = [], []
    gc.collect()
    gc.disable()      # no cyclic-GC pauses inside the timed steps
    t_ev0.record()
    wall0 = time.perf_counter()
    for _ in range(args.steps):
        t0 = time.perf_counter()
        rep = step()
        per_step.append(time.perf_counter() - t0)
        rep.solution = None     # free the device solution now: no pool growth across steps
        reports.append(rep)
    torch.cuda.synchronize()
    t_ev1.record()
    torch.cuda.synchronize()
    wall = time.perf_counter() - wall0
    gc.enable()
    barrier()
    launches = _lib.launch_count() - launches0
    clk = clocks.stop()
    dev_ms = t_ev0.elapsed_time(t_ev1)
    # whole-region device time (events on the default stream bracket all work,
    # the solve's own streams are synchronised inside each step)
    total_s = max(dev_ms / 1e3, wall)
    if ws > 1:
        t = torch.tensor([total_s], device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        total_s = float(t.item())
    value = total_s / args.steps

    # --- kernel timing: separate instrumented steps (CUDA events around every
    # SpMV and Arnoldi launch on the solver stream); kept out of `value`
    # because recording events per launch adds host work to the step
    timer = EventTimer()
    timer.active = True
    prof_steps = max(1, min(args.steps, 3))
    prof_reports = []
    for _ in range(prof_steps):
        r = step(timer)
        r.solution = None
        prof_reports.append(r)
    kern = timer.summary()

    # --- per-kernel roofline ----------------------------------------------------
    hbm, peak_kind = peaks()
    infos = {}
    last = reports[-1]
    for swap in last.config_timeline:
        tok = swap.config.token()
        rep = A if swap.config.format is P.FormatTag.CSR else P.convert(A, swap.config.format)
        inf = rep._device().info
        infos[tok] = {"nnz": int(inf.nnz), "ndiag": int(inf.ndiag), "width": int(inf.width),
                      "spill": int(inf.spill_nnz)}
    groups = {}
    for tag, ms in kern.items():
        tot = sum(ms)
        if tag.startswith("spmv:"):
            tok = tag.split(":", 1)[1]
            if tok not in infos:
                continue
            byts = algorithmic_bytes(tag, infos[tok], n) * len(ms)
        elif tag == "mgs":
            # j cycles 0..restart-1 across steps; the column of each call is
            # reconstructed from the iteration schedule of the reports
            js = []
            for r in prof_reports:
                js += [it % RESTART for it in range(r.iterations)]
            resident = os.environ.get("SPMVTUNE_MGS") != "stream"
            byts = sum(mgs_bytes(n, j, resident) for j in js[:len(ms)])
        else:
            continue
        groups[tag] = {"launches": len(ms), "ms_total": tot, "ms_avg": tot / len(ms),
                       "gbs": byts / (tot / 1e3) / 1e9, "bytes_per_launch": byts / len(ms)}
    step_ms = value * 1e3
    for g in groups.values():
        g["share_of_step"] = g["ms_total"] / prof_steps / step_ms
    dom_tag = max(groups, key=lambda t: groups[t]["ms_total"]) if groups else None
    traffic = None
    prof = ROOT / "profiles" / "ncu_traffic.json"
    if prof.exists() and dom_tag:
        tr = json.loads(prof.read_text())
        traffic = tr.get(dom_tag)
    roofline = None
    if dom_tag:
        g = groups[dom_tag]
        roofline = {"kernel": dom_tag, "bound": "hbm", "achieved": round(g["gbs"], 1),
                    "peak": hbm, "unit": "GB/s", "frac": round(g["gbs"] / hbm, 4),
                    "traffic": traffic, "peak_kind": peak_kind,
                    "bytes_per_launch": g["bytes_per_launch"], "avg_launch_ms": g["ms_avg"]}

    # --- end-to-end through the public API from pinned host buffers -----------------
    e2e = None
    if rank == 0 or ws > 1:
        rp = np.asarray(A.row_ptr)
        ci = np.asarray(A.col_idx)
        vv = np.asarray(A.values)
        bh = b_dev.to_numpy(s)
        pin = {}
        for k, arr in (("rp", rp), ("ci", ci), ("vv", vv), ("b", bh)):
            t = torch.empty(arr.size, dtype=torch.from_numpy(arr[:1]).dtype, pin_memory=True)
            t.numpy()[:] = arr
            pin[k] = t
        Ah = P.CsrMatrix(n, n, pin["rp"].numpy(), pin["ci"].numpy(), pin["vv"].numpy())
        b_host = pin["b"].numpy()

        def e2e_step():
            Ah._dev = None                     # drop the device copy: upload inside the clock
            rep = P.async_solve(Ah, b_host, params, models, initial_config=start_cfg)
            return rep
        e2e_step()
        torch.cuda.synchronize()
        k_e2e = max(1, min(args.steps, 5))
        t0 = time.perf_counter()
        for _ in range(k_e2e):
            rep_e = e2e_step()
        torch.cuda.synchronize()
        e2e_s = (time.perf_counter() - t0) / k_e2e
        h2d = rp.nbytes + ci.nbytes + vv.nbytes + bh.nbytes
        d2h = rep_e.solution.nbytes + 48 * (rep_e.iterations + 4)
        e2e = {"value": e2e_s, "unit": "s", "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "steps": k_e2e,
               "note": "CsrMatrix from pinned host int64/f64 arrays (upload + narrowing inside "
                       "the clock) -> async_solve -> solution to host"}

    # --- comparison solves (not timed as `value`) ---------------------------
    detail = {}
    if rank == 0:
        with DeviceOptions(keep_solution_on_device=True):
            def timed(fn, reps=3):          # median of `reps` warm runs
                ts, rep = [], None
                for _ in range(reps):
                    torch.cuda.synchronize()
                    t0 = time.perf_counter()
                    rep = fn()
                    torch.cuda.synchronize()
                    ts.append(time.perf_counter() - t0)
                    rep.solution = None
                return statistics.median(ts), rep
            dt, d = timed(lambda: P.gmres_solve(A, b_dev, params, initial_config=start_cfg))
            detail["default_csr_vector_gpu_s"] = dt
            detail["default_iterations"] = d.iterations
            st, sq = timed(lambda: P.sequential_predict_solve(A, b_dev, params, models))
            detail["sequential_gpu_s"] = st
            detail["sequential_phases"] = sq.phases
        if not args.no_extra:
            detail["config1_cg"] = config1_cg(P, device, _lib, models, start_cfg)
    detail.update({
        "iterations": last.iterations, "converged": last.converged,
        "final_residual": last.final_residual,
        "timeline": [sw.to_dict() for sw in last.config_timeline],
        "advisor_outcome": last.advisor_outcome, "per_step_wall_s": per_step,
        "per_step_swaps": [[(sw.iteration, sw.config.token(), round(sw.swap_cost_seconds, 5))
                            for sw in r.config_timeline] for r in reports],
        "device_region_ms": dev_ms, "wall_region_s": wall, "kernels": groups})

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu:
        try:
            r = run_cpu_sample(1, 0, last.iterations)
            cpu = {"value": r["value"], "unit": "s", "cores": r["cores"], "kind": r["kind"],
                   "sample": r["sample"], "phases": r["phases"], "cpu_model": r.get("cpu_model")}
        except Exception as exc:  # measurement must not kill the bench line
            cpu = {"value": None, "unit": "s", "cores": os.cpu_count(), "kind": "port",
                   "sample": f"failed: {exc}"[:300]}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "s", "n_gpus": ws, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": value * 1e3, "higher_is_better": False,
                # one fixed system at every N (N > 1: row-partitioned, dist_arm)
                "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {"workload": WORKLOAD, "mode": "async",
                           "parallelism": f"replicas{ws}" if ws > 1 else "single",
                           "l2": "inputs larger than L2 (CSR 448 MB + Krylov basis 992 MB vs 126 MB L2)"},
                "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
                "gpu_launches": int(launches), "clocks": clk, "detail": detail}
        print(json.dumps(line), flush=True)
    if ws > 1:
        torch.distributed.destroy_process_group()


# ---------------------------------------------------------------------------
# row-partitioned arm (torchrun, N > 1; or --workload config5 at any N)
# ---------------------------------------------------------------------------
def stencil_problem(workload: str):
    if workload == "config5":
        offs, wts = [], []
        for dz in (-1, 0, 1):
            for dy in (-1, 0, 1):
                for dx in (-1, 0, 1):
                    offs.append((dz, dy, dx))
                    wts.append(26.0 if (dx, dy, dz) == (0, 0, 0) else -1.0)
        n3 = int(os.environ.get("SPMVTUNE_CONFIG5_N", "600"))
        return ("cg", (n3, n3, n3), offs, wts,
                f"config5: CG fp64, tol {TOL:g}, b=A*1, 3-D 27-point Laplacian {n3}^3 "
                f"(n={n3 ** 3:,}, nnz={(3 * n3 - 2) ** 3:,}), row-partitioned z-slabs generated "
                "per rank on the device, cascade on exact global features, NCCL halo + all-reduce")
    offs, wts = [], []
    for dy in (-1, 0, 1):
        for dx in (-1, 0, 1):
            offs.append((dy, dx))
            wts.append(8.5 if (dx, dy) == (0, 0) else -1.0 - 0.25 * (dx + dy))
    return ("gmres", (NX, NX), offs, wts, WORKLOAD.replace("async predict-while-solve starting on "
            "CSR/LibA/32", "row-partitioned predict-then-solve (cascade on exact global features, "
            "NCCL halo + all-reduce)"))


def dist_arm(args, ws, rank, local):
    """Time-to-solution of the row-partitioned solve (distributed.py): each
    rank generates its slab on its GPU (outside the clock, like the single-GPU
    arm's matrix), then every step runs global features -> cascade ->
    conversion -> solve.  Strong scaling: the problem is fixed as N grows."""
    import torch
    import torch.distributed as dist

    import paper_2411_10143_b200 as P
    from paper_2411_10143_b200 import _lib, device
    from paper_2411_10143_b200.distributed import HostStagedComm, distributed_stencil_solve, \
        stencil_block, stencil_partition

    comm_class = HostStagedComm if os.environ.get("SPMVTUNE_DIST_BACKEND") == "gloo" else None

    method, dims, offs, wts, workload = stencil_problem(args.workload)
    models = P.CascadeModelSet.load_dir(ROOT / "tests" / "golden" / "models")
    params = P.GmresParams(restart_m=RESTART, tol=TOL, max_iters=20000)
    bounds = stencil_partition(dims, ws)
    s = device.thread_stream(0)
    t0 = time.perf_counter()
    blk = stencil_block(dims, offs, wts, int(bounds[rank]), int(bounds[rank + 1]), s)
    gen_s = time.perf_counter() - t0

    def step():
        t = {}
        res, _ = distributed_stencil_solve(method, dims, offs, wts, params, models=models, blk=blk,
                                           comm_class=comm_class,
                                           timings=t)
        return res, t

    for _ in range(args.warmup):
        step()
    try:
        clocks = NvmlClockSampler(local)
    except Exception:
        clocks = ClockSampler(local)
    launches0 = _lib.launch_count()
    dist.barrier()
    torch.cuda.synchronize()
    steps, results = [], []
    t_all = time.perf_counter()
    for _ in range(args.steps):
        res, t = step()
        steps.append(t)
        results.append({k: res[k] for k in ("converged", "iterations", "final", "config")})
    torch.cuda.synchronize()
    wall = time.perf_counter() - t_all
    dist.barrier()
    clk = clocks.stop()
    launches = _lib.launch_count() - launches0
    tt = torch.tensor([wall], device="cpu" if comm_class else "cuda")
    dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    value = float(tt.item()) / args.steps

    # roofline: the local SpMV in the predicted configuration, events on our stream
    cfg = P.SpmvConfig.from_token(results[-1]["config"])
    csr = blk._dev_csr
    mat = csr if cfg.format is P.FormatTag.CSR else P.convert(csr, cfg.format)
    inf = mat._device().info
    xw = device.DeviceVector(blk.window)
    _lib.check(_lib.lib().svb_fill(xw.ptr, blk.window, 1.0, s.handle))
    yl = device.DeviceVector(blk.nloc)
    ext = torch.cuda.ExternalStream(s.handle)
    from paper_2411_10143_b200.kernels import default_workers, launch
    for _ in range(3):
        launch(cfg, mat, xw.ptr, yl.ptr, workers=default_workers(), stream=s)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 20
    e0.record(ext)
    for _ in range(reps):
        launch(cfg, mat, xw.ptr, yl.ptr, workers=default_workers(), stream=s)
    e1.record(ext)
    torch.cuda.synchronize()
    spmv_ms = e0.elapsed_time(e1) / reps
    n_loc = blk.nloc
    info = {"nnz": int(inf.nnz), "ndiag": int(inf.ndiag), "width": int(inf.width),
            "spill": int(inf.spill_nnz)}
    byts = algorithmic_bytes("spmv:" + cfg.token(), info, n_loc)
    byts += 8 * (blk.window - n_loc)          # x is the window, not just the local rows
    hbm, peak_kind = peaks()
    gbs = byts / (spmv_ms / 1e3) / 1e9
    roofline = {"kernel": "spmv:" + cfg.token(), "bound": "hbm", "achieved": round(gbs, 1), "peak": hbm,
                "unit": "GB/s", "frac": round(gbs / hbm, 4), "traffic": None, "peak_kind": peak_kind,
                "bytes_per_launch": byts, "avg_launch_ms": spmv_ms}
    its = results[-1]["iterations"]
    per_iter = {k: v / max(1, its) for k, v in steps[-1].items() if k == "solve_s"}
    gathered = [None] * ws
    dist.all_gather_object(gathered, {"rank": rank, "rows": [int(bounds[rank]), int(bounds[rank + 1])],
                                      "spmv_ms": spmv_ms, "gbs": gbs, "gen_s": gen_s,
                                      "last_step": steps[-1]})
    cpu = None
    if rank == 0 and ws == 1 and args.workload == "config5" and not args.no_cpu:
        try:
            env = dict(os.environ)
            env["OPENBLAS_NUM_THREADS"] = str(os.cpu_count() or 1)
            env.pop("CUDA_VISIBLE_DEVICES", None)
            cmd = [sys.executable, "-m", "oracle.bench_cpu", "--laplace27", "120", "--iters", "4",
                   "--total-iters", str(results[-1]["iterations"]), "--target", str(dims[0])]
            o = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
            r = json.loads(o.stdout.strip().splitlines()[-1])
            cpu = {k: r[k] for k in ("value", "unit", "cores", "kind", "sample", "cpu_model")}
        except Exception as exc:  # measurement must not kill the bench line
            cpu = {"value": None, "unit": "s", "cores": os.cpu_count(), "kind": "port",
                   "sample": f"failed: {exc}"[:300]}
    if rank == 0:
        line = {"metric": METRIC5 if args.workload == "config5" else METRIC,
                "value": value, "unit": "s", "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": value * 1e3, "higher_is_better": False, "scaling": "strong",
                "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {"workload": workload, "parallelism": f"row-partitioned x{ws}",
                           "comm": "gloo, host-staged (path validation, not a performance number)"
                           if comm_class else "nccl",
                           "l2": "inputs larger than L2"},
                "roofline": roofline, "cpu_baseline": cpu,
                "e2e": None, "gpu_launches": int(launches), "clocks": clk,
                "detail": {"results": results[-1], "per_step": steps, "per_rank": gathered,
                           "per_iteration_solve_s": per_iter,
                           "cpu_baseline_note": "the reference arm's CPU path cannot hold this "
                           "matrix (int64 CSR >= 140 GB) — see BASELINE configs[4]"
                           if args.workload == "config5" else "single-GPU line carries it"}}
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--total-iters", type=int, default=77,
                    help="reference arm: GMRES iterations the solve takes (77 at config 2)")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-extra", action="store_true", help="skip the config-1 CG side measurement")
    ap.add_argument("--workload", default="config2", choices=["config2", "config5"],
                    help="config5 = row-partitioned CG on the 27-point Laplacian 600^3 (any N); "
                         "N > 1 always runs the row-partitioned solver")
    args = ap.parse_args(argv)
    if args.warmup < 0 or args.steps < 1:
        raise SystemExit("--steps >= 1 and --warmup >= 0")
    if args.impl == "reference":
        reference_arm(args)
    else:
        b200_arm(args)


if __name__ == "__main__":
    main()
