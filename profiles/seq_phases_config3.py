"""Config 3 (8 M-row power-law CG): repeated predict-then-solve phases and
CSR->HYB conversions interleaved with solves, to locate intermittent stalls.
    python profiles/seq_phases_config3.py [nogc]"""
import gc
import json
import sys
import time
sys.path.insert(0, ".")
import paper_2411_10143_b200 as P  # noqa: E402
from paper_2411_10143_b200 import generators as G, device  # noqa: E402
from paper_2411_10143_b200.solver import DeviceOptions  # noqa: E402
if "nogc" in sys.argv:
    gc.disable()
A = P.CsrMatrix(*G.powerlaw_spd(8_000_000, seed=0))
A._device()
models = P.CascadeModelSet.load_dir(P.B200_MODELS_DIR)
params = P.GmresParams(tol=1e-8, max_iters=20000, rhs="random", seed=0)
with DeviceOptions(keep_solution_on_device=True):
    for k in range(4):
        t0 = time.perf_counter()
        r = P.convert(A, P.FormatTag.HYB)
        device.thread_stream(0).sync()
        t1 = time.perf_counter()
        rep = P.cg_solve(r, None, params, initial_config=P.SpmvConfig.from_token("HYB/LibA"))
        t2 = time.perf_counter()
        del r, rep
        t3 = time.perf_counter()
        print(f"convert {1e3 * (t1 - t0):8.2f} ms  solve {1e3 * (t2 - t1):8.2f} ms  del {1e3 * (t3 - t2):6.2f} ms",
              flush=True)
    for k in range(3):
        s = P.sequential_predict_solve(A, None, params, models, method="cg")
        print(json.dumps(s.phases), s.wall_seconds, flush=True)
