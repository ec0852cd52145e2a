"""Config-1 async CG timing inside one long process: fresh, after the
config-2 leg, and with a thread per advisor instead of reused workers —
locates the difference between the standalone and the full-bench number.
    python profiles/c1_ab.py"""
import argparse
import json
import sys
import threading
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
import paper_2411_10143_b200 as P  # noqa: E402
from paper_2411_10143_b200 import _lib, device, solver  # noqa: E402

models = P.CascadeModelSet.load_dir(ROOT / "tests" / "golden" / "models")
args = argparse.Namespace(steps=10, warmup=3)


def c1(tag):
    d = bench.config1_detail(args, P, device, _lib, models)
    print(json.dumps({tag: {k: d[k] for k in ("async_s", "default_csr_vector_s", "swaps")},
                      "threads": threading.active_count()}), flush=True)


c1("fresh")
c1("fresh_again")
bench.config2_detail(args, P, device, _lib, models)
c1("after_config2")
orig = solver._AdvisorThreads.run
solver._AdvisorThreads.run = classmethod(lambda cls, job: threading.Thread(target=job, daemon=True).start())
c1("thread_per_job")
solver._AdvisorThreads.run = orig
c1("reused_again")
