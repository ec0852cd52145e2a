"""Config-5 e2e path alone (profiling aid): the slab copied to pinned host
memory once, then distributed_solve_slab N times with its phase timings
(upload / predict / convert / solve) — the e2e leg of bench.py."""
import argparse
import json
import os
import socket
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

s = socket.socket()
s.bind(("127.0.0.1", 0))
os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(s.getsockname()[1]), RANK="0", WORLD_SIZE="1")
s.close()
torch.cuda.set_device(0)
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
import bench  # noqa: E402
import paper_2411_10143_b200 as P  # noqa: E402
from paper_2411_10143_b200 import device  # noqa: E402
from paper_2411_10143_b200.distributed import stencil_block  # noqa: E402

n3 = int(os.environ.get("SPMVTUNE_CONFIG5_N", "600"))
dims = (n3,) * 3
offs, w = bench.stencil27()
blk = stencil_block(dims, offs, w, 0, n3 ** 3, device.thread_stream(0))
models = P.CascadeModelSet.load_dir(ROOT / "tests" / "golden" / "models")
params = P.GmresParams(tol=1e-8, max_iters=20000)
k = int(os.environ.get("SPMVTUNE_E2E_STEPS", "4"))
args = argparse.Namespace(steps=k, e2e_steps=k)
import paper_2411_10143_b200.distributed as D  # noqa: E402
_solve = D.distributed_solve_slab


def traced(*a, **kw):                    # pool state around every solve (fragmentation check)
    i0 = device.device_info()
    r = _solve(*a, **kw)
    i1 = device.device_info()
    t = kw.get("timings")
    if t is not None:
        t["pool_gb"] = [round(i0["pool_reserved_bytes"] / 1e9, 2), round(i1["pool_reserved_bytes"] / 1e9, 2),
                        round(i1["free_bytes"] / 1e9, 2)]
    return r


D.distributed_solve_slab = traced
out = bench.e2e_slab(args, blk, 0, n3 ** 3, params, models, None, 1)
print(json.dumps({"value": out["value"], "phases": out["phases"]}))
dist.destroy_process_group()
