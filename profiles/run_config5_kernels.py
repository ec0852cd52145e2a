"""Config 5 (27-point Laplacian n3^3, row-partitioned CG at world 1) for ncu:
generate the slab on the device, then run a truncated predict-then-solve CG
(`--iters` iterations) so a launch list / `--set full` capture sees the
per-iteration kernels (local DIA SpMV, dot, fused x/r update, p update).

    python profiles/run_config5_kernels.py [--n3 600] [--iters 12]
"""
import argparse
import os
import socket
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

ap = argparse.ArgumentParser()
ap.add_argument("--n3", type=int, default=600)
ap.add_argument("--iters", type=int, default=12)
a = ap.parse_args()

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

s = socket.socket()
s.bind(("127.0.0.1", 0))
os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(s.getsockname()[1]), RANK="0", WORLD_SIZE="1")
s.close()
torch.cuda.set_device(0)
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))

import paper_2411_10143_b200 as P  # noqa: E402
from paper_2411_10143_b200 import device  # noqa: E402
from paper_2411_10143_b200.distributed import distributed_stencil_solve, stencil_block  # noqa: E402

offs, w = [], []
for dz in (-1, 0, 1):
    for dy in (-1, 0, 1):
        for dx in (-1, 0, 1):
            offs.append((dz, dy, dx))
            w.append(26.0 if (dx, dy, dz) == (0, 0, 0) else -1.0)
dims = (a.n3,) * 3
n = a.n3 ** 3
blk = stencil_block(dims, offs, w, 0, n, device.thread_stream(0))
models = P.CascadeModelSet.load_dir(ROOT / "tests" / "golden" / "models")
params = P.GmresParams(tol=1e-300, max_iters=a.iters)
for _ in range(2):
    res, _ = distributed_stencil_solve("cg", dims, offs, w, params, models=models, blk=blk)
torch.cuda.synchronize()
print("iterations", res["iterations"], "config", res["config"])
dist.destroy_process_group()
