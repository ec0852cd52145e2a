"""Peer-memory collectives (csrc/peer.cu, distributed.PeerComm) with two
processes on the one test GPU, mailboxes mapped through CUDA IPC as on a
multi-GPU box: the all-reduce gives every rank the same bits over many
epochs (both slot banks), and a rank that stops participating surfaces as
an error on the waiting rank after the deadline — never a hang."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, port, mode, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), SPMVTUNE_PEER_DEADLINE_MS="1500")
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=2)
    try:
        from paper_2411_10143_b200 import device
        from paper_2411_10143_b200.distributed import HostStagedComm, PeerComm
        s = device.thread_stream(0)
        comm = PeerComm(HostStagedComm(s), s, ipc=True)
        sc = device.DeviceVector(8)
        got = []
        if mode == "sum":
            rng = np.random.default_rng(rank)
            for it in range(40):                       # both parity banks, many epochs
                vals = rng.standard_normal(5) * (it + 1)
                device.copy(sc.ptr, vals.ctypes.data, vals.nbytes, s)
                comm.allreduce(sc, 0, 5)
                got.append((vals, sc.to_numpy(s)[:5]))
            comm.check()
            q.put((rank, "ok", got))
        else:                                           # rank 1 never joins the all-reduce
            err = None
            if rank == 0:
                comm.allreduce(sc, 0, 1)
                s.sync()
                try:
                    comm.check()
                except RuntimeError as exc:
                    err = str(exc)
            q.put((rank, "ok", err))
        comm.close()
    except Exception as exc:
        import traceback
        q.put((rank, "error", repr(exc) + traceback.format_exc()[-1500:]))
    finally:
        dist.destroy_process_group()


def _run(mode):
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, port, mode, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = sorted([q.get(timeout=300) for _ in range(2)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
    assert all(o[1] == "ok" for o in out), out
    return out


def test_peer_allreduce_same_bits_on_every_rank():
    (_, _, g0), (_, _, g1) = _run("sum")
    for (v0, r0), (v1, r1) in zip(g0, g1):
        assert np.array_equal(r0, r1)                  # bit-identical totals
        assert np.array_equal(r0, v0 + v1)             # rank order: slot 0 + slot 1


def test_peer_wait_deadline_raises_instead_of_hanging():
    (_, _, err0), _ = _run("stall")
    assert err0 is not None and "timed out" in err0
