"""svb_copy_host (device.copy_host): the staged pageable host <-> device
copies behind gmres_solve's b upload / x download and DeviceVector's
numpy conversions — byte-exact at every size class (direct below 1 MB,
staged, more than one 64 MB staging window, odd lengths), pinned buffers,
and stream order (a D2H sees the work enqueued before it)."""
import numpy as np
import pytest
import torch

from paper_2411_10143_b200 import device

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("nbytes", [8, 1 << 19, (3 << 20) + 8, (16 << 20) - 8, (70 << 20) + 24])
def test_round_trip_bit_exact(nbytes):
    n = nbytes // 8
    a = np.random.default_rng(nbytes).standard_normal(n)
    s = device.thread_stream(0)
    d = device.DeviceVector(n)
    device.copy_host(d.ptr, a.ctypes.data, a.nbytes, True, s)
    a_copy = a.copy()
    a[:] = 0.0                            # the call returned: the source may be reused
    out = np.empty(n)
    device.copy_host(out.ctypes.data, d.ptr, out.nbytes, False, s)
    assert np.array_equal(out.view(np.uint64), a_copy.view(np.uint64))
    assert np.array_equal(d.to_numpy(s).view(np.uint64), a_copy.view(np.uint64))
    assert np.array_equal(device.DeviceVector.from_numpy(a_copy, s).to_numpy(s), a_copy)


def test_pinned_buffers_and_stream_order():
    n = 4 << 20
    pinned = torch.empty(n, dtype=torch.float64, pin_memory=True).numpy()
    pinned[:] = np.arange(n, dtype=np.float64)
    s = device.thread_stream(0)
    d = device.DeviceVector(n)
    device.copy_host(d.ptr, pinned.ctypes.data, pinned.nbytes, True, s)
    back = np.empty(n)
    device.copy_host(back.ctypes.data, d.ptr, back.nbytes, False, s)
    assert np.array_equal(back, pinned)
    device.memset(d.ptr, 0, d.nbytes, s)          # enqueued, not waited for
    device.copy_host(back.ctypes.data, d.ptr, back.nbytes, False, s)
    assert not back.any()
