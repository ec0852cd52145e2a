"""Advisor kernels for ncu: the feature pass and the CSR->DIA conversion on
config 2 (convdiff 2000^2), then the feature pass on a 4 M-row power-law
matrix — each launched twice (the second launch is the one to read)."""
import sys
sys.path.insert(0, ".")
import paper_2411_10143_b200 as P  # noqa: E402
from paper_2411_10143_b200 import device  # noqa: E402
from paper_2411_10143_b200 import generators as G  # noqa: E402

offs = [(dy, dx) for dy in (-1, 0, 1) for dx in (-1, 0, 1)]
w = [8.5 if o == (0, 0) else -1.0 - 0.25 * (o[1] + o[0]) for o in offs]
A = P.CsrMatrix.stencil((2000, 2000), offs, w)
for _ in range(2):
    P.extract_features(A)
for _ in range(2):
    d = P.convert(A, P.FormatTag.DIA)
    d._device()
    device.thread_stream(0).sync()
    del d
B = P.CsrMatrix(*G.powerlaw_spd(4_000_000, seed=0))
for _ in range(2):
    P.extract_features(B)
print("ok")
