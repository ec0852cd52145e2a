"""CPU oracle for the spmvtune hot path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
``--impl reference`` leg may import this package, and only as the checker or
as the timed CPU reference.  The product package
(``paper_2411_10143_b200``) never imports it: its compute path is the CUDA
library and fails loudly when that library is missing.

Parity status: PINNED.  ``tests/golden/make_golden.py`` imports the real
reference (``/root/reference/pkg/src/spmvtune``) in the build container and
records its outputs; ``tests/test_oracle_golden.py`` checks this oracle
against those fixtures bit-for-bit (SpMV, conversions, features, cascade) and
by iteration count / solution for GMRES.
"""
from .cpu_oracle import *  # noqa: F401,F403
