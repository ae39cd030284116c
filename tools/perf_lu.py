"""Profiling driver for the LU trailing update at the headline size: cfg4
(N = 15360) batch of B frequencies (default 2) through the BEM handle, one
warm-up evaluate and one profiled evaluate. Run under ncu, e.g.

    ncu --set full -k regex:lu_gemm3m_tma -s 160 -c 1 python tools/perf_lu.py

(120 super-panel updates per factorization; -s 160 lands in the second
factorization at rest ~ 10000)."""
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_1511_04355_b200 as P  # noqa: E402
from paper_1511_04355_b200 import mesh  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 2
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
V, F = mesh.icosphere(4)
sysb = P.BemSystem(V, F, mesh.random_traction(F.shape[0], seed=0), channels=list(range(48)), max_batch=B)
s = 0.25 + 1j * 2 * np.pi / 20.0 * np.arange(1, B + 1)  # contour frequencies 1..B (cfg4: T = 20)
for _ in range(reps):
    sysb.evaluate_batch_device(s)
    print(sysb.last_timing())
