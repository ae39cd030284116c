"""BASELINE config 4 AFS at the reference defaults on the LU path.

5120-triangle sphere (N = 15360), random traction seed 0, T = 20, N_s = 512,
eta = 5/T, Omega = Omega_s = pi N_s / T. Channels pinned per SURVEY.md A.4:
the 3 displacement components of 16 collocation points drawn with the
reference's draw_indices(N_e, 16, 0) (48 channels); the driver draws its 5
ORFs from them with the seed (afs.cpp:234-236) and tests all 48 (afs.cpp:239-242).
Reference defaults otherwise (afs.hpp:21-39: J0 16, thresholds 1e-4 / 2e-3,
max_iterations 500). Writes one JSON object to stdout.

Usage: python tools/run_cfg4_afs.py [max_iterations] [e1] [e2]
"""
import json
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_1511_04355_b200 as P  # noqa: E402
from paper_1511_04355_b200 import BemSystem, mesh  # noqa: E402

T, NS = 20.0, 512
ETA = 5.0 / T
max_iter = int(sys.argv[1]) if len(sys.argv) > 1 else 500
e1 = float(sys.argv[2]) if len(sys.argv) > 2 else 1e-4
e2 = float(sys.argv[3]) if len(sys.argv) > 3 else 2e-3

V, F = mesh.icosphere(4)
trac = mesh.random_traction(F.shape[0], seed=0)
pts = mesh.draw_indices(F.shape[0], 16, 0)
dofs = [3 * p + i for p in pts for i in range(3)]
cfg = dict(omega_max=np.pi * NS / T, eta=ETA, period=T, max_iterations=max_iter, e1_threshold=e1,
           e2_threshold=e2)
out = {"config": "cfg4 AFS: icosphere(4), N=15360, random traction seed 0, T=20, Ns=512, eta=5/T, "
                 "Omega=Omega_s, 48 channels (16 points x 3), ORFs drawn by the driver, LU solves",
       "max_iterations": max_iter, "e1_threshold": e1, "e2_threshold": e2}
sysb = BemSystem(V, F, trac, channels=dofs, max_batch=16)
t0 = time.perf_counter()
try:
    r = P.run_afs(sysb, **cfg)
    out.update(wall_s=time.perf_counter() - t0, n_c=r["n_c"], converged=r["converged"],
               solver_calls=r["solver_calls"], order=int(len(r["poles"])),
               history=r["history"].tolist())
except P.Error as e:
    out.update(wall_s=time.perf_counter() - t0, error=f"{type(e).__name__}: {e}")
print(json.dumps(out))
