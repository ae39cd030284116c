"""Single-matrix LU beyond configs[2]: unit-cube cavity with g x g squares per face
(N = 36 g^2 unknowns, 16 N^2 bytes), Heaviside pressure, one frequency: assembly + LU +
solve, backward error of the solution against the re-assembled matrix.
usage: python tools/run_large_n.py 36 44"""
import json, sys, time
sys.path.insert(0, ".")
import numpy as np
import paper_1511_04355_b200 as P
from paper_1511_04355_b200 import BemSystem, mesh

s = 0.25 + 2.199114857512855j  # contour(7) of the T = 20 sweep
for g in [int(a) for a in sys.argv[1:]] or [36]:
    V, F = mesh.cube_cavity(g)
    tr = mesh.pressure_traction(V, F)
    n = 3 * F.shape[0]
    t0 = time.perf_counter()
    sysb = BemSystem(V, F, tr, max_batch=1)
    t_create = time.perf_counter() - t0
    u = sysb.evaluate(s)
    t = sysb.last_timing()
    nr = sysb.residual(s, u)
    back = nr["res"] / (nr["a_inf"] * nr["u"] + nr["b"])
    print(json.dumps(dict(g=g, n=n, elements=int(F.shape[0]), matrix_gb=16.0 * n * n / 1e9, create_s=t_create,
                          timing=t, lu_tflops=8.0 * n ** 3 / 3 / (t["lu_ms"] * 1e-3) / 1e12,
                          backward_error=back, res_over_b=nr["res"] / nr["b"])), flush=True)
    sysb.close()
