"""LU vs GMRES on the config-2 batch (129 frequencies, N = 3840): where the
iterative path stops paying (per-frequency GMRES is launch/sync-bound at this
size, so the batched LU stays the default)."""
import sys, math, time, json
sys.path.insert(0, ".")
import numpy as np
import paper_1511_04355_b200 as P
from paper_1511_04355_b200 import mesh
V, F = mesh.icosphere(3)
sysb = P.BemSystem(V, F, mesh.pressure_traction(V, F), channels=list(range(48)), max_batch=129)
s = 0.25 + 1j * 2 * math.pi / 20.0 * np.arange(129)
ul = sysb.evaluate_batch(s)
t = sysb.last_timing()
sysb.set_solver("gmres", tol=1e-12)
sysb.evaluate_batch(s)
ug = sysb.evaluate_batch(s)
tg = sysb.last_timing()
print(json.dumps({"lu": t, "gmres": tg, "gm": sysb.last_gmres(), "diff": float(np.linalg.norm(ug - ul) / np.linalg.norm(ul))}))
