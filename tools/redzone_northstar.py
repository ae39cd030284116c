"""Red-zone run at the north_star sizes (FDSWEEP_REDZONE=1 python tools/redzone_northstar.py):
cfg4 (N = 15360) as a batch of 8 and as a single matrix (look-ahead), the cfg3 cube (N = 36864,
global-slot panels, banded 3M update); prints fds_debug_redzone_check's counts."""
import json, sys
sys.path.insert(0, ".")
import numpy as np
import paper_1511_04355_b200 as P
from paper_1511_04355_b200 import BemSystem, mesh

out = {}
V, F = mesh.icosphere(4)
tr = mesh.random_traction(F.shape[0], seed=0)
for B in (8, 1):
    s = BemSystem(V, F, tr, channels=list(range(48)), max_batch=B)
    y = np.asarray(s.evaluate_batch(0.25 + 1j * 2 * np.pi / 20.0 * (1 + np.arange(B))))
    out[f"cfg4_batch{B}"] = {"resp_norm": float(np.linalg.norm(y)), **P.api.redzone_check()}
    s.close()
V, F = mesh.cube_cavity(32)
s = BemSystem(V, F, mesh.pressure_traction(V, F), channels=list(range(32)), max_batch=1)
y = np.asarray(s.evaluate_batch(np.array([0.25 + 2.0j])))
out["cfg3_single"] = {"resp_norm": float(np.linalg.norm(y)), **P.api.redzone_check()}
s.close()
out["after_close"] = P.api.redzone_check()
print(json.dumps(out))
