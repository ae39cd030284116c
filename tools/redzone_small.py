import sys
sys.path.insert(0, ".")
import numpy as np
import paper_1511_04355_b200 as P
from paper_1511_04355_b200 import BemSystem, mesh
V, F = mesh.icosphere(2)
for B in (2, 1):
    s = BemSystem(V, F, mesh.pressure_traction(V, F), channels=list(range(48)), max_batch=B)
    try:
        y = np.asarray(s.evaluate_batch(0.25 + 1j * (1.0 + np.arange(B))))
        print("B", B, "ok", np.isfinite(y).all(), P.api.redzone_check())
    except Exception as e:
        print("B", B, "FAIL", e); break
