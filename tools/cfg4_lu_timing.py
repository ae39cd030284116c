"""cfg4 single-matrix LU timing (N = 15360), three repeats; FDSWEEP_LOOKAHEAD=0/1 compares the
schedules (3M update: look-ahead 306 ms, super-panels without look-ahead 326 ms)."""
import sys, json
sys.path.insert(0, ".")
import numpy as np
from paper_1511_04355_b200 import BemSystem, mesh
V, F = mesh.icosphere(4)
s = BemSystem(V, F, mesh.random_traction(F.shape[0], seed=0), channels=list(range(48)), max_batch=1)
r = []
for _ in range(3):
    s.evaluate_batch_device(np.array([0.25 + 1j * 2 * np.pi / 20.0]))
    r.append(s.last_timing()["lu_ms"])
print(json.dumps({"lu_ms": r}))
