"""One cfg4 solve (N = 15360) for launch-list / ncu captures (development tool)."""
import sys
import numpy as np
sys.path.insert(0, ".")
from paper_1511_04355_b200 import BemSystem, mesh

V, F = mesh.icosphere(4)
sysb = BemSystem(V, F, mesh.random_traction(F.shape[0], seed=0), channels=list(range(48)), max_batch=1)
sysb.evaluate_batch_device(np.array([0.25 + 1j * 2 * np.pi / 20.0]))
sysb.close()
