"""One cfg2 assembly+solve batch (for ncu captures of the assembly kernels)."""
import sys
import numpy as np
sys.path.insert(0, ".")
from paper_1511_04355_b200 import BemSystem, mesh

V, F = mesh.icosphere(3)
sysb = BemSystem(V, F, mesh.pressure_traction(V, F), channels=list(range(48)), max_batch=129)
s = 0.25 + 1j * 2 * np.pi / 20.0 * np.arange(129)
sysb.evaluate_batch_device(s)
sysb.close()
