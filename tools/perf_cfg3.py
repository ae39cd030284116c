"""cfg3 single solve (cube cavity, N = 36864) LU timing, two evaluates."""
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_1511_04355_b200 import BemSystem, mesh  # noqa: E402

V, F = mesh.cube_cavity(32)
sysb = BemSystem(V, F, mesh.pressure_traction(V, F), channels=list(range(48)), max_batch=1)
s = np.array([complex(0.25, 2 * np.pi / 20.0 * 7)])
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 2):
    sysb.evaluate_batch_device(s)
    print(sysb.last_timing())
