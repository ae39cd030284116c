"""Config 3: unit-cube cavity, 32x32 squares per face (12288 triangles, N = 36864,
A = 21.7 GB), one Heaviside-pressure frequency solve: assembly + LU + solve on one B200."""
import json, math, sys, time
sys.path.insert(0, ".")
import numpy as np
import paper_1511_04355_b200 as P
from paper_1511_04355_b200 import BemSystem, mesh

V, F = mesh.cube_cavity(32)
tr = mesh.pressure_traction(V, F)
t0 = time.perf_counter()
sysb = BemSystem(V, F, tr, channels=list(range(48)), max_batch=1)
t_create = time.perf_counter() - t0
s = np.array([0.25 + 0.5j])
out = {}
for rep in range(2):
    sysb.evaluate_batch_device(s)
    t = sysb.last_timing()
    out[f"run{rep}"] = t
n = 3 * F.shape[0]
t = out["run1"]
out.update(n=n, elements=F.shape[0], matrix_gb=2 * 8 * n * n / 1e9, create_s=t_create,
           lu_tflops=8.0 * n ** 3 / 3 / (t["lu_ms"] * 1e-3) / 1e12,
           solves_per_s=1e3 / (t["assembly_ms"] + t["lu_ms"] + t["solve_ms"]))
print(json.dumps(out))
