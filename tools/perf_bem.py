"""Quick per-stage timing of the BEM path on one B200 (development tool)."""
import sys, time, json
import numpy as np
sys.path.insert(0, ".")
from paper_1511_04355_b200 import BemSystem, mesh

def run(level, B, reps=2):
    V, F = mesh.icosphere(level)
    tr = mesh.pressure_traction(V, F)
    sysb = BemSystem(V, F, tr, channels=list(range(48)), max_batch=B)
    T = 20.0
    s = 0.25 + 1j * 2 * np.pi / T * np.arange(B)
    sysb.evaluate_batch_device(s)
    out = []
    for _ in range(reps):
        sysb.evaluate_batch_device(s)
        out.append(sysb.last_timing())
    n = 3 * F.shape[0]
    t = out[-1]
    fl = B * 8 * n**3 / 3
    print(json.dumps(dict(n=n, B=B, **t, lu_tflops=fl / (t["lu_ms"] * 1e-3) / 1e12)), flush=True)

for lvl, B in [(2, 129), (3, 129), (4, 1)]:
    run(lvl, B)
