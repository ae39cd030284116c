"""Per-stage timing of the BEM path on one B200 (development tool)."""
import ctypes, json, sys
import numpy as np
sys.path.insert(0, ".")
import paper_1511_04355_b200 as P
from paper_1511_04355_b200 import BemSystem, mesh

L = P.lib()

def prof(kind):
    c, ms, wk = ctypes.c_int(), ctypes.c_double(), ctypes.c_double()
    P.api._check(L.fds_profile_read(kind, ctypes.byref(c), ctypes.byref(ms), ctypes.byref(wk)))
    return ms.value, wk.value

def run(level, B, reps=2):
    V, F = mesh.icosphere(level)
    tr = mesh.pressure_traction(V, F)
    sysb = BemSystem(V, F, tr, channels=list(range(48)), max_batch=B)
    T = 20.0
    s = 0.25 + 1j * 2 * np.pi / T * np.arange(B)
    sysb.evaluate_batch_device(s)
    for _ in range(reps):
        sysb.evaluate_batch_device(s)
    t = sysb.last_timing()
    P.api._check(L.fds_profile_enable(1))
    sysb.evaluate_batch_device(s)
    g, gw = prof(0); pn, _ = prof(1); tr_, _ = prof(2)
    P.api._check(L.fds_profile_enable(0))
    n = 3 * F.shape[0]
    fl = B * 8 * n**3 / 3
    print(json.dumps(dict(n=n, B=B, **{k: round(v, 2) for k, v in t.items()}, lu_tflops=round(fl / (t["lu_ms"] * 1e-3) / 1e12, 2),
                          gemm_ms=round(g, 1), gemm_tflops=round(gw / (g * 1e-3) / 1e12, 2), panel_ms=round(pn, 1), trsm_ms=round(tr_, 1))), flush=True)
    sysb.close()

for lvl, B in [(2, 129), (3, 129), (4, 1)]:
    run(lvl, B)
