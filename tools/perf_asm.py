"""BEM assembly stage split (far / near kernels) at cfg2 size (development tool)."""
import ctypes, json, sys
import numpy as np
sys.path.insert(0, ".")
import paper_1511_04355_b200 as P
from paper_1511_04355_b200 import BemSystem, mesh

L = P.lib()


def prof(kind):
    c, ms, wk = ctypes.c_int(), ctypes.c_double(), ctypes.c_double()
    P.api._check(L.fds_profile_read(kind, ctypes.byref(c), ctypes.byref(ms), ctypes.byref(wk)))
    return ms.value


for lvl, B in [(3, 129), (4, 1)]:
    V, F = mesh.icosphere(lvl)
    tr = mesh.pressure_traction(V, F)
    sysb = BemSystem(V, F, tr, channels=list(range(48)), max_batch=B)
    s = 0.25 + 1j * 2 * np.pi / 20.0 * np.arange(B)
    sysb.evaluate_batch_device(s)
    sysb.evaluate_batch_device(s)
    t = sysb.last_timing()
    P.api._check(L.fds_profile_enable(1))
    sysb.evaluate_batch_device(s)
    far, near = prof(3), prof(4)
    P.api._check(L.fds_profile_enable(0))
    print(json.dumps(dict(n=3 * F.shape[0], B=B, assembly_ms=round(t["assembly_ms"], 2), far_ms=round(far, 2),
                          near_ms=round(near, 2))), flush=True)
    sysb.close()
