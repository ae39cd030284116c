import sys, math, time
sys.path[:0] = ['.', 'oracle', 'tests']
import numpy as np
import paper_1511_04355_b200 as P
from paper_1511_04355_b200 import mesh
for lvl in (2, 3):
    V, F = mesh.icosphere(lvl); tr = mesh.random_traction(F.shape[0], seed=0)
    pts = mesh.draw_indices(F.shape[0], 16, 0); dofs = [3*p+i for p in pts for i in range(3)]
    g = P.BemSystem(V, F, tr, channels=dofs)
    for e1, e2 in ((1e-4, 2e-3), (1e-3, 1e-2)):
        t = time.time()
        try:
            r = P.run_afs(g, omega_max=math.pi*256/20.0, eta=0.25, period=20.0, initial_count=16, e1_threshold=e1, e2_threshold=e2, max_iterations=200)
            print(lvl, e1, e2, "nc", r["n_c"], r["converged"], "%.1fs" % (time.time()-t), r["history"][-4:, [0, 6, 7]].tolist(), flush=True)
        except Exception as ex:
            print(lvl, e1, e2, type(ex).__name__, ex, "%.1fs" % (time.time()-t), flush=True)
