"""Iterative vs direct BEM solves on one B200: cfg4
(sphere, N = 15360, random traction) and cfg3 (cube, N = 36864, pressure), one
frequency each: assembly + LU + substitution against assembly + GMRES
(tol 1e-12, restart 60, block-Jacobi). Prints one JSON object."""
import json, math, sys, time
sys.path.insert(0, ".")
import numpy as np
import paper_1511_04355_b200 as P
from paper_1511_04355_b200 import mesh

out = {}
for name, (V, F), load in [("cfg4_N15360", mesh.icosphere(4), "random"), ("cfg3_N36864", mesh.cube_cavity(32), "pressure")]:
    tr = mesh.random_traction(F.shape[0], seed=0) if load == "random" else mesh.pressure_traction(V, F)
    sysb = P.BemSystem(V, F, tr, max_batch=1)
    s = np.array([0.25 + 1j * 2 * math.pi / 20.0 * 7])
    res = {}
    for solver in ("lu", "gmres"):
        sysb.set_solver(solver, tol=1e-12, restart=60, max_iter=2000)
        sysb.evaluate_batch(s)  # warm
        t0 = time.perf_counter()
        u = sysb.evaluate_batch(s)
        wall = time.perf_counter() - t0
        t = sysb.last_timing()
        res[solver] = dict(u=u, wall_s=wall, **t)
        if solver == "gmres":
            res[solver].update(sysb.last_gmres())
    du = float(np.linalg.norm(res["gmres"]["u"] - res["lu"]["u"]) / np.linalg.norm(res["lu"]["u"]))
    for r in res.values():
        r.pop("u")
    n = 3 * F.shape[0]
    out[name] = {"n": n, "lu": res["lu"], "gmres": res["gmres"], "rel_diff_gmres_vs_lu": du,
                 "matvec_bytes": 16.0 * n * n,
                 "speedup_device": (res["lu"]["assembly_ms"] + res["lu"]["lu_ms"] + res["lu"]["solve_ms"]) /
                                   (res["gmres"]["assembly_ms"] + res["gmres"]["lu_ms"] + res["gmres"]["solve_ms"])}
    sysb.close()
print(json.dumps(out))
