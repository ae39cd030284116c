"""AFS driver cost split on a BEM system (development tool): wall time of
run_afs vs the time spent in BEM solves, for a small and an all-DOF channel set."""
import json, math, sys, time
sys.path.insert(0, ".")
import numpy as np
import paper_1511_04355_b200 as P
from paper_1511_04355_b200 import mesh

V, F = mesh.icosphere(3)
tr = mesh.random_traction(F.shape[0], seed=0)
out = {}
for name, chans in (("16_points", list(range(0, 1280, 80))), ("all_dofs", None)):
    sysb = P.BemSystem(V, F, tr, channels=[3 * e + i for e in chans for i in range(3)] if chans else None)
    for solver in ("lu", "gmres"):
        sysb.set_solver(solver)
        cfg = dict(omega_max=math.pi * 256 / 20.0, eta=0.25, period=20.0, initial_count=12, validation_steps=6,
                   e1_threshold=float("inf"), e2_threshold=float("inf"))
        P.run_afs(sysb, **cfg)  # warm
        t0 = time.perf_counter()
        r = P.run_afs(sysb, **cfg)
        wall = time.perf_counter() - t0
        # solve-only time: the same frequencies evaluated (J0 batched + singles)
        s = np.asarray(r["samples"] if isinstance(r, dict) else r.samples)
        t1 = time.perf_counter()
        sysb.evaluate_batch(s[:12])
        for z in s[12:]:
            sysb.evaluate(z)
        solve = time.perf_counter() - t1
        out[f"{name}_{solver}"] = {"channels": sysb.descriptor().channel_count, "n_c": len(s), "afs_wall_s": wall,
                                   "solves_wall_s": solve, "driver_overhead_s": wall - solve}
    # driver-only cost: replay the recorded samples through a Python system (dict lookup)
    r = P.run_afs(sysb, **cfg)
    s = np.asarray(r["samples"]); vals = np.asarray(r["values"]).reshape(len(s), -1)
    table = {complex(z): vals[i] for i, z in enumerate(s)}

    class Replay:
        def descriptor(self):
            return P.api.SystemDescriptor(vals.shape[1], [])

        def evaluate(self, z):
            return table[complex(z)]

    P.run_afs(Replay(), **cfg)
    t0 = time.perf_counter()
    rr = P.run_afs(Replay(), **cfg)
    out[f"{name}_replay"] = {"channels": vals.shape[1], "n_c": len(rr["samples"]),
                             "driver_wall_s": time.perf_counter() - t0,
                             "same_samples": bool(np.array_equal(np.asarray(rr["samples"]), s))}
    sysb.close()
print(json.dumps(out))
