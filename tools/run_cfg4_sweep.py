"""BASELINE config 4: 5120-triangle sphere (N = 15360), seeded random traction,
full FSM sweep (N_s = 512 -> N_c = 257 frequencies) versus AFS, timing assembly,
LU, solve and reconstruction separately. Writes one JSON object to stdout.

Usage: python tools/run_cfg4_sweep.py [max_afs_iterations]
"""
import json
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_1511_04355_b200 as P  # noqa: E402
from paper_1511_04355_b200 import BemSystem, mesh  # noqa: E402

T, NS = 20.0, 512
ETA = 5.0 / T
NC = NS // 2 + 1
max_iter = int(sys.argv[1]) if len(sys.argv) > 1 else 40

V, F = mesh.icosphere(4)
trac = mesh.random_traction(F.shape[0], seed=0)
out = {"config": "cfg4: icosphere(4), 5120 triangles, N = 15360, random traction seed 0, T = 20, N_s = 512, "
                 "eta = 5/T", "n": 3 * F.shape[0]}

# ---- full FSM sweep: 257 frequencies in batches of 32 (32 x 3.77 GB matrices)
sysb = BemSystem(V, F, trac, max_batch=32)
sk = ETA + 1j * 2 * np.pi / T * np.arange(NC)
stage = dict(assembly_ms=0.0, lu_ms=0.0, solve_ms=0.0)
spectra = np.zeros((NC, sysb.descriptor().channel_count), np.complex128)
t0 = time.perf_counter()
for c0 in range(0, NC, 32):
    spectra[c0:c0 + 32] = sysb.evaluate_batch(sk[c0:c0 + 32])
    lt = sysb.last_timing()
    for key in stage:
        stage[key] += lt[key]
sweep_s = time.perf_counter() - t0
t1 = time.perf_counter()
h = P.fsm_invert(T, NS, ETA, spectra.T.copy())  # (K, N_s) displacement histories
fsm_api_ms = (time.perf_counter() - t1) * 1e3
out["fsm_sweep"] = {"frequencies": NC, "batch": 32, "wall_s": sweep_s, **stage,
                    "fsm_invert_api_ms": fsm_api_ms, "channels": spectra.shape[1],
                    "solves_per_s": NC / sweep_s,
                    "max_abs_displacement": float(np.max(np.abs(h)))}

# ---- AFS on the same system (reference defaults, omega_max = Omega_s, 5 ORFs drawn by the driver)
cfg = dict(omega_max=np.pi * NS / T, eta=ETA, period=T, max_iterations=max_iter)
t0 = time.perf_counter()
try:
    r = P.run_afs(BemSystem(V, F, trac, max_batch=16), **cfg)
    afs = {"wall_s": time.perf_counter() - t0, "n_c": r["n_c"], "converged": r["converged"],
           "solver_calls": r["solver_calls"], "order": int(len(r["poles"])),
           "last_history": r["history"][-1].tolist() if len(r["history"]) else None}
except P.Error as e:  # the reference algorithm's own failure modes
    afs = {"wall_s": time.perf_counter() - t0, "error": f"{type(e).__name__}: {e}"}
afs["max_iterations"] = max_iter
out["afs"] = afs
print(json.dumps(out))
