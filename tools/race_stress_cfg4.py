"""Race stress at the north_star size (development evidence, complements
tests/test_gpu_race_stress.py, which runs small systems inside the test budget):
cfg4 (N = 15360) solved as a batch of 2 (super-panel schedule, global-slot and
cluster panels, 3M GEMM ring, dataflow solve) and as a single matrix
(look-ahead schedule with the side-stream panel), and cfg3 (N = 36864) as a
single matrix (a 144-CTA global-slot panel behind one software barrier), a
36 x 36 cube (N = 46656: 183 panel CTAs, more than one per SM), twice
under the product build
and twice under the timing-perturbed FDS_JITTER build. Correct synchronisation
means identical SHA-256 digests. Prints one JSON object."""
import json
import os
import subprocess
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
CODE = r'''
import sys, json, hashlib, time
sys.path[:0] = [ROOT]
import numpy as np
import paper_1511_04355_b200 as P
from paper_1511_04355_b200 import mesh
h = lambda a: hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()
V, F = mesh.icosphere(4)
g = P.BemSystem(V, F, mesh.random_traction(F.shape[0], seed=0), max_batch=2)
s2 = 0.25 + 1j * (2 * np.pi / 20.0) * np.array([7.0, 200.0])
out = {"batch2": [], "single": []}
t0 = time.perf_counter()
for rep in range(2):
    out["batch2"].append(h(g.evaluate_batch(s2)))
    out["single"].append(h(g.evaluate(s2[0])))
g.close()
V3, F3 = mesh.cube_cavity(32)
g3 = P.BemSystem(V3, F3, mesh.pressure_traction(V3, F3), max_batch=1)
out["cfg3_single"] = [h(g3.evaluate(s2[0])) for _ in range(2)]  # P = 144 CTAs behind one software barrier
g3.close()
V5, F5 = mesh.cube_cavity(36)
g5 = P.BemSystem(V5, F5, mesh.pressure_traction(V5, F5), max_batch=1)
out["n46656_single"] = [h(g5.evaluate(s2[0])) for _ in range(2)]  # P = 183 CTAs, several per SM
g5.close()
out["wall_s"] = time.perf_counter() - t0
out["library"] = str(P.library_path())
print("RESULT" + json.dumps(out))
'''


def run(variant):
    env = dict(os.environ)
    env.pop("FDSWEEP_LIB_VARIANT", None)
    if variant:
        env["FDSWEEP_LIB_VARIANT"] = variant
    r = subprocess.run([sys.executable, "-c", CODE.replace("ROOT", repr(str(ROOT)))], env=env,
                       capture_output=True, text=True, timeout=3000)
    if r.returncode != 0:
        raise SystemExit(r.stderr[-3000:])
    return json.loads([l for l in r.stdout.splitlines() if l.startswith("RESULT")][-1][6:])


base, jit = run(None), run("jitter")
ok = all(len(set(base[k])) == 1 and set(jit[k]) == set(base[k]) for k in ("batch2", "single", "cfg3_single", "n46656_single"))
print(json.dumps({"workload": "cfg4 N=15360: batch of 2 (k = 7, 200) and a single matrix (k = 7); cfg3 N=36864 single "
                              "matrix (k = 7); N=46656 cube single matrix (panel CTAs share SMs); 2 runs per build",
                  "product": base, "jitter": jit, "bit_identical": ok}))
