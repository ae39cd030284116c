"""API-level timing of the VF least-squares steps at AFS-like sizes:
relocate_poles on 5 ORF channels and identify_residues on 48 channels for
(J, M) from the cfg5 size up to the J ~ 200 the cfg4 AFS reaches."""
import json
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_1511_04355_b200 as P  # noqa: E402

rng = np.random.default_rng(0)
out = {}
for J, M in ((40, 48), (80, 40), (120, 60), (160, 80), (210, 104)):
    s = 0.25 + 1j * np.linspace(0.0, 80.0, J)
    pairs = M // 2
    p = []
    for m in range(pairs):
        a = complex(-0.3 - 0.01 * m, 0.3 + 80.0 * (m + 0.5) / pairs)
        p += [a, a.conjugate()]
    p = np.array(p)
    v5 = rng.normal(size=(J, 5)) + 1j * rng.normal(size=(J, 5))
    v48 = rng.normal(size=(J, 48)) + 1j * rng.normal(size=(J, 48))
    P.relocate_poles(s, v5, p)
    t0 = time.perf_counter()
    for _ in range(5):
        P.relocate_poles(s, v5, p)
    tr = (time.perf_counter() - t0) / 5
    P.identify_residues(s, v48, p)
    t0 = time.perf_counter()
    for r in range(5):
        P.identify_residues(s, v48, p * (1.0 + 1e-12 * (r + 1)))  # new (s, poles): the solve operator is formed
    ti = (time.perf_counter() - t0) / 5
    out[f"J{J}_M{M}"] = {"relocate_ms": tr * 1e3, "identify_cold_ms": ti * 1e3}
print(json.dumps(out))
