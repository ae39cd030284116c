"""cfg2 batch (129 frequencies, N = 3840) LU timing and per-stage profile."""
import ctypes
import json
import sys

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_1511_04355_b200 as P  # noqa: E402
from paper_1511_04355_b200 import BemSystem  # noqa: E402

V, F, tr, dofs, s = bench.cfg2_inputs()
sysb = BemSystem(V, F, tr, channels=dofs, max_batch=len(s))
for _ in range(3):
    sysb.evaluate_batch_device(s)
    print(sysb.last_timing())
L = P.lib()
P.api._check(L.fds_profile_enable(1))
sysb.evaluate_batch_device(s)
print(json.dumps(bench.profile_stages(P, L)))
P.api._check(L.fds_profile_enable(0))
