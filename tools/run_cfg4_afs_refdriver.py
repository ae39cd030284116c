"""cfg4 AFS at the reference defaults, product vs the reference's own driver.

Both sides see the same responses: the product's run_afs (GPU BEM + GPU VF,
csrc/afs.cpp) and the REFERENCE run_afs (/root/reference/proj/src/afs.cpp:226-396,
compiled unmodified into the oracle, with the oracle's CPU restatement of
vecfit.cpp) driving a callback system whose evaluate(s) is the product's GPU
BEM solve (N = 15360 solves are ~10 s each on the oracle's CPU path; the GPU
solution matches the oracle's OpenBLAS solve to ~1e-14, tests/test_gpu_northstar.py).
Reports each side's outcome (n_c / error class / J at failure) and the length of
the identical sampled-frequency prefix. Config as tools/run_cfg4_afs.py.

Usage: python tools/run_cfg4_afs_refdriver.py [max_iterations]
"""
import json
import sys
import time

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "oracle")
import paper_1511_04355_b200 as P  # noqa: E402
import pyoracle as O  # noqa: E402
from paper_1511_04355_b200 import BemSystem, mesh  # noqa: E402

T, NS = 20.0, 512
max_iter = int(sys.argv[1]) if len(sys.argv) > 1 else 500
V, F = mesh.icosphere(4)
trac = mesh.random_traction(F.shape[0], seed=0)
pts = mesh.draw_indices(F.shape[0], 16, 0)
dofs = [3 * p + i for p in pts for i in range(3)]
cfg = dict(omega_max=np.pi * NS / T, eta=5.0 / T, period=T, max_iterations=max_iter)
out = {"config": "cfg4 AFS at the reference defaults (afs.hpp:21-39), N=15360, random traction seed 0, "
                  "T=20, Omega=pi*512/T, eta=5/T, 48 channels (16 points x 3), ORFs drawn with seed 0",
       "max_iterations": max_iter}

sysb = BemSystem(V, F, trac, channels=dofs, max_batch=16)
t0 = time.perf_counter()
try:
    r = P.run_afs(sysb, **cfg)
    prod = dict(n_c=r["n_c"], converged=r["converged"], samples=r["samples"], error=None)
    cache = {}
except P.Error as e:
    part = getattr(e, "partial", {}) or {}
    prod = dict(error=type(e).__name__, msg=str(e), samples=part.get("samples", np.zeros(0)),
                n_c=part.get("n_c"), history_last=part.get("history", np.zeros((1, 8)))[-1:].tolist())
    # the product's responses at the frequencies it sampled (served to the
    # reference driver when it asks for the same s, so both see identical data)
    cache = {complex(sv): part["values"][i] for i, sv in enumerate(part.get("samples", []))}
prod["wall_s"] = time.perf_counter() - t0

single = BemSystem(V, F, trac, channels=dofs, max_batch=1)
calls = [0]


def fn(s):
    if s in cache:
        return cache[s]
    calls[0] += 1
    return single.evaluate(s)


sysr = O.System.callback(len(dofs), fn)
t0 = time.perf_counter()
try:
    rr = O.run_afs(sysr, **cfg)
    ref = dict(n_c=rr["n_c"], converged=rr["converged"], samples=rr["samples"], error=None)
except O.OracleError as e:
    rpart = getattr(e, "partial", {}) or {}
    ref = dict(error=str(e).split(":")[0], msg=str(e), samples=rpart.get("samples", np.zeros(0)),
               n_c=rpart.get("n_c"))
ref["wall_s"] = time.perf_counter() - t0
ref["fresh_gpu_solves"] = calls[0]

a, b = np.asarray(prod["samples"]), np.asarray(ref["samples"])
same = 0
while same < min(len(a), len(b)) and a[same] == b[same]:
    same += 1
# Why the sequences part: refit the iteration at the first differing selection
# (J = same samples, identical on both sides) with both VF implementations and
# report how far their relocated poles are apart and how close the oracle's last
# stacked sigma system is to Eigen's rank threshold (afs.cpp:337-340,
# vecfit.cpp:281-285).
diag = {}
if prod.get("error") and "part" in dir() and same >= 16:
    hist = np.asarray(part.get("history", np.zeros((0, 8))))
    row = [h for h in hist if int(h[0]) == same]
    vals = part["values"][:same]
    orf = list(part.get("orf", []))
    if row and orf:
        mh, ml = int(row[0][1]), int(row[0][2])
        for tag, order in (("high", mh), ("low", ml)):
            mg, _ = P.vector_fit(a[:same], vals, orf, order, 3)
            mo = O.vector_fit(a[:same], vals, orf, order, 3)
            po = np.asarray(mo["poles"])
            worst = max(min(abs(g - w) / abs(w) for g in mg.poles) for w in po)
            A_, b_, _ = O.last_relocation()
            qr = O.colpivqr(A_, b_)
            rd = np.abs(qr["rdiag"])
            diag[tag] = dict(order=order, worst_pole_rel_diff=worst, sigma_rows=int(A_.shape[0]),
                             sigma_cols=int(A_.shape[1]), rank=qr["rank"],
                             min_over_max_rdiag=float(rd.min() / rd.max()))
for d in (prod, ref):
    d["samples_count"] = int(len(d["samples"]))
    d["samples"] = None
out.update(product=prod, reference=ref, identical_prefix=same, divergence_refit=diag)
print(json.dumps(out, default=lambda x: x.tolist() if hasattr(x, "tolist") else str(x)))
