"""Dumps the cfg4 product AFS samples (reference defaults, tools/run_cfg4_afs.py
config) and, at the iteration with J samples, the pole relocation trajectory of
vector_fit (vecfit.cpp:410-488) on the ORF channels as the product computes it
and as the oracle computes it, from the same initial poles; plus the product's
single relocation step applied to each oracle iterate (isolates the per-step
difference from its propagation). The numpy/LAPACK leg is added on the CPU by
tools/afs_divergence_compare.py. Writes gpurun_out/cfg4_afs_dump.npz.

Usage: python tools/afs_divergence_dump.py [J=165]"""
import sys

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "oracle")
import paper_1511_04355_b200 as P  # noqa: E402
import pyoracle as O  # noqa: E402
from paper_1511_04355_b200 import BemSystem, mesh  # noqa: E402

J = int(sys.argv[1]) if len(sys.argv) > 1 else 165
T, NS = 20.0, 512
V, F = mesh.icosphere(4)
trac = mesh.random_traction(F.shape[0], seed=0)
pts = mesh.draw_indices(F.shape[0], 16, 0)
dofs = [3 * p + i for p in pts for i in range(3)]
sysb = BemSystem(V, F, trac, channels=dofs, max_batch=16)
try:
    P.run_afs(sysb, omega_max=np.pi * NS / T, eta=5.0 / T, period=T)
    raise SystemExit("expected the reference defaults to fail at cfg4")
except P.Error as e:
    part = e.partial
s, v, hist, orf = part["samples"], part["values"], part["history"], np.array(part["orf"])
row = [h for h in hist if int(h[0]) == J][0]
out = dict(samples=s, values=v, history=hist, orf=orf, J=J, mh=int(row[1]), ml=int(row[2]))
sj, vj = s[:J], v[:J][:, orf]
for tag, order in (("high", int(row[1])), ("low", int(row[2]))):
    p0 = O.initial_poles(max(abs(sj.imag)), order)
    po, pp = [p0], [p0]
    one = []
    for _ in range(3):
        po.append(O.canonical_poles(O.relocate_poles(sj, vj, po[-1])[0]))
        pp.append(O.canonical_poles(P.relocate_poles(sj, vj, pp[-1])[0]))
        one.append(O.canonical_poles(P.relocate_poles(sj, vj, po[-2])[0]))
    out[f"{tag}_oracle"] = np.array(po)
    out[f"{tag}_product"] = np.array(pp)
    out[f"{tag}_product_one_step"] = np.array(one)
np.savez("gpurun_out/cfg4_afs_dump.npz", **out)
print("saved", {k: np.shape(x) for k, x in out.items()})
