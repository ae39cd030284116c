import sys, math
sys.path[:0] = ['.', 'oracle', 'tests']
import numpy as np
import paper_1511_04355_b200 as P, pyoracle as O
from paper_1511_04355_b200 import mesh
from helpers import worst_match
V, F = mesh.icosphere(2); tr = mesh.pressure_traction(V, F)
pts = mesh.draw_indices(F.shape[0], 16, 0); dofs = [3*p+i for p in pts for i in range(3)]
g = P.BemSystem(V, F, tr, channels=dofs)
wmax = math.pi*256/20
s = O.initial_frequencies(12, 0.25, wmax)
vals = g.evaluate_batch(s)
orf = mesh.draw_indices(48, 5, 0)
for M in (6, 5):
    mg, rg = P.vector_fit(s, vals, orf, M, 3)
    mo = O.vector_fit(s, vals, orf, M, 3)
    print("M", M, "poles", worst_match(mg.poles, mo["poles"]), "iters", rg["iterations"], mo["iterations"])
    print("  poles g", np.sort_complex(mg.poles))
    print("  poles o", np.sort_complex(mo["poles"]))
    # residues compare (match pole order)
    idx = [int(np.argmin(np.abs(mg.poles - p))) for p in mo["poles"]]
    d = np.abs(mg.residues[:, idx] - mo["residues"]).max() / np.abs(mo["residues"]).max()
    print("  residue max rel diff", d, "rms g/o", rg["rms"][:4], mo["rms"][:4])
grid = 0.25 + 1j*wmax*np.arange(4096)/4095
mh = P.vector_fit(s, vals, orf, 6, 3)[0]; ml = P.vector_fit(s, vals, orf, 5, 3)[0]
oh = O.vector_fit(s, vals, orf, 6, 3); ol = O.vector_fit(s, vals, orf, 5, 3)
eg = P.channel_errors(mh, ml, grid)
eo = O.channel_errors(oh["poles"], oh["residues"], ol["poles"], ol["residues"], grid)
print("errors g", eg[:8]); print("errors o", eo[:8])
# cross: oracle models evaluated by GPU channel_errors
ec = P.channel_errors(P.RationalModel(oh["poles"], oh["residues"]), P.RationalModel(ol["poles"], ol["residues"]), grid)
print("errors gpu-on-oracle-models", ec[:8])
