import sys, numpy as np, time
sys.path.insert(0, ".")
import paper_1511_04355_b200 as P
rng = np.random.default_rng(0)
J, M = 210, 104
s = 0.25 + 1j * np.linspace(0.0, 80.0, J)
p = []
for m in range(M // 2):
    a = complex(-0.3 - 0.01 * m, 0.3 + 80.0 * (m + 0.5) / (M // 2)); p += [a, a.conjugate()]
p = np.array(p)
v5 = rng.normal(size=(J, 5)) + 1j * rng.normal(size=(J, 5))
v48 = rng.normal(size=(J, 48)) + 1j * rng.normal(size=(J, 48))
for r in range(2):
    P.relocate_poles(s, v5, p)
    P.identify_residues(s, v48, p * (1 + 1e-12 * (r + 1)))
