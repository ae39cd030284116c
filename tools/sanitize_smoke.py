"""Small end-to-end run of every kernel family, for compute-sanitizer."""
import sys
sys.path[:0] = [".", "oracle", "tests"]
import numpy as np
import paper_1511_04355_b200 as P
from paper_1511_04355_b200 import mesh
from helpers import ModalFixture, contour_points

V, F = mesh.icosphere(1)
g = P.BemSystem(V, F, mesh.pressure_traction(V, F))
u = g.evaluate_batch(np.array([0.25 + 0.5j, 0.25 + 1.5j, 0.3 + 2j, 0.3 + 3j, 0.3 + 4j, 0.3 + 5j, 0.3 + 6j, 0.3 + 7j]))
u1 = g.evaluate(0.5 + 0.5j)
rng = np.random.default_rng(0)
A = rng.normal(size=(5, 70, 70)) + 1j * rng.normal(size=(5, 70, 70))
x = P.zgesv_batch(A, rng.normal(size=(5, 70)) + 0j)
fx = ModalFixture(6)
s, v = fx.samples(contour_points(0.35, 1.5 * fx.band, 40))
m, rep = P.vector_fit(s, v, [0, 1], 12, 3)
grid = contour_points(0.35, 40.0, 256)
ml, _ = P.vector_fit(s, v, [0, 1], 10, 3)
e = P.channel_errors(m, ml, grid)
sn = P.select_new_frequency(m, ml, grid, s, [0, 1], 0.01)
h = P.rational_invert(m, np.linspace(0, 5, 100))
f = P.fsm_invert(4.0, 512, 1.7, v.T[:, :1].repeat(257, axis=1))
f2 = P.fsm_invert(4.0, 218, 1.7, v.T[:, :1].repeat(110, axis=1))
print("ok", np.isfinite(u).all(), np.isfinite(x).all(), np.isfinite(h).all())
