"""End-to-end run of every kernel family at sizes that take the production
code paths, for compute-sanitizer (memcheck / racecheck / synccheck).

    compute-sanitizer --tool racecheck python tools/sanitize_smoke.py [small|large]

small (default): BEM batch of 8 at N = 960 (cluster/DSMEM panels, super-panels,
the 3M TMA GEMM and its operand prep, L11^-1 strips, dataflow solve), one
single-matrix solve (look-ahead schedule), zgesv batches, the VF chain (device
pivoted-QR least squares, bulk-copy residue kernel, channel errors, selection),
rational_invert, FSM on frequency-major N_s = 512 spectra (TMA kernel),
channel-major and N_s = 218.
large: one n = 4500 matrix (panels wider than a 16-CTA cluster: the global-slot
panel kernel with its software group barrier, look-ahead on a side stream).
"""
import sys

sys.path[:0] = [".", "oracle", "tests"]
import numpy as np  # noqa: E402

import paper_1511_04355_b200 as P  # noqa: E402
from helpers import ModalFixture, contour_points  # noqa: E402
from paper_1511_04355_b200 import mesh  # noqa: E402

mode = sys.argv[1] if len(sys.argv) > 1 else "small"
rng = np.random.default_rng(0)
if mode == "large":
    n = 4500
    A = rng.normal(size=(1, n, n)) + 1j * rng.normal(size=(1, n, n))
    x = P.zgesv_batch(A, rng.normal(size=(1, n)) + 0j)
    print("ok large", np.isfinite(x).all())
    sys.exit(0)

V, F = mesh.icosphere(2)  # 320 triangles, N = 960
g = P.BemSystem(V, F, mesh.random_traction(F.shape[0], seed=0))
s8 = 0.25 + 1j * (2 * np.pi / 20.0) * np.arange(1, 9)
u = g.evaluate_batch(s8)  # batch of 8: super-panels + 3M TMA GEMM + dataflow solve
u1 = g.evaluate(0.5 + 0.5j)  # single matrix: look-ahead schedule
A = rng.normal(size=(5, 70, 70)) + 1j * rng.normal(size=(5, 70, 70))
x = P.zgesv_batch(A, rng.normal(size=(5, 70)) + 0j)
A2 = rng.normal(size=(3, 700, 700)) + 1j * rng.normal(size=(3, 700, 700))
x2 = P.zgesv_batch(A2, rng.normal(size=(3, 700)) + 0j)
fx = ModalFixture(6)
s, v = fx.samples(contour_points(0.35, 1.5 * fx.band, 40))
m, rep = P.vector_fit(s, v, [0, 1], 12, 3)
grid = contour_points(0.35, 40.0, 256)
ml, _ = P.vector_fit(s, v, [0, 1], 10, 3)
e = P.channel_errors(m, ml, grid)
sn = P.select_new_frequency(m, ml, grid, s, [0, 1], 0.01)
vb = rng.normal(size=(40, 300)) + 1j * rng.normal(size=(40, 300))
R, rms = P.identify_residues(s, vb, m.poles)  # 300 channels: ragged last 64-channel tile
h = P.rational_invert(m, np.linspace(0, 5, 100))
half = rng.normal(size=(37, 257)) + 1j * rng.normal(size=(37, 257))
f = P.fsm_invert(4.0, 512, 1.7, half)  # channel-major
import ctypes  # noqa: E402

import torch  # noqa: E402

hd = torch.tensor(np.ascontiguousarray(half.T), device="cuda")  # frequency-major [i][k] (TMA kernel)
od = torch.empty((37, 512), dtype=torch.float64, device="cuda")
P.api._check(P.lib().fds_fsm_invert_device_strided(ctypes.c_double(4.0), 512, ctypes.c_double(1.7), 37,
                                                   ctypes.c_void_p(hd.data_ptr()), ctypes.c_longlong(1),
                                                   ctypes.c_longlong(37), 1, ctypes.c_void_p(od.data_ptr()), None))
fdev = od.cpu().numpy()
f2 = P.fsm_invert(4.0, 218, 1.7, v.T[:, :1].repeat(110, axis=1))
print("ok small", np.isfinite(u).all(), np.isfinite(x).all(), np.isfinite(x2).all(), np.isfinite(h).all(),
      np.abs(f - fdev).max())
