"""Race / synchronisation stress for the hand-rolled protocols (compute-sanitizer
is closed on this GPU pool: profiles/r02_compute_sanitizer_closed.log).

libfdsweep_b200_jitter.so is the product code compiled with FDS_JITTER: every
hand-rolled synchronisation point sleeps a pseudo-random 0-8 us before it
proceeds (common.cuh fds_jitter):
  * the 3M GEMM's barrier-free stage ring ("last warp out refills",
    lu_gemm3m_tma_kernel) at every k-chunk;
  * the cluster/DSMEM panel before every per-column cluster barrier and the
    global-slot panel's software group barrier;
  * the dataflow substitution's flag publication and readiness polls;
  * the producer/consumer mbarrier rings of the bulk-copy residue kernel and
    the TMA FSM kernel.
Every reduction in the library has a fixed order, so correct synchronisation
means the perturbed build returns results BIT-IDENTICAL to the product build on
the same inputs; a missing fence, barrier or release/acquire would surface as
corrupted or merely different bits under the changed interleavings. Each
workload runs several times in a subprocess per library build.
"""
import json
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parent.parent

WORKLOAD = r'''
import sys, json, hashlib
sys.path[:0] = [ROOT, ROOT + "/oracle", ROOT + "/tests"]
import numpy as np, ctypes, torch
import paper_1511_04355_b200 as P
from paper_1511_04355_b200 import mesh
from helpers import ModalFixture, contour_points
out = {}
def h(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()
V, F = mesh.icosphere(2)
g = P.BemSystem(V, F, mesh.random_traction(F.shape[0], seed=0))
s8 = 0.25 + 1j * (2 * np.pi / 20.0) * np.arange(1, 9)
for rep in range(REPS):
    out.setdefault("bem_batch8", []).append(h(g.evaluate_batch(s8)))     # cluster panels, super-panels, 3M GEMM, dataflow
    out.setdefault("bem_single", []).append(h(g.evaluate(0.5 + 0.5j)))    # look-ahead schedule
rng = np.random.default_rng(0)
n = 4500
A = rng.normal(size=(1, n, n)) + 1j * rng.normal(size=(1, n, n))
b = rng.normal(size=(1, n)) + 0j
for rep in range(2):
    out.setdefault("zgesv_4500", []).append(h(P.zgesv_batch(A, b)))      # global-slot panel (P > 16), software barrier
fx = ModalFixture(6)
s, v = fx.samples(contour_points(0.35, 1.5 * fx.band, 40))
m, _ = P.vector_fit(s, v, [0, 1], 12, 3)
vb = rng.normal(size=(40, 20000)) + 1j * rng.normal(size=(40, 20000))
for rep in range(REPS):
    R, _ = P.identify_residues(s, vb, m.poles)                          # bulk-copy residue ring
    out.setdefault("residues", []).append(h(R))
half = rng.normal(size=(3001, 257)) + 1j * rng.normal(size=(3001, 257))
hd = torch.tensor(np.ascontiguousarray(half.T), device="cuda")
od = torch.empty((3001, 512), dtype=torch.float64, device="cuda")
for rep in range(REPS):
    P.api._check(P.lib().fds_fsm_invert_device_strided(ctypes.c_double(4.0), 512, ctypes.c_double(1.7), 3001,
        ctypes.c_void_p(hd.data_ptr()), ctypes.c_longlong(1), ctypes.c_longlong(3001), 1,
        ctypes.c_void_p(od.data_ptr()), None))
    out.setdefault("fsm_freq_major", []).append(h(od.cpu().numpy()))    # TMA FSM ring
out["library"] = str(P.library_path())
print("RESULT" + json.dumps(out))
'''


def _run(variant, reps):
    env = dict(os.environ)
    if variant:
        env["FDSWEEP_LIB_VARIANT"] = variant
    else:
        env.pop("FDSWEEP_LIB_VARIANT", None)
    code = WORKLOAD.replace("ROOT", repr(str(ROOT))).replace("REPS", str(reps))
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=1200)
    assert r.returncode == 0, r.stderr[-3000:]
    line = [l for l in r.stdout.splitlines() if l.startswith("RESULT")][-1]
    return json.loads(line[len("RESULT"):])


def test_jitter_build_is_bit_identical_to_product():
    lib = ROOT / "paper_1511_04355_b200" / "libfdsweep_b200_jitter.so"
    assert lib.exists(), "build the stress library: make -C paper_1511_04355_b200"
    base = _run(None, 2)
    jit = _run("jitter", 4)
    assert base["library"].endswith("libfdsweep_b200.so") and jit["library"].endswith("_jitter.so")
    for key, hashes in base.items():
        if key == "library":
            continue
        assert len(set(hashes)) == 1, f"{key}: product build not deterministic"
        assert set(jit[key]) == set(hashes), f"{key}: timing-perturbed build differs (synchronisation bug)"
