"""Generates tests/golden/afs_defaults_pressurised_sphere.json: the outcome of
the REFERENCE run_afs (/root/reference/proj/src/afs.cpp:226-396, compiled
unmodified into oracle/_ref, with the oracle's restatement of vecfit.cpp) at
the reference defaults (afs.hpp:21-39) on the pressurised cfg1 sphere
(icosphere(2), 320 triangles, every one of the 960 DOFs a channel, 5 ORFs
drawn with seed 0), solved by the oracle BEM.

The oracle run takes ~12 min of host CPU, too long for the GPU test budget,
so tests/test_gpu_northstar.py compares the product against this fixture.
Run from the repo root: python tests/golden/make_afs_defaults_fixture.py
"""
import json
import math
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path[:0] = [str(ROOT), str(ROOT / "oracle")]
import pyoracle as O  # noqa: E402
from paper_1511_04355_b200 import mesh  # noqa: E402

T_PERIOD = 20.0
V, F = mesh.icosphere(2)
tr = mesh.pressure_traction(V, F)
kw = dict(omega_max=math.pi * 256 / T_PERIOD, eta=0.25, period=T_PERIOD)
t0 = time.perf_counter()
out = {"what": __doc__.strip().splitlines()[0], "mesh": "icosphere(2) pressure_traction", "config": kw,
       "channels": 3 * F.shape[0]}
try:
    r = O.run_afs(O.System.bem(O.Bem(V, F, tr), list(range(3 * F.shape[0]))), **kw)
    out.update(error=None, n_c=r["n_c"], samples=[[z.real, z.imag] for z in r["samples"]])
except O.OracleError as e:
    p = e.partial
    out.update(error=e.kind, message=str(e), n_c=p["n_c"], solver_calls=p["solver_calls"],
               samples=[[z.real, z.imag] for z in p["samples"]])
out["oracle_wall_s"] = round(time.perf_counter() - t0, 1)
(Path(__file__).parent / "afs_defaults_pressurised_sphere.json").write_text(json.dumps(out, indent=0) + "\n")
print(out["error"], out["n_c"], out["oracle_wall_s"])
