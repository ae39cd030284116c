"""The drop-in boundary end to end: the reference's OWN run_afs / system factory
(proj/src/afs.cpp, systems.cpp — compiled unmodified into integration/_build/
demo_afs) linked against libfdsweep_b200 through include/fdsweep_b200_shim.hpp
must sample exactly the frequencies the all-CPU oracle samples."""
import json
import math
import struct
import subprocess
from pathlib import Path

import numpy as np
import pytest

import pyoracle as O
from helpers import ModalFixture
from paper_1511_04355_b200 import mesh

pytestmark = pytest.mark.gpu
DEMO = Path(__file__).resolve().parent.parent / "integration" / "_build" / "demo_afs"


def _run(args):
    if not DEMO.exists():
        pytest.skip("integration demo not built (needs /root/reference at build time)")
    out = subprocess.run([str(DEMO)] + args, capture_output=True, text=True, timeout=600)
    d = json.loads(out.stdout.strip().splitlines()[-1])
    assert "error" not in d, d
    return d


def test_reference_run_afs_modal_on_gpu_fits(tmp_path):
    fx = ModalFixture(6)
    p = tmp_path / "modal.json"
    p.write_text(fx.system_json())
    d = _run(["modal", str(p)])
    o = O.run_afs(O.System.from_json(fx.system_json()), omega_max=1.5 * 29.8, eta=0.35, period=20.0,
                  orf=[0, 1, 2], test=[3, 4, 5], grid_points=1024, time_points=256, e1_threshold=1e-2,
                  e2_threshold=5e-2)
    got = np.array([complex(a, b) for a, b in d["samples"]])
    assert d["n_c"] == o["n_c"] and d["converged"] == o["converged"]
    np.testing.assert_array_equal(got, o["samples"])


def test_reference_run_afs_on_gpu_bem_system(tmp_path):
    V, F = mesh.icosphere(2)
    tr = mesh.random_traction(F.shape[0], seed=0)
    pts = mesh.draw_indices(F.shape[0], 16, 0)
    dofs = np.array([3 * p + i for p in pts for i in range(3)], np.int32)
    f = tmp_path / "mesh.bin"
    with open(f, "wb") as fh:
        fh.write(struct.pack("ii", V.shape[0], F.shape[0]))
        fh.write(np.ascontiguousarray(V, np.float64).tobytes())
        fh.write(np.ascontiguousarray(F, np.int32).tobytes())
        fh.write(np.ascontiguousarray(tr, np.float64).tobytes())
        fh.write(struct.pack("i", len(dofs)))
        fh.write(dofs.tobytes())
    d = _run(["bem", str(f)])
    o = O.run_afs(O.System.bem(O.Bem(V, F, tr), dofs), omega_max=math.pi * 256 / 20.0, eta=0.25, period=20.0,
                  initial_count=12, e1_threshold=float("inf"), e2_threshold=float("inf"), validation_steps=6)
    got = np.array([complex(a, b) for a, b in d["samples"]])
    assert d["n_c"] == o["n_c"] == 18 and d["solver_calls"] == 18
    np.testing.assert_array_equal(got, o["samples"])
