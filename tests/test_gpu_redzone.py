"""Out-of-bounds write check of the device library (memcheck stand-in: compute-sanitizer is closed on
this GPU pool, profiles/r02_compute_sanitizer_closed.log). A child pytest process runs the functional
GPU suites with FDSWEEP_REDZONE=1: every cudaMalloc of the library then carries a 4 KB guard zone on
each side (csrc/common.cuh), compared on every free and, for the allocations still live, at session
end (tests/conftest.py); fresh allocations are pre-filled with 0xFF (NaN / -1), so the suites' parity
assertions also fail on any dependence on memory the library never wrote. The suites cover the odd sizes where an overrun would show: LU n = 1 ... 3001
with forced pivoting and every 64/128/256 boundary, ragged VF / FSM tiles, batches that do not fill a
chunk, GMRES restarts, the AFS driver."""
import os
import re
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
SUITES = ["tests/test_gpu_bem.py", "tests/test_gpu_vf.py", "tests/test_gpu_edge_cases.py", "tests/test_gpu_gmres.py",
          "tests/test_gpu_fullsize.py"]


@pytest.mark.gpu
def test_no_write_outside_any_device_allocation():
    env = dict(os.environ, FDSWEEP_REDZONE="1")
    r = subprocess.run([sys.executable, "-m", "pytest", *SUITES, "-m", "gpu", "-q", "-x", "-s", "-p", "no:cacheprovider"],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=1500)
    tail = (r.stdout + r.stderr)[-3000:]
    m = re.search(r"redzone: enabled=1 overwritten_bytes=(\d+) checks=(\d+) live=(\d+)", r.stdout)
    assert m, tail
    assert int(m.group(1)) == 0, tail
    assert int(m.group(2)) > 100 and int(m.group(3)) > 0, tail  # the mode was live and zones were compared
    assert r.returncode == 0, tail


_CONTROL = r"""
import ctypes, sys
import numpy as np
sys.path.insert(0, ".")
import paper_1511_04355_b200 as P
from paper_1511_04355_b200 import BemSystem, mesh
V, F = mesh.icosphere(2)
K, B = 48, 2
sysb = BemSystem(V, F, mesh.pressure_traction(V, F), channels=list(range(K)), max_batch=B)
ptr = sysb.evaluate_batch_device(0.25 + 1j * np.array([1.0, 2.0]))
clean = P.api.redzone_check()
import torch  # its CUDA runtime shares the primary context: an 8-byte write just past the K x B result buffer
rt = ctypes.CDLL("libcudart.so.12")
rt.cudaMemset.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_size_t]
assert rt.cudaMemset(ctypes.c_void_p(ptr + B * K * 16), 0, 8) == 0
assert rt.cudaDeviceSynchronize() == 0
dirty = P.api.redzone_check()
print("control", int(clean["enabled"]), clean["overwritten_bytes"], dirty["overwritten_bytes"])
"""


@pytest.mark.gpu
def test_redzone_detects_a_deliberate_overrun():
    """Negative control: 8 bytes written just past the library's response buffer are reported."""
    env = dict(os.environ, FDSWEEP_REDZONE="1")
    r = subprocess.run([sys.executable, "-c", _CONTROL], cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    m = re.search(r"control 1 0 (\d+)", r.stdout)
    assert m and int(m.group(1)) == 8, (r.stdout + r.stderr)[-2000:]
