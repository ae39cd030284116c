"""CPU-side checks of the drop-in boundary: the C-ABI library loads and exports
every entry point include/fdsweep_b200.h declares (no compute without a GPU),
host-side mesh/load generators, and the multi-rank bench plumbing (gloo).
"""
import ctypes
import os
import re
import socket
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

import paper_1511_04355_b200 as P
import pyoracle as O
from paper_1511_04355_b200 import mesh

ROOT = Path(__file__).resolve().parent.parent


def declared_symbols():
    text = (ROOT / "include" / "fdsweep_b200.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(fds_[a-z0-9_]+)\s*\(", text)) - {"fds_system_fn"})


def test_library_exports_every_declared_symbol():
    lib = P.lib()
    syms = declared_symbols()
    assert len(syms) >= 25
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    assert lib.fds_version().decode().startswith("fdsweep_b200")


def test_library_built_for_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", str(P.library_path())], capture_output=True, text=True)
    assert "sm_100a" in out.stdout


def test_library_has_dmma_tma_and_cluster_sass():
    out = subprocess.run(["cuobjdump", "-sass", str(P.library_path())], capture_output=True, text=True).stdout
    assert "DMMA" in out  # LU trailing GEMM, TRSM, residues, rational inversion on the FP64 tensor pipe
    assert "UTMALDG" in out  # TMA-fed trailing GEMM (cp.async.bulk.tensor)
    assert "UCGABAR_ARV" in out and "UCGABAR_WAIT" in out  # cluster barrier of the DSMEM pivot exchange


def test_no_gpu_fails_loudly():
    """Without a GPU the product must raise, never fall back to a CPU path."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(P.CudaError):
        V, F = mesh.icosphere(0)
        P.BemSystem(V, F, mesh.pressure_traction(V, F))


def test_draw_indices_matches_reference():
    # the reference's draw_indices (afs.cpp:28-46) picks the ORFs when none are given
    fx_json = '{"type": "modal", "omega": [1.0, 2.0], "zeta": [0.1, 0.1], "participation": ' + \
              "{" + ", ".join(f'"c{k}": [1.0, {k + 1.0}]' for k in range(12)) + "}}"
    sysm = O.System.from_json(fx_json)
    r = O.run_afs(sysm, omega_max=3.0, eta=0.3, period=10.0, initial_count=8, e1_threshold=float("inf"),
                  e2_threshold=float("inf"), grid_points=64, time_points=32, seed=11, validation_steps=0,
                  test=[0])
    assert list(r["orf"]) == mesh.draw_indices(12, 5, 11)


def test_meshes():
    V, F = mesh.icosphere(4)
    assert F.shape == (5120, 3)
    V, F = mesh.cube_cavity(32)
    assert F.shape == (12288, 3)
    c, n, a = mesh.element_geometry(V, F)
    assert abs(a.sum() - 6.0) < 1e-12
    tr = mesh.random_traction(10, 0)
    assert tr.shape == (10, 3) and abs(tr.mean()) < 1.5


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_bench_replica_reduction_gloo():
    """bench.py's N > 1 plumbing over world_size 2 (gloo, CPU): the contour's
    sub-batches are dealt to the replicas without overlap inside a step, the
    step time is the max over ranks and the value is the whole-job aggregate."""
    code = r'''
import os, sys, numpy as np, torch.distributed as dist
sys.path.insert(0, os.environ["FDS_ROOT"])
import bench
dist.init_process_group("gloo")
r, w = dist.get_rank(), dist.get_world_size()
s = bench.contour(bench.NS4)
mine = [bench.sub_batch(s, i, r, w) for i in range(4)]
assert all(len(b) == bench.SUB for b in mine)
# every step: the two replicas hold different frequencies of the contour
import torch
for b in mine:
    first = torch.tensor([b[0].imag], dtype=torch.float64)
    both = [torch.zeros(1, dtype=torch.float64) for _ in range(w)]
    dist.all_gather(both, first)
    assert len({float(x) for x in both}) == w
# over NSUB / w steps the replicas cover the 8 full sub-batches exactly once
cover = torch.zeros(bench.NSUB, dtype=torch.float64)
for i in range(bench.NSUB // w):
    cover[(i * w + r) % bench.NSUB] += 1
dist.all_reduce(cover)
assert cover.tolist() == [1.0] * bench.NSUB
total_ms = bench.allreduce_max(dist, 1000.0 + 500.0 * r)   # slowest rank wins
assert total_ms == 1500.0
v = bench.whole_job_rate(bench.SUB, w, 3, total_ms)
assert abs(v - bench.SUB * w * 3 / 1.5) < 1e-12
bench.barrier(dist)
if r == 0: print("OK", w)
dist.destroy_process_group()
'''
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()), FDS_ROOT=str(ROOT))
    procs = []
    for r in range(2):
        e = dict(env, RANK=str(r), WORLD_SIZE="2", LOCAL_RANK=str(r))
        procs.append(subprocess.Popen([sys.executable, "-c", code], env=e, stdout=subprocess.PIPE,
                                      stderr=subprocess.PIPE, text=True))
    outs = [p.communicate(timeout=180) for p in procs]
    assert all(p.returncode == 0 for p in procs), [o[1][-2000:] for o in outs]
    assert "OK 2" in outs[0][0]


def test_version_string_names_the_target():
    import paper_1511_04355_b200 as P

    assert "sm_100a" in P.api.version()


@pytest.mark.parametrize("case", ["vertex_index", "degenerate", "material", "channel", "nan_vertex", "nan_traction"])
def test_bem_create_validates_on_the_host(case):
    """fds_bem_create rejects bad meshes / loads / materials / channels with
    ValidationError before touching the device (so also without a GPU)."""
    import numpy as np

    import paper_1511_04355_b200 as P
    from paper_1511_04355_b200 import mesh

    V, F = mesh.icosphere(1)
    tr = mesh.pressure_traction(V, F)
    kw = {}
    if case == "vertex_index":
        F = F.copy()
        F[3, 1] = len(V) + 5
    elif case == "degenerate":
        F = F.copy()
        F[2] = [F[2, 0], F[2, 0], F[2, 1]]
    elif case == "material":
        kw = dict(nu=0.5)
    elif case == "channel":
        kw = dict(channels=[0, 3 * len(F)])
    elif case == "nan_vertex":
        V = V.copy()
        V[0, 0] = np.nan
    elif case == "nan_traction":
        tr = tr.copy()
        tr[1, 2] = np.inf
    with pytest.raises(P.ValidationError):
        P.BemSystem(V, F, tr, **kw)


def test_default_3m_gemm_kernel_is_tma_fed_dmma():
    """The default trailing update (lu_gemm3m_tma_kernel<128, 32, 4, 2, 256, 1, 16, 2>)
    issues only DMMA for its products (no FP64 adds in the k-loop: the operand
    sums come from lu_g3_prep_kernel), is fed by TMA tensor loads and moves
    its A fragments and the C tile in 16-byte accesses."""
    fn = "_ZN4fdsb20lu_gemm3m_tma_kernelILi128ELi32ELi4ELi2ELi256ELi1ELi16ELi2EEEv14CUtensorMap_stS1_S1_S1_Pdmmiiiii"
    out = subprocess.run(["cuobjdump", "-sass", "-fun", fn, str(P.library_path())], capture_output=True,
                         text=True).stdout
    assert "UTMALDG" in out
    n_dmma = out.count("DMMA.8x8x4")
    # 3 products x 4 k-steps x (MI = 2) x (NI = 2) per unrolled k-chunk, twice: the
    # steady-state chunk and the P-first first chunk (P alone, then Q and R)
    assert n_dmma == 2 * 3 * 4 * 2 * 2
    lines = out.splitlines()
    last_dmma = max(i for i, ln in enumerate(lines) if "DMMA.8x8x4" in ln)
    dadd = [i for i, ln in enumerate(lines) if "DADD" in ln]
    assert dadd and min(dadd) > last_dmma  # epilogue only: Q - P, R - P
    assert "LDS.128" in out and "STG.E.128" in out and "LDG.E.128" in out
