"""The CLI (SPEC.md cli module; §8f row f1): integration/_build/fdsweep_b200 (the
product: reference io/systems/afs + the B200 library) against
oracle/_ref/fdsweep_oracle_cli (the same main linked with the CPU oracle).

CPU tests exercise the contract on the oracle build (file set, hashes, exit
codes, determinism, compare); GPU tests require the two builds to agree: BEM
spectra within 1e-9, time series within 1e-8 (rel. L2), identical AFS
frequency sequences, fitted poles within 1e-6.
"""
import json
import math
import os
import subprocess
from pathlib import Path

import numpy as np
import pytest

import pyoracle as O
from helpers import ModalFixture

ROOT = Path(__file__).resolve().parent.parent
GPU_CLI = ROOT / "integration" / "_build" / "fdsweep_b200"
CPU_CLI = ROOT / "oracle" / "_ref" / "fdsweep_oracle_cli"


def run(cli, *args, timeout=900):
    if not cli.exists():
        pytest.skip(f"{cli.name} not built (needs /root/reference at build time)")
    env = dict(os.environ)
    if cli == CPU_CLI:  # oracle BEM solves through OpenBLAS zgetrf when available
        try:
            env["FDSWEEP_ORACLE_OPENBLAS"] = O.openblas_path()
        except Exception:  # noqa: BLE001
            pass
    return subprocess.run([str(cli)] + [str(a) for a in args], capture_output=True, text=True, timeout=timeout,
                          env=env)


def fnv1a64(b: bytes) -> str:
    """io.cpp:394-403 (content_hash); note its offset basis is 1469598103934665603."""
    h = 1469598103934665603
    for x in b:
        h ^= x
        h = (h * 0x100000001B3) & ((1 << 64) - 1)
    return f"fnv1a64:{h:016x}"


def write(p: Path, obj) -> Path:
    p.write_text(json.dumps(obj))
    return p


def read_time(path: Path):
    lines = path.read_text().strip().splitlines()
    labels = lines[0].split(",")[1:]
    data = np.array([[float(x) for x in ln.split(",")] for ln in lines[1:]])
    return labels, data[:, 0], data[:, 1:]


def read_spectrum(path: Path):
    rows = [ln.split(",") for ln in path.read_text().strip().splitlines()[1:]]
    return {(float(r[0]), r[1]): complex(float(r[2]), float(r[3])) for r in rows}


@pytest.fixture
def modal(tmp_path):
    return write(tmp_path / "modal.json", json.loads(ModalFixture(6).system_json()))


AFS_MODAL = {"omega_max": 1.5 * 29.8, "eta": 0.35, "period": 20.0, "orf_indices": [0, 1, 2],
             "test_indices": [3, 4, 5], "grid_points": 1024, "time_points": 256, "e1_threshold": 1e-2,
             "e2_threshold": 5e-2, "samples": 64}


# ------------------------------------------------------------------ contract (CPU oracle build)
def test_sweep_fsm_files_and_hashes(tmp_path, modal):
    cfg = write(tmp_path / "fsm.json", {"period": 20.0, "samples": 64, "kappa": 3})
    out = tmp_path / "o"
    r = run(CPU_CLI, "sweep-fsm", "--system", modal, "--config", cfg, "--out", out)
    assert r.returncode == 0, r.stderr
    rep = json.loads((out / "report.json").read_text())
    assert rep["n_c"] == 33 and rep["samples"] == 64
    for name, h in rep["files"].items():
        assert fnv1a64((out / name).read_bytes()) == h
    labels, t, x = read_time(out / "time.csv")
    assert len(t) == 64 and labels == [f"ch{k}" for k in range(6)]
    # the series is fsm_invert of the sampled contour spectra
    fx = ModalFixture(6)
    eta = 3 * math.log(10) / 20.0
    s = eta + 1j * 2 * math.pi / 20.0 * np.arange(33)
    half = np.array([fx.evaluate(z) for z in s]).T.copy()
    ref = O.fsm_invert(20.0, 64, eta, half)
    np.testing.assert_allclose(x.T, ref, rtol=0, atol=1e-12 * np.abs(ref).max())


def test_sweep_fsm_odd_samples_is_validation_error(tmp_path, modal):
    cfg = write(tmp_path / "fsm.json", {"period": 20.0, "samples": 63})
    r = run(CPU_CLI, "sweep-fsm", "--system", modal, "--config", cfg, "--out", tmp_path / "o")
    assert r.returncode == 3, (r.returncode, r.stderr)


def test_sweep_afs_deterministic_and_matches_run_afs(tmp_path, modal):
    cfg = write(tmp_path / "afs.json", AFS_MODAL)
    a, b = tmp_path / "a", tmp_path / "b"
    for d in (a, b):
        r = run(CPU_CLI, "sweep-afs", "--system", modal, "--config", cfg, "--out", d, "--seed", 7)
        assert r.returncode == 0, r.stderr
    assert (a / "report.json").read_bytes() == (b / "report.json").read_bytes()
    rep = json.loads((a / "report.json").read_text())
    o = O.run_afs(O.System.from_json(ModalFixture(6).system_json()), omega_max=1.5 * 29.8, eta=0.35, period=20.0,
                  orf=[0, 1, 2], test=[3, 4, 5], grid_points=1024, time_points=256, e1_threshold=1e-2,
                  e2_threshold=5e-2, seed=7)
    assert rep["n_c"] == o["n_c"] and rep["converged"] == o["converged"]
    got = np.array([complex(x, y) for x, y in rep["frequencies"]])
    np.testing.assert_array_equal(got, o["samples"])


def test_compare_identical_and_mismatch(tmp_path, modal):
    fsm = tmp_path / "fsm"
    r = run(CPU_CLI, "sweep-fsm", "--system", modal, "--config",
            write(tmp_path / "c.json", {"period": 20.0, "samples": 64}), "--out", fsm)
    assert r.returncode == 0, r.stderr
    r = run(CPU_CLI, "compare", "--config", write(tmp_path / "cmp.json", {"fsm": str(fsm), "afs": str(fsm)}),
            "--out", tmp_path / "cmp")
    assert r.returncode == 0, r.stderr
    c = json.loads((tmp_path / "cmp" / "comparison.json").read_text())
    assert c["nc_ratio"] == 1.0 and all(v["rms_diff"] == 0.0 for v in c["per_channel"].values())
    other = tmp_path / "fsm2"
    run(CPU_CLI, "sweep-fsm", "--system", modal, "--config",
        write(tmp_path / "c2.json", {"period": 10.0, "samples": 64}), "--out", other)
    r = run(CPU_CLI, "compare", "--config", write(tmp_path / "cmp2.json", {"fsm": str(fsm), "afs": str(other)}),
            "--out", tmp_path / "cmp2")
    assert r.returncode == 3 and "grid mismatch" in r.stderr


def test_fit_then_invert(tmp_path, modal):
    fit = tmp_path / "fit"
    r = run(CPU_CLI, "fit", "--system", modal, "--config",
            write(tmp_path / "f.json", {"period": 20.0, "samples": 128, "eta": 0.35, "order": 16}), "--out", fit)
    assert r.returncode == 0, r.stderr
    rep = json.loads((fit / "report.json").read_text())
    assert max(rep["e_vf"]) < 1e-6  # exactly rational data, true order
    inv = tmp_path / "inv"
    r = run(CPU_CLI, "invert", "--config",
            write(tmp_path / "i.json", {"model": str(fit / "model.json"), "period": 20.0, "samples": 128}),
            "--out", inv)
    assert r.returncode == 0, r.stderr
    _, t, x = read_time(inv / "time.csv")
    assert x.shape == (128, 6)


def test_bem_system_matches_python_oracle(tmp_path):
    from paper_1511_04355_b200 import mesh

    sysj = write(tmp_path / "bem.json", {"type": "bem", "mesh": {"kind": "icosphere", "level": 1},
                                         "load": {"kind": "random", "seed": 3}, "collocation_points": [0, 7]})
    out = tmp_path / "o"
    r = run(CPU_CLI, "sweep-fsm", "--system", sysj, "--config",
            write(tmp_path / "c.json", {"period": 20.0, "samples": 8, "eta": 0.25}), "--out", out)
    assert r.returncode == 0, r.stderr
    spec = read_spectrum(out / "spectrum.csv")
    V, F = mesh.icosphere(1)
    bem = O.Bem(V, F, mesh.random_traction(F.shape[0], seed=3))
    for k in range(5):
        s = 0.25 + 1j * 2 * math.pi / 20.0 * k
        u = bem.solve(s)
        for dof in (0, 1, 2, 21, 22, 23):
            got = spec[(s.imag, f"u{dof}")]
            assert abs(got - u[dof]) <= 1e-12 * np.abs(u).max()


# ------------------------------------------------------------------ product vs oracle (GPU)
@pytest.mark.gpu
def test_gpu_cli_sweep_fsm_bem_matches_oracle_cli(tmp_path):
    sysj = write(tmp_path / "bem.json", {"type": "bem", "mesh": {"kind": "icosphere", "level": 2},
                                         "load": {"kind": "pressure"}, "collocation_points": list(range(16))})
    cfg = write(tmp_path / "c.json", {"period": 20.0, "samples": 32, "eta": 0.25})
    g, c = tmp_path / "g", tmp_path / "c"
    r = run(GPU_CLI, "sweep-fsm", "--system", sysj, "--config", cfg, "--out", g)
    assert r.returncode == 0, r.stderr
    r = run(CPU_CLI, "sweep-fsm", "--system", sysj, "--config", cfg, "--out", c)
    assert r.returncode == 0, r.stderr
    assert json.loads((g / "report.json").read_text())["solver"] == "b200"
    sg, sc = read_spectrum(g / "spectrum.csv"), read_spectrum(c / "spectrum.csv")
    assert sg.keys() == sc.keys()
    a = np.array([sg[k] for k in sorted(sg)])
    b = np.array([sc[k] for k in sorted(sc)])
    assert np.linalg.norm(a - b) / np.linalg.norm(b) < 1e-9
    _, tg, xg = read_time(g / "time.csv")
    _, tc, xc = read_time(c / "time.csv")
    np.testing.assert_array_equal(tg, tc)
    assert np.linalg.norm(xg - xc) / np.linalg.norm(xc) < 1e-8


@pytest.mark.gpu
def test_gpu_cli_sweep_afs_modal_identical_sequence(tmp_path, modal):
    cfg = write(tmp_path / "afs.json", AFS_MODAL)
    g, c = tmp_path / "g", tmp_path / "c"
    assert run(GPU_CLI, "sweep-afs", "--system", modal, "--config", cfg, "--out", g).returncode == 0
    assert run(CPU_CLI, "sweep-afs", "--system", modal, "--config", cfg, "--out", c).returncode == 0
    rg, rc = json.loads((g / "report.json").read_text()), json.loads((c / "report.json").read_text())
    assert rg["n_c"] == rc["n_c"] and rg["converged"] == rc["converged"]
    assert rg["frequencies"] == rc["frequencies"]


@pytest.mark.gpu
def test_gpu_cli_sweep_afs_bem_identical_sequence(tmp_path):
    sysj = write(tmp_path / "bem.json", {"type": "bem", "mesh": {"kind": "icosphere", "level": 2},
                                         "load": {"kind": "random", "seed": 0},
                                         "collocation_points": [3, 40, 77, 150, 222, 301]})
    cfg = write(tmp_path / "afs.json", {"omega_max": math.pi * 256 / 20.0, "eta": 0.25, "period": 20.0,
                                        "initial_count": 10, "validation_steps": 4, "e1_threshold": "inf",
                                        "e2_threshold": "inf", "samples": 256})
    g, c = tmp_path / "g", tmp_path / "c"
    rg = run(GPU_CLI, "sweep-afs", "--system", sysj, "--config", cfg, "--out", g)
    rc = run(CPU_CLI, "sweep-afs", "--system", sysj, "--config", cfg, "--out", c, timeout=1800)
    assert rg.returncode == rc.returncode, (rg.stderr, rc.stderr)
    jg, jc = json.loads((g / "report.json").read_text()), json.loads((c / "report.json").read_text())
    assert jg["n_c"] == jc["n_c"] == 14
    assert jg["frequencies"] == jc["frequencies"]
    _, _, xg = read_time(g / "time.csv")
    _, _, xc = read_time(c / "time.csv")
    assert np.linalg.norm(xg - xc) / np.linalg.norm(xc) < 1e-8


@pytest.mark.gpu
def test_gpu_cli_fit_poles_match_oracle(tmp_path, modal):
    cfg = write(tmp_path / "f.json", {"period": 20.0, "samples": 128, "eta": 0.35, "order": 16})
    g, c = tmp_path / "g", tmp_path / "c"
    assert run(GPU_CLI, "fit", "--system", modal, "--config", cfg, "--out", g).returncode == 0
    assert run(CPU_CLI, "fit", "--system", modal, "--config", cfg, "--out", c).returncode == 0
    pg = np.array([complex(*p) for p in json.loads((g / "model.json").read_text())["poles"]])
    pc = np.array([complex(*p) for p in json.loads((c / "model.json").read_text())["poles"]])
    for p in pc:
        assert np.min(np.abs(pg - p)) / abs(p) < 1e-6


def _resume_roundtrip(cli, tmp_path, sysj, cfg_full, cfg_short):
    full, part, res = tmp_path / "full", tmp_path / "part", tmp_path / "res"
    r = run(cli, "sweep-afs", "--system", sysj, "--config", cfg_full, "--out", full, timeout=1800)
    assert r.returncode == 0, r.stderr
    r = run(cli, "sweep-afs", "--system", sysj, "--config", cfg_short, "--out", part, "--checkpoint", timeout=1800)
    assert r.returncode == 6, (r.returncode, r.stderr)  # ConvergenceError: iteration budget exhausted
    arch = json.loads((part / "archive.json").read_text())
    r = run(cli, "sweep-afs", "--system", sysj, "--config", cfg_full, "--out", res, "--resume",
            part / "archive.json", timeout=1800)
    assert r.returncode == 0, r.stderr
    jf, jr = json.loads((full / "report.json").read_text()), json.loads((res / "report.json").read_text())
    assert jr["frequencies"] == jf["frequencies"] and jr["n_c"] == jf["n_c"]
    assert jr["solver_calls"] == jf["n_c"] - len(arch["samples"])  # resumed samples are never re-solved
    return jf


def test_sweep_afs_resume_equivalence(tmp_path, modal):
    """SPEC.md io invariant: interrupted + archived + resumed == uninterrupted."""
    full = dict(AFS_MODAL)
    short = dict(AFS_MODAL, max_iterations=3)
    _resume_roundtrip(CPU_CLI, tmp_path, modal, write(tmp_path / "f.json", full), write(tmp_path / "s.json", short))


@pytest.mark.gpu
def test_gpu_cli_bem_resume_equivalence(tmp_path):
    sysj = write(tmp_path / "bem.json", {"type": "bem", "mesh": {"kind": "icosphere", "level": 2},
                                         "load": {"kind": "random", "seed": 0},
                                         "collocation_points": [3, 40, 77, 150, 222, 301]})
    base = {"omega_max": math.pi * 256 / 20.0, "eta": 0.25, "period": 20.0, "initial_count": 10,
            "validation_steps": 4, "e1_threshold": "inf", "e2_threshold": "inf", "samples": 256}
    jf = _resume_roundtrip(GPU_CLI, tmp_path, sysj, write(tmp_path / "f.json", base),
                           write(tmp_path / "s.json", dict(base, max_iterations=2)))
    assert jf["n_c"] == 14


@pytest.mark.gpu
def test_gpu_cli_bem_gmres_solver_matches_lu(tmp_path):
    base = {"type": "bem", "mesh": {"kind": "icosphere", "level": 2}, "load": {"kind": "pressure"},
            "collocation_points": list(range(16))}
    cfg = write(tmp_path / "c.json", {"period": 20.0, "samples": 32, "eta": 0.25})
    a, b = tmp_path / "lu", tmp_path / "gm"
    assert run(GPU_CLI, "sweep-fsm", "--system", write(tmp_path / "s1.json", base), "--config", cfg,
               "--out", a).returncode == 0
    r = run(GPU_CLI, "sweep-fsm", "--system",
            write(tmp_path / "s2.json", dict(base, solver={"kind": "gmres", "tol": 1e-13})), "--config", cfg,
            "--out", b)
    assert r.returncode == 0, r.stderr
    sa, sb = read_spectrum(a / "spectrum.csv"), read_spectrum(b / "spectrum.csv")
    x = np.array([sa[k] for k in sorted(sa)])
    y = np.array([sb[k] for k in sorted(sb)])
    assert np.linalg.norm(x - y) / np.linalg.norm(x) < 1e-10
