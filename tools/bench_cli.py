"""CLI end-to-end timing (SPEC.md cli module, §8f row f1): the product CLI
(integration/_build/fdsweep_b200, B200) against the same main linked with the
CPU oracle (oracle/_ref/fdsweep_oracle_cli, OpenMP assembly + OpenBLAS zgetrf
on every host core), on the config-2 FSM sweep (1280-triangle sphere, 129
contour frequencies, 16 collocation points) and an AFS sweep on the config-2 mesh (random traction, 16 points, J0 = 12,
J_c = 6, thresholds off so both builds take the same 18 samples).
Writes profiles/r01_cli_timing.json."""
import json, os, subprocess, sys, tempfile, time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT / "oracle"))
import pyoracle as O  # noqa: E402

GPU = ROOT / "integration" / "_build" / "fdsweep_b200"
CPU = ROOT / "oracle" / "_ref" / "fdsweep_oracle_cli"


def run(cli, args, env=None):
    t0 = time.perf_counter()
    r = subprocess.run([str(cli)] + args, capture_output=True, text=True, env=env)
    dt = time.perf_counter() - t0
    assert r.returncode in (0, 6), r.stderr
    return dt


def main():
    env = dict(os.environ, FDSWEEP_ORACLE_OPENBLAS=O.openblas_path())
    out = {"cores": os.cpu_count()}
    with tempfile.TemporaryDirectory() as d:
        d = Path(d)
        (d / "cfg2.json").write_text(json.dumps({"type": "bem", "mesh": {"kind": "icosphere", "level": 3},
                                                 "load": {"kind": "pressure"}, "collocation_points": list(range(16))}))
        (d / "fsm.json").write_text(json.dumps({"period": 20.0, "samples": 256, "eta": 0.25}))
        args = ["sweep-fsm", "--system", str(d / "cfg2.json"), "--config", str(d / "fsm.json")]
        g = run(GPU, args + ["--out", str(d / "g")])
        c = run(CPU, args + ["--out", str(d / "c")], env)
        rg = json.loads((d / "g" / "report.json").read_text())
        out["sweep_fsm_cfg2"] = {"n_c": rg["n_c"], "gpu_wall_s": g, "gpu_system_s": rg["system_s"], "gpu_solve_s": rg["solve_s"], "cpu_wall_s": c, "speedup": c / g,
                                 "gpu_solves_per_s": rg["n_c"] / g, "cpu_solves_per_s": rg["n_c"] / c}
        (d / "cfg1.json").write_text(json.dumps({"type": "bem", "mesh": {"kind": "icosphere", "level": 3},
                                                 "load": {"kind": "random", "seed": 0},
                                                 "collocation_points": list(range(0, 1280, 80))}))
        (d / "afs.json").write_text(json.dumps({"omega_max": 3.141592653589793 * 256 / 20.0, "eta": 0.25,
                                                "period": 20.0, "initial_count": 12, "validation_steps": 6,
                                                "e1_threshold": "inf", "e2_threshold": "inf", "samples": 256}))
        args = ["sweep-afs", "--system", str(d / "cfg1.json"), "--config", str(d / "afs.json")]
        g = run(GPU, args + ["--out", str(d / "ga")])
        c = run(CPU, args + ["--out", str(d / "ca")], env)
        ra = json.loads((d / "ga" / "report.json").read_text())
        rc = json.loads((d / "ca" / "report.json").read_text())
        out["sweep_afs_cfg2_mesh"] = {"n_c": ra["n_c"], "gpu_wall_s": g, "cpu_wall_s": c, "speedup": c / g,
                                 "identical_frequencies": ra["frequencies"] == rc["frequencies"]}
    (ROOT / "profiles" / "r01_cli_timing.json").write_text(json.dumps(out, indent=1))
    print(json.dumps(out))


if __name__ == "__main__":
    main()
