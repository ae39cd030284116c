#!/usr/bin/env python
"""Benchmark of the B200 BEM / VF / FSM hot path (BASELINE.json metric).

Headline workload (configs[3], the north_star's N = 15360): spherical cavity,
5120-triangle icosphere (N = 15360 unknowns, 3.77 GB per complex matrix) under
the seeded random traction (xorshift64 + Box-Muller, seed 0), Heaviside in
time; the full FSM contour of T = 20, N_s = 512 (N_c = N_s/2 + 1 = 257
frequencies, s_k = 5/T + i k 2 pi/T). One step = one 32-frequency sub-batch of
that contour (step i takes frequencies 32 (i mod 8) ... 32 (i mod 8) + 31),
solved as independent dense systems: assembly + batched LU + solve, with the
displacement of 16 collocation points (48 DOFs, draw_indices(5120, 16, 0)) as
the channels.

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]

Under torchrun (N > 1) every rank solves its own sub-batches (replicas only:
the path has no exchange step), the step time is the max over
ranks, and value = total solves / time ("scaling": "weak").
``--impl reference`` times the CPU oracle port of the same path (OpenMP
assembly + OpenBLAS zgetrf/zgetrs on all host cores), one cfg4 frequency per
step — the reference has no BEM.
"""
from __future__ import annotations

import argparse
import faulthandler
import json
import math
import os
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "BEM frequency solves/sec (assembly+LU)"
UNIT = "solves/s"
T_PERIOD = 20.0
ETA = 5.0 / T_PERIOD
NS4 = 512                 # cfg4: N_s = 512 -> N_c = 257 contour frequencies
SUB = 32                  # one step = one 32-frequency sub-batch of the contour
NSUB = (NS4 // 2 + 1) // SUB  # 8 full sub-batches (frequencies 0..255)


def contour(ns):
    return ETA + 1j * (2 * math.pi / T_PERIOD) * np.arange(ns // 2 + 1)


def cfg4_inputs():
    """configs[3]: icosphere(4) (5120 triangles, N = 15360), random traction seed 0,
    16 collocation points x 3 DOFs as channels, the N_s = 512 contour."""
    from paper_1511_04355_b200 import mesh

    V, F = mesh.icosphere(4)
    tr = mesh.random_traction(F.shape[0], seed=0)
    pts = mesh.draw_indices(F.shape[0], 16, 0)
    dofs = [3 * p + i for p in pts for i in range(3)]
    return V, F, tr, dofs, contour(NS4)


def sub_batch(s, i, rank=0, world=1):
    """Step i of replica `rank`: the contour's sub-batches are dealt round-robin
    over the replicas (no data-path collective: every frequency is an independent
    system), so N ranks walk N distinct sub-batches per step."""
    j = (i * world + rank) % NSUB
    return s[SUB * j: SUB * (j + 1)]


def whole_job_rate(units_per_rank_step, world, steps, max_total_ms):
    """Aggregate throughput: units all ranks processed / the slowest rank's time."""
    return units_per_rank_step * world * steps / (max_total_ms * 1e-3)


def cfg2_inputs():
    from paper_1511_04355_b200 import mesh

    V, F = mesh.icosphere(3)
    tr = mesh.pressure_traction(V, F)
    pts = mesh.draw_indices(F.shape[0], 16, 0)
    dofs = [3 * p + i for p in pts for i in range(3)]
    return V, F, tr, dofs, contour(256)


class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        self.lines = []
        if self.proc is not None:
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.proc.kill()
                out = ""
            self.lines = [l for l in out.splitlines() if l.strip()]

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in self.lines:
            parts = [p.strip() for p in l.split(",")]
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except (ValueError, IndexError):
                continue
            for nm, v in zip(names, parts[3:]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


def measured_fp64_peak():
    p = ROOT / "profiles" / "r01_fp64_peak.json"
    try:
        d = json.loads(p.read_text())
        return float(d["fp64_peak_tflops"]), "measured (profiles/r01_fp64_peak.json: DMMA microbench / cuBLAS ZGEMM)"
    except Exception:
        return 36.9, "fallback (B200 FP64 datasheet class)"


def ncu_traffic(kernel: str):
    p = ROOT / "profiles" / "ncu_traffic.json"
    try:
        return json.loads(p.read_text()).get(kernel)
    except Exception:
        return None


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    if world > 1:
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    return world, rank, local, dist


def allreduce_max(dist, x: float) -> float:
    if dist is None:
        return x
    import torch

    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"  # gloo: the CPU plumbing test
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(dist):
    if dist is not None:
        dist.barrier()


# ------------------------------------------------------------------ CPU legs
def _oracle():
    sys.path.insert(0, str(ROOT / "oracle"))
    import pyoracle as O

    return O


def cpu_warmup(O):
    """Spins up OpenMP / OpenBLAS threads on a small system (cfg1 mesh) — untimed."""
    from paper_1511_04355_b200 import mesh

    V, F = mesh.icosphere(2)
    O.Bem(V, F, mesh.pressure_traction(V, F)).solve_openblas(complex(ETA, 1.0), O.openblas_path())


def cpu_cfg4_solve(O, bem, s):
    """Oracle port of one cfg4 frequency: OpenMP assembly + OpenBLAS zgetrf/zgetrs
    on all host cores. Returns (seconds, [assembly_s, factor+solve_s])."""
    t0 = time.perf_counter()
    _, t = bem.solve_openblas(s, O.openblas_path())
    return time.perf_counter() - t0, [float(t[0]), float(t[1])]


def run_reference(args, world, rank):
    """Reference arm: the CPU path on the box's host cores, one cfg4 frequency
    (N = 15360) per step, the frequencies walking the same contour sub-batches."""
    if rank != 0:
        return
    O = _oracle()
    V, F, tr, dofs, s = cfg4_inputs()
    cpu_warmup(O)
    bem = O.Bem(V, F, tr)
    per, split = [], []
    for i in range(args.steps):
        dt, sp = cpu_cfg4_solve(O, bem, sub_batch(s, i)[i % SUB])
        per.append(dt)
        split.append(sp)
    dt = float(np.mean(per))
    v = 1.0 / dt
    cores = os.cpu_count()
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "c128", "data": "synthetic",
        "config": {"workload": "cfg4: sphere cavity, 5120-tri icosphere, N=15360, random traction seed 0, "
                               "FSM contour T=20 Ns=512 eta=5/T (257 frequencies), 48 channels",
                   "sample": "1 contour frequency per step (bounded CPU sample of the 32-frequency sub-batch step)",
                   "warmup": "one untimed cfg1-size solve (thread pools); a cfg4 warm-up solve would add ~30 s each"},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": "oracle BEM assembly (OpenMP, all cores) + OpenBLAS zgetrf/zgetrs (all cores), "
                                   "1 cfg4 frequency per step"},
        "stage_s": {"assembly": float(np.mean([x[0] for x in split])),
                    "factor_solve": float(np.mean([x[1] for x in split]))},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ GPU leg
# FP64 work per far-field kernel evaluation: executed thread instructions of
# bem_far_kernel at HEAD (ncu sm__sass_thread_inst_executed_op_{dfma,dadd,dmul}
# on cfg2: 2 DFMA + DADD + DMUL flops, DFMA + DADD + DMUL issue slots) divided by
# its 7 N_e (N_e - 1) B evaluations (profiles/r02_far_ncu.json, round2_op_counts).
# A DADD or DMUL takes the same FP64-pipe slot as a DFMA, so the pipe fraction
# (instructions against peak / 2 flops per slot) is the bound; the flop fraction
# is reported beside it.
ASM_FLOPS_PER_EVAL = 425.8
ASM_FP64_INST_PER_EVAL = 274.1


def profile_stages(P, L):
    import ctypes

    out = {}
    for name, kind in (("gemm", 0), ("panel", 1), ("trsm", 2), ("far", 3), ("near", 4)):
        c, ms, wk = ctypes.c_int(), ctypes.c_double(), ctypes.c_double()
        P.api._check(L.fds_profile_read(kind, ctypes.byref(c), ctypes.byref(ms), ctypes.byref(wk)))
        out[name] = dict(launches=c.value, ms=ms.value, work=wk.value)
    return out


def gemm_roofline(prof, n, B, label):
    peak, peak_src = measured_fp64_peak()
    g = prof["gemm"]
    # the library's GEMM work counter is the conventional complex count 8 rest^2 w;
    # the 3M kernel executes three real products per complex MAC (6 rest^2 w)
    effective = g["work"] / (g["ms"] * 1e-3) / 1e12
    achieved = 0.75 * effective
    return {"bound": "tensor",
            "kernel": "lu_gemm3m_tma_kernel (TMA-fed DMMA complex GEMM, 3 real products per complex MAC; "
                      "timing includes lu_g3_prep_kernel)",
            "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
            "peak_source": peak_src, "traffic": ncu_traffic("lu_gemm3m_tma_kernel@" + label),
            "traffic_def": "ncu dram__bytes_read.sum + dram__bytes_write.sum of one rank-128 launch "
                           "(profiles/ncu_traffic.json)",
            "work_def": "6*rest^2*w FP64 flops executed per launch (A22 -= L21 U12 as 3 real GEMMs), "
                        "summed over the step's launches / their CUDA-event time on the launching stream",
            "effective_complex_tflops": effective,
            "effective_work_def": "8*rest^2*w (conventional complex GEMM count) / time",
            "launches_per_step": g["launches"],
            "share_of_lu": g["ms"] / max(g["ms"] + prof["panel"]["ms"] + prof["trsm"]["ms"], 1e-9),
            "lu_tflops_conventional": B * 8.0 * n ** 3 / 3.0}


def run_ours(args, world, rank, local, dist):
    import paper_1511_04355_b200 as P
    from paper_1511_04355_b200 import BemSystem

    L = P.lib()
    P.api._check(L.fds_set_device(local))
    V, F, tr, dofs, s = cfg4_inputs()
    n = 3 * F.shape[0]
    sysb = BemSystem(V, F, tr, channels=dofs, max_batch=SUB)
    for i in range(args.warmup):
        sysb.evaluate_batch_device(sub_batch(s, i, rank, world))
    barrier(dist)
    launches0 = P.kernel_launches()
    dev_ms, stage = [], dict(assembly_ms=0.0, lu_ms=0.0, solve_ms=0.0)
    with ClockSampler(local) as clk:
        t0 = time.perf_counter()
        for i in range(args.steps):
            sysb.evaluate_batch_device(sub_batch(s, i, rank, world))
            t = sysb.last_timing()
            dev_ms.append(t["assembly_ms"] + t["lu_ms"] + t["solve_ms"])
            for k in stage:
                stage[k] += t[k] / args.steps
        wall = time.perf_counter() - t0
    launches = (P.kernel_launches() - launches0) // args.steps
    total_ms = allreduce_max(dist, float(np.sum(dev_ms)))
    ms_step = total_ms / args.steps
    value = whole_job_rate(SUB, world, args.steps, total_ms)

    # end to end through the public C-ABI with host buffers: the 8 full sub-batches
    # of the contour (frequencies 0..255), H2D of s and D2H of the 48-channel
    # responses inside the timed region; frequency 256 is solved untimed so the
    # full 257-frequency spectra feed the FSM reconstruction below
    barrier(dist)
    spectra = np.zeros((len(s), len(dofs)), np.complex128)
    e2e_stage = dict(assembly_ms=0.0, lu_ms=0.0, solve_ms=0.0)
    t0 = time.perf_counter()
    for i in range(NSUB):
        spectra[SUB * i: SUB * (i + 1)] = sysb.evaluate_batch(sub_batch(s, i))
        t = sysb.last_timing()
        for k in e2e_stage:
            e2e_stage[k] += t[k]
    e2e_s = allreduce_max(dist, time.perf_counter() - t0) / NSUB
    e2e = {"value": SUB * world / e2e_s, "unit": UNIT, "h2d_bytes_per_step": 16 * SUB,
           "d2h_bytes_per_step": 16 * SUB * len(dofs), "steps": NSUB,
           "note": "the 8 full 32-frequency sub-batches of the contour through fds_bem_evaluate_batch"}
    t1 = time.perf_counter()
    spectra[NSUB * SUB:] = sysb.evaluate_batch(s[NSUB * SUB:])
    tail_s = time.perf_counter() - t1
    t1 = time.perf_counter()
    hist = P.fsm_invert(T_PERIOD, NS4, ETA, spectra.T.copy())
    fsm_api_ms = (time.perf_counter() - t1) * 1e3
    fsm_sweep = {"frequencies": len(s), "wall_s": e2e_s * NSUB + tail_s,
                 "solves_per_s": len(s) / (e2e_s * NSUB + tail_s),
                 "assembly_s": e2e_stage["assembly_ms"] * 1e-3, "lu_s": e2e_stage["lu_ms"] * 1e-3,
                 "solve_s": e2e_stage["solve_ms"] * 1e-3,
                 "reconstruction_ms": fsm_api_ms, "channels": len(dofs), "time_steps": NS4,
                 "max_abs_displacement": float(np.max(np.abs(hist))),
                 "note": "frequencies 0..255 from the e2e loop (stage times summed) + frequency 256 alone; "
                         "reconstruction = fsm_invert (host API, incl. copies)"}

    # roofline of the dominant kernel (the LU trailing GEMM on the FP64 tensor pipe)
    P.api._check(L.fds_profile_enable(1))
    sysb.evaluate_batch_device(sub_batch(s, 0))
    prof = profile_stages(P, L)
    P.api._check(L.fds_profile_enable(0))
    sysb.close()
    roof = gemm_roofline(prof, n, SUB, "cfg4")
    lu_flops = SUB * 8.0 * n ** 3 / 3.0
    far = prof["far"]
    result = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "c128",
        "data": "synthetic",
        "config": {"workload": "cfg4: sphere cavity, 5120-tri icosphere, N=15360, random traction seed 0, "
                               "32-frequency sub-batch of the FSM contour (T=20, Ns=512, eta=5/T, 257 frequencies) "
                               "per step, 16 collocation points x 3 DOFs",
                   "global_batch": SUB * world, "parallelism": f"replicas x{world}",
                   "l2": "inputs larger than L2 (32 x 3.77 GB matrices per step)"},
        "e2e": e2e,
        "roofline": roof,
        "stages_ms": {"assembly": stage["assembly_ms"], "lu": stage["lu_ms"], "solve": stage["solve_ms"],
                      "lu_panel": prof["panel"]["ms"], "lu_trsm": prof["trsm"]["ms"], "lu_gemm": prof["gemm"]["ms"]},
        "lu_tflops": lu_flops / (stage["lu_ms"] * 1e-3) / 1e12,
        "assembly_far": {"ms": far["ms"], "kernel_evaluations": far["work"],
                         "flops_per_evaluation": ASM_FLOPS_PER_EVAL,
                         "tflops": ASM_FLOPS_PER_EVAL * far["work"] / max(far["ms"], 1e-9) / 1e9,
                         "fp64_frac": ASM_FLOPS_PER_EVAL * far["work"] / max(far["ms"], 1e-9) / 1e9 /
                         measured_fp64_peak()[0],
                         "fp64_instructions_per_evaluation": ASM_FP64_INST_PER_EVAL,
                         "fp64_pipe_frac": ASM_FP64_INST_PER_EVAL * far["work"] / max(far["ms"], 1e-9) / 1e9 /
                         (measured_fp64_peak()[0] / 2.0)},
        "wall_ms_per_step": wall * 1e3 / args.steps,
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
    }
    if rank == 0 and world == 1 and not args.no_extra:
        result["extra"] = extra_configs(args, fsm_sweep)
    if rank == 0 and world == 1 and not args.no_cpu:
        O = _oracle()
        cpu_warmup(O)
        dt, sp = cpu_cfg4_solve(O, O.Bem(V, F, tr), s[7])
        result["cpu_baseline"] = {"value": 1.0 / dt, "unit": UNIT, "cores": os.cpu_count(), "kind": "port",
                                  "sample": "1 cfg4 frequency (k=7, N=15360): oracle BEM assembly (OpenMP) "
                                            f"{sp[0]:.1f} s + OpenBLAS zgetrf/zgetrs {sp[1]:.1f} s, all host cores"}
        try:
            result.setdefault("extra", {})["cfg5_cpu_baseline"] = cpu_vf_fsm_baseline(O)
        except Exception as e:  # noqa: BLE001
            result.setdefault("extra", {})["cfg5_cpu_error"] = repr(e)
    if rank == 0:
        print(json.dumps(result), flush=True)


def cfg5_vf_fsm(D=300_000, J=40, pairs=24, T_steps=512, reps=3):
    """Config 5: VF + reconstruction alone at 300k DOFs (device-resident inputs).

    Pinned synthetic data: 24 stable pole pairs Re~U[-0.5,-0.01],
    Im~U[0,40]; per-DOF residues N(0,1) complex; N(0,1e-3) additive noise; seed 0
    (torch CUDA generator); Omega_s = 1.2 max Im a, T = pi*512/Omega_s,
    eta = 3 ln10 / T; J = 40 Chebyshev contour samples (initial_frequencies(40, ...))
    stand in for the "40 adaptively chosen" ones. Stages timed with CUDA events
    inside the library: residue identification for all D DOFs (after relocation
    on 5 ORF DOFs), rational_invert to 512 steps, and the FSM C2R inversion of the
    D x 257 contour spectra (N_s = 512).
    """
    import ctypes

    import torch

    import paper_1511_04355_b200 as P

    L = P.lib()
    g = torch.Generator(device="cuda").manual_seed(0)
    dev = "cuda"
    re = -(0.01 + 0.49 * torch.rand(pairs, generator=g, device=dev, dtype=torch.float64))
    im = 40.0 * torch.rand(pairs, generator=g, device=dev, dtype=torch.float64)
    heads = torch.complex(re, im)
    poles = torch.stack([heads, heads.conj()], 1).reshape(-1)  # canonical: pairs adjacent
    rh = torch.complex(torch.randn(D, pairs, generator=g, device=dev, dtype=torch.float64),
                       torch.randn(D, pairs, generator=g, device=dev, dtype=torch.float64))
    res = torch.stack([rh, rh.conj()], 2).reshape(D, -1)  # (D, M)
    wmax = 1.2 * float(im.max())
    Tper = math.pi * 512 / wmax
    eta = 3.0 * math.log(10.0) / Tper
    j = np.arange(J)
    s_np = eta + 1j * wmax * (1.0 - np.cos(j * math.pi / (2.0 * (J - 1))))
    s = torch.tensor(s_np, device=dev)
    vals = (res @ (1.0 / (s[None, :] - poles[:, None]))).T.contiguous()  # (J, D)
    vals += 1e-3 * torch.complex(torch.randn(J, D, generator=g, device=dev, dtype=torch.float64),
                                 torch.randn(J, D, generator=g, device=dev, dtype=torch.float64))
    # relocation on 5 ORF DOFs (host-visible samples) -> common poles
    orf = list(range(5))
    t0 = time.perf_counter()
    model, rep = P.vector_fit(s_np, vals[:, :5].cpu().numpy(), orf, 2 * pairs, 3)
    t_reloc = time.perf_counter() - t0
    M = len(model.poles)
    ph = np.ascontiguousarray(model.poles, np.complex128)
    res_dev = torch.empty((M, D), dtype=torch.complex128, device=dev)
    out_dev = torch.empty((D, T_steps), dtype=torch.float64, device=dev)
    tgrid = np.ascontiguousarray(np.arange(T_steps) * Tper / T_steps)
    ms = ctypes.c_double()

    def best(fn):
        b = 1e30
        for _ in range(reps):
            fn()
            b = min(b, ms.value)
        return b

    # cold: the solve operator W formed from scratch (the vector fit above left the
    # ORF fit's operator for the same (s, poles) cached, which the warm timings reuse)
    P.api._check(L.fds_vf_release_workspace())
    P.api._check(L.fds_vf_identify_residues_device(
        J, D, s_np.ctypes.data_as(ctypes.c_void_p), ctypes.c_void_p(vals.data_ptr()), M,
        ph.ctypes.data_as(ctypes.c_void_p), ctypes.c_void_p(res_dev.data_ptr()), ctypes.byref(ms)))
    t_res_cold = ms.value
    t_res = best(lambda: P.api._check(L.fds_vf_identify_residues_device(
        J, D, s_np.ctypes.data_as(ctypes.c_void_p), ctypes.c_void_p(vals.data_ptr()), M,
        ph.ctypes.data_as(ctypes.c_void_p), ctypes.c_void_p(res_dev.data_ptr()), ctypes.byref(ms))))
    # pair heads only (the conjugate rows carry no information; rational_invert reads heads)
    t_res_h = best(lambda: P.api._check(L.fds_vf_identify_residues_device_heads(
        J, D, s_np.ctypes.data_as(ctypes.c_void_p), ctypes.c_void_p(vals.data_ptr()), M,
        ph.ctypes.data_as(ctypes.c_void_p), ctypes.c_void_p(res_dev.data_ptr()), ctypes.byref(ms))))
    t_rat = best(lambda: P.api._check(L.fds_rational_invert_device(
        M, ph.ctypes.data_as(ctypes.c_void_p), D, ctypes.c_void_p(res_dev.data_ptr()), T_steps,
        tgrid.ctypes.data_as(ctypes.c_void_p), ctypes.c_void_p(out_dev.data_ptr()), ctypes.byref(ms))))
    # FSM: exact contour spectra of the synthetic model (N_s = 512 -> 257 frequencies), [i][k]
    Ns = 512
    sk = eta + 1j * (2 * math.pi / Tper) * torch.arange(Ns // 2 + 1, device=dev, dtype=torch.float64)
    half = (res @ (1.0 / (sk[None, :] - poles[:, None]))).T.contiguous()  # (Nc, D)
    vals_keep = vals
    t_fsm = best(lambda: P.api._check(L.fds_fsm_invert_device(
        ctypes.c_double(Tper), Ns, ctypes.c_double(eta), D, ctypes.c_void_p(half.data_ptr()), 1, ctypes.c_void_p(out_dev.data_ptr()),
        ctypes.byref(ms))))
    # kernel-only device times (CUDA events around the launches, library profiler)
    P.api._check(L.fds_profile_enable(1))
    for _ in range(reps):
        P.api._check(L.fds_vf_identify_residues_device(
            J, D, s_np.ctypes.data_as(ctypes.c_void_p), ctypes.c_void_p(vals_keep.data_ptr()), M,
            ph.ctypes.data_as(ctypes.c_void_p), ctypes.c_void_p(res_dev.data_ptr()), ctypes.byref(ms)))
        P.api._check(L.fds_rational_invert_device(
            M, ph.ctypes.data_as(ctypes.c_void_p), D, ctypes.c_void_p(res_dev.data_ptr()), T_steps,
            tgrid.ctypes.data_as(ctypes.c_void_p), ctypes.c_void_p(out_dev.data_ptr()), ctypes.byref(ms)))
        P.api._check(L.fds_fsm_invert_device(
            ctypes.c_double(Tper), Ns, ctypes.c_double(eta), D, ctypes.c_void_p(half.data_ptr()), 1,
            ctypes.c_void_p(out_dev.data_ptr()), ctypes.byref(ms)))
    kern = {}
    for name, kind in (("residue", 5), ("rational", 6), ("fsm", 7)):
        c, kms, wk = ctypes.c_int(), ctypes.c_double(), ctypes.c_double()
        P.api._check(L.fds_profile_read(kind, ctypes.byref(c), ctypes.byref(kms), ctypes.byref(wk)))
        kern[name] = kms.value / max(c.value, 1)
    P.api._check(L.fds_profile_enable(0))
    P.api._check(L.fds_profile_enable(1))
    for _ in range(reps):
        P.api._check(L.fds_vf_identify_residues_device_heads(
            J, D, s_np.ctypes.data_as(ctypes.c_void_p), ctypes.c_void_p(vals_keep.data_ptr()), M,
            ph.ctypes.data_as(ctypes.c_void_p), ctypes.c_void_p(res_dev.data_ptr()), ctypes.byref(ms)))
    c, kms, wk = ctypes.c_int(), ctypes.c_double(), ctypes.c_double()
    P.api._check(L.fds_profile_read(5, ctypes.byref(c), ctypes.byref(kms), ctypes.byref(wk)))
    kern["residue_heads"] = kms.value / max(c.value, 1)
    P.api._check(L.fds_profile_enable(0))
    # channel-major spectra (the reference's per-channel fsm_invert layout)
    cmaj = half.T.contiguous()
    del half

    def fsm_cm():
        P.api._check(L.fds_fsm_invert_device_strided(
            ctypes.c_double(Tper), Ns, ctypes.c_double(eta), D, ctypes.c_void_p(cmaj.data_ptr()),
            ctypes.c_longlong(Ns // 2 + 1), ctypes.c_longlong(1), 1, ctypes.c_void_p(out_dev.data_ptr()),
            ctypes.byref(ms)))

    t_fsm_cm = best(fsm_cm)
    P.api._check(L.fds_profile_enable(1))
    for _ in range(reps):
        fsm_cm()
    c, kms, wk = ctypes.c_int(), ctypes.c_double(), ctypes.c_double()
    P.api._check(L.fds_profile_read(7, ctypes.byref(c), ctypes.byref(kms), ctypes.byref(wk)))
    kern["fsm_chan_major"] = kms.value / max(c.value, 1)
    P.api._check(L.fds_profile_enable(0))
    del cmaj
    hbm = 6543.4
    try:
        hbm = float(json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"])
    except Exception:
        pass
    fp64, _ = measured_fp64_peak()
    b_res = D * (16.0 * J + 16.0 * M / 2)
    b_fsm = D * (16.0 * (Ns // 2 + 1) + 8.0 * Ns)
    f_rat = D * 2.0 * M * T_steps
    kr, kt, kf, kc = kern["residue"], kern["rational"], kern["fsm"], kern["fsm_chan_major"]
    f_res = D * 4.0 * J * M  # W (M x 2J) times the 2J real samples of each DOF
    out = {
        "dofs": D, "J": J, "M": M, "time_steps": T_steps, "relocation_s": t_reloc,
        "api_ms": {"residue_id": t_res, "residue_id_cold": t_res_cold, "residue_id_heads": t_res_h,
                   "rational_invert": t_rat, "fsm": t_fsm, "fsm_chan_major": t_fsm_cm},
        "api_note": "residue_id* warm: the shared solve operator for (s, poles) is reused from the preceding call "
                    "(as run_afs's final all-channel fit reuses its last high-order fit); residue_id_cold forms it "
                    "on the device from scratch (one-CTA pivoted QR)",
        "kernel_ms": {"residue_id": kr, "rational_invert": kt, "fsm": kf, "fsm_chan_major": kc},
        "residue_id_dof_per_s": D / (kr * 1e-3), "residue_id_gbs": b_res / (kr * 1e-3) / 1e9,
        "residue_id_hbm_frac": b_res / (kr * 1e-3) / 1e9 / hbm,
        "residue_id_tflops": f_res / (kr * 1e-3) / 1e12, "residue_id_fp64_frac": f_res / (kr * 1e-3) / 1e12 / fp64,
        "rational_invert_dof_per_s": D / (kt * 1e-3), "rational_invert_tflops": f_rat / (kt * 1e-3) / 1e12,
        "rational_invert_fp64_frac": f_rat / (kt * 1e-3) / 1e12 / fp64,
        "fsm_dof_per_s": D / (kf * 1e-3), "fsm_gbs": b_fsm / (kf * 1e-3) / 1e9,
        "fsm_hbm_frac": b_fsm / (kf * 1e-3) / 1e9 / hbm,
        "fsm_chan_major_gbs": b_fsm / (kc * 1e-3) / 1e9, "fsm_chan_major_hbm_frac": b_fsm / (kc * 1e-3) / 1e9 / hbm,
        "fsm_layouts": "fsm = frequency-major [i][k] spectra as the batched BEM emits them (gather-bound); "
                       "fsm_chan_major = per-channel [k][i] spectra, the reference fsm_invert layout",
        "vf_fsm_dof_per_s": D / ((t_res_h + t_rat) * 1e-3),
        "vf_fsm_dof_per_s_def": "D / (API-level residue identification (pair heads) + rational_invert time: CUDA "
                                "events around the whole C-ABI calls, including the shared QR and the W operator)",
        "residue_heads": {"api_ms": t_res_h, "kernel_ms": kern["residue_heads"],
                          "bytes_per_dof": 16.0 * J + 8.0 * M,
                          "hbm_frac": D * (16.0 * J + 8.0 * M) / (kern["residue_heads"] * 1e-3) / 1e9 / hbm,
                          "fp64_frac": D * 4.0 * J * M / (kern["residue_heads"] * 1e-3) / 1e12 / fp64,
                          "binding_roofline_frac": max(D * 4.0 * J * M / (fp64 * 1e12),
                                                       D * (16.0 * J + 8.0 * M) / (hbm * 1e9)) /
                          (kern["residue_heads"] * 1e-3),
                          "note": "fds_vf_identify_residues_device_heads: conjugate rows of pole pairs not written "
                                  "(SURVEY §8d's 16 J + 16 M/2 bytes per DOF)"},
        "api_dof_per_s": {"residue_id": D / (t_res * 1e-3), "residue_id_heads": D / (t_res_h * 1e-3),
                          "rational_invert": D / (t_rat * 1e-3),
                          "fsm": D / (t_fsm * 1e-3), "fsm_chan_major": D / (t_fsm_cm * 1e-3)},
        "api_hbm_frac": {"residue_id": b_res / (t_res * 1e-3) / 1e9 / hbm, "fsm": b_fsm / (t_fsm * 1e-3) / 1e9 / hbm,
                         "fsm_chan_major": b_fsm / (t_fsm_cm * 1e-3) / 1e9 / hbm},
        "kernel_dof_per_s_vf_fsm": D / ((kr + kt) * 1e-3),
        "bytes_per_dof": {"residue_id": b_res / D, "fsm": b_fsm / D}, "flops_per_dof_rational": f_rat / D,
        "pinned": "Chebyshev J=40, Omega_s=1.2 max Im a, T=pi*512/Omega_s, eta=3ln10/T, torch CUDA seed 0",
    }
    return out


def cfg4_afs(fsm_sweep):
    """cfg4 FSM sweep versus AFS at the reference defaults on the LU path
    (afs.hpp:21-39: J0 16, E1 1e-4, E2 2e-3, max_iterations 500, 5 ORFs drawn with
    seed 0, all 48 channels tested; Omega = Omega_s of the N_s = 512 contour)."""
    import paper_1511_04355_b200 as P
    from paper_1511_04355_b200 import BemSystem

    V, F, tr, dofs, s = cfg4_inputs()
    sysb = BemSystem(V, F, tr, channels=dofs, max_batch=16)
    cfg = dict(omega_max=math.pi * NS4 / T_PERIOD, eta=ETA, period=T_PERIOD, max_iterations=500)
    t0 = time.perf_counter()
    try:
        r = P.run_afs(sysb, **cfg)
        res = {"converged": r["converged"], "n_c": r["n_c"], "solver_calls": r["solver_calls"],
               "order": int(len(r["poles"])), "iterations": int(len(r["history"])), "orf": r["orf"]}
    except P.Error as e:  # the reference algorithm's own failure classes (types.hpp:14-36)
        pa = getattr(e, "partial", {})
        hist = pa.get("history", np.zeros((0, 8)))
        res = {"error_class": type(e).__name__, "error": str(e), "n_c": pa.get("n_c"),
               "solver_calls": pa.get("solver_calls"), "iterations_completed": int(len(hist)),
               "failed_at_J": int(pa.get("n_c", 0)), "orf": pa.get("orf"),
               "last_history": hist[-1].tolist() if len(hist) else None}
    wall = time.perf_counter() - t0
    ct = sysb.cumulative_timing()
    sysb.close()
    solver_s = (ct["assembly_ms"] + ct["lu_ms"] + ct["solve_ms"]) * 1e-3
    res.update(wall_s=wall, assembly_s=ct["assembly_ms"] * 1e-3, lu_s=ct["lu_ms"] * 1e-3,
               solve_s=ct["solve_ms"] * 1e-3, frequencies_solved=ct["frequencies"],
               vf_and_driver_s=wall - solver_s,
               config="reference defaults (afs.hpp:21-39), Omega = pi*512/T, eta = 5/T, 48 channels "
                      "(16 points x 3), LU solves (batch of the J0 initial frequencies, then one per iteration)")
    return {"fsm_sweep": fsm_sweep, "afs": res,
            "fsm_solves": fsm_sweep["frequencies"], "afs_solves": res.get("frequencies_solved")}


def extra_configs(args, fsm_sweep):
    """Secondary measurements (not the headline)."""
    from paper_1511_04355_b200 import BemSystem, mesh

    out = {}
    try:
        out["cfg5_vf_fsm_300k"] = cfg5_vf_fsm()
    except Exception as e:  # noqa: BLE001
        out["cfg5_error"] = repr(e)
    try:  # configs[1]: the round-1 headline (129-frequency batch, N = 3840)
        V, F, tr, dofs, s = cfg2_inputs()
        sysb = BemSystem(V, F, tr, channels=dofs, max_batch=len(s))
        for _ in range(2):
            sysb.evaluate_batch_device(s)
        ms = []
        for _ in range(3):
            sysb.evaluate_batch_device(s)
            t = sysb.last_timing()
            ms.append(t["assembly_ms"] + t["lu_ms"] + t["solve_ms"])
        t = sysb.last_timing()
        n = 3 * F.shape[0]
        out["cfg2_N3840_batch129"] = {**t, "solves_per_s": len(s) / (np.mean(ms) * 1e-3),
                                      "lu_tflops": len(s) * 8.0 * n ** 3 / 3 / (t["lu_ms"] * 1e-3) / 1e12}
        sysb.close()
    except Exception as e:  # noqa: BLE001
        out["cfg2_error"] = repr(e)
    try:  # configs[3] one frequency: the single-matrix (look-ahead) LU schedule, plus GMRES
        V, F, tr, dofs, s = cfg4_inputs()
        tc = time.perf_counter()
        sysb = BemSystem(V, F, tr, channels=dofs, max_batch=1)
        create_s = time.perf_counter() - tc
        for _ in range(2):
            sysb.evaluate_batch_device(s[7:8])
        t = sysb.last_timing()
        n = 3 * F.shape[0]
        out["cfg4_N15360_single_solve"] = {**t, "lu_tflops": 8.0 * n ** 3 / 3 / (t["lu_ms"] * 1e-3) / 1e12,
                                           "handle_create_s": create_s,
                                           "note": "handle_create_s: host geometry + near-pair lists + device upload"}
        sysb.set_solver("gmres", tol=1e-12, restart=60, max_iter=2000)
        for _ in range(2):
            sysb.evaluate_batch_device(s[7:8])
        tg = sysb.last_timing()
        gm = sysb.last_gmres()
        out["cfg4_N15360_gmres"] = {**tg, **gm,
                                    "matvec_gbs_effective": 16.0 * n * n * (gm["iterations"] + 1) /
                                    (tg["lu_ms"] * 1e-3) / 1e9,
                                    "note": "lu_ms is the GMRES time (iterations + restarts' true residual products)"}
        sysb.close()
    except Exception as e:  # noqa: BLE001
        out["cfg4_error"] = repr(e)
    try:  # configs[2] one frequency: N = 36864 (21.7 GB), the largest single-GPU config
        V, F = mesh.cube_cavity(32)
        tc = time.perf_counter()
        sysb = BemSystem(V, F, mesh.pressure_traction(V, F), channels=list(range(48)), max_batch=1)
        create_s = time.perf_counter() - tc
        s3 = np.array([complex(ETA, 2 * math.pi / T_PERIOD * 7)])
        for _ in range(2):
            sysb.evaluate_batch_device(s3)
        t = sysb.last_timing()
        n = 3 * F.shape[0]
        out["cfg3_N36864_single_solve"] = {**t, "lu_tflops": 8.0 * n ** 3 / 3 / (t["lu_ms"] * 1e-3) / 1e12,
                                           "handle_create_s": create_s,
                                           "solves_per_s": 1e3 / (t["assembly_ms"] + t["lu_ms"] + t["solve_ms"])}
        sysb.close()
    except Exception as e:  # noqa: BLE001
        out["cfg3_error"] = repr(e)
    try:
        out["cfg4_fsm_vs_afs"] = cfg4_afs(fsm_sweep)
    except Exception as e:  # noqa: BLE001
        out["cfg4_afs_error"] = repr(e)
    return out


def cpu_vf_fsm_baseline(O, D_sample=3000):
    """CPU baseline of the cfg5 VF + FSM stages on a DOF subset (the reference
    path is single-threaded: vecfit.cpp:356-408 per channel, laplace.cpp:89-125
    with one FFTW plan per channel, :127-164). identify_residues runs the oracle
    restatement per channel on 1 thread and on all cores; fsm_invert and
    rational_invert run as vectorised numpy ports on one thread (numpy's
    pocketfft stands in for FFTW; the oracle's own DFT is a direct O(N^2) sum).
    DOF/s extrapolate linearly (every DOF is independent)."""
    import threadpoolctl

    rng = np.random.default_rng(0)
    pairs, J, Ts, Ns = 24, 40, 512, 512
    heads = -(0.01 + 0.49 * rng.random(pairs)) + 1j * 40.0 * rng.random(pairs)
    poles = np.stack([heads, heads.conj()], 1).reshape(-1)
    wmax = 1.2 * heads.imag.max()
    T = math.pi * 512 / wmax
    eta = 3 * math.log(10) / T
    s = eta + 1j * wmax * (1 - np.cos(np.arange(J) * math.pi / (2 * (J - 1))))
    rh = rng.normal(size=(D_sample, pairs)) + 1j * rng.normal(size=(D_sample, pairs))
    res = np.stack([rh, rh.conj()], 2).reshape(D_sample, -1)
    vals = (1.0 / (s[:, None] - poles[None, :])) @ res.T
    vals += 1e-3 * (rng.normal(size=vals.shape) + 1j * rng.normal(size=vals.shape))
    out = {"dofs_sampled": D_sample, "cores_all": os.cpu_count()}
    t0 = time.perf_counter()
    O.identify_residues_many(s, vals, poles, threads=1)
    t1 = time.perf_counter() - t0
    t0 = time.perf_counter()
    R = O.identify_residues_many(s, vals, poles, threads=os.cpu_count())
    tN = time.perf_counter() - t0
    out["residue_id_dof_per_s_1core"] = D_sample / t1
    out["residue_id_dof_per_s_allcores"] = D_sample / tN
    tgrid = np.arange(Ts) * T / Ts
    sk = eta + 1j * (2 * math.pi / T) * np.arange(Ns // 2 + 1)
    half = res @ (1.0 / (sk[None, :] - poles[:, None]))  # (D, 257)
    with threadpoolctl.threadpool_limits(1):
        t0 = time.perf_counter()
        E = np.exp(np.outer(poles, tgrid))  # laplace.cpp:127-164: h = Re sum r e^{a t}
        np.real(R @ E)
        tr = time.perf_counter() - t0
        t0 = time.perf_counter()
        k = np.arange(Ns // 2 + 1)
        w = 0.5 * (1 + np.cos(2 * math.pi * k / Ns))  # laplace.cpp:67-72 Hanning on the half spectrum
        w[0] = 1.0
        h = np.fft.irfft(half * w[None, :], n=Ns, axis=1) * (Ns / T)  # conjugate fill + inverse DFT
        h *= np.exp(eta * np.arange(Ns) * (T / Ns))[None, :]
        tf = time.perf_counter() - t0
    out["rational_invert_dof_per_s_1core"] = D_sample / tr
    out["fsm_dof_per_s_1core"] = D_sample / tf
    out["vf_fsm_dof_per_s_1core"] = D_sample / (t1 + tr)
    out["kind"] = "port"
    out["sample"] = (f"{D_sample} DOFs of the cfg5 distribution (J=40, M=48, 512 steps); oracle identify_residues "
                     "per channel (C, 1 thread / all cores); numpy rational_invert and irfft-based FSM on 1 thread")
    return out


def main():
    faulthandler.enable()
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-extra", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    world, rank, local, dist = dist_setup()
    if args.impl == "reference":
        run_reference(args, world, rank)
    else:
        run_ours(args, world, rank, local, dist)
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
