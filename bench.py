#!/usr/bin/env python
"""Benchmark of the B200 BEM / VF / FSM hot path (BASELINE.json metric).

Headline workload (configs[1]): spherical cavity, 1280-triangle icosphere
(N = 3840 unknowns), Heaviside pressure, the full FSM contour of T = 20,
N_s = 256 (N_c = N_s/2 + 1 = 129 frequencies, s_k = 5/T + i k 2π/T) solved as one
batch of independent dense systems; displacement at 16 collocation points
(48 DOFs). One step = assembly + batched LU + solve of all 129 systems.

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]

Under torchrun (N > 1) every rank solves its own 129-frequency sweep (replicas
only: the path has no exchange step), the step time is the max
over ranks, and value = total solves / time ("scaling": "weak").
``--impl reference`` times the CPU oracle port of the same path (OpenMP
assembly + OpenBLAS zgetrf on all host cores) — the reference has no BEM.
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
T_PERIOD, NS = 20.0, 256
ETA = 5.0 / T_PERIOD


def cfg2_inputs():
    from paper_1511_04355_b200 import mesh

    V, F = mesh.icosphere(3)
    tr = mesh.pressure_traction(V, F)
    pts = mesh.draw_indices(F.shape[0], 16, 0)
    dofs = [3 * p + i for p in pts for i in range(3)]
    nc = NS // 2 + 1
    s = ETA + 1j * (2 * math.pi / T_PERIOD) * np.arange(nc)
    return V, F, tr, dofs, s


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

    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(dist):
    if dist is not None:
        dist.barrier()


# ------------------------------------------------------------------ CPU legs
def cpu_oracle_solves(n_freq: int, warm: int = 0):
    """Oracle port: OpenMP assembly + OpenBLAS zgetrf/zgetrs, all host cores."""
    sys.path.insert(0, str(ROOT / "oracle"))
    import pyoracle as O

    V, F, tr, dofs, s = cfg2_inputs()
    bem = O.Bem(V, F, tr)
    ob = O.openblas_path()
    for i in range(warm):
        bem.solve_openblas(s[1 + i], ob)
    t0 = time.perf_counter()
    for i in range(n_freq):
        bem.solve_openblas(s[1 + (i % (len(s) - 1))], ob)
    return time.perf_counter() - t0


def run_reference(args, world, rank):
    if rank != 0:
        return
    per = []
    cpu_oracle_solves(0, warm=min(args.warmup, 1))
    for _ in range(args.steps):
        per.append(cpu_oracle_solves(1))
    dt = float(np.mean(per))
    v = 1.0 / dt
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "c128", "data": "synthetic",
        "config": {"workload": "cfg2 sphere 1280 tri N=3840, one FSM frequency per step (bounded CPU sample)",
                   "sample": "1 frequency solve per step"},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": os.cpu_count(), "kind": "port",
                         "sample": "oracle BEM (OpenMP assembly) + OpenBLAS zgetrf/zgetrs, 1 frequency of cfg2 per step"},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ GPU leg
# FP64 flops per far-field kernel evaluation: 32 x (2 DFMA + DMUL + DADD) warp
# instructions of bem_far_kernel (ncu sass__inst_executed_per_opcode on cfg2)
# divided by its 7 N_e (N_e - 1) B evaluations (profiles/r01_assembly_ncu_full.json).
ASM_FLOPS_PER_EVAL = 439.0


def run_ours(args, world, rank, local, dist):
    import paper_1511_04355_b200 as P
    from paper_1511_04355_b200 import BemSystem

    L = P.lib()
    P.api._check(L.fds_set_device(local))
    V, F, tr, dofs, s = cfg2_inputs()
    B = len(s)
    sysb = BemSystem(V, F, tr, channels=dofs, max_batch=B)
    for _ in range(args.warmup):
        sysb.evaluate_batch_device(s)
    barrier(dist)
    launches0 = P.kernel_launches()
    dev_ms = []
    with ClockSampler(local) as clk:
        t0 = time.perf_counter()
        for _ in range(args.steps):
            sysb.evaluate_batch_device(s)
            t = sysb.last_timing()
            dev_ms.append(t["assembly_ms"] + t["lu_ms"] + t["solve_ms"])
        wall = time.perf_counter() - t0
    launches = (P.kernel_launches() - launches0) // args.steps
    stage = sysb.last_timing()
    total_ms = allreduce_max(dist, float(np.sum(dev_ms)))
    ms_step = total_ms / args.steps
    value = B * world / (ms_step * 1e-3)

    # end to end through the public C-ABI with host buffers (H2D s, D2H values)
    barrier(dist)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        sysb.evaluate_batch(s)
    e2e_s = allreduce_max(dist, time.perf_counter() - t0) / args.steps
    e2e = {"value": B * world / e2e_s, "unit": UNIT, "h2d_bytes_per_step": 16 * B,
           "d2h_bytes_per_step": 16 * B * len(dofs)}

    # roofline of the dominant kernel (LU trailing GEMM on the FP64 tensor pipe)
    P.api._check(L.fds_profile_enable(1))
    sysb.evaluate_batch_device(s)
    import ctypes

    c, ms, wk = ctypes.c_int(), ctypes.c_double(), ctypes.c_double()
    P.api._check(L.fds_profile_read(0, ctypes.byref(c), ctypes.byref(ms), ctypes.byref(wk)))
    gemm = dict(launches=c.value, ms=ms.value, flops=wk.value)
    P.api._check(L.fds_profile_read(1, ctypes.byref(c), ctypes.byref(ms), ctypes.byref(wk)))
    panel = dict(launches=c.value, ms=ms.value)
    P.api._check(L.fds_profile_read(2, ctypes.byref(c), ctypes.byref(ms), ctypes.byref(wk)))
    trsm = dict(launches=c.value, ms=ms.value)
    P.api._check(L.fds_profile_read(3, ctypes.byref(c), ctypes.byref(ms), ctypes.byref(wk)))
    far = dict(ms=ms.value, evaluations=wk.value)
    P.api._check(L.fds_profile_enable(0))
    peak, peak_src = measured_fp64_peak()
    # the library's GEMM work counter is the algorithmic complex count 8 rest^2 w; the
    # default 3M kernel executes three real products per complex MAC (6 rest^2 w)
    four_m = os.environ.get("FDSWEEP_GEMM", "") in ("4m", "cpasync")
    executed = 1.0 if four_m else 0.75
    effective = gemm["flops"] / (gemm["ms"] * 1e-3) / 1e12 if gemm["ms"] > 0 else None
    achieved = effective * executed if effective else None
    gemm_kernel = "lu_gemm_tma_kernel" if four_m else "lu_gemm3m_tma_kernel"
    traffic = ncu_traffic(gemm_kernel)
    n = 3 * F.shape[0]
    lu_flops = B * 8.0 * n ** 3 / 3.0
    result = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "c128",
        "data": "synthetic",
        "config": {"workload": "cfg2: sphere cavity, 1280-tri icosphere, N=3840, 129-frequency FSM batch "
                               "(T=20, Ns=256, eta=5/T), 16 collocation points",
                   "global_batch": B * world, "parallelism": f"replicas x{world}",
                   "l2": "inputs larger than L2 (129 x 236 MB matrices)"},
        "e2e": e2e,
        "roofline": {"bound": "tensor",
                     "kernel": (gemm_kernel + (" (TMA-fed DMMA complex GEMM)" if four_m else
                                               " (TMA-fed DMMA complex GEMM, 3 real products per complex MAC; "
                                               "timing includes lu_g3_prep_kernel)")),
                     "achieved": achieved,
                     "peak": peak, "unit": "TFLOP/s", "frac": (achieved / peak) if achieved else None,
                     "peak_source": peak_src, "traffic": traffic,
                     "work_def": ("8*rest^2*w FP64 flops per launch (A22 -= L21 U12)" if four_m else
                                  "6*rest^2*w FP64 flops executed per launch (A22 -= L21 U12 as 3 real GEMMs)"),
                     "effective_complex_tflops": effective,
                     "effective_work_def": "8*rest^2*w (conventional complex GEMM count) / time",
                     "share_of_lu": gemm["ms"] / max(gemm["ms"] + panel["ms"] + trsm["ms"], 1e-9)},
        "stages_ms": {"assembly": stage["assembly_ms"], "lu": stage["lu_ms"], "solve": stage["solve_ms"],
                      "lu_panel": panel["ms"], "lu_trsm": trsm["ms"], "lu_gemm": gemm["ms"]},
        "lu_tflops": lu_flops / (stage["lu_ms"] * 1e-3) / 1e12,
        # assembly far field: kernel evaluations x a per-evaluation FP64 flop
        # constant taken from the kernel's SASS op counts (DFMA = 2), profiles/r01_assembly_ncu_full.json
        "assembly_far": {"ms": far["ms"], "kernel_evaluations": far["evaluations"],
                         "flops_per_evaluation": ASM_FLOPS_PER_EVAL,
                         "tflops": ASM_FLOPS_PER_EVAL * far["evaluations"] / max(far["ms"], 1e-9) / 1e9,
                         "fp64_frac": ASM_FLOPS_PER_EVAL * far["evaluations"] / max(far["ms"], 1e-9) / 1e9 / peak},
        "wall_ms_per_step": wall * 1e3 / args.steps,
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
    }
    sysb.close()
    if rank == 0 and world == 1 and not args.no_extra:
        result["extra"] = extra_configs(args)
    if rank == 0 and world == 1 and not args.no_cpu:
        ncpu = 2
        dt = cpu_oracle_solves(ncpu, warm=1)
        result["cpu_baseline"] = {"value": ncpu / dt, "unit": UNIT, "cores": os.cpu_count(), "kind": "port",
                                  "sample": f"{ncpu} frequencies of cfg2 (N=3840): oracle BEM assembly (OpenMP) "
                                            "+ OpenBLAS zgetrf/zgetrs"}
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

    t_res = best(lambda: P.api._check(L.fds_vf_identify_residues_device(
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
        "api_ms": {"residue_id": t_res, "rational_invert": t_rat, "fsm": t_fsm, "fsm_chan_major": t_fsm_cm},
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
        "vf_fsm_dof_per_s": D / ((kr + kt) * 1e-3),
        "bytes_per_dof": {"residue_id": b_res / D, "fsm": b_fsm / D}, "flops_per_dof_rational": f_rat / D,
        "pinned": "Chebyshev J=40, Omega_s=1.2 max Im a, T=pi*512/Omega_s, eta=3ln10/T, torch CUDA seed 0",
    }
    return out


def extra_configs(args):
    """Secondary measurements (not the headline): cfg4 single N=15360 solve, cfg5 VF/FSM."""
    from paper_1511_04355_b200 import BemSystem, mesh

    out = {}
    try:  # the headline batch through the iterative solver (not the BASELINE metric)
        V, F = mesh.icosphere(3)
        sysg = BemSystem(V, F, mesh.pressure_traction(V, F), channels=list(range(48)), max_batch=129)
        sysg.set_solver("gmres", tol=1e-12, restart=60, max_iter=2000)
        sg = 0.25 + 1j * 2 * math.pi / 20.0 * np.arange(129)
        sysg.evaluate_batch_device(sg)
        sysg.evaluate_batch_device(sg)
        tg = sysg.last_timing()
        out["cfg2_gmres_batch"] = {**tg, **sysg.last_gmres(),
                                   "solves_per_s": 129.0 / ((tg["assembly_ms"] + tg["lu_ms"] + tg["solve_ms"]) * 1e-3),
                                   "note": "lu_ms is the lockstep GMRES time for all 129 systems (tol 1e-12)"}
        sysg.close()
    except Exception as e:  # noqa: BLE001
        out["cfg2_gmres_error"] = repr(e)
    try:
        out["cfg5_vf_fsm_300k"] = cfg5_vf_fsm()
    except Exception as e:  # noqa: BLE001
        out["cfg5_error"] = repr(e)
    try:
        V, F = mesh.icosphere(4)
        tr = mesh.random_traction(F.shape[0], seed=0)
        sysb = BemSystem(V, F, tr, channels=list(range(48)), max_batch=1)
        s = np.array([0.25 + 1j * 2 * math.pi / 20.0])
        sysb.evaluate_batch_device(s)
        sysb.evaluate_batch_device(s)
        t = sysb.last_timing()
        n = 3 * F.shape[0]
        out["cfg4_N15360_single_solve"] = {**{k: v for k, v in t.items()},
                                           "lu_tflops": 8.0 * n ** 3 / 3 / (t["lu_ms"] * 1e-3) / 1e12}
        # iterative alternative: restarted GMRES on the same assembled system
        sysb.set_solver("gmres", tol=1e-12, restart=60, max_iter=2000)
        sysb.evaluate_batch_device(s)
        sysb.evaluate_batch_device(s)
        tg = sysb.last_timing()
        gm = sysb.last_gmres()
        out["cfg4_N15360_gmres"] = {**{k: v for k, v in tg.items()}, **gm,
                                    "matvec_gbs_effective": 16.0 * n * n * (gm["iterations"] + 1) / (tg["lu_ms"] * 1e-3) / 1e9,
                                    "note": "lu_ms is the GMRES time (iterations + restarts' true residual products)"}
        sysb.close()
    except Exception as e:  # noqa: BLE001
        out["cfg4_error"] = repr(e)
    return out


def main():
    faulthandler.enable()
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
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
