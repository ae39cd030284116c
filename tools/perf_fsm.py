"""FSM C2R kernel at cfg5 size (300k DOFs, N_s = 512): time + oracle agreement,
for the frequency-major layout (as the batched BEM produces spectra) and the
channel-major layout (the reference's per-channel fsm_invert input).

Usage: FDSWEEP_FSM=<variant> FSM_D=<dofs> python tools/perf_fsm.py
"""
import ctypes, json, math, os, sys
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "oracle"))
import numpy as np
import torch
import paper_1511_04355_b200 as P
import pyoracle as O

D, Ns = int(os.environ.get("FSM_D", 300_000)), 512
Nc = Ns // 2 + 1
L = P.lib()
g = torch.Generator(device="cuda").manual_seed(0)
fm = torch.complex(torch.randn(Nc, D, generator=g, device="cuda", dtype=torch.float64),
                   torch.randn(Nc, D, generator=g, device="cuda", dtype=torch.float64))
cm = fm.T.contiguous()
out = torch.empty((D, Ns), dtype=torch.float64, device="cuda")
Tper, eta = 20.0, 0.3
res = {"variant": os.environ.get("FDSWEEP_FSM", "default"), "D": D}
sub = np.arange(0, D, 9973)
ref = O.fsm_invert(Tper, Ns, eta, fm[:, sub].T.cpu().numpy().copy())
for name, buf, sk, si in (("freq_major", fm, 1, D), ("chan_major", cm, Nc, 1)):
    def call():
        P.api._check(L.fds_fsm_invert_device_strided(
            ctypes.c_double(Tper), Ns, ctypes.c_double(eta), D, ctypes.c_void_p(buf.data_ptr()),
            ctypes.c_longlong(sk), ctypes.c_longlong(si), 1, ctypes.c_void_p(out.data_ptr()), None))
    for _ in range(3):
        call()
    ev = []
    for _ in range(5):
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); call(); b.record(); torch.cuda.synchronize(); ev.append(a.elapsed_time(b))
    ms = min(ev)
    got = out[sub].cpu().numpy()
    res[name] = {"call_ms": ms, "GBps": D * (16 * Nc + 8 * Ns) / (ms * 1e6),
                 "rel_vs_oracle": float(np.linalg.norm(got - ref) / np.linalg.norm(ref))}
print(json.dumps(res))
