"""cuBLAS reference for the LU trailing update shape: C(mxm) -= A(mx64) B(64xm), complex128."""
import json, torch
out = {}
for (m, b) in [(3776, 129), (2560, 129), (15296, 1), (7680, 1)]:
    A = torch.randn(b, m, 64, dtype=torch.complex128, device="cuda")
    B = torch.randn(b, 64, m, dtype=torch.complex128, device="cuda")
    C = torch.randn(b, m, m, dtype=torch.complex128, device="cuda")
    for _ in range(3): torch.baddbmm(C, A, B, beta=1, alpha=-1, out=C)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e30
    for _ in range(5):
        e0.record(); torch.baddbmm(C, A, B, beta=1, alpha=-1, out=C); e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    out[f"m{m}_b{b}"] = round(8.0 * m * m * 64 * b / (best * 1e-3) / 1e12, 2)
    del A, B, C
print(json.dumps(out))
