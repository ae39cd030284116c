"""cuBLAS FP64 reference throughput (DGEMM / ZGEMM via torch.matmul) on one B200.

Used once to pin the FP64 roofline denominator alongside fp64_peak.cu.
"""
import json, torch

def bench(dtype, n, reps=10):
    a = torch.randn(n, n, dtype=dtype, device="cuda")
    b = torch.randn(n, n, dtype=dtype, device="cuda")
    for _ in range(3):
        c = a @ b
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); c = a @ b; e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    flops = (8.0 if dtype.is_complex else 2.0) * n ** 3
    return flops / (best * 1e-3) / 1e12

out = {}
for n in (4096, 8192):
    out[f"dgemm_{n}_tflops"] = round(bench(torch.float64, n), 3)
    out[f"zgemm_{n}_tflops"] = round(bench(torch.complex128, n), 3)
a = torch.randn(15360, 15360, dtype=torch.complex128, device="cuda")
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
lu = torch.linalg.lu_factor(a[:3840, :3840].contiguous()); torch.cuda.synchronize()
for n in (3840, 15360):
    m = a[:n, :n].contiguous()
    torch.linalg.lu_factor(m); torch.cuda.synchronize()
    e0.record(); torch.linalg.lu_factor(m); e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    out[f"torch_zgetrf_{n}_ms"] = round(ms, 3)
    out[f"torch_zgetrf_{n}_tflops"] = round(8.0 * n ** 3 / 3 / (ms * 1e-3) / 1e12, 3)
print(json.dumps(out))
