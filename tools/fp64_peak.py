"""Measure the FP64 GEMM peak on the box (cuBLAS DGEMM via torch.matmul float64),
the same way MEASURED_PEAKS.json measures bf16: best of 10 (burst) and back-to-back
for ~4 s (sustained). Prints one JSON line. Tooling only, not part of the product."""
import json, time, torch
n = 8192
a = torch.randn(n, n, dtype=torch.float64, device="cuda")
b = torch.randn(n, n, dtype=torch.float64, device="cuda")
for _ in range(3):
    torch.matmul(a, b)
torch.cuda.synchronize()
best = 1e9
for _ in range(10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); torch.matmul(a, b); e1.record(); torch.cuda.synchronize()
    best = min(best, e0.elapsed_time(e1))
burst = 2 * n**3 / (best * 1e-3) / 1e12
t0 = time.time(); k = 0
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record()
while time.time() - t0 < 4.0:
    torch.matmul(a, b); k += 1
    if k % 4 == 0: torch.cuda.synchronize()
e1.record(); torch.cuda.synchronize()
sus = 2 * n**3 * k / (e0.elapsed_time(e1) * 1e-3) / 1e12
print(json.dumps({"dgemm_tflops_burst": round(burst, 2), "dgemm_tflops_sustained": round(sus, 2), "n": n}))
