"""Measured dense TF32 GEMM rate of this B200 through cuBLAS (torch.matmul, fp32 inputs with
TF32 tensor cores allowed), 8192^3, for context next to the nominal-ratio peak bench.py uses."""
import torch
torch.backends.cuda.matmul.allow_tf32 = True
n = 8192
a = torch.randn(n, n, device="cuda")
b = torch.randn(n, n, device="cuda")
for _ in range(3):
    a @ b
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
best = 0.0
for _ in range(5):
    e0.record()
    for _ in range(10):
        a @ b
    e1.record()
    torch.cuda.synchronize()
    best = max(best, 10 * 2 * n ** 3 / (e0.elapsed_time(e1) / 1e3) / 1e12)
print(f"cuBLAS TF32 8192^3: {best:.1f} TFLOP/s (best of 5 x 10)")
