"""cuBLAS DGEMM (torch.matmul float64) on the ACI contraction shapes, for comparison only."""
import torch
for (m, k, n) in [(1024, 256, 1024), (512, 256, 512), (1024, 512, 1024), (2048, 256, 2048), (8192, 8192, 8192)]:
    a = torch.randn(m, k, dtype=torch.float64, device="cuda")
    b = torch.randn(k, n, dtype=torch.float64, device="cuda")
    for _ in range(3):
        torch.matmul(a, b)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 50 if m < 8192 else 5
    e0.record()
    for _ in range(reps):
        torch.matmul(a, b)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(f"cuBLAS {m}x{k}x{n}: {ms*1e3:8.1f} us {2*m*n*k/ms/1e9:6.2f} TF/s")
