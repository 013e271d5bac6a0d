set -x
timeout 120 ./tools/gemm_bench2 > gpurun_out/r02m_gemm.txt 2>&1
timeout 120 python -c "
import torch
a = torch.randn(1024, 256, dtype=torch.float64, device='cuda'); b = torch.randn(256, 1024, dtype=torch.float64, device='cuda')
c = a @ b
best = 1e9
for _ in range(5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20): torch.matmul(a, b, out=c)
    e1.record(); torch.cuda.synchronize(); best = min(best, e0.elapsed_time(e1) / 20)
print('cuBLAS DGEMM 1024x256x1024: %.2f us %.2f TF/s' % (best * 1e3, 2 * 1024 * 1024 * 256 / best / 1e9))
" >> gpurun_out/r02m_gemm.txt 2>&1
