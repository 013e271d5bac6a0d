"""Measure cuBLAS DGEMM (torch.matmul float64) as the achievable FP64 ceiling.

Not part of the product path: it sizes the roofline denominator that
MEASURED_PEAKS.json does not carry (FP64). Prints one JSON line.
"""
import json
import subprocess
import time

import torch


def main():
    n = 8192
    a = torch.randn(n, n, dtype=torch.float64, device="cuda")
    b = torch.randn(n, n, dtype=torch.float64, device="cuda")
    for _ in range(3):
        torch.matmul(a, b)
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(10):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        torch.matmul(a, b)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    # sustained for ~4 s with clocks sampled
    smi = subprocess.Popen(
        ["nvidia-smi", "--query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active",
         "--format=csv,noheader,nounits", "-lms", "200"], stdout=subprocess.PIPE, text=True)
    t0 = time.time()
    cnt = 0
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    while time.time() - t0 < 4.0:
        torch.matmul(a, b)
        cnt += 1
        if cnt % 4 == 0:
            torch.cuda.synchronize()
    e1.record()
    torch.cuda.synchronize()
    smi.terminate()
    out = smi.communicate()[0].strip().splitlines()
    sust_ms = e0.elapsed_time(e1) / cnt
    clocks = [float(x.split(",")[0]) for x in out if x.strip()]
    clocks.sort()
    print(json.dumps({
        "dgemm_n": n,
        "dgemm_tflops_burst": 2 * n ** 3 / best / 1e9,
        "dgemm_tflops_sustained": 2 * n ** 3 / sust_ms / 1e9,
        "sm_mhz_median": clocks[len(clocks) // 2] if clocks else None,
        "smi_tail": out[-3:],
    }))


if __name__ == "__main__":
    main()
