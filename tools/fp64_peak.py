"""Measure cuBLAS DGEMM (torch.float64 matmul) throughput: burst and sustained.

Writes one JSON line per measurement; used to fill the FP64 roofline
denominator that MEASURED_PEAKS.json does not carry.
"""
import json
import time

import torch


def main():
    dev = torch.device("cuda:0")
    n = 8192
    a = torch.randn(n, n, dtype=torch.float64, device=dev)
    b = torch.randn(n, n, dtype=torch.float64, device=dev)
    c = torch.empty(n, n, dtype=torch.float64, device=dev)
    for _ in range(3):
        torch.matmul(a, b, out=c)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    best = 1e30
    for _ in range(5):
        e0.record()
        torch.matmul(a, b, out=c)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    print(json.dumps({"bench": "dgemm_burst", "n": n, "ms": best, "tflops": 2 * n**3 / best / 1e9}))
    t0 = time.time()
    cnt = 0
    e0.record()
    while time.time() - t0 < 6.0:
        torch.matmul(a, b, out=c)
        cnt += 1
        if cnt % 4 == 0:
            torch.cuda.synchronize()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(json.dumps({"bench": "dgemm_sustained", "n": n, "iters": cnt, "ms": ms,
                      "tflops": 2 * n**3 * cnt / ms / 1e9}))


if __name__ == "__main__":
    main()
