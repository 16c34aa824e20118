"""cuBLAS DGEMM throughput probe via torch.matmul(float64) -- measurement only (roofline context).

Prints one JSON line per size: burst (best of 5) and sustained (back to back for ~4 s).
"""
import json
import time

import torch


def main():
    dev = torch.device("cuda:0")
    for n in (8192, 16384):
        a = torch.randn(n, n, dtype=torch.float64, device=dev)
        b = torch.randn(n, n, dtype=torch.float64, device=dev)
        c = torch.empty(n, n, dtype=torch.float64, device=dev)
        for _ in range(2):
            torch.matmul(a, b, out=c)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        best = 1e30
        for _ in range(5):
            e0.record()
            torch.matmul(a, b, out=c)
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        flops = 2.0 * n ** 3
        t0 = time.time()
        reps = 0
        e0.record()
        while time.time() - t0 < 4.0:
            torch.matmul(a, b, out=c)
            reps += 1
            if reps % 4 == 0:
                torch.cuda.synchronize()
        e1.record()
        torch.cuda.synchronize()
        sus = e0.elapsed_time(e1) / reps
        print(json.dumps({"kernel": "cublas_dgemm", "n": n, "burst_tflops": flops / best / 1e9,
                          "sustained_tflops": flops / sus / 1e9, "reps": reps}), flush=True)


if __name__ == "__main__":
    main()
