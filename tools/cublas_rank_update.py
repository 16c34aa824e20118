"""cuBLAS reference point for the LU Schur update shape (a7): C[M x M] -= A[M x K] B[K x M] in FP64 with
K = nb = 256, through torch.addmm (cuBLAS DGEMM), CUDA events, best and mean of 10 after 3 warm-ups.
Prints one JSON line per M.  python tools/cublas_rank_update.py [M ...]"""
import json
import sys

import torch


def main():
    Ms = [int(a) for a in sys.argv[1:]] or [32512, 16128, 8192]
    K = 256
    for M in Ms:
        A = torch.randn(M, K, dtype=torch.float64, device="cuda")
        B = torch.randn(K, M, dtype=torch.float64, device="cuda")
        C = torch.randn(M, M, dtype=torch.float64, device="cuda")
        for _ in range(3):
            C.addmm_(A, B, alpha=-1.0)
        torch.cuda.synchronize()
        ts = []
        for _ in range(10):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            C.addmm_(A, B, alpha=-1.0)
            e1.record()
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        fl = 2.0 * M * M * K
        print(json.dumps({"kernel": "cublas_dgemm_addmm", "M": M, "N": M, "K": K,
                          "best_ms": min(ts), "mean_ms": sum(ts) / len(ts),
                          "tflops_best": fl / min(ts) / 1e9, "tflops_mean": fl / (sum(ts) / len(ts)) / 1e9}),
              flush=True)
        del A, B, C
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
