"""The library's Schur update kernel alone on the C3 step-1 shape (hlq_test_schur: A[K:, K:] -=
A[K:, :K] A[:K, K:], M = N - K), TMA-fed (k_dgemm_tma) and cp.async (k_dgemm), CUDA events, best and
mean of 10 after 3 warm-ups; the same shape as tools/cublas_rank_update.py.
python tools/schur_bench.py [N ...]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1401_5522_b200 as H  # noqa: E402


def main():
    Ns = [int(a) for a in sys.argv[1:]] or [32768, 16384, 8448]
    K = 256
    for N in Ns:
        A = torch.empty(N * N, dtype=torch.float64, device="cuda")
        H.hlq_generate_uniform(A, N, N, N, 3, 0, N)
        s = torch.cuda.current_stream()
        for tma in (1, 0):
            for _ in range(3):
                H.hlq_test_schur(A, N, N, 0, K, bool(tma), stream=s)
            ts = []
            for _ in range(10):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(s)
                ran = H.hlq_test_schur(A, N, N, 0, K, bool(tma), stream=s)
                e1.record(s)
                e1.synchronize()
                ts.append(e0.elapsed_time(e1))
            M = N - K
            fl = 2.0 * M * M * K
            print(json.dumps({"kernel": "k_dgemm_tma" if ran == 1 else "k_dgemm", "M": M, "N": M,
                              "K": K, "best_ms": min(ts), "mean_ms": sum(ts) / len(ts),
                              "tflops_best": fl / min(ts) / 1e9,
                              "tflops_mean": fl / (sum(ts) / len(ts)) / 1e9}), flush=True)
        del A
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
