"""GFLOP/s of trinv_lower / trinv_upper / inv_from_lu over n (device-resident inputs,
CUDA events, per-call median of a few reps; small n replayed from a CUDA graph).

    python tools/sweep_n.py > profiles/r01_sweep_n.txt
"""
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_2307_07611_b200 as P  # noqa: E402


def bench(fn, reps):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    if reps >= 20:  # latency-bound sizes: graph replay
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            fn()
        run = g.replay
    else:
        run = fn
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); run(); e1.record(); e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)


def main():
    dev = torch.device("cuda:0")
    print(f"{'op':6s} {'n':>6s} {'ms':>10s} {'GFLOP/s':>10s} {'%DMMA peak':>10s}")
    for n in (64, 128, 256, 512, 1024, 2048, 4096, 8192, 16384, 32768):
        reps = 50 if n <= 1024 else (10 if n <= 8192 else 3)
        for uplo in ("L", "U"):
            A = torch.empty((n, n), dtype=torch.float64, device=dev)
            synth.device_fill(A, n, uplo=uplo, diag="signed" if uplo == "L" else "pos")
            X = torch.empty_like(A)
            f = P.trinv_lower if uplo == "L" else P.trinv_upper
            ms = bench(lambda: f(A, out=X), reps)
            gf = n ** 3 / 3 / (ms / 1e3) / 1e9
            print(f"{'trinv' + uplo:6s} {n:6d} {ms:10.4f} {gf:10.1f} {100 * gf / 37085:9.1f}%", flush=True)
            del A, X
        if 128 <= n <= 16384:
            L = torch.empty((n, n), dtype=torch.float64, device=dev)
            U = torch.empty_like(L)
            synth.device_fill(L, n, tag="L", diag="one")
            synth.device_fill(U, n, tag="U", uplo="U", diag="pos")
            X = torch.empty_like(L)
            ms = bench(lambda: P.inv_from_lu(L, U, out=X), reps)
            gf = 4 * n ** 3 / 3 / (ms / 1e3) / 1e9
            print(f"{'lu':6s} {n:6d} {ms:10.4f} {gf:10.1f} {100 * gf / 37085:9.1f}%", flush=True)
            del L, U, X
        torch.cuda.empty_cache()




def sweep_beta4():
    dev = torch.device("cuda:0")
    print(f"{'op':8s} {'n':>6s} {'beta2 ms':>10s} {'beta4 ms':>10s} {'b4/b2':>7s}")
    for n in (256, 512, 1024, 2048, 4096, 8192, 16384):
        reps = 50 if n <= 1024 else (10 if n <= 8192 else 3)
        for uplo in ("L", "U"):
            A = torch.empty((n, n), dtype=torch.float64, device=dev)
            synth.device_fill(A, n, uplo=uplo, diag="signed" if uplo == "L" else "pos")
            X = torch.empty_like(A)
            t2 = bench(lambda: P.trinv_beta(A, uplo, 2, out=X), reps)
            t4 = bench(lambda: P.trinv_beta(A, uplo, 4, out=X), reps)
            print(f"{'trinv' + uplo:8s} {n:6d} {t2:10.4f} {t4:10.4f} {t4 / t2:7.3f}", flush=True)
            del A, X
        torch.cuda.empty_cache()


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "beta4":
        sweep_beta4()
    else:
        main()
