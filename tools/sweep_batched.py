"""Batched small-order throughput (trinv_batched, device-resident synthetic inputs, CUDA
events): python tools/sweep_batched.py [n ...].  HBM fraction on the algorithmic bytes
n(n+1)/2 read + n^2 written per matrix, against MEASURED_PEAKS.json hbm_gbs."""
import json
import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
import paper_2307_07611_b200 as P  # noqa: E402


def main():
    ns = [int(v) for v in sys.argv[1:]] or [16, 32, 48, 64, 96, 128]
    try:
        hbm = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    except Exception:
        hbm = 6550.4
    dev = torch.device("cuda:0")
    print(f"{'n':>4} {'batch':>8} {'us':>9} {'inv/s':>10} {'GB/s':>8} {'frac':>6} {'GFLOP/s':>9}")
    for n in ns:
        B = max(1, (1 << 30) // (n * n * 8))  # ~1 GiB of input (larger than L2)
        A = torch.empty((B, n, n), dtype=torch.float64, device=dev)
        synth.device_fill(A, n)
        X = torch.empty_like(A)
        for _ in range(3):
            P.trinv_batched(A, out=X)
        torch.cuda.synchronize()
        ts = []
        for _ in range(20):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); P.trinv_batched(A, out=X); e1.record(); e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        ms = statistics.median(ts)
        byts = B * (n * (n + 1) / 2 + n * n) * 8
        gbs = byts / ms / 1e6
        print(f"{n:4d} {B:8d} {ms * 1e3:9.1f} {B / ms * 1e3:10.3e} {gbs:8.1f} {gbs / hbm:6.3f} "
              f"{B * n ** 3 / 3 / ms / 1e6:9.1f}")
        del A, X


if __name__ == "__main__":
    main()
