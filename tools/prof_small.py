"""Small-order probes for ncu / timing: single trinv_lower at n = 64, 128, 256 and
batched orders 64 / 128 (device-resident synthetic inputs).

    python tools/prof_small.py            # CUDA-event timings (graph replay)
    ncu ... python tools/prof_small.py --once
"""
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_2307_07611_b200 as P  # noqa: E402


def timed(fn, reps=200):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); g.replay(); e1.record(); e1.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    return statistics.median(ts)


def main():
    once = "--once" in sys.argv
    dev = torch.device("cuda:0")
    cases = []
    for n in (64, 128, 256):
        A = torch.from_numpy(synth.host(n, seed=0)).to(dev)
        X = torch.empty_like(A)
        cases.append((f"trinv_lower n={n}", lambda A=A, X=X: P.trinv_lower(A, out=X)))
    for n, B in ((64, 148), (128, 148), (128, 4096), (64, 16384)):
        A = torch.empty((B, n, n), dtype=torch.float64, device=dev)
        synth.device_fill(A, n)
        X = torch.empty_like(A)
        cases.append((f"batched n={n} B={B}", lambda A=A, X=X: P.trinv_batched(A, out=X)))
    for name, fn in cases:
        if once:
            fn()
            torch.cuda.synchronize()
        else:
            print(f"{name:28s} {timed(fn):9.2f} us")


if __name__ == "__main__":
    main()
