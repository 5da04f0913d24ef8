"""Per-kernel time breakdown of one library call via torch.profiler (CUPTI activity
records, no replay): python tools/kprof.py A 16384   (ops as in tools/prof_one.py, plus A)."""
import os
import sys
from collections import defaultdict

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_2307_07611_b200 as P  # noqa: E402


def main():
    op, n = sys.argv[1], int(sys.argv[2])
    dev = torch.device("cuda:0")
    if op == "A":
        L = torch.empty((n, n), dtype=torch.float64, device=dev)
        U = torch.empty_like(L)
        synth.device_fill(L, n, uplo="L", diag="one", tag="L")
        synth.device_fill(U, n, uplo="U", diag="pos", tag="U")
        A = L @ U
        X = torch.empty_like(A)
        fn = lambda: P.inv_general(A, out=X)  # noqa: E731
    elif op in "LU":
        A = torch.empty((n, n), dtype=torch.float64, device=dev)
        synth.device_fill(A, n, uplo=op, diag="signed" if op == "L" else "pos")
        X = torch.empty_like(A)
        fn = (lambda: P.trinv_lower(A, out=X)) if op == "L" else (lambda: P.trinv_upper(A, out=X))
    elif op == "G":
        L = torch.empty((n, n), dtype=torch.float64, device=dev)
        U = torch.empty_like(L)
        synth.device_fill(L, n, uplo="L", diag="one", tag="L")
        synth.device_fill(U, n, uplo="U", diag="pos", tag="U")
        X = torch.empty_like(L)
        fn = lambda: P.inv_from_lu(L, U, unit_l=True, out=X)  # noqa: E731
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); fn(); e1.record(); e1.synchronize()
    wall = e0.elapsed_time(e1)
    with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
        fn(); torch.cuda.synchronize()
    evs = sorted([e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA],
                 key=lambda e: e.time_range.start)
    if "--gaps" in sys.argv:
        prev = None
        for e in evs:
            if prev is not None:
                gap = (e.time_range.start - prev.time_range.end) / 1e3
                if gap > 0.05:
                    print(f"  gap {gap:8.3f} ms before {e.name.split('(')[0][:50]} (after {prev.name.split('(')[0][:40]})")
            prev = e
    agg = defaultdict(lambda: [0, 0.0])
    for ev in prof.events():
        if ev.device_type == torch.autograd.DeviceType.CUDA:
            name = ev.name.split("(")[0][:70]
            agg[name][0] += 1
            agg[name][1] += ev.device_time_total / 1e3
    tot = sum(v[1] for v in agg.values())
    print(f"{op} n={n}: call {wall:.2f} ms (events), kernels sum {tot:.2f} ms, {sum(v[0] for v in agg.values())} launches")
    for name, (c, ms) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"  {ms:9.3f} ms {c:6d}x  {name}")


if __name__ == "__main__":
    main()
