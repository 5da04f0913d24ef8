"""Launch timeline of one library call (torch.profiler / CUPTI activity records, no replay):
start offset, duration and the gap before each kernel.
    python tools/timeline.py L 2048 [reps]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_2307_07611_b200 as P  # noqa: E402


def main():
    op, n = sys.argv[1], int(sys.argv[2])
    dev = torch.device("cuda:0")
    if op in "LU":
        A = torch.empty((n, n), dtype=torch.float64, device=dev)
        synth.device_fill(A, n, uplo=op, diag="signed" if op == "L" else "pos")
        X = torch.empty_like(A)
        f = P.trinv_lower if op == "L" else P.trinv_upper
        fn = lambda: f(A, out=X)  # noqa: E731
    else:
        L = torch.empty((n, n), dtype=torch.float64, device=dev)
        U = torch.empty_like(L)
        synth.device_fill(L, n, uplo="L", diag="one", tag="L")
        synth.device_fill(U, n, uplo="U", diag="pos", tag="U")
        X = torch.empty_like(L)
        fn = lambda: P.inv_from_lu(L, U, unit_l=True, out=X)  # noqa: E731
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    # graph replay: launch overhead of the host out of the picture
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    g.replay(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(20):
        e0.record(); g.replay(); e1.record(); e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    print(f"{op} n={n}: graph replay median {ts[len(ts) // 2] * 1e3:.1f} us, min {ts[0] * 1e3:.1f} us; "
          f"{n ** 3 / 3 / (ts[len(ts) // 2] / 1e3) / 1e12:.2f} TF/s at n^3/3")
    with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
        g.replay(); torch.cuda.synchronize()
    evs = sorted([e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA],
                 key=lambda e: e.time_range.start)
    t0 = evs[0].time_range.start
    prev_end = t0
    busy = 0.0
    for e in evs:
        st, en = e.time_range.start, e.time_range.end
        busy += (en - st)
        print(f"  {st - t0:9.1f} us  dur {en - st:8.1f} us  gap {st - prev_end:6.1f}  {e.name.split('(')[0][:60]}")
        prev_end = max(prev_end, en)
    print(f"  span {prev_end - t0:.1f} us, kernels busy {busy:.1f} us")


if __name__ == "__main__":
    main()
