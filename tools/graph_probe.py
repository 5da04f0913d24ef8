"""Per-call device time of a small trinv when R calls are captured in one CUDA graph
(replayed once), vs one call per graph replay: separates kernel + launch latency on the
device from host-side replay overhead.   python tools/graph_probe.py [n=64] [R=100]"""
import sys
import time

import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
import paper_2307_07611_b200 as P  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
R = int(sys.argv[2]) if len(sys.argv) > 2 else 100
dev = torch.device("cuda:0")
A = torch.empty((n, n), dtype=torch.float64, device=dev)
synth.device_fill(A, n, diag="signed")
X = torch.empty_like(A)
P.trinv_lower(A, out=X); torch.cuda.synchronize()
for reps in (1, R):
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(reps):
            P.trinv_lower(A, out=X)
    g.replay(); torch.cuda.synchronize()
    N = max(1, 2000 // reps)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    for _ in range(N):
        g.replay()
    e1.record(); e1.synchronize()
    t1 = time.perf_counter()
    print(f"n={n}: {reps:4d} calls per graph: {e0.elapsed_time(e1) * 1e3 / (N * reps):7.2f} us per call (device), "
          f"{(t1 - t0) * 1e6 / N:8.2f} us host per replay")
