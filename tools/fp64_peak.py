"""FP64 peak measurement on the B200 box.

Runs tools/fp64_peak (register-only DMMA / DFMA loops) and times cuBLAS DGEMM
(torch.matmul on float64, reference only) best-of-10 and back-to-back ~4 s.
Writes one JSON object to stdout.
"""
import json, subprocess, sys, time, os
import torch

here = os.path.dirname(os.path.abspath(__file__))
res = json.loads(subprocess.check_output([os.path.join(here, "fp64_peak")]).decode())
dev = torch.device("cuda:0")
for n in (8192, 16384):
    a = torch.randn(n, n, dtype=torch.float64, device=dev)
    b = torch.randn(n, n, dtype=torch.float64, device=dev)
    for _ in range(2):
        torch.matmul(a, b)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e30
    for _ in range(5 if n == 16384 else 10):
        e0.record(); torch.matmul(a, b); e1.record(); e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    res[f"cublas_dgemm_{n}_tflops_best"] = 2 * n**3 / (best * 1e-3) / 1e12
    if n == 8192:
        t0 = time.time(); k = 0
        e0.record()
        while time.time() - t0 < 4.0:
            torch.matmul(a, b); k += 1
            if k % 4 == 0:
                torch.cuda.synchronize()
        e1.record(); e1.synchronize()
        res[f"cublas_dgemm_{n}_tflops_sustained"] = 2 * n**3 * k / (e0.elapsed_time(e1) * 1e-3) / 1e12
    del a, b
res["torch"] = torch.__version__
print(json.dumps(res))
