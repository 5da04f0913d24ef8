"""Timing of configs 3 / 4 / 5 single calls (CUDA events, median of 3 after 1 warm-up):
    python tools/trmm_time.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_2307_07611_b200 as P  # noqa: E402


def t(fn, reps=3):
    fn(); torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    return sorted(ts)[len(ts) // 2]


dev = "cuda:0"
n = 32768
U = torch.empty((n, n), dtype=torch.float64, device=dev)
synth.device_fill(U, n, uplo="U", diag="pos")
X = torch.empty_like(U)
print(f"config3 U n=32768: {t(lambda: P.trinv_upper(U, out=X)):.2f} ms")
del U, X
n = 16384
L = torch.empty((n, n), dtype=torch.float64, device=dev)
Uf = torch.empty_like(L)
synth.device_fill(L, n, uplo="L", diag="one", tag="L")
synth.device_fill(Uf, n, uplo="U", diag="pos", tag="U")
X = torch.empty_like(L)
print(f"config4 inv_from_lu n=16384: {t(lambda: P.inv_from_lu(L, Uf, unit_l=True, out=X)):.2f} ms")
A = L @ Uf
print(f"config5 inv_general n=16384: {t(lambda: P.inv_general(A, out=X)):.2f} ms")
