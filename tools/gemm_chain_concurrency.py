"""Concurrency check of the DMMA GEMM engine when each product reads the previous product's output
(two CUDA streams, disjoint buffers): chains C1 = A B, C2 = C1 B, ... per stream, against cuBLAS.
    python tools/gemm_chain_concurrency.py [reps]"""
import sys

import torch

sys.path.insert(0, '.')
import paper_2307_07611_b200 as P  # noqa: E402

dev = torch.device('cuda:0')
g = torch.Generator(device=dev).manual_seed(1)
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
for n in (256, 512, 1024, 2048):
    L = 6
    A = [torch.rand((n, n), dtype=torch.float64, device=dev, generator=g) / n for _ in range(2)]
    B = [torch.rand((n, n), dtype=torch.float64, device=dev, generator=g) for _ in range(2)]
    ref = []
    for k in range(2):
        c, chain = A[k], []
        for _ in range(L):
            c = c @ B[k]
            chain.append(c)
        ref.append(chain)
    ss = [torch.cuda.Stream(), torch.cuda.Stream()]
    for mode in ("serial", "concurrent"):
        bad = 0
        for r in range(reps):
            Cs = [[torch.full_like(A[0], float('nan')) for _ in range(L)] for _ in range(2)]
            torch.cuda.synchronize()
            for step in range(L):
                for k in range(2):
                    with torch.cuda.stream(ss[k] if mode == "concurrent" else ss[0]):
                        P.gemm(A[k] if step == 0 else Cs[k][step - 1], B[k], C=Cs[k][step])
            torch.cuda.synchronize()
            for k in range(2):
                for step in range(L):
                    rf = ref[k][step]
                    if not (((Cs[k][step] - rf).abs().max() / rf.abs().max()).item() < 1e-12):
                        bad += 1
        print(f"n={n} {mode}: {bad} wrong of {reps * 2 * L}", flush=True)
