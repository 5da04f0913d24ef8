"""Concurrency check of the Strassen path (two CUDA streams, disjoint buffers): each stream runs
gemm_strassen calls back to back; results against cuBLAS (torch.matmul).  Prints the number of
wrong products per setting.     python tools/strassen_concurrency.py [reps]"""
import sys

import torch

sys.path.insert(0, '.')
import paper_2307_07611_b200 as P  # noqa: E402

dev = torch.device('cuda:0')
g = torch.Generator(device=dev).manual_seed(0)
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
for n in [int(x) for x in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["1024", "2048", "4096"])]:
    k = 4
    As = [torch.rand((n, n), dtype=torch.float64, device=dev, generator=g) for _ in range(k)]
    Bs = [torch.rand((n, n), dtype=torch.float64, device=dev, generator=g) for _ in range(k)]
    ref = [a @ b for a, b in zip(As, Bs)]
    ss = [torch.cuda.Stream(), torch.cuda.Stream()]
    wsb = P.lib().trinv_strassen_workspace_bytes(n)
    GUARD = 64 << 20
    wsfull = [torch.full((wsb + 2 * GUARD,), 0x5A, dtype=torch.uint8, device=dev) for _ in range(k)]
    ws = [w[GUARD:GUARD + wsb] for w in wsfull]
    for mode in ("serial", "concurrent"):
        bad = 0
        for r in range(reps):
            Cs = [torch.full_like(As[0], float('nan')) for _ in range(k)]
            torch.cuda.synchronize()
            for i in range(k):
                st = ss[i % 2] if mode == "concurrent" else ss[0]
                P.lib().trinv_gemm_strassen(n, As[i].data_ptr(), n, Bs[i].data_ptr(), n, Cs[i].data_ptr(), n,
                                            ws[i].data_ptr(), ws[i].numel(), st.cuda_stream)
            torch.cuda.synchronize()
            for i, (c, rf) in enumerate(zip(Cs, ref)):
                if not (((c - rf).abs().max() / rf.abs().max()).item() < 1e-12):
                    bad += 1
                    h = n // 2
                    qe = [((c[a:a + h, b:b + h] - rf[a:a + h, b:b + h]).abs().max() / rf.abs().max()).item()
                          for a in (0, h) for b in (0, h)]
                    if bad <= 3:
                        print(f"   rep {r} product {i} (stream {i % 2}): quadrant errors " + " ".join(f"{x:.1e}" for x in qe))
        gbad = sum(int((w[:GUARD] != 0x5A).sum().item() + (w[GUARD + wsb:] != 0x5A).sum().item()) for w in wsfull)
        print(f"n={n} {mode}: {bad} wrong of {reps * k}; workspace guard bytes changed: {gbad}", flush=True)
