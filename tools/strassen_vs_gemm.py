"""Stream 0 runs Strassen products (trinv_gemm_strassen), stream 1 runs plain DMMA GEMMs or a
memset loop at the same time; counts wrong Strassen products.  python tools/strassen_vs_gemm.py"""
import sys

import torch

sys.path.insert(0, '.')
import paper_2307_07611_b200 as P  # noqa: E402

dev = torch.device('cuda:0')
g = torch.Generator(device=dev).manual_seed(0)
for other in ("none", "gemm", "memset", "strassen"):
    for n in (1024, 2048):
        k = 4
        As = [torch.rand((n, n), dtype=torch.float64, device=dev, generator=g) for _ in range(k)]
        Bs = [torch.rand((n, n), dtype=torch.float64, device=dev, generator=g) for _ in range(k)]
        ref = [a @ b for a, b in zip(As, Bs)]
        wsb = P.lib().trinv_strassen_workspace_bytes(n)
        ws = [torch.empty(wsb, dtype=torch.uint8, device=dev) for _ in range(k + 4)]
        X = torch.rand((n, n), dtype=torch.float64, device=dev, generator=g)
        Y = [torch.empty_like(X) for _ in range(4)]
        big = torch.empty(1 << 28, dtype=torch.uint8, device=dev)
        s0, s1 = torch.cuda.Stream(), torch.cuda.Stream()
        bad = 0
        for r in range(30):
            Cs = [torch.full_like(As[0], float('nan')) for _ in range(k)]
            torch.cuda.synchronize()
            for i in range(k):
                P.lib().trinv_gemm_strassen(n, As[i].data_ptr(), n, Bs[i].data_ptr(), n, Cs[i].data_ptr(), n,
                                            ws[i].data_ptr(), wsb, s0.cuda_stream)
                with torch.cuda.stream(s1):
                    if other == "gemm":
                        P.gemm(X, X, C=Y[i % 4])
                    elif other == "memset":
                        big.zero_()
                    elif other == "strassen":
                        P.lib().trinv_gemm_strassen(n, X.data_ptr(), n, X.data_ptr(), n, Y[i % 4].data_ptr(), n,
                                                    ws[k + i % 4].data_ptr(), wsb, s1.cuda_stream)
            torch.cuda.synchronize()
            bad += sum(not (((c - rf).abs().max() / rf.abs().max()).item() < 1e-12) for c, rf in zip(Cs, ref))
        print(f"other={other:8s} n={n}: {bad} wrong of {30 * k}", flush=True)
