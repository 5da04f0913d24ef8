"""DMMA GEMM engine rates for the product shapes of inv_general / inv_from_lu (dense and one
triangular operand), CUDA events around graph-free calls, median of 5 after 2 warm-up:
    python tools/gemm_probe.py            (TRINV_GEMM_W128 / TRINV_GEMM_WAVES select the tile)"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2307_07611_b200 as P  # noqa: E402


def main():
    dev = torch.device("cuda:0")
    g = torch.Generator(device=dev).manual_seed(0)
    for n in (2048, 4096, 8192):
        A = torch.rand((n, n), dtype=torch.float64, device=dev, generator=g)
        B = torch.rand((n, n), dtype=torch.float64, device=dev, generator=g)
        C = torch.empty_like(A)
        for sa, sb in (("N", "N"), ("L", "N"), ("N", "U")):
            Au = A.tril() if sa == "L" else A
            Bu = B.triu() if sb == "U" else B
            fl = 2.0 * n ** 3 / (2 if (sa != "N" or sb != "N") else 1)
            ts = []
            for i in range(7):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                P.gemm(Au, Bu, C=C, struct_a=sa, struct_b=sb)
                e1.record()
                e1.synchronize()
                if i >= 2:
                    ts.append(e0.elapsed_time(e1))
            ts.sort()
            ms = ts[len(ts) // 2]
            print(f"n={n:5d} {sa}{sb}: {ms:8.3f} ms  {fl / ms / 1e9:6.2f} TF/s")


if __name__ == "__main__":
    main()
