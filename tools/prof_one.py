"""One call of a chosen operation on device-resident synthetic input (for ncu launch lists).

    python tools/prof_one.py L 8192        # trinv_lower n = 8192 (also U, G = inv_from_lu, A = inv_general)
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_2307_07611_b200 as P  # noqa: E402


def main():
    op, n = sys.argv[1], int(sys.argv[2])
    reps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
    dev = torch.device("cuda:0")
    if op in "LU":
        A = torch.empty((n, n), dtype=torch.float64, device=dev)
        synth.device_fill(A, n, uplo=op, diag="signed" if op == "L" else "pos")
        X = torch.empty_like(A)
        fn = (lambda: P.trinv_lower(A, out=X)) if op == "L" else (lambda: P.trinv_upper(A, out=X))
    elif op == "G":
        L = torch.empty((n, n), dtype=torch.float64, device=dev)
        U = torch.empty_like(L)
        synth.device_fill(L, n, uplo="L", diag="unit", tag="L")
        synth.device_fill(U, n, uplo="U", diag="pos", tag="U")
        X = torch.empty_like(L)
        fn = lambda: P.inv_from_lu(L, U, unit_l=True, out=X)  # noqa: E731
    elif op == "A":
        L = torch.empty((n, n), dtype=torch.float64, device=dev)
        U = torch.empty_like(L)
        synth.device_fill(L, n, uplo="L", diag="one", tag="L")
        synth.device_fill(U, n, uplo="U", diag="pos", tag="U")
        A = L @ U
        X = torch.empty_like(A)
        fn = lambda: P.inv_general(A, out=X)  # noqa: E731
    else:
        raise SystemExit(f"unknown op {op}")
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    print("ok")


if __name__ == "__main__":
    main()
