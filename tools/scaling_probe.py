"""Accuracy of the product engines on power-of-two row / column scaled triangular matrices:
inv(D1 T D2) vs D2^-1 inv(T) D1^-1 (both computed by the library), for scalings 2^k with
|k| <= R.  Prints the largest entry error mapped back to the unscaled problem.
    python tools/scaling_probe.py"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
import paper_2307_07611_b200 as P  # noqa: E402

n = 1024
T = synth.host(n, seed=9, diag="signed")
for engine in ("dmma", "int8crt"):
    P.set_product_engine(engine, min_block=256)
    Y = P.trinv_lower(torch.from_numpy(T).cuda()).cpu().numpy()
    for R in (0, 2, 4, 8, 16, 30, 60):
        rng = np.random.default_rng(11)
        k1 = rng.integers(-R, R + 1, n); k2 = rng.integers(-R, R + 1, n)
        S = np.ldexp(np.ldexp(T, k1[:, None]), k2[None, :])
        X = P.trinv_lower(torch.from_numpy(S).cuda()).cpu().numpy()
        Z = np.ldexp(np.ldexp(Y, -k2[:, None]), -k1[None, :])
        E = np.ldexp(np.ldexp(np.abs(X - Z), k2[:, None]), k1[None, :])
        print(f"{engine:8s} |k| <= {R:2d}: max error (unscaled units) {E.max():.3e}, bitwise equal {np.array_equal(X, Z)}")
P.set_product_engine()
