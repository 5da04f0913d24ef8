"""Normwise error of gemm_oz(digits=0) on shapes the CTA-pair kernel takes (run with
TRINV_OZ2_PAIR=256 to route them through it)."""
import sys, numpy as np, torch
sys.path.insert(0, ".")
import paper_2307_07611_b200 as P
rng = np.random.default_rng(1)
for (M, N, K, sa, sb) in [(256, 256, 128, "N", "N"), (512, 512, 512, "N", "N"), (1024, 512, 768, "L", "N"), (512, 1024, 1024, "N", "L"), (1024, 1024, 1024, "U", "N"), (1024, 1024, 1024, "N", "U")]:
    A = rng.uniform(-1, 1, (M, K)); B = rng.uniform(-1, 1, (K, N))
    if sa == "L": A = np.tril(A)
    if sa == "U": A = np.triu(A)
    if sb == "L": B = np.tril(B)
    if sb == "U": B = np.triu(B)
    C = P.gemm_oz(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), digits=0, struct_a=sa, struct_b=sb).cpu().numpy()
    R = A @ B
    sc = np.abs(A).max(1, keepdims=True) * np.abs(B).max(0, keepdims=True) * K
    print(M, N, K, sa, sb, "err", float(np.max(np.abs(C - R) / sc)), flush=True)
