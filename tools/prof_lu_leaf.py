"""One Crout leaf (lu_leaf_kernel<128>) per call, for ncu / timing:
    python tools/prof_lu_leaf.py [n=128] [reps=20]"""
import sys

import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
import paper_2307_07611_b200 as P  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
dev = torch.device("cuda:0")
L = torch.empty((n, n), dtype=torch.float64, device=dev)
U = torch.empty_like(L)
synth.device_fill(L, n, seed=5, tag="L", diag="pos")
synth.device_fill(U, n, seed=5, tag="U", uplo="U", diag="one")
A0 = L @ U
A = A0.clone()
P.lu_crout(A); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    P.lu_crout(A)  # refactors the (already factored) matrix: same work per call
e1.record(); e1.synchronize()
print(f"lu_crout n={n}: {e0.elapsed_time(e1) / reps * 1e3:.1f} us per call")
A = A0.clone(); P.lu_crout(A)
print("max |L - L_ref| =", (torch.tril(A) - L).abs().max().item())
