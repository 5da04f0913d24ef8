import sys, torch
sys.path.insert(0, ".")
import synth, paper_2307_07611_b200 as P
dev = torch.device("cuda:0")
for n in (64, 128):
    A = torch.empty((n, n), dtype=torch.float64, device=dev)
    synth.device_fill(A, n, diag="signed")
    X = torch.empty_like(A)
    for i in range(4):
        P.trinv_lower(A, out=X); torch.cuda.synchronize()
