import sys, torch
sys.path.insert(0, '/root/repo')
import paper_2307_07611_b200 as P
n = int(sys.argv[1]); dg = int(sys.argv[2])
A = torch.rand((n, n), dtype=torch.float64, device="cuda") * 2 - 1
B = torch.rand((n, n), dtype=torch.float64, device="cuda") * 2 - 1
P.gemm_oz(A, B, digits=dg); torch.cuda.synchronize()
