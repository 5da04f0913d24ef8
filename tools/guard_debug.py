"""Scaling-guard check on a BASELINE-style input and its diagonal halves, with the true row /
column maxima for comparison (python tools/guard_debug.py)."""
import sys, torch
sys.path.insert(0, ".")
import synth, paper_2307_07611_b200 as P
n = 32768; h = n // 2
T = torch.empty((n, n), dtype=torch.float64, device="cuda"); synth.device_fill(T, n)
print("engine", P.product_engine(), "min_block", P.product_min_block())
print("T ok", P.int8_scaling_ok(T, "L"))
A = T[:h, :h].contiguous(); B = T[h:, h:].contiguous()
print("A ok", P.int8_scaling_ok(A, "L"), "B ok", P.int8_scaling_ok(B, "L"))
Bd = torch.diagonal(B); print("B diag min/max", Bd.abs().min().item(), Bd.abs().max().item())
rm = B.tril().abs().amax(dim=1); print("B rowmax min/max", rm.min().item(), rm.max().item())
cm = B.tril().abs().amax(dim=0); print("B colmax min/max", cm.min().item(), cm.max().item())
