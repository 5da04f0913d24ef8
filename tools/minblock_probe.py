"""INT8 CRT threshold probe: device time of the config 2 / 3 / 4 / 5 calls with the modular
engine taking blocks >= min_block (the library default 4096) vs 2048 / 8192.
Usage: python tools/minblock_probe.py"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
import paper_2307_07611_b200 as P

dev = "cuda:0"


def timed(fn, reps=5):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = []
    for _ in range(reps):
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        best.append(e0.elapsed_time(e1))
    best.sort()
    return best[len(best) // 2]


cases = []
T8 = torch.empty((8192, 8192), dtype=torch.float64, device=dev); synth.device_fill(T8, 8192, diag="signed")
cases.append(("c2 trinv_lower n=8192", lambda: P.trinv_lower(T8)))
T32 = torch.empty((32768, 32768), dtype=torch.float64, device=dev); synth.device_fill(T32, 32768, uplo="U", diag="pos")
cases.append(("c3 trinv_upper n=32768", lambda: P.trinv_upper(T32)))
n = 16384
Lm = torch.empty((n, n), dtype=torch.float64, device=dev); synth.device_fill(Lm, n, tag="L", diag="one")
Um = torch.empty((n, n), dtype=torch.float64, device=dev); synth.device_fill(Um, n, tag="U", uplo="U", diag="pos")
X16 = torch.empty((n, n), dtype=torch.float64, device=dev)
cases.append(("c4 inv_from_lu n=16384", lambda: P.inv_from_lu(Lm, Um, unit_l=True, out=X16)))
Lg = torch.empty((n, n), dtype=torch.float64, device=dev); synth.device_fill(Lg, n, seed=5, tag="L", diag="pos")
Ug = torch.empty((n, n), dtype=torch.float64, device=dev); synth.device_fill(Ug, n, seed=5, tag="U", uplo="U", diag="one")
A16 = Lg @ Ug
del Lg, Ug
cases.append(("c5 inv_general n=16384", lambda: P.inv_general(A16, out=X16)))
for name, fn in cases:
    for mb in (1024, 2048, 4096):
        P.set_product_engine("int8crt", min_block=mb)
        print(f"{name:28s} min_block={mb:5d}  {timed(fn):9.3f} ms", flush=True)
P.set_product_engine()
