"""Device / host time per dist.trinv_split call on one process (n = 32768)."""
import sys, time, torch
sys.path.insert(0, ".")
import synth, paper_2307_07611_b200 as P
from paper_2307_07611_b200.dist import trinv_split
n = 32768
T = torch.empty((n, n), dtype=torch.float64, device="cuda"); synth.device_fill(T, n)
for i in range(4):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter(); e0.record()
    X = trinv_split(T, "L")
    e1.record(); t1 = time.perf_counter(); e1.synchronize(); t2 = time.perf_counter()
    print(f"call {i}: device {e0.elapsed_time(e1):.1f} ms, host enqueue {1e3*(t1-t0):.1f} ms, total {1e3*(t2-t0):.1f} ms, "
          f"reserved {torch.cuda.memory_reserved()/1e9:.1f} GB", flush=True)
    del X
