"""Kernel breakdown and gaps of one dist.trinv_split call on one process (n = 32768)."""
import sys, torch
sys.path.insert(0, ".")
import synth, paper_2307_07611_b200 as P
from paper_2307_07611_b200.dist import trinv_split
from collections import defaultdict
n = 32768
T = torch.empty((n, n), dtype=torch.float64, device="cuda"); synth.device_fill(T, n)
X = trinv_split(T, "L"); torch.cuda.synchronize(); del X
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    X = trinv_split(T, "L"); torch.cuda.synchronize()
agg = defaultdict(lambda: [0, 0.0])
for ev in prof.events():
    if ev.device_type == torch.autograd.DeviceType.CUDA:
        a = agg[ev.name.split("(")[0][:60]]; a[0] += 1; a[1] += ev.device_time_total / 1e3
for k, (c, ms) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:14]:
    print(f"{ms:9.3f} ms {c:5d}x {k}")
evs = sorted([e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA], key=lambda e: e.time_range.start)
prev = None
for e in evs:
    if prev is not None:
        gap = (e.time_range.start - prev.time_range.end) / 1e3
        if gap > 2.0:
            print(f"  gap {gap:8.3f} ms before {e.name.split('(')[0][:50]} (after {prev.name.split('(')[0][:40]})")
    prev = e
print("span", (evs[-1].time_range.end - evs[0].time_range.start) / 1e3, "ms")
agg2 = defaultdict(lambda: [0, 0.0])
for e in evs:
    a = agg2[e.name.split("(")[0][:60]]; a[0] += 1; a[1] += (e.time_range.end - e.time_range.start) / 1e3
for k, (c, ms) in sorted(agg2.items(), key=lambda kv: -kv[1][1])[:10]:
    print(f"span-sum {ms:9.3f} ms {c:5d}x {k}")
