"""Host-side timing of one large triangular inverse: device time per call (events), host
time spent inside the call, and the GPU idle time between consecutive kernels."""
import sys
import time

import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
import paper_2307_07611_b200 as P  # noqa: E402


def main():
    uplo, n = sys.argv[1], int(sys.argv[2])
    dev = torch.device("cuda:0")
    A = torch.empty((n, n), dtype=torch.float64, device=dev)
    synth.device_fill(A, n, uplo=uplo, diag="pos" if uplo == "U" else "signed")
    X = torch.empty_like(A)
    f = P.trinv_upper if uplo == "U" else P.trinv_lower
    ws = torch.empty(P.workspace_bytes(uplo, n, A, n, X, n), dtype=torch.uint8, device=dev)
    lib = P.lib()
    fn_c = lib.trinv_upper if uplo == "U" else lib.trinv_lower
    import ctypes

    def raw():
        fn_c(n, ctypes.c_void_p(A.data_ptr()), n, ctypes.c_void_p(X.data_ptr()), n, 0,
             ctypes.c_void_p(ws.data_ptr()), ws.numel(), None, ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))

    for name, fn in (("python", lambda: f(A, out=X)), ("c-abi", raw)):
        fn(); torch.cuda.synchronize()
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); t0 = time.perf_counter(); fn(); t1 = time.perf_counter(); e1.record(); e1.synchronize()
            print(f"{name}: device {e0.elapsed_time(e1):8.2f} ms, host in call {1e3 * (t1 - t0):8.2f} ms")
    with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA,
                                            torch.profiler.ProfilerActivity.CPU]) as prof:
        raw(); torch.cuda.synchronize()
    evs = sorted([e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA],
                 key=lambda e: e.time_range.start)
    idle = sum(max(0, b.time_range.start - a.time_range.end) for a, b in zip(evs, evs[1:])) / 1e3
    span = (evs[-1].time_range.end - evs[0].time_range.start) / 1e3
    busy = sum(e.time_range.end - e.time_range.start for e in evs) / 1e3
    print(f"profiled: span {span:.2f} ms, kernels {busy:.2f} ms, idle between kernels {idle:.2f} ms, {len(evs)} events")
    cpu = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CPU]
    agg = {}
    for e in cpu:
        a = agg.setdefault(e.name, [0, 0.0]); a[0] += 1; a[1] += (e.time_range.end - e.time_range.start) / 1e3
    for k, (c, ms) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:12]:
        print(f"  host {ms:9.3f} ms {c:5d}x {k[:70]}")


if __name__ == "__main__":
    main()
