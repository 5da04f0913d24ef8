import sys, torch, ctypes
sys.path.insert(0, '.')
import synth, paper_2307_07611_b200 as P
B, n = 131072, 32
A = synth.host(n, batch=B)
h_in = torch.from_numpy(A).pin_memory(); h_out = torch.empty_like(h_in).pin_memory()
dev = torch.device('cuda:0'); s = torch.cuda.current_stream()
for chunk in (2048, 4096, 8192, 16384, 32768):
    ws = torch.empty(P.lib().trinv_batched_host_workspace_bytes(n, chunk), dtype=torch.uint8, device=dev)
    def step():
        st = P.lib().trinv_batched_host(b"L", n, B, ctypes.c_void_p(h_in.data_ptr()), ctypes.c_void_p(h_out.data_ptr()), 0, chunk,
                                        ctypes.c_void_p(ws.data_ptr()), ws.numel(), None, ctypes.c_void_p(s.cuda_stream))
        assert st == 0
    step(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(5): step()
    e1.record(s); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(f"chunk {chunk:6d}: {ms:.3f} ms per step, {B / ms * 1e3:.3e} inverses/s, {B * 8192 / ms / 1e6:.1f} GB/s each way")
    del ws
