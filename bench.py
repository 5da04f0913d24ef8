#!/usr/bin/env python
"""bench.py — throughput of the FP64 triangular-inverse hot path on B200.

Default workload (BASELINE.json configs[1], the metric's batched case):
131072 independent lower-triangular 32x32 fp64 matrices, matrix b seeded by
its global index b, row-major contiguous, inverted by trinv_batched (one
launch per step).  `value` = matrices inverted by all ranks / max-over-ranks
device time, inverses/s.  At N = 1 the same line carries an "fp64" block:
BASELINE configs 2, 3 and 4 (the metric's FP64 half) timed in the same run on
the DMMA engine, with their fraction of the FP64 tensor-core peak measured
live (trinv_probe_dmma_tflops).  --config 0|2|3|4 runs a single-matrix
configuration as the main line instead.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl reference]

Multi-GPU: launched by torchrun, one rank per GPU; config 1 is sharded by
batch as BASELINE states ("sharded by batch over 1/2/4/8 GPUs", strong
scaling: rank r inverts dist.shard_range(131072, N, r), 131072/N matrices,
generated locally from their global indices); no collective touches the
timed data path.  After the timed region the shards are gathered on rank 0
(NCCL gather, timed apart with its NVLink roofline) and rank 0 checks that the
gathered batch equals, bit for bit, its own single-GPU inversion of all 131072
matrices (sharding invariance, SURVEY P-l).  --scaling weak gives every rank
its own 131072 matrices instead.

--impl reference times the CPU oracle (oracle/, test infrastructure) on the
host cores on a bounded sample of the same workload; it is the tier's
reference arm, not the product.
"""
import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "fp64 trinv GFLOP/s (n^3/3) and % FP64 TC peak; batched 32x32 inverses/s"
FP64_PEAK_FALLBACK = 37.1  # TF/s, measured register-only DMMA peak (profiles/fp64_peaks_r01.json)
HBM_FALLBACK = 6550.4      # GB/s, MEASURED_PEAKS.json at round start
BATCH = 131072

CONFIGS = {
    0: dict(workload="config0: single fp64 lower n=64, seed 0", kind="L", n=64, diag="signed"),
    1: dict(workload="config1: batch 131072 x fp64 lower 32x32, seed b per matrix", kind="B", n=32),
    2: dict(workload="config2: single fp64 lower n=8192 (128-wide diagonal blocks: 16-wide leaves + in-CTA "
                     "DMMA merges, then beta=2 levels b=128..4096)", kind="L", n=8192, diag="signed"),
    3: dict(workload="config3: single fp64 upper n=32768", kind="U", n=32768, diag="pos"),
    4: dict(workload="config4: inv_from_lu n=16384, L unit", kind="G", n=16384),
    5: dict(workload="NEXT f2: general fp64 inverse from A, n=16384 (A = L U with U unit; Crout LU without "
                     "pivoting + U^-1 L^-1), 2n^3 flops", kind="A", n=16384),
    6: dict(workload="NEXT f1: one fp64 lower n=32768 split across the ranks (diagonal halves on ranks 0/1, "
                     "2G balanced column panels of the off-diagonal block, gather on rank 0)", kind="S", n=32768,
            diag="signed"),
}


def n_of(cfg):
    return cfg.get("n", 0)


def peaks():
    hbm, src_h = HBM_FALLBACK, "fallback"
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        try:
            hbm, src_h = float(json.load(open(p))["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs"
        except Exception:
            pass
    fp64, src_f = FP64_PEAK_FALLBACK, "fallback"
    q = os.path.join(ROOT, "profiles", "fp64_peaks_r01.json")
    if os.path.exists(q):
        try:
            d = json.load(open(q))
            fp64, src_f = float(d["dmma_tflops_sustained"]), "profiles/fp64_peaks_r01.json dmma_tflops_sustained"
        except Exception:
            pass
    return hbm, src_h, fp64, src_f


def _bf16_sustained():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        return float(json.load(open(p))["bf16_tflops_sustained"])
    except Exception:
        return 1363.9


I8_PER_BF16_SUSTAINED = _bf16_sustained()  # TF/s; x 2 = int8 TOPS (nominal 4.5 POPS / 2.25 PF dense ratio)


def ncu_traffic(kernel_key):
    """dram bytes (read+write) per launch from the committed ncu --set full summary, if any."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(p):
        return None
    try:
        return json.load(open(p)).get(kernel_key)
    except Exception:
        return None


class ClockSampler:
    """NVML SM-clock / throttle-reason sampler running during the timed region."""

    REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
               "sw_power_cap": 0x4, "hw_power_brake_slowdown": 0x80}

    def __init__(self, index, period=0.0001):
        self.index, self.period = index, period
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        self._t = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for name, bit in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.nv is not None:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": 0}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# ----------------------------------------------------------------------------- reference arm
def run_reference(args):
    world, rank, _ = dist_setup()
    if rank != 0:
        return  # the oracle arm runs on rank 0 only
    import numpy as np
    import oracle
    import synth
    cfg = CONFIGS[args.config]
    # the other ranks exit at once: rank 0 runs the oracle on every host core it may use (torchrun
    # sets OMP_NUM_THREADS=1 per process); `cores` is the OpenMP thread count actually used
    oracle.set_threads(len(os.sched_getaffinity(0)))
    cores = oracle.max_threads()
    if cfg["kind"] == "B":
        sample = BATCH  # the whole 131072-matrix batch per step (about 0.1-0.5 s on the host cores)
        A = synth.host(32, batch=sample)
        def step():
            oracle.crit_batched(A)
        unit, work, what = "inverses/s", sample, f"all {sample} config-1 matrices per step, OpenMP over matrices"
    elif cfg["kind"] in ("A",):
        m = 1024
        Lg = synth.host(m, seed=5, tag="L", diag="pos"); Ug = synth.host(m, seed=5, tag="U", uplo="U", diag="one")
        Am = Lg @ Ug
        def step():
            oracle.inv_general(Am)
        unit, work, what = "GFLOP/s", 2 * m ** 3 / 1e9, f"SKUL + S K at n={m} per step (n={cfg['n']} takes hours)"
    else:
        n = cfg["n"]
        cols = np.arange(0, n, max(1, n // 64))[:64]
        if cfg["kind"] == "G":
            L = synth.host(n, tag="L", diag="one")
            U = synth.host(n, tag="U", uplo="U", diag="pos")
            def step():
                oracle.lu_columns(L, U, cols, unit_l=True)
            cost = lambda j: (n - j) ** 2 + n ** 2  # noqa: E731
            total_flops = 4 * n ** 3 / 3
        else:
            kind = "L" if cfg["kind"] == "S" else cfg["kind"]
            T = synth.host(n, uplo=kind, diag=cfg["diag"])
            def step():
                oracle.columns(T, kind, cols)
            cost = (lambda j: (n - j) ** 2) if kind == "L" else (lambda j: j ** 2)  # noqa: E731
            total_flops = n ** 3 / 3
        frac = sum(cost(j) for j in cols) / sum(cost(j) for j in range(n))
        work = total_flops * frac / 1e9
        unit, what = "GFLOP/s", f"{len(cols)} columns per step (extrapolated by the column cost model)"
    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    dt = (time.perf_counter() - t0) / args.steps
    value = work / dt
    line = {"metric": METRIC, "value": value, "unit": unit, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True,
            "scaling": "strong" if cfg["kind"] == "B" else "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
            "config": {"workload": cfg["workload"], "n": cfg["n"]},
            "cpu_baseline": {"value": value, "unit": unit, "cores": cores, "kind": "oracle", "sample": what},
            "e2e": {"value": value, "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- CPU baseline leg
def one_thread(fn):
    """Seconds of fn() with the oracle's OpenMP loops on one thread (restored after)."""
    import oracle
    prev = oracle.max_threads()
    oracle.set_threads(1)
    try:
        fn()
        t0 = time.perf_counter()
        fn()
        return time.perf_counter() - t0
    finally:
        oracle.set_threads(prev)


def cpu_baseline(cfg):
    import numpy as np
    import oracle
    import synth
    cores = oracle.max_threads()  # the OpenMP threads the oracle's loops use in this process
    if cfg["kind"] == "B":
        sample = 32768
        A = synth.host(32, batch=sample)
        oracle.crit_batched(A[:1024])
        t0 = time.perf_counter(); reps = 0
        while True:
            oracle.crit_batched(A); reps += 1
            if time.perf_counter() - t0 > 2.0:
                break
        dt = (time.perf_counter() - t0) / reps
        t1 = one_thread(lambda: oracle.crit_batched(A[:4096]))
        return {"value": sample / dt, "unit": "inverses/s", "cores": cores, "kind": "oracle",
                "sample": f"{sample} of the 131072 config-1 matrices x {reps} reps, OpenMP over matrices",
                "value_1thread": 4096 / t1, "sample_1thread": "4096 of the config-1 matrices, 1 OpenMP thread"}
    n = cfg["n"]
    if cfg["kind"] == "A":  # SKUL oracle (O(n^3)) on a smaller order, GFLOP/s at 2n^3
        m = 1024
        Lg = synth.host(m, seed=5, tag="L", diag="pos"); Ug = synth.host(m, seed=5, tag="U", uplo="U", diag="one")
        A = Lg @ Ug
        t0 = time.perf_counter(); oracle.inv_general(A)
        dt = time.perf_counter() - t0
        return {"value": 2 * m ** 3 / dt / 1e9, "unit": "GFLOP/s", "cores": cores, "kind": "oracle",
                "sample": f"SKUL + S K at n={m} (the n={n} workload would take hours on the host)"}
    if n <= 2048:
        uplo = "L" if cfg["kind"] != "U" else "U"
        T = synth.host(n, uplo=uplo, diag=cfg.get("diag", "signed"))
        reps = 200 if n <= 128 else 1
        t0 = time.perf_counter()
        for _ in range(reps):
            oracle.trinv(T, uplo)
        dt = (time.perf_counter() - t0) / reps
        t1 = one_thread(lambda: [oracle.trinv(T, uplo) for _ in range(reps)]) / reps
        return {"value": n ** 3 / 3 / dt / 1e9, "unit": "GFLOP/s", "cores": cores, "kind": "oracle",
                "sample": f"full inverse n={n} x {reps}", "value_1thread": n ** 3 / 3 / t1 / 1e9,
                "us_per_call": dt * 1e6, "us_per_call_1thread": t1 * 1e6}
    cols = np.arange(0, n, n // 16)[:16]
    if cfg["kind"] == "G":
        L = synth.host(n, tag="L", diag="one"); U = synth.host(n, tag="U", uplo="U", diag="pos")
        t0 = time.perf_counter(); oracle.lu_columns(L, U, cols)
        dt = time.perf_counter() - t0
        cost = lambda j: (n - j) ** 2 + n ** 2  # noqa: E731
        total = 4 * n ** 3 / 3
    else:
        kind = "L" if cfg["kind"] == "S" else cfg["kind"]
        T = synth.host(n, uplo=kind, diag=cfg["diag"])
        t0 = time.perf_counter(); oracle.columns(T, kind, cols)
        dt = time.perf_counter() - t0
        cost = (lambda j: (n - j) ** 2) if kind == "L" else (lambda j: j ** 2)  # noqa: E731
        total = n ** 3 / 3
    frac = sum(cost(j) for j in cols) / sum(cost(j) for j in range(n))
    return {"value": total * frac / dt / 1e9, "unit": "GFLOP/s", "cores": cores, "kind": "oracle",
            "sample": f"{len(cols)} sampled columns, extrapolated to the full inverse by the column cost model"}


# ----------------------------------------------------------------------------- config 1 at N > 1
NVLINK_PEER_GBS = 770.0  # measured peer copy per direction (B200_PROFILING.md); 900 nominal


def gather_and_check(X, count, strong, world, rank, dev, stream, backend, n, barrier, max_over_ranks, P, torch,
                     dist):
    """Gather every rank's shard on rank 0 (NCCL gather = one send per rank into rank 0), timed
    apart from the throughput with its NVLink roofline (rank 0's ingress bytes / the measured
    peer-copy bandwidth), then rank 0 inverts the whole 131072-matrix batch itself and compares
    the gathered result bit for bit (sharding invariance, SURVEY P-l)."""
    import hashlib
    import synth
    nccl = backend == "nccl"
    send = X if nccl else X.cpu()
    recv = [torch.empty_like(send) for _ in range(world)] if rank == 0 else None
    for _ in range(2):  # warm the communicator
        dist.gather(send, recv, dst=0)
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record(stream)
    dist.gather(send, recv, dst=0)
    e1.record(stream)
    barrier()
    wall = time.perf_counter() - t0
    g_ms = max_over_ranks(e0.elapsed_time(e1) if nccl else wall * 1e3)
    ingress = (world - 1) * count * n * n * 8
    out = {"op": "dist.gather to rank 0" + (" (NCCL)" if nccl else f" ({backend}, host-staged)"),
           "ms": g_ms, "rank0_ingress_bytes": ingress,
           "achieved_gbs": ingress / (g_ms / 1e3) / 1e9 if g_ms > 0 else None,
           "peak_gbs": NVLINK_PEER_GBS, "peak_source": "B200_PROFILING.md measured peer copy per direction",
           "frac": ingress / (g_ms / 1e3) / 1e9 / NVLINK_PEER_GBS if g_ms > 0 else None,
           "in_throughput": False}
    if rank == 0 and strong:
        G = torch.cat([r.to(dev) for r in recv], dim=0)
        Af = torch.empty((BATCH, n, n), dtype=torch.float64, device=dev)
        synth.device_fill(Af, n, b0=0)
        Xf = P.trinv_batched(Af, "L")
        torch.cuda.synchronize()
        h = lambda t: hashlib.sha256(t.cpu().numpy().tobytes()).hexdigest()[:16]  # noqa: E731
        hg, h1 = h(G), h(Xf)
        out.update({"hash_gathered": hg, "hash_g1": h1, "hash_equal_g1": hg == h1,
                    "hash_note": "sha256 of the 131072 x 32 x 32 fp64 result: gathered shards vs one rank "
                                 "inverting the whole batch"})
        del G, Af, Xf
    return out


# ----------------------------------------------------------------------------- fp64 block (N = 1)
def fp64_block(args, dev, stream, P, synth, torch, barrier):
    """BASELINE configs 2, 3, 4 on the default DMMA engine in the same run: GFLOP/s (n^3/3 per
    triangular inverse, 4n^3/3 for inv_from_lu) and the fraction of the FP64 tensor-core peak
    measured live (register-only DMMA loop) before and after the block."""
    peak0 = P.lib().trinv_probe_dmma_tflops(200.0, ctypes_stream(stream))
    out = {"engine": P.product_engine(), "configs": {}}
    W = max(3, args.warmup)
    for c in (2, 3, 4):
        cfg = CONFIGS[c]
        n = cfg["n"]
        if cfg["kind"] == "G":
            Lm = torch.empty((n, n), dtype=torch.float64, device=dev)
            Um = torch.empty((n, n), dtype=torch.float64, device=dev)
            synth.device_fill(Lm, n, tag="L", diag="one")
            synth.device_fill(Um, n, tag="U", uplo="U", diag="pos")
            X = torch.empty((n, n), dtype=torch.float64, device=dev)
            step = lambda: P.inv_from_lu(Lm, Um, unit_l=True, out=X)  # noqa: E731
            flops = 4 * n ** 3 / 3
        else:
            A = torch.empty((n, n), dtype=torch.float64, device=dev)
            synth.device_fill(A, n, uplo=cfg["kind"], diag=cfg["diag"])
            X = torch.empty((n, n), dtype=torch.float64, device=dev)
            f = P.trinv_lower if cfg["kind"] == "L" else P.trinv_upper
            step = lambda: f(A, out=X)  # noqa: E731
            flops = n ** 3 / 3
        for _ in range(W):
            step()
        barrier()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.fp64_steps + 1)]
        with ClockSampler(dev.index) as clk:
            ev[0].record(stream)
            for i in range(args.fp64_steps):
                step()
                ev[i + 1].record(stream)
            barrier()
        ms = [ev[i].elapsed_time(ev[i + 1]) for i in range(args.fp64_steps)]
        med = statistics.median(ms)
        tf = flops / (med / 1e3) / 1e12
        out["configs"][f"config{c}"] = {
            "workload": cfg["workload"], "n": n, "flops_per_call": flops,
            "ms": {"median": med, "min": min(ms), "max": max(ms)}, "steps": args.fp64_steps, "warmup": W,
            "gflops": tf * 1e3, "clocks": clk.summary()}
        del X
        if cfg["kind"] == "G":
            del Lm, Um
        else:
            del A
        torch.cuda.empty_cache()
    peak1 = P.lib().trinv_probe_dmma_tflops(200.0, ctypes_stream(stream))
    peak = max(peak0, peak1)
    out["fp64_tc_peak"] = {"tflops": peak, "before": peak0, "after": peak1,
                           "source": "trinv_probe_dmma_tflops: register-only mma.sync m8n8k4 f64 (DMMA.8x8x4) "
                                     "loop on all SMs, measured in this run (max of before / after the block)"}
    for v in out["configs"].values():
        v["frac_of_fp64_tc_peak"] = v["gflops"] / 1e3 / peak if peak > 0 else None
    return out


def ctypes_stream(stream):
    import ctypes
    return ctypes.c_void_p(stream.cuda_stream)


# ----------------------------------------------------------------------------- GPU arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", type=int, default=1, choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--no-graph", action="store_true", help="never replay steps from a CUDA graph")
    ap.add_argument("--products", default="dmma", choices=["dmma", "int8crt"],
                    help="engine for the level products: FP64 DMMA for every level (dmma, default) or the opt-in "
                         "FP64-emulated (Ozaki-II) INT8 tensor-core engine, 16 moduli + CRT, for blocks >= 2048")
    ap.add_argument("--min-block", type=int, default=0, help="INT8 engines: smallest level block (0: 2048)")
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"],
                    help="config 1 at N > 1: shard the 131072-matrix batch over the ranks (strong, BASELINE) "
                         "or give every rank its own 131072 matrices (weak)")
    ap.add_argument("--no-fp64", action="store_true", help="config 1 at N = 1: skip the FP64 configs 2-4 block")
    ap.add_argument("--fp64-steps", type=int, default=3, help="timed steps per FP64 config of the fp64 block")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    assert args.warmup >= 3 or os.environ.get("BENCH_ALLOW_SHORT"), "timing rules need >= 3 warm-up steps"

    import torch
    import torch.distributed as dist
    import synth
    import paper_2307_07611_b200 as P

    world, rank, local = dist_setup()
    # BENCH_DIST_BACKEND=gloo + BENCH_ONE_GPU=1 exercise the multi-rank logic on a single GPU
    # (test only: ranks never wait on each other inside a kernel).
    backend = os.environ.get("BENCH_DIST_BACKEND", "nccl")
    dev_index = 0 if (world == 1 or os.environ.get("BENCH_ONE_GPU")) else local
    dev = torch.device("cuda", dev_index)
    if world > 1:
        torch.cuda.set_device(dev)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    torch.cuda.set_device(dev)
    stream = torch.cuda.current_stream()
    cfg = CONFIGS[args.config]
    hbm_peak, hbm_src, fp64_peak, fp64_src = peaks()
    mb = args.min_block or 2048
    P.set_product_engine(args.products, min_block=mb)
    if cfg["kind"] not in ("B",) and n_of(cfg) > 128:
        if args.products == "dmma":
            cfg = dict(cfg, workload=cfg["workload"] + " [FP64 DMMA products]")
        else:
            desc = "16 moduli + CRT"
            cfg = dict(cfg, workload=cfg["workload"] + f" [products of blocks >= {mb} on the INT8 tensor cores "
                                                       f"({desc}), smaller ones on FP64 DMMA]")

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev if backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    n = cfg["n"]
    strong = cfg["kind"] == "B" and args.scaling == "strong"
    if cfg["kind"] == "B":
        from paper_2307_07611_b200.dist import shard_range
        b0, B = shard_range(BATCH, world, rank) if strong else (rank * BATCH, BATCH)
        A = torch.empty((B, n, n), dtype=torch.float64, device=dev)
        synth.device_fill(A, n, b0=b0)  # matrix b seeded by its global index (shard-invariant)
        X = torch.empty_like(A)
        def step():
            P.trinv_batched(A, "L", out=X)
        units_per_rank, unit = B, "inverses/s"
        total_units = BATCH if strong else BATCH * world
        algo_bytes_per_launch = B * (n * (n + 1) / 2 + n * n) * 8  # triangle in + full matrix out
        flops_per_step = B * n ** 3 / 3
    else:
        if cfg["kind"] == "S":
            from paper_2307_07611_b200.dist import trinv_split, trinv_split_p2p
            # BENCH_SPLIT=p2p: the broadcast / gather fused into the kernels over peer memory
            split = trinv_split_p2p if os.environ.get("BENCH_SPLIT") == "p2p" else trinv_split
            cfg = dict(cfg, workload=cfg["workload"] + (" [peer-memory transport]" if split is trinv_split_p2p
                                                        else " [process-group transport]"))
            A = torch.empty((n, n), dtype=torch.float64, device=dev)
            synth.device_fill(A, n, diag=cfg["diag"])  # replicated input on every rank
            X = torch.empty((n, n), dtype=torch.float64, device=dev)
            def step():
                Y = split(A, "L")
                if Y is not None:
                    X.copy_(Y)
            flops_per_step = n ** 3 / 3
        elif cfg["kind"] == "A":
            Lg = torch.empty((n, n), dtype=torch.float64, device=dev)
            Ug = torch.empty_like(Lg)
            synth.device_fill(Lg, n, seed=5, tag="L", diag="pos")
            synth.device_fill(Ug, n, seed=5, tag="U", uplo="U", diag="one")
            A = Lg @ Ug  # input construction (library DGEMM), outside the timed region
            del Lg, Ug
            X = torch.empty((n, n), dtype=torch.float64, device=dev)
            def step():
                P.inv_general(A, out=X)
            flops_per_step = 2 * n ** 3
        elif cfg["kind"] == "G":
            Lm = torch.empty((n, n), dtype=torch.float64, device=dev)
            Um = torch.empty((n, n), dtype=torch.float64, device=dev)
            synth.device_fill(Lm, n, tag="L", diag="one")
            synth.device_fill(Um, n, tag="U", uplo="U", diag="pos")
            X = torch.empty((n, n), dtype=torch.float64, device=dev)
            ws = torch.empty(P.workspace_bytes("G", n, Lm, n, X, n), dtype=torch.uint8, device=dev)
            def step():
                import ctypes
                st = P.lib().inv_from_lu(n, ctypes.c_void_p(Lm.data_ptr()), n, ctypes.c_void_p(Um.data_ptr()), n,
                                         ctypes.c_void_p(X.data_ptr()), n, 1, 0, ctypes.c_void_p(ws.data_ptr()),
                                         ws.numel(), None, ctypes.c_void_p(stream.cuda_stream))
                assert st == 0, P.status_string(st)
            flops_per_step = 4 * n ** 3 / 3
        else:
            A = torch.empty((n, n), dtype=torch.float64, device=dev)
            synth.device_fill(A, n, uplo=cfg["kind"], diag=cfg["diag"])
            X = torch.empty((n, n), dtype=torch.float64, device=dev)
            f = P.trinv_lower if cfg["kind"] == "L" else P.trinv_upper
            def step():
                f(A, out=X)
            flops_per_step = n ** 3 / 3
        units_per_rank, unit = flops_per_step / 1e9, "GFLOP/s"
        if cfg["kind"] == "S":  # one matrix for the whole job (strong scaling): count it once
            units_per_rank /= world

    for _ in range(args.warmup):
        step()
    barrier()
    # ---- timed region: K steps, per-step events on the launching stream ----
    # Small single matrices are launch-latency bound: their steps are replayed from a
    # CUDA graph captured from the same public call (no Python between launches).
    use_graph = cfg["kind"] != "B" and n <= 1024 and not args.no_graph
    graph = None
    if use_graph:
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):  # captured on torch's side stream, replayed on `stream`
            step()
        graph.replay()
        barrier()
        launches_per_step = None
    run = graph.replay if graph is not None else step
    # the timed region carries no per-launch profiling events (they add ~1-3% to the
    # multi-launch configs); the roofline's per-kernel figures come from a separate profiled pass
    P.reset_launch_count()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    with ClockSampler(dev.index) as clk:
        barrier()
        ev[0].record(stream)
        for i in range(args.steps):
            run()
            if graph is None or i == args.steps - 1:  # graph-replayed latency steps: no event between them
                ev[i + 1].record(stream)
        barrier()
    launches = P.launch_count()
    if graph is not None:
        # count the kernels inside one captured step, then scale to the timed steps
        P.reset_launch_count(); step(); barrier()
        launches = P.launch_count() * args.steps
    step_ms = [ev[i].elapsed_time(ev[i + 1]) for i in range(args.steps)] if graph is None else None
    total_ms = ev[0].elapsed_time(ev[-1])
    total_ms = max_over_ranks(total_ms)
    ms_per_step = total_ms / args.steps
    if cfg["kind"] == "B":
        value = total_units * args.steps / (total_ms / 1e3)
    else:
        value = units_per_rank * world * args.steps / (total_ms / 1e3)

    line = {"metric": METRIC, "value": value, "unit": unit, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong" if (cfg["kind"] == "S" or strong) else "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (counter-based SplitMix64, synth/)"}
    conf = {"workload": cfg["workload"], "n": n, "per_rank_units": units_per_rank,
            "l2_policy": "inputs larger than L2 (126 MB)" if (cfg["kind"] == "B" or n >= 4096)
            else "input smaller than L2, not flushed (latency config)",
            "parallelism": f"batch partition x{world}" if cfg["kind"] == "B" else "replicas (single matrix per GPU)"}
    if step_ms:
        line["step_ms_stats"] = {"median": statistics.median(step_ms), "min": min(step_ms), "max": max(step_ms),
                                 "rank": rank}
    if cfg["kind"] == "B":
        conf["batch_per_rank"] = B
        conf["batch_total"] = total_units
        conf["parallelism"] = (f"batch shards of {B} over {world} rank(s) (dist.shard_range)" if strong
                               else f"batch partition x{world}, {BATCH} matrices per rank (weak)")
    elif n > 128:
        conf["arithmetic"] = ("FP64 (DMMA mma.sync) for every level product" if args.products == "dmma" else
                              "FP64 results; level products of blocks >= %d computed exactly in int8 x int8 -> int32 "
                              "on the tcgen05 tensor cores (%s) and reconstructed in FP64, smaller ones on FP64 DMMA"
                              % (mb, "16 moduli + CRT"))
        if cfg["kind"] in ("G", "A") and args.products == "int8crt":
            conf["arithmetic"] += ("; U^-1 L^-1 as its diagonal terms (one elementwise pass) plus the strictly "
                                   "triangular product on the INT8 engine" +
                                   ("; LU products of blocks >= %d on the INT8 engine" % mb if cfg["kind"] == "A" else ""))
    line["config"] = conf

    # ---- roofline of the dominant kernel ----
    if cfg["kind"] == "B":
        avg_ms = statistics.mean(step_ms)  # one launch per step: the leaf kernel
        achieved = algo_bytes_per_launch / (avg_ms / 1e3) / 1e9
        traffic = ncu_traffic("leaf32_tma_kernel")
        traffic_per_launch = traffic * B / BATCH if traffic else None  # the ncu capture is of a 131072 launch
        line["roofline"] = {"bound": "hbm", "kernel": "leaf32_tma_kernel (trinv_batched)", "achieved": achieved,
                            "peak": hbm_peak, "unit": "GB/s", "frac": achieved / hbm_peak,
                            "traffic": traffic_per_launch, "peak_source": hbm_src,
                            "traffic_frac": (traffic_per_launch / (avg_ms / 1e3) / 1e9 / hbm_peak
                                             if traffic_per_launch else None),
                            "traffic_note": "DRAM moves 128-byte lines: the referenced triangle costs 6144 B of "
                                            "reads per matrix (48 lines), not 4224 (tools/sector_probe.cu: 32 B "
                                            "read per line still moves the whole line), so the frac ceiling on "
                                            "the 12416 B algorithmic bytes is 12416 / 14336 = 0.866 at the copy "
                                            "peak; traffic_frac is the same launch on the bytes DRAM moves",
                            "algorithmic_bytes_per_launch": algo_bytes_per_launch,
                            "launch_ms": avg_ms, "fp64_gflops": flops_per_step / (avg_ms / 1e3) / 1e9}
    else:
        # a separate profiled pass of K eager steps (per-launch CUDA events on each kernel's stream,
        # trinv_profile_*): the dominant kernel's device time and algorithmic flops
        P._lib.profile_begin()
        pe0, pe1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        pe0.record(stream)
        for _ in range(args.steps):
            step()
        pe1.record(stream)
        barrier()
        prof_step_ms = pe0.elapsed_time(pe1) / args.steps  # denominator of the *_share_of_step fields
        ms_d, n_d, fl_d, _ = P._lib.profile_read(1)
        ms_l, n_l, fl_l, _ = P._lib.profile_read(0)
        ms_o, n_o, fl_o, ops_o = P._lib.profile_read(2)  # INT8 engine: FP64-equivalent flops, int8 ops
        ms_x, n_x, _, by_x = P._lib.profile_read(3)  # CRT engine's scaling / residue / reconstruction kernels
        P._lib.profile_end()
        achieved = fl_d / (ms_d / 1e3) / 1e12 if ms_d > 0 else 0.0
        if n_o > 0 and ms_o + ms_x >= ms_d:  # the INT8 engine carries the dominant products
            i8_peak = 2.0 * I8_PER_BF16_SUSTAINED
            ach = ops_o / (ms_o / 1e3) / 1e12
            kname = "oz2_gemm_kernel (INT8 tcgen05, 16 moduli + CRT; FP64-emulated, Ozaki-II)"
            line["roofline"] = {"bound": "tensor", "kernel": kname,
                                "achieved": ach, "peak": i8_peak, "unit": "TOPS (int8)", "frac": ach / i8_peak,
                                "traffic": ncu_traffic("oz2_gemm_kernel") if args.products == "int8crt" else None,
                                "traffic_note": "DRAM bytes of one top-level product launch of config 3 (ncu --set "
                                                "full); a tensor-bound kernel: for comparison with its operand bytes",
                                "peak_source": "MEASURED_PEAKS.json bf16_tflops_sustained x 2 (nominal int8 / bf16)",
                                "int8_share_of_step": ms_o / (args.steps * prof_step_ms),
                                "int8_fp64_equivalent_tflops": fl_o / (ms_o / 1e3) / 1e12,
                                "crt_aux_kernels": None if n_x == 0 else {
                                    "kernels": "oz2_split_rows / colmax / split_cols / reconstruct",
                                    "achieved_gbs": by_x / (ms_x / 1e3) / 1e9, "peak_gbs": hbm_peak,
                                    "frac": by_x / (ms_x / 1e3) / 1e9 / hbm_peak,
                                    "share_of_step": ms_x / (args.steps * prof_step_ms),
                                    "note": "algorithmic bytes (operands in the GEMM's K range: 8 B read + 16 B "
                                            "residues written; outputs: 16 B residues read + 8 B written); "
                                            "integer-ALU bound"},
                                "dmma_part": {"achieved_tflops": achieved, "peak": fp64_peak,
                                              "frac": achieved / fp64_peak,
                                              "share_of_step": ms_d / (args.steps * prof_step_ms)},
                                "whole_step_tflops": flops_per_step / (ms_per_step / 1e3) / 1e12,
                                "whole_step_frac_of_fp64_peak": flops_per_step / (ms_per_step / 1e3) / 1e12 / fp64_peak}
        elif n_d == 0:  # a single block launch (n <= 128): latency-bound, no level products
            line["roofline"] = {"bound": "latency", "kernel": "blk_kernel (single launch)", "achieved": None,
                                "peak": None, "unit": None, "frac": None, "traffic": None,
                                "leaf_us_per_launch": 1e3 * ms_l / max(n_l, 1),
                                "note": "one 64x64 inverse per launch in one CTA; bounded by launch latency and "
                                        "the dependent phases (load, leaves, two merge levels, store), not by HBM "
                                        "or the tensor pipe"}
        else:
            line["roofline"] = {"bound": "tensor", "kernel": "dmma_level_kernel (all product launches)",
                              "achieved": achieved, "peak": fp64_peak, "unit": "TFLOP/s",
                              "frac": achieved / fp64_peak, "traffic": ncu_traffic("dmma_level_kernel"),
                              "peak_source": fp64_src + " (FP64 DMMA, register-only loop)",
                              "dmma_share_of_step": ms_d / (args.steps * prof_step_ms) if prof_step_ms else None,
                              "dmma_launches_per_step": n_d / args.steps, "leaf_ms_per_step": ms_l / args.steps,
                              "whole_step_tflops": flops_per_step / (ms_per_step / 1e3) / 1e12,
                              "whole_step_frac_of_peak": flops_per_step / (ms_per_step / 1e3) / 1e12 / fp64_peak}
        line["config"]["cuda_graph"] = graph is not None
    line["gpu_launches"] = launches
    line["clocks"] = clk.summary()

    # ---- end-to-end through the public API with host buffers ----
    if cfg["kind"] == "B" and args.e2e_steps > 0:
        # host buffers through the library's pipelined host entry point (trinv_batched_host:
        # chunked H2D / invert / D2H on overlapping streams); copies are inside the timed region
        h_in = torch.empty((B, n, n), dtype=torch.float64).pin_memory()
        h_out = torch.empty_like(h_in).pin_memory()
        h_in.copy_(A.cpu())
        ws = torch.empty(P.lib().trinv_batched_host_workspace_bytes(n, 0), dtype=torch.uint8, device=dev)
        import ctypes
        def e2e_step():
            st = P.lib().trinv_batched_host(b"L", n, B, ctypes.c_void_p(h_in.data_ptr()),
                                            ctypes.c_void_p(h_out.data_ptr()), 0, 0,
                                            ctypes.c_void_p(ws.data_ptr()), ws.numel(), None,
                                            ctypes.c_void_p(stream.cuda_stream))
            assert st == 0, P.status_string(st)
        e2e_step(); barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        barrier(); e0.record(stream)
        for _ in range(args.e2e_steps):
            e2e_step()
        e1.record(stream); barrier()
        e_ms = max_over_ranks(e0.elapsed_time(e1)) / args.e2e_steps
        nbytes = h_in.numel() * 8
        line["e2e"] = {"value": total_units / (e_ms / 1e3), "unit": unit, "h2d_bytes_per_step": nbytes,
                       "d2h_bytes_per_step": nbytes, "bytes_are": "per rank (its shard)" if world > 1 else "whole job",
                       "ms_per_step": e_ms, "steps": args.e2e_steps,
                       "path": "pinned host -> trinv_batched_host (C-ABI; 4096-matrix chunks, H2D / invert / "
                               "D2H overlapped on 3 streams) -> pinned host",
                       "pcie_gbs_each_way": nbytes / (e_ms / 1e3) / 1e9}
        del h_in, h_out, ws
    elif cfg["kind"] not in ("B", "S"):
        # host buffers: H2D of the input factor(s), the call, D2H of the inverse
        ins = [Lm, Um] if cfg["kind"] == "G" else [A]  # config 5: A
        h_ins = [t.cpu().pin_memory() for t in ins]
        h_out = torch.empty((n, n), dtype=torch.float64).pin_memory()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        barrier(); e0.record(stream)
        steps_e = max(1, min(args.e2e_steps, 3))
        for _ in range(steps_e):
            for d, h in zip(ins, h_ins):
                d.copy_(h, non_blocking=True)
            step()
            h_out.copy_(X, non_blocking=True)
        e1.record(stream); barrier()
        e_ms = max_over_ranks(e0.elapsed_time(e1)) / steps_e
        line["e2e"] = {"value": units_per_rank * world / (e_ms / 1e3), "unit": unit,
                       "h2d_bytes_per_step": sum(h.numel() * 8 for h in h_ins), "d2h_bytes_per_step": n * n * 8,
                       "ms_per_step": e_ms, "steps": steps_e}

    if cfg["kind"] == "B" and world > 1:
        line["gather"] = gather_and_check(X, B, strong, world, rank, dev, stream, backend, n, barrier,
                                          max_over_ranks, P, torch, dist)
    if cfg["kind"] == "B" and world == 1 and not args.no_fp64:
        del A, X
        torch.cuda.empty_cache()
        line["fp64"] = fp64_block(args, dev, stream, P, synth, torch, barrier)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(cfg)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
