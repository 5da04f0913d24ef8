"""Config-1 kernel variants on one box (each in its own process: the env is read once).
    python tools/leaf_sweep.py [steps]"""
import json
import os
import subprocess
import sys

steps = sys.argv[1] if len(sys.argv) > 1 else "20"
MMA = {"TRINV_LEAF32": "mma"}
variants = [("pipe 8x3", dict(MMA, TRINV_LEAF32_CFG="1083")), ("pipe 6x3", dict(MMA, TRINV_LEAF32_CFG="1063")),
            ("pipe 6x4", dict(MMA, TRINV_LEAF32_CFG="1064")), ("pipe 4x3", dict(MMA, TRINV_LEAF32_CFG="1043")),
            ("mma 8x3", dict(MMA, TRINV_LEAF32_CFG="83")), ("mma 8x2", dict(MMA, TRINV_LEAF32_CFG="82")),
            ("mma 12x2", dict(MMA, TRINV_LEAF32_CFG="122")), ("mma 6x4", dict(MMA, TRINV_LEAF32_CFG="64")),
            ("mma 6x2", dict(MMA, TRINV_LEAF32_CFG="62")), ("mma 4x2", dict(MMA, TRINV_LEAF32_CFG="42")),
            ("band16", {})]
for name, env in variants:
    e = dict(os.environ, **env)
    r = subprocess.run([sys.executable, "bench.py", "--steps", steps, "--warmup", "5", "--no-cpu-baseline",
                        "--e2e-steps", "0", "--no-fp64"], env=e, capture_output=True, text=True)
    try:
        d = json.loads(r.stdout.strip().splitlines()[-1])
        print(f"{name:10s} {d['ms_per_step']:.4f} ms  {d['value']:.4e} inv/s  frac {d['roofline']['frac']:.3f}  "
              f"median {d['step_ms_stats']['median']:.4f}", flush=True)
    except Exception:
        print(name, "failed", r.stderr[-500:], flush=True)
