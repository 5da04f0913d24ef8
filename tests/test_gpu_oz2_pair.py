"""The CTA-pair CRT GEMM (oz2_gemm_pair_kernel, cta_group::2) at small sizes: a
subprocess with TRINV_OZ2_PAIR=256 routes every product with M % 256 == 0 through it
(the default only takes products >= 8192), and its results must equal the single-CTA
kernel's bit for bit (both compute the same exact integer products) on dense, triangular
and both-triangular operands, with alpha / beta, ragged K and non-square shapes."""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, %(root)r)
import paper_2307_07611_b200 as P
rng = np.random.default_rng(5)
out = []
for (M, N, K, sa, sb) in [(256, 256, 128, "N", "N"), (512, 768, 384, "N", "N"), (1024, 512, 1024, "L", "N"),
                          (768, 1024, 1024, "U", "N"), (1024, 1024, 1024, "N", "L"), (512, 1024, 1024, "N", "U"),
                          (1024, 1024, 1024, "U", "L")]:
    A = rng.uniform(-1, 1, (M, K)); B = rng.uniform(-1, 1, (K, N)); C0 = rng.uniform(-1, 1, (M, N))
    if sa == "L": A = np.tril(A)
    if sa == "U": A = np.triu(A)
    if sb == "L": B = np.tril(B)
    if sb == "U": B = np.triu(B)
    C = P.gemm_oz(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), C=torch.from_numpy(C0).cuda(),
                  alpha=-1.5, beta=0.25, digits=0, struct_a=sa, struct_b=sb).cpu().numpy()
    out.append(C)
np.savez(sys.argv[1], *out)
"""


def _run(tmp_path, pair):
    f = tmp_path / ("pair.npz" if pair else "single.npz")
    env = dict(os.environ, TRINV_OZ2_PAIR="256" if pair else "0")
    code = SCRIPT % {"root": ROOT}
    r = subprocess.run([sys.executable, "-c", code, str(f)], env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    z = np.load(f)
    return [z[k] for k in sorted(z.files, key=lambda s: int(s.split("_")[1]))]


def test_pair_kernel_matches_single_cta_kernel(tmp_path):
    single = _run(tmp_path, False)
    pair = _run(tmp_path, True)
    assert len(single) == len(pair) == 7
    for a, b in zip(single, pair):
        assert np.array_equal(a, b)
