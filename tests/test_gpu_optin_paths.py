"""The opt-in experimental launch paths (each measured slower than the default and kept
behind an environment variable read once per process, hence one subprocess per setting):
serial split-K (TRINV_SPLITK=1, 64x64 and 32x32 tiles), split-K with the last-chunk fix-up
(TRINV_SPLITK=2), fused level launches (TRINV_FUSED=1), stream-order launches without
programmatic dependent launch (TRINV_PDL=0; PDL is the default since round 2's last session), stream-K level launches (TRINV_SK=1; WMIN=2 cuts tiles into several pieces) and the
persistent dependency-driven level chain (TRINV_CHAIN=1; OCC=1 makes every CTA walk many tiles), and the
128-register level kernels off (TRINV_R128=0) or on for every 64x64 / 64x32 level (TRINV_R128=3, WAVES=0).  Each must still match the oracle: full parity at n = 1024 / 2048 (lower and
upper, ragged n = 1500) and bit-for-bit determinism."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

_SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import oracle, synth, paper_2307_07611_b200 as P
from gpu_common import REL_TOL, RES_TOL
bad = []
for n, uplo in ((1024, 'L'), (2048, 'U'), (2048, 'L'), (1500, 'U')):
    T = synth.host(n, seed=n + 7, uplo=uplo, diag='signed' if uplo == 'L' else 'pos')
    f = P.trinv_lower if uplo == 'L' else P.trinv_upper
    Td = torch.from_numpy(T).cuda()
    X1 = f(Td).cpu().numpy(); X2 = f(Td).cpu().numpy()
    R = oracle.trinv(T, uplo)
    Tt = np.tril(T) if uplo == 'L' else np.triu(T)
    e = oracle.floored_rel_err(X1, R); r = oracle.residual_ratio(Tt, X1)
    opp = np.triu(X1, 1) if uplo == 'L' else np.tril(X1, -1)
    if not (e <= REL_TOL and r <= RES_TOL and np.all(opp == 0) and np.array_equal(X1, X2)):
        bad.append((n, uplo, e, r))
print('BAD', bad)
"""


@pytest.mark.parametrize("env", [{"TRINV_SPLITK": "1"}, {"TRINV_SPLITK": "1", "TRINV_SPLITK_T": "32", "TRINV_SPLITK_KC": "256"},
                                 {"TRINV_SPLITK": "2", "TRINV_SPLITK_T": "32", "TRINV_SPLITK_KC": "256"},
                                 {"TRINV_SPLITK": "2"}, {"TRINV_FUSED": "1"}, {"TRINV_PDL": "0"},
                                 {"TRINV_SK": "1", "TRINV_SK_BMIN": "128"},
                                 {"TRINV_SK": "1", "TRINV_SK_TILE": "12864", "TRINV_SK_BMIN": "128", "TRINV_SK_WMIN": "2"},
                                 {"TRINV_CHAIN": "1"}, {"TRINV_CHAIN": "1", "TRINV_CHAIN_OCC": "1"},
                                 {"TRINV_R128": "0"}, {"TRINV_R128": "3", "TRINV_R128_WAVES": "0"}],
                         ids=["splitk1", "splitk1-t32", "splitk2-t32", "splitk2", "fused", "pdl", "sk64", "sk128x64",
                              "chain", "chain-occ1", "r128-off", "r128-all"])
def test_optin_path_parity(env):
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", _SCRIPT], cwd=root, env=dict(os.environ, **env), capture_output=True,
                       text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-2000:]
    assert "BAD []" in r.stdout, r.stdout + r.stderr[-2000:]
