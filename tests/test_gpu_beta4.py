"""NEXT row f4: COMBRIT with beta = 4 at the top level (Alg. 1) —
parity with the CPU oracle and with the beta = 2 path."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
import oracle  # noqa: E402
import synth  # noqa: E402
import paper_2307_07611_b200 as P  # noqa: E402
from gpu_common import check_full  # noqa: E402

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


@pytest.mark.parametrize("n", [128, 256, 512, 1024, 2048])
@pytest.mark.parametrize("uplo", ["L", "U"])
@pytest.mark.parametrize("unit", [False, True])
def test_beta4_parity(n, uplo, unit):
    T = synth.host(n, seed=n + unit, uplo=uplo, diag="one" if unit else ("signed" if uplo == "L" else "pos"))
    Td = torch.from_numpy(T).to(DEV)
    X4 = P.trinv_beta(Td, uplo, 4, unit=unit).cpu().numpy()
    check_full(T, X4, uplo, unit=unit)
    X2 = P.trinv_beta(Td, uplo, 2, unit=unit).cpu().numpy()
    assert oracle.floored_rel_err(X4, X2) <= 1e-10


def test_beta4_exact_pins():
    n = 256
    for s in (0.5, -1.0):
        L = np.eye(n) - s * np.eye(n, k=-1)
        i, j = np.indices((n, n))
        ref = np.where(i >= j, float(s) ** (i - j).astype(float), 0.0)
        assert np.array_equal(P.trinv_beta(torch.from_numpy(L).to(DEV), "L", 4).cpu().numpy(), ref)
        assert np.array_equal(P.trinv_beta(torch.from_numpy(L.T.copy()).to(DEV), "U", 4).cpu().numpy(), ref.T)


def test_beta4_unsupported_sizes():
    A = torch.from_numpy(synth.host(300, seed=1)).to(DEV)
    with pytest.raises(P.TrinvError):
        P.trinv_beta(A, "L", 4)
