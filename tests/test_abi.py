"""The C-ABI library loads, exports every symbol include/trinv.h declares, and
rejects bad arguments synchronously (no GPU needed: nothing is enqueued)."""
import ctypes

import pytest

import paper_2307_07611_b200 as P
from paper_2307_07611_b200 import _lib


def test_exports_every_declared_symbol():
    L = P.lib()
    names = _lib.declared_symbols()
    assert {"trinv_lower", "trinv_upper", "trinv_batched", "inv_from_lu", "trinv_workspace_bytes"} <= set(names)
    for name in names:
        assert hasattr(L, name), name


def test_version_and_status_strings():
    assert b"sm_100a" in P.lib().trinv_version()
    for st in range(6):
        assert P.status_string(st).startswith("TRINV_")


FAKE = ctypes.c_void_p(1 << 20)
FAKE2 = ctypes.c_void_p(1 << 30)


@pytest.mark.parametrize("fn", ["trinv_lower", "trinv_upper"])
def test_tri_argument_validation(fn):
    f = getattr(P.lib(), fn)
    assert f(0, None, 0, None, 0, 0, None, 0, None, None) == _lib.TRINV_OK  # n == 0 no-op
    assert f(-1, FAKE, 1, FAKE2, 1, 0, None, 0, None, None) == _lib.TRINV_INVALID_ARG
    assert f(4, None, 4, FAKE2, 4, 0, None, 0, None, None) == _lib.TRINV_INVALID_ARG
    assert f(4, FAKE, 3, FAKE2, 4, 0, None, 0, None, None) == _lib.TRINV_INVALID_ARG  # lda < n
    assert f(4, FAKE, 4, FAKE2, 4, 7, None, 0, None, None) == _lib.TRINV_INVALID_ARG  # bad diag
    assert f(4, FAKE, 4, FAKE, 4, 0, None, 0, None, None) == _lib.TRINV_ALIASING
    over = ctypes.c_void_p((1 << 20) + 8 * 5)
    assert f(4, FAKE, 4, over, 4, 0, None, 0, None, None) == _lib.TRINV_ALIASING
    assert f(200, FAKE, 200, FAKE2, 200, 0, None, 0, None, None) == _lib.TRINV_WORKSPACE_TOO_SMALL


def test_batched_argument_validation():
    f = P.lib().trinv_batched
    assert f(b"L", 32, 0, None, 32, 1024, None, 32, 1024, 0, None, None) == _lib.TRINV_OK
    assert f(b"X", 32, 4, FAKE, 32, 1024, FAKE2, 32, 1024, 0, None, None) == _lib.TRINV_INVALID_ARG
    assert f(b"L", 32, 4, FAKE, 32, 1000, FAKE2, 32, 1024, 0, None, None) == _lib.TRINV_INVALID_ARG
    assert f(b"L", 129, 4, FAKE, 129, 129 * 129, FAKE2, 129, 129 * 129, 0, None, None) == _lib.TRINV_NOT_SUPPORTED


def test_inv_from_lu_argument_validation():
    f = P.lib().inv_from_lu
    assert f(0, None, 0, None, 0, None, 0, 1, 0, None, 0, None, None) == _lib.TRINV_OK
    assert f(8, FAKE, 8, FAKE2, 8, FAKE, 8, 1, 0, None, 0, None, None) == _lib.TRINV_ALIASING
    assert f(8, FAKE, 8, FAKE2, 8, ctypes.c_void_p(1 << 25), 8, 1, 0, None, 0, None, None) == \
        _lib.TRINV_WORKSPACE_TOO_SMALL


def test_workspace_sizes():
    ws = P.lib().trinv_workspace_bytes
    assert ws(b"L", 64, None, 64, None, 64) == 0
    n = 32768
    P.set_product_engine()  # default: DMMA for every product
    assert P.product_engine() == "dmma"
    assert P.strassen_levels() == 2  # default: Strassen in the top merge's dense quadrants (f3)
    h = n // 4  # the top merge's quadrant order
    sync = 65536  # split-K tickets / semaphores, fused-level flags (LEVEL_SYNC_BYTES)
    # Strassen scratch: 17 quadrant temps (5 + 5 operand sums, M1..M7) per level, 2 levels
    assert ws(b"L", n, None, n, None, n) == (n // 2) ** 2 * 8 + 17 * (h // 2) ** 2 * 8 + 17 * (h // 4) ** 2 * 8 + sync
    P.set_strassen(0)
    assert ws(b"L", n, None, n, None, n) == (n // 2) ** 2 * 8 + sync  # W = one (n/2)^2 block
    try:
        P.set_product_engine("int8crt")  # opt-in INT8 CRT engine for blocks >= 2048 adds its residue scratch
        h = n // 2
        assert ws(b"L", n, None, n, None, n) >= h * h * 8 + 16 * 3 * h * h
        assert P.product_engine() == "int8crt"
    finally:
        P.set_product_engine()
    assert ws(b"L", n, None, n, None, n) == (n // 2) ** 2 * 8 + sync
    P.set_strassen()
    assert ws(b"U", 1000, None, 1000, None, 1000) > 0
    # odd leading dimensions stage through the workspace
    assert ws(b"L", 999, None, 999, None, 999) > ws(b"L", 999, None, 1000, None, 1000)
    assert ws(b"G", 1024, None, 1024, None, 1024) >= 2 * 1024 * 1024 * 8
