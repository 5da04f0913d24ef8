"""paper_2307_07611_b200 — B200-native FP64 triangular inversion (arXiv 2307.07611 hot path).

Thin Python binding over the C ABI in include/trinv.h (libtrinv.so, built in-tree
for sm_100a).  This module only marshals arguments: shapes, leading dimensions,
device pointers, the current CUDA stream and a workspace allocated through torch.
Every arithmetic step runs in the library's CUDA kernels; there is no CPU or
PyTorch fallback — if libtrinv.so is missing or no GPU is present the calls raise.

    X = trinv_lower(L)            # L^{-1}, full matrix, +0.0 above the diagonal
    X = trinv_upper(U)            # U^{-1}
    X = trinv_batched(A, "L")     # A: [B, n, n] on the device, n <= 128
    X = trinv_batched_host(Ah)    # Ah: host [B, n, n]; pipelined H2D / invert / D2H
    X = inv_from_lu(L, U)         # (L U)^{-1} = U^{-1} L^{-1}, L unit by default
"""
import ctypes
import os

from ._lib import (TRINV_OK, TRINV_UNIT, TRINV_NON_UNIT, TrinvError, SingularMatrixError,  # noqa: F401
                   lib, so_path, status_string, launch_count, reset_launch_count)

__all__ = ["trinv_lower", "trinv_upper", "trinv_batched", "trinv_batched_host", "inv_from_lu", "inv_general",
           "lu_crout", "gemm", "gemm_oz", "gemm_strassen", "set_product_engine", "product_engine", "product_min_block",
           "int8_scaling_ok", "trinv_beta", "workspace_bytes",
           "TrinvError", "SingularMatrixError", "lib", "so_path", "launch_count", "reset_launch_count"]


def _torch():
    import torch
    return torch


def _ld(t):
    """Leading dimension of a row-major 2-D (or [B, n, n]) CUDA float64 tensor."""
    torch = _torch()
    if not isinstance(t, torch.Tensor) or t.dtype != torch.float64:
        raise TypeError("expected a torch.float64 tensor")
    if not t.is_cuda:
        raise ValueError("expected a CUDA tensor (device memory); host buffers: copy with .cuda() first")
    if t.shape[-1] > 1 and t.stride(-1) != 1:
        raise ValueError("row-major layout required (stride(-1) == 1)")
    if t.shape[-2] > 1 or t.stride(-2) >= t.shape[-1]:
        return max(t.stride(-2), t.shape[-1])
    return t.shape[-1]


def _on_stream(fn):
    """Run a binding call with its `stream` (if given) as torch's current stream, so that the
    workspace, info and output tensors the call allocates belong to that stream's memory pool
    (the caching allocator may otherwise hand a freed workspace to another stream while this
    call's kernels still use it) and a synchronous read of `info` is ordered after them."""
    import functools

    @functools.wraps(fn)
    def wrapper(*args, **kwargs):
        stream = kwargs.get("stream")
        if stream is None:
            return fn(*args, **kwargs)
        with _torch().cuda.stream(stream):
            return fn(*args, **kwargs)
    return wrapper


def _stream(stream):
    torch = _torch()
    s = torch.cuda.current_stream() if stream is None else stream
    return ctypes.c_void_p(s.cuda_stream)


def _check(st):
    if st != TRINV_OK:
        raise TrinvError(st)


def workspace_bytes(op, n, A=None, lda=None, X=None, ldx=None):
    """Device workspace bytes for op 'L' | 'U' | 'G' (see trinv_workspace_bytes)."""
    pa = ctypes.c_void_p(A.data_ptr()) if A is not None else None
    px = ctypes.c_void_p(X.data_ptr()) if X is not None else None
    lda = n if lda is None else lda
    ldx = n if ldx is None else ldx
    return lib().trinv_workspace_bytes(op.encode(), n, pa, lda, px, ldx)


def _alloc_ws(nbytes, device):
    torch = _torch()
    if nbytes == 0:
        return None, 0
    w = torch.empty(nbytes, dtype=torch.uint8, device=device)
    return w, nbytes


def _info(check, device):
    torch = _torch()
    return torch.zeros(1, dtype=torch.int32, device=device) if check else None


def _raise_info(info, what):
    if info is not None:
        v = int(info.item())
        if v != 0:
            raise SingularMatrixError(v, what)


def _tri(uplo, A, unit, out, check, stream):
    torch = _torch()
    n = A.shape[-1]
    if A.dim() != 2 or A.shape[0] != n:
        raise ValueError("expected a square 2-D matrix")
    lda = _ld(A)
    X = torch.empty((n, n), dtype=torch.float64, device=A.device) if out is None else out
    ldx = _ld(X)
    ws, wsb = _alloc_ws(workspace_bytes(uplo, n, A, lda, X, ldx), A.device)
    info = _info(check, A.device)
    f = lib().trinv_lower if uplo == "L" else lib().trinv_upper
    _check(f(n, ctypes.c_void_p(A.data_ptr()), lda, ctypes.c_void_p(X.data_ptr()), ldx,
             TRINV_UNIT if unit else TRINV_NON_UNIT,
             ctypes.c_void_p(ws.data_ptr()) if ws is not None else None, wsb,
             ctypes.c_void_p(info.data_ptr()) if info is not None else None, _stream(stream)))
    _raise_info(info, "trinv_lower" if uplo == "L" else "trinv_upper")
    return X


@_on_stream
def trinv_lower(A, *, unit=False, out=None, check=False, stream=None):
    """X = A^{-1} for lower-triangular A (only the lower triangle is used)."""
    return _tri("L", A, unit, out, check, stream)


@_on_stream
def trinv_upper(A, *, unit=False, out=None, check=False, stream=None):
    """X = A^{-1} for upper-triangular A (only the upper triangle is used)."""
    return _tri("U", A, unit, out, check, stream)


@_on_stream
def trinv_batched(A, uplo="L", *, unit=False, out=None, info=False, stream=None):
    """X[b] = A[b]^{-1} for A of shape [B, n, n], n <= 128.  Returns X, or (X, info[B]) if info."""
    torch = _torch()
    if A.dim() != 3 or A.shape[1] != A.shape[2]:
        raise ValueError("expected [B, n, n]")
    B, n = A.shape[0], A.shape[1]
    lda = _ld(A)
    X = torch.empty_like(A, memory_format=torch.contiguous_format) if out is None else out
    ldx = _ld(X)
    sa = A.stride(0) if B > 1 else n * lda
    sx = X.stride(0) if B > 1 else n * ldx
    inf = torch.empty(B, dtype=torch.int32, device=A.device) if info else None
    _check(lib().trinv_batched(uplo.encode(), n, B, ctypes.c_void_p(A.data_ptr()), lda, sa,
                               ctypes.c_void_p(X.data_ptr()), ldx, sx,
                               TRINV_UNIT if unit else TRINV_NON_UNIT,
                               ctypes.c_void_p(inf.data_ptr()) if inf is not None else None,
                               _stream(stream)))
    return (X, inf) if info else X


@_on_stream
def trinv_batched_host(A_host, uplo="L", *, unit=False, out=None, chunk=0, info=False, device=None,
                       stream=None):
    """Invert a HOST batch [B, n, n] (contiguous, ideally pinned): chunked H2D / invert / D2H
    pipeline on the current CUDA device.  Returns the host tensor X (or (X, info[B] on device))."""
    torch = _torch()
    if A_host.is_cuda or A_host.dim() != 3 or A_host.shape[1] != A_host.shape[2]:
        raise ValueError("expected a host tensor [B, n, n]")
    if A_host.dtype != torch.float64 or not A_host.is_contiguous():
        raise ValueError("expected a contiguous float64 host tensor")
    B, n = A_host.shape[0], A_host.shape[1]
    X = torch.empty_like(A_host, pin_memory=A_host.is_pinned()) if out is None else out
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    wsb = lib().trinv_batched_host_workspace_bytes(n, chunk)
    ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
    inf = torch.empty(B, dtype=torch.int32, device=dev) if info else None
    _check(lib().trinv_batched_host(uplo.encode(), n, B, ctypes.c_void_p(A_host.data_ptr()),
                                    ctypes.c_void_p(X.data_ptr()), TRINV_UNIT if unit else TRINV_NON_UNIT,
                                    chunk, ctypes.c_void_p(ws.data_ptr()), wsb,
                                    ctypes.c_void_p(inf.data_ptr()) if inf is not None else None,
                                    _stream(stream)))
    # keep the workspace alive until the stream has consumed it
    ws.record_stream(torch.cuda.current_stream() if stream is None else stream)
    return (X, inf) if info else X


@_on_stream
def trinv_beta(A, uplo="L", beta=4, *, unit=False, out=None, check=False, stream=None):
    """Triangular inverse with a COMBRIT top level of block count beta (2 or 4; NEXT row f4)."""
    torch = _torch()
    n = A.shape[-1]
    lda = _ld(A)
    X = torch.empty((n, n), dtype=torch.float64, device=A.device) if out is None else out
    ldx = _ld(X)
    ws, wsb = _alloc_ws(lib().trinv_tri_ex_workspace_bytes(beta, n), A.device)
    info = _info(check, A.device)
    _check(lib().trinv_tri_ex(uplo.encode(), beta, n, ctypes.c_void_p(A.data_ptr()), lda,
                              ctypes.c_void_p(X.data_ptr()), ldx, TRINV_UNIT if unit else TRINV_NON_UNIT,
                              ctypes.c_void_p(ws.data_ptr()) if ws is not None else None, wsb,
                              ctypes.c_void_p(info.data_ptr()) if info is not None else None, _stream(stream)))
    _raise_info(info, "trinv_beta")
    return X


@_on_stream
def gemm(A, B, *, C=None, alpha=1.0, beta=0.0, struct_a="N", struct_b="N", stream=None):
    """C = alpha A B + beta C on the DMMA engine; A [.., M, K], B [.., K, N] (optionally batched
    with a leading batch dimension); struct_a / struct_b = 'L' / 'U' declare a triangular operand."""
    torch = _torch()
    batched = A.dim() == 3
    if batched != (B.dim() == 3):
        raise ValueError("A and B must both be 2-D or both 3-D")
    M, K = A.shape[-2], A.shape[-1]
    N = B.shape[-1]
    if B.shape[-2] != K:
        raise ValueError("inner dimensions differ")
    bs = A.shape[0] if batched else 1
    if C is None:
        C = torch.zeros((bs, M, N) if batched else (M, N), dtype=torch.float64, device=A.device)
    lda, ldb, ldc = _ld(A), _ld(B), _ld(C)
    sa = A.stride(0) if batched else M * lda
    sb = B.stride(0) if batched else K * ldb
    sc = C.stride(0) if batched else M * ldc
    _check(lib().trinv_gemm(M, N, K, bs, float(alpha), ctypes.c_void_p(A.data_ptr()), lda, sa, struct_a.encode(),
                            ctypes.c_void_p(B.data_ptr()), ldb, sb, struct_b.encode(), float(beta),
                            ctypes.c_void_p(C.data_ptr()), ldc, sc, _stream(stream)))
    return C


@_on_stream
def gemm_oz(A, B, *, C=None, alpha=1.0, beta=0.0, struct_a="N", struct_b="N", digits=0, stream=None):
    """C = alpha A B + beta C, FP64-emulated (Ozaki-II) on the INT8 tensor cores: 16 moduli
    + CRT (trinv_gemm_oz; digits must be 0, the digit-splitting variant was retired)."""
    torch = _torch()
    M, K = A.shape
    N = B.shape[1]
    if B.shape[0] != K:
        raise ValueError("inner dimensions differ")
    if C is None:
        C = torch.zeros((M, N), dtype=torch.float64, device=A.device)
    ws, wsb = _alloc_ws(lib().trinv_gemm_oz_workspace_bytes(M, N, K, digits), A.device)
    _check(lib().trinv_gemm_oz(M, N, K, float(alpha), ctypes.c_void_p(A.data_ptr()), _ld(A), struct_a.encode(),
                               ctypes.c_void_p(B.data_ptr()), _ld(B), struct_b.encode(), float(beta),
                               ctypes.c_void_p(C.data_ptr()), _ld(C), digits,
                               ctypes.c_void_p(ws.data_ptr()) if ws is not None else None, wsb, _stream(stream)))
    return C


_MIN_BLOCK = 2048  # the engines' block threshold as last set through set_product_engine


def set_product_engine(engine="dmma", min_block=2048):
    """Engine of the level products: "dmma" (default: FP64 mma.sync for every product) or
    "int8crt" (opt-in, FP64-emulated (Ozaki-II) on the INT8 tensor cores, 16 moduli + CRT,
    for the levels with block size >= min_block; one host synchronisation per call for its
    scaling guard)."""
    global _MIN_BLOCK
    e = {"dmma": 0, "int8crt": 2}[engine]
    _check(lib().trinv_set_product_engine(e, 0, min_block))
    _MIN_BLOCK = int(min_block)


def set_strassen(levels=2, min_h=4096):
    """NEXT row f3: Strassen levels in the dense quadrant products of the top merge of a
    triangular inverse and of inv_from_lu's U^-1 L^-1 (trinv_set_strassen; library default
    2 levels from h = 4096; 0 = off)."""
    _check(lib().trinv_set_strassen(int(levels), int(min_h)))


def strassen_levels():
    return int(lib().trinv_get_strassen())


def product_min_block():
    return _MIN_BLOCK


@_on_stream
def int8_scaling_ok(A, uplo="N", unit=False, stream=None):
    """The INT8 engine's scaling guard (trinv_int8_scaling_ok): True when A's row / column
    maxima span at most 8 binades and every entry is finite (only the `uplo` triangle read
    for "L" / "U"); False under stream capture (the guard cannot run)."""
    n = A.shape[-1]
    r = lib().trinv_int8_scaling_ok(n, ctypes.c_void_p(A.data_ptr()), _ld(A), uplo.encode(), int(bool(unit)),
                                    _stream(stream))
    if r < 0:
        _check(-r)
    return r == 1


def product_engine():
    return {0: "dmma", 2: "int8crt"}[lib().trinv_get_product_engine()]


@_on_stream
def gemm_strassen(A, B, *, C=None, stream=None):
    """C = A B (dense n x n) with one Strassen level over the DMMA GEMM (NEXT row f3, measurement)."""
    torch = _torch()
    n = A.shape[-1]
    C = torch.empty((n, n), dtype=torch.float64, device=A.device) if C is None else C
    ws, wsb = _alloc_ws(lib().trinv_strassen_workspace_bytes(n), A.device)
    _check(lib().trinv_gemm_strassen(n, ctypes.c_void_p(A.data_ptr()), _ld(A), ctypes.c_void_p(B.data_ptr()), _ld(B),
                                     ctypes.c_void_p(C.data_ptr()), _ld(C),
                                     ctypes.c_void_p(ws.data_ptr()) if ws is not None else None, wsb,
                                     _stream(stream)))
    return C


@_on_stream
def lu_crout(A, *, check=False, stream=None):
    """In-place Crout factorisation without pivoting (SKUL): A <- L\\U packed,
    L lower with its diagonal, U unit upper (strict upper part stored)."""
    n = A.shape[-1]
    lda = _ld(A)
    ws, wsb = _alloc_ws(workspace_bytes("F", n), A.device)
    info = _info(check, A.device)
    _check(lib().lu_crout(n, ctypes.c_void_p(A.data_ptr()), lda,
                          ctypes.c_void_p(ws.data_ptr()) if ws is not None else None, wsb,
                          ctypes.c_void_p(info.data_ptr()) if info is not None else None, _stream(stream)))
    _raise_info(info, "lu_crout")
    return A


@_on_stream
def inv_general(A, *, out=None, check=False, stream=None):
    """X = A^{-1} for a general matrix with non-zero leading principal minors (Crout LU without
    pivoting, then U^{-1} L^{-1})."""
    torch = _torch()
    n = A.shape[-1]
    lda = _ld(A)
    X = torch.empty((n, n), dtype=torch.float64, device=A.device) if out is None else out
    ldx = _ld(X)
    ws, wsb = _alloc_ws(workspace_bytes("A", n, A, lda, X, ldx), A.device)
    info = _info(check, A.device)
    _check(lib().inv_general(n, ctypes.c_void_p(A.data_ptr()), lda, ctypes.c_void_p(X.data_ptr()), ldx,
                             ctypes.c_void_p(ws.data_ptr()) if ws is not None else None, wsb,
                             ctypes.c_void_p(info.data_ptr()) if info is not None else None, _stream(stream)))
    _raise_info(info, "inv_general")
    return X


@_on_stream
def inv_from_lu(L, U, *, unit_l=True, unit_u=False, out=None, check=False, stream=None):
    """X = (L U)^{-1} = U^{-1} L^{-1} from a lower factor L and an upper factor U."""
    torch = _torch()
    n = L.shape[-1]
    if L.shape != (n, n) or U.shape != (n, n):
        raise ValueError("expected two n x n factors")
    ldl, ldu = _ld(L), _ld(U)
    X = torch.empty((n, n), dtype=torch.float64, device=L.device) if out is None else out
    ldx = _ld(X)
    nb = workspace_bytes("G", n, L, ldl, X, ldx)
    nb = max(nb, lib().trinv_workspace_bytes(b"G", n, ctypes.c_void_p(U.data_ptr()), ldu,
                                             ctypes.c_void_p(X.data_ptr()), ldx))
    ws, wsb = _alloc_ws(nb, L.device)
    info = _info(check, L.device)
    _check(lib().inv_from_lu(n, ctypes.c_void_p(L.data_ptr()), ldl, ctypes.c_void_p(U.data_ptr()), ldu,
                             ctypes.c_void_p(X.data_ptr()), ldx,
                             TRINV_UNIT if unit_l else TRINV_NON_UNIT,
                             TRINV_UNIT if unit_u else TRINV_NON_UNIT,
                             ctypes.c_void_p(ws.data_ptr()) if ws is not None else None, wsb,
                             ctypes.c_void_p(info.data_ptr()) if info is not None else None,
                             _stream(stream)))
    _raise_info(info, "inv_from_lu")
    return X
