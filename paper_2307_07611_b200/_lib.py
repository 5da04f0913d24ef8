"""ctypes loader for libtrinv.so (the C ABI of include/trinv.h).  Loading fails
loudly when the library has not been built: there is no fallback path."""
import ctypes
import os
import re

HERE = os.path.dirname(os.path.abspath(__file__))
HEADER = os.path.join(HERE, "..", "include", "trinv.h")
# TRINV_LIB may point at another build of the same ABI (A/B measurements only)
_SO = os.environ.get("TRINV_LIB") or os.path.join(HERE, "libtrinv.so")

TRINV_OK, TRINV_INVALID_ARG, TRINV_ALIASING, TRINV_WORKSPACE_TOO_SMALL, TRINV_CUDA_ERROR, TRINV_NOT_SUPPORTED = range(6)
TRINV_NON_UNIT, TRINV_UNIT = 0, 1
_lib = None

_i64, _vp, _sz, _i32 = ctypes.c_int64, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int


class TrinvError(RuntimeError):
    def __init__(self, status):
        self.status = status
        msg = status_string(status)
        if status == TRINV_CUDA_ERROR:
            msg += f" (cudaError {lib().trinv_last_cuda_error()})"
        super().__init__(msg)


class SingularMatrixError(ArithmeticError):
    def __init__(self, info, what=""):
        self.info = info
        super().__init__(f"{what}: exact zero on the diagonal (info = {info})")


def so_path():
    return _SO


def lib():
    """Load libtrinv.so (build it with __graft_entry__.build())."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(_SO):
        raise ImportError(f"{_SO} is missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
    L = ctypes.CDLL(_SO)
    def sig(name, args, res=None):
        try:
            f = getattr(L, name)
        except AttributeError:
            if os.environ.get("TRINV_LIB"):  # an older build under A/B test: skip newer entry points
                return
            raise
        if args is not None:
            f.argtypes = args
        if res is not None:
            f.restype = res

    sig("trinv_workspace_bytes", [ctypes.c_char, _i64, _vp, _i64, _vp, _i64], _sz)
    for name in ("trinv_lower", "trinv_upper"):
        sig(name, [_i64, _vp, _i64, _vp, _i64, _i32, _vp, _sz, _vp, _vp], _i32)
    sig("trinv_batched", [ctypes.c_char, _i64, _i64, _vp, _i64, _i64, _vp, _i64, _i64, _i32, _vp, _vp], _i32)
    sig("trinv_batched_host_workspace_bytes", [_i64, _i64], _sz)
    sig("trinv_batched_host", [ctypes.c_char, _i64, _i64, _vp, _vp, _i32, _i64, _vp, _sz, _vp, _vp], _i32)
    sig("inv_from_lu", [_i64, _vp, _i64, _vp, _i64, _vp, _i64, _i32, _i32, _vp, _sz, _vp, _vp], _i32)
    sig("lu_crout", [_i64, _vp, _i64, _vp, _sz, _vp, _vp], _i32)
    sig("inv_general", [_i64, _vp, _i64, _vp, _i64, _vp, _sz, _vp, _vp], _i32)
    sig("trinv_gemm", [_i64, _i64, _i64, _i64, ctypes.c_double, _vp, _i64, _i64, ctypes.c_char, _vp, _i64,
                             _i64, ctypes.c_char, ctypes.c_double, _vp, _i64, _i64, _vp], _i32)
    sig("trinv_tri_ex_workspace_bytes", [_i32, _i64], _sz)
    sig("trinv_tri_ex", [ctypes.c_char, _i32, _i64, _vp, _i64, _vp, _i64, _i32, _vp, _sz, _vp, _vp], _i32)
    sig("trinv_strassen_workspace_bytes", [_i64], _sz)
    sig("trinv_gemm_strassen", [_i64, _vp, _i64, _vp, _i64, _vp, _i64, _vp, _sz, _vp], _i32)
    sig("trinv_gemm_oz_workspace_bytes", [_i64, _i64, _i64, _i32], _sz)
    sig("trinv_gemm_oz", [_i64, _i64, _i64, ctypes.c_double, _vp, _i64, ctypes.c_char, _vp, _i64, ctypes.c_char,
                          ctypes.c_double, _vp, _i64, _i32, _vp, _sz, _vp], _i32)
    sig("trinv_set_product_engine", [_i32, _i32, _i64], _i32)
    sig("trinv_get_product_engine", None, _i32)
    sig("trinv_set_strassen", [_i32, _i64], _i32)
    sig("trinv_get_strassen", None, _i32)
    sig("trinv_int8_scaling_ok", [_i64, ctypes.c_void_p, _i64, ctypes.c_char, _i32, ctypes.c_void_p], _i32)
    sig("trinv_status_string", [_i32], ctypes.c_char_p)
    sig("trinv_last_cuda_error", None, _i32)
    sig("trinv_version", None, ctypes.c_char_p)
    sig("trinv_probe_dmma_tflops", [ctypes.c_double, ctypes.c_void_p], ctypes.c_double)
    sig("trinv_launch_count", None, _i64)
    sig("trinv_profile_read", [_i32, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(_i64),
                                     ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double)], _i32)
    _lib = L
    return L


def status_string(st):
    return lib().trinv_status_string(st).decode()


def launch_count():
    return lib().trinv_launch_count()


def reset_launch_count():
    lib().trinv_reset_launch_count()


def profile_begin():
    lib().trinv_profile_begin()


def profile_end():
    lib().trinv_profile_end()


def profile_read(kind):
    """(ms, launches, flops, bytes) summed over the profiled launches of `kind` (0 leaf, 1 DMMA)."""
    ms, n, f, b = ctypes.c_double(), _i64(), ctypes.c_double(), ctypes.c_double()
    st = lib().trinv_profile_read(kind, ctypes.byref(ms), ctypes.byref(n), ctypes.byref(f), ctypes.byref(b))
    if st != TRINV_OK:
        raise TrinvError(st)
    return ms.value, n.value, f.value, b.value


def declared_symbols():
    """Function names declared in include/trinv.h."""
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(\w+)\s*\(", src)) - {"if", "defined", "sizeof"})
