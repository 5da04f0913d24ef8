"""Seeded synthetic inputs for tests and bench (no method arithmetic; see synth.h).

Host generator: libsynth.so (C, OpenMP).  Device twin: libsynth_cuda.so.
`entry_py` is a pure-Python restatement used to pin both on tiny cases.
"""
import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "libsynth.so")
_SO_CUDA = os.path.join(_HERE, "libsynth_cuda.so")
DIAG = {"signed": 0, "pos": 1, "one": 2}
TAGS = {None: 0, "L": ord("L"), "U": ord("U")}
_lib = None
_libc = None
M64 = (1 << 64) - 1
G = 0x9E3779B97F4A7C15


def build(force=False, cuda=True):
    src = os.path.join(_HERE, "synth.c")
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(src):
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fopenmp", "-fPIC", "-shared",
                               "-o", _SO, src])
    if cuda:
        csrc = os.path.join(_HERE, "synth_cuda.cu")
        if force or not os.path.exists(_SO_CUDA) or os.path.getmtime(_SO_CUDA) < os.path.getmtime(csrc):
            subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3",
                                   "-fmad=false", "-Xcompiler", "-fPIC", "-shared", "-o", _SO_CUDA,
                                   csrc])


def _host():
    global _lib
    if _lib is None:
        build(cuda=False)
        L = ctypes.CDLL(_SO)
        L.synth_fill_host.argtypes = [ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_uint64,
                                      ctypes.c_uint64, ctypes.c_char, ctypes.c_int,
                                      ctypes.POINTER(ctypes.c_double), ctypes.c_int64, ctypes.c_int64]
        _lib = L
    return _lib


def _dev():
    global _libc
    if _libc is None:
        if not os.path.exists(_SO_CUDA):
            build(cuda=True)
        L = ctypes.CDLL(_SO_CUDA)
        L.synth_fill_device.argtypes = [ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_uint64,
                                        ctypes.c_uint64, ctypes.c_char, ctypes.c_int, ctypes.c_void_p,
                                        ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p]
        L.synth_fill_device.restype = ctypes.c_int
        _libc = L
    return _libc


def host(n, batch=None, b0=0, seed=0, tag=None, uplo="L", diag="signed"):
    """numpy [batch, n, n] (or [n, n] if batch is None) on the host."""
    cnt = 1 if batch is None else batch
    out = np.empty((cnt, n, n), dtype=np.float64)
    _host().synth_fill_host(n, b0, cnt, seed, TAGS.get(tag, tag if isinstance(tag, int) else 0),
                            uplo.encode(), DIAG[diag],
                            out.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), n, n * n)
    return out[0] if batch is None else out


def device_fill(t, n, b0=0, seed=0, tag=None, uplo="L", diag="signed", ld=None, stride=None, stream=None):
    """Fill a CUDA torch tensor (float64) in place with the same values as host()."""
    import torch
    cnt = 1 if t.dim() == 2 else t.shape[0]
    ld = n if ld is None else ld
    stride = n * ld if stride is None else stride
    s = torch.cuda.current_stream().cuda_stream if stream is None else stream
    rc = _dev().synth_fill_device(n, b0, cnt, seed, TAGS.get(tag, 0), uplo.encode(), DIAG[diag],
                                  ctypes.c_void_p(t.data_ptr()), ld, stride, ctypes.c_void_p(s))
    if rc != 0:
        raise RuntimeError(f"synth_fill_device failed: cuda error {rc}")
    return t


# --- pure-Python restatement (tiny sizes only) ---------------------------------
def _mix(z):
    z &= M64
    z ^= z >> 30; z = (z * 0xBF58476D1CE4E5B9) & M64
    z ^= z >> 27; z = (z * 0x94D049BB133111EB) & M64
    z ^= z >> 31
    return z


def entry_py(seed, tag, n, i, j, uplo="L", diag="signed"):
    if (uplo == "L" and i < j) or (uplo == "U" and i > j):
        return 0.0
    key = _mix(_mix(seed ^ G) ^ TAGS.get(tag, 0))
    idx = i * n + j
    h = _mix((key + (2 * idx + 1) * G) & M64)
    u = (h >> 11) * 2.0 ** -53
    if i != j:
        return (2.0 * u - 1.0) / n
    if diag == "one":
        return 1.0
    d = 1.0 + u
    if diag == "signed" and (_mix((key + (2 * idx + 2) * G) & M64) >> 63):
        d = -d
    return d
