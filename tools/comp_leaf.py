"""Config-1 leaf kernel with its output in compressible device memory (experiment).

The full-matrix output contract writes +0.0 over the upper triangle of every 32x32 inverse
(496 of 1024 entries, 16 of the 64 128-byte lines entirely zero).  tools/comp_probe.cu
showed that a cuMemCreate allocation with CU_MEM_ALLOCATION_COMP_GENERIC cuts the DRAM
write traffic of that pattern to 0.68.  This times trinv_batched into a cudaMalloc
(torch) output and into a compressible one, alternating, and checks the two results are
bitwise equal.  Usage: python tools/comp_leaf.py [steps]
"""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2307_07611_b200 as P  # noqa: E402
import synth  # noqa: E402


class _CompBuf:
    """cuMemCreate(CU_MEM_ALLOCATION_COMP_GENERIC) allocation exposed to torch through
    __cuda_array_interface__ (experiment only; libcuda through ctypes)."""

    def __init__(self, shape, device_index=0):
        cu = ctypes.CDLL("libcuda.so.1")
        self.cu = cu
        nbytes = int(np.prod(shape)) * 8

        class Loc(ctypes.Structure):
            _fields_ = [("type", ctypes.c_int), ("id", ctypes.c_int)]

        class Flags(ctypes.Structure):
            _fields_ = [("compressionType", ctypes.c_ubyte), ("gpuDirectRDMACapable", ctypes.c_ubyte),
                        ("usage", ctypes.c_ushort), ("reserved", ctypes.c_ubyte * 4)]

        class Prop(ctypes.Structure):
            _fields_ = [("type", ctypes.c_int), ("requestedHandleTypes", ctypes.c_int), ("location", Loc),
                        ("win32HandleMetaData", ctypes.c_void_p), ("allocFlags", Flags)]

        class Access(ctypes.Structure):
            _fields_ = [("location", Loc), ("flags", ctypes.c_int)]

        prop = Prop()
        prop.type = 1  # CU_MEM_ALLOCATION_TYPE_PINNED
        prop.location.type = 1  # CU_MEM_LOCATION_TYPE_DEVICE
        prop.location.id = device_index
        prop.allocFlags.compressionType = 1  # CU_MEM_ALLOCATION_COMP_GENERIC
        gran = ctypes.c_size_t()
        assert cu.cuMemGetAllocationGranularity(ctypes.byref(gran), ctypes.byref(prop), 1) == 0
        size = (nbytes + gran.value - 1) // gran.value * gran.value
        h = ctypes.c_ulonglong()
        assert cu.cuMemCreate(ctypes.byref(h), ctypes.c_size_t(size), ctypes.byref(prop), ctypes.c_ulonglong(0)) == 0
        got = Prop()
        assert cu.cuMemGetAllocationPropertiesFromHandle(ctypes.byref(got), h) == 0
        self.compressed = got.allocFlags.compressionType
        ptr = ctypes.c_ulonglong()
        assert cu.cuMemAddressReserve(ctypes.byref(ptr), ctypes.c_size_t(size), ctypes.c_size_t(0),
                                      ctypes.c_ulonglong(0), ctypes.c_ulonglong(0)) == 0
        assert cu.cuMemMap(ptr, ctypes.c_size_t(size), ctypes.c_size_t(0), h, ctypes.c_ulonglong(0)) == 0
        acc = Access()
        acc.location.type = 1
        acc.location.id = device_index
        acc.flags = 3  # READWRITE
        assert cu.cuMemSetAccess(ptr, ctypes.c_size_t(size), ctypes.byref(acc), ctypes.c_size_t(1)) == 0
        self.ptr, self.size, self.h = ptr.value, size, h
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": "<f8", "data": (self.ptr, False),
                                         "version": 2, "strides": None}


def main():
    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
    B, n = 131072, 32
    dev = torch.device("cuda:0")
    A = torch.from_numpy(synth.host(n, batch=B)).to(dev)
    Xp = torch.empty_like(A)
    buf = _CompBuf((B, n, n))
    Xc = torch.as_tensor(buf, device=dev)
    print("compressionType:", buf.compressed, "ptr", hex(Xc.data_ptr()), Xc.shape, Xc.dtype)
    s = torch.cuda.current_stream()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    res = {"plain": [], "compressible": []}
    for rep in range(3):
        for name, X in (("plain", Xp), ("compressible", Xc)):
            for _ in range(3):
                P.trinv_batched(A, out=X)
            torch.cuda.synchronize()
            for _ in range(steps):
                ev[0].record(s)
                P.trinv_batched(A, out=X)
                ev[1].record(s)
                ev[1].synchronize()
                res[name].append(ev[0].elapsed_time(ev[1]))
    eq = torch.equal(Xp, Xc)
    for name, t in res.items():
        med = float(np.median(t))
        print(f"{name:13s} median {med:.4f} ms  min {min(t):.4f}  inv/s {B / med * 1e3:.3e}  "
              f"frac(12416 B, 6549 GB/s) {B * 12416 / med / 1e6 / 6549.1:.3f}")
    print("bitwise equal:", eq)


if __name__ == "__main__":
    main()
