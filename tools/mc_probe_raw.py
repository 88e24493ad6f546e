"""Experiment helper (GPU box): cuMulticastCreate straight through libcuda
with a grid of (numDevices, size, handleTypes)."""
import ctypes as C

cuda = C.CDLL("libcuda.so.1")
print("init", cuda.cuInit(0))
dev = C.c_int()
cuda.cuDeviceGet(C.byref(dev), 0)
ctx = C.c_void_p()
print("retain primary", cuda.cuDevicePrimaryCtxRetain(C.byref(ctx), dev), "set", cuda.cuCtxSetCurrent(ctx))


class Prop(C.Structure):
    _fields_ = [("numDevices", C.c_uint), ("size", C.c_size_t), ("handleTypes", C.c_ulonglong),
                ("flags", C.c_ulonglong)]


for ht in (0, 1, 8):
    p = Prop(1, 2 << 20, ht, 0)
    g = C.c_size_t()
    r0 = cuda.cuMulticastGetGranularity(C.byref(g), C.byref(p), 0)
    r1 = cuda.cuMulticastGetGranularity(C.byref(g), C.byref(p), 1)
    print("ht", ht, "gran rc", r0, r1, "gran", g.value)
    for ndev in (1, 2):
        for size in (2 << 20, g.value or (2 << 20), 1 << 30):
            p = Prop(ndev, size, ht, 0)
            h = C.c_ulonglong()
            r = cuda.cuMulticastCreate(C.byref(h), C.byref(p))
            print(f"  ndev {ndev} size {size}: {r}")
            if r == 0:
                cuda.cuMemRelease(h)
