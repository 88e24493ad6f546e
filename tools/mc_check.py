import ctypes as C
cuda = C.CDLL("libcuda.so.1")
cuda.cuInit(0)
dev = C.c_int()
cuda.cuDeviceGet(C.byref(dev), 0)
v = C.c_int()
# CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED = 132
r = cuda.cuDeviceGetAttribute(C.byref(v), 132, dev)
print("multicast supported:", r, v.value)
# fabric handle / nvlink
r = cuda.cuDeviceGetAttribute(C.byref(v), 128, dev); print("attr128 (HANDLE_TYPE_FABRIC?):", r, v.value)
