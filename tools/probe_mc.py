"""Probe NVLS multicast object creation on this GPU (driver API via ctypes).  Tooling only."""
import ctypes
cuda = ctypes.CDLL("libcuda.so.1")
print("cuInit", cuda.cuInit(0))
dev = ctypes.c_int()
cuda.cuDeviceGet(ctypes.byref(dev), 0)
ctx = ctypes.c_void_p()
print("ctx", cuda.cuDevicePrimaryCtxRetain(ctypes.byref(ctx), dev), cuda.cuCtxSetCurrent(ctx))
class Prop(ctypes.Structure):
    _fields_ = [("numDevices", ctypes.c_uint), ("size", ctypes.c_size_t), ("handleTypes", ctypes.c_ulonglong), ("flags", ctypes.c_ulonglong)]
for ht in (0, 1, 8):  # NONE, POSIX_FD, FABRIC
    for nd in (1, 2):
        p = Prop(nd, 1 << 21, ht, 0)
        g = ctypes.c_size_t()
        r1 = cuda.cuMulticastGetGranularity(ctypes.byref(g), ctypes.byref(p), 0)
        g2 = ctypes.c_size_t()
        r2 = cuda.cuMulticastGetGranularity(ctypes.byref(g2), ctypes.byref(p), 1)
        p.size = max(g.value, g2.value, 1 << 21)
        h = ctypes.c_ulonglong()
        r = cuda.cuMulticastCreate(ctypes.byref(h), ctypes.byref(p))
        print(f"handleTypes={ht} numDevices={nd} gran_min={g.value} (rc {r1}) gran_rec={g2.value} (rc {r2}) size={p.size} -> cuMulticastCreate rc {r}")
        if r == 0:
            print("  addDevice", cuda.cuMulticastAddDevice(h, dev))
            cuda.cuMemRelease(h)
v = ctypes.c_int()
for a in (132, 128, 103, 102):
    cuda.cuDeviceGetAttribute(ctypes.byref(v), a, dev); print("attr", a, v.value)
