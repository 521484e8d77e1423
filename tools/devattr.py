import ctypes
rt = ctypes.CDLL("libcudart.so.12") if True else None
def attr(a):
    v = ctypes.c_int()
    rt.cudaDeviceGetAttribute(ctypes.byref(v), a, 0)
    return v.value
print("L2 bytes", attr(89), "max persisting L2", attr(108), "SMs", attr(16), "max smem/block optin", attr(97))
