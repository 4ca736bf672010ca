import ctypes
rt = ctypes.CDLL("libcudart.so")
def attr(a):
    v = ctypes.c_int()
    rt.cudaDeviceGetAttribute(ctypes.byref(v), a, 0)
    return v.value
# cudaDevAttrL2CacheSize=89, cudaDevAttrMaxPersistingL2CacheSize=108, cudaDevAttrMaxAccessPolicyWindowSize=109
print("L2", attr(89), "maxPersist", attr(108), "maxWindow", attr(109))
