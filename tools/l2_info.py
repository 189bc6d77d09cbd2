from cuda.bindings import runtime as rt
for name in ("cudaDevAttrL2CacheSize", "cudaDevAttrMaxPersistingL2CacheSize", "cudaDevAttrMaxAccessPolicyWindowSize",
             "cudaDevAttrMaxSharedMemoryPerMultiprocessor", "cudaDevAttrMaxSharedMemoryPerBlockOptin"):
    err, v = rt.cudaDeviceGetAttribute(getattr(rt.cudaDeviceAttr, name), 0)
    print(name, v, v / 2**20, "MiB")
