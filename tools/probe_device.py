"""Print device attributes relevant to kernel design (L2 persistence etc.)."""
from cuda.bindings import runtime as rt

attrs = ["cudaDevAttrL2CacheSize", "cudaDevAttrMaxPersistingL2CacheSize",
         "cudaDevAttrMaxAccessPolicyWindowSize", "cudaDevAttrMultiProcessorCount",
         "cudaDevAttrMaxSharedMemoryPerBlockOptin", "cudaDevAttrMaxSharedMemoryPerMultiprocessor",
         "cudaDevAttrClockRate", "cudaDevAttrMemoryClockRate", "cudaDevAttrGlobalMemoryBusWidth"]
for a in attrs:
    err, v = rt.cudaDeviceGetAttribute(getattr(rt.cudaDeviceAttr, a), 0)
    print(a, v)
