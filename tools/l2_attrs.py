import torch
from cuda.bindings import runtime as rt   # cuda-python
for name in ["cudaDevAttrMaxPersistingL2CacheSize", "cudaDevAttrMaxAccessPolicyWindowSize", "cudaDevAttrL2CacheSize"]:
    err, v = rt.cudaDeviceGetAttribute(getattr(rt.cudaDeviceAttr, name), 0)
    print(name, err, v)
