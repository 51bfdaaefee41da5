import torch
p=torch.cuda.get_device_properties(0)
import ctypes
lib=ctypes.CDLL("libcudart.so.12") if False else None
from cuda.bindings import runtime as rt
for a in ["cudaDevAttrPageableMemoryAccess","cudaDevAttrPageableMemoryAccessUsesHostPageTables","cudaDevAttrConcurrentManagedAccess","cudaDevAttrHostRegisterSupported"]:
    err,v=rt.cudaDeviceGetAttribute(getattr(rt.cudaDeviceAttr,a),0); print(a,v)
