import ctypes, numpy as np, torch
cudart = ctypes.CDLL("libcudart.so.12") if False else None
torch.cuda.init()
from cuda.bindings import runtime as rt
err, v = rt.cudaDeviceGetAttribute(rt.cudaDeviceAttr.cudaDevAttrPageableMemoryAccess, 0); print("pageableMemoryAccess", v)
err, v = rt.cudaDeviceGetAttribute(rt.cudaDeviceAttr.cudaDevAttrPageableMemoryAccessUsesHostPageTables, 0); print("usesHostPageTables", v)
err, v = rt.cudaDeviceGetAttribute(rt.cudaDeviceAttr.cudaDevAttrConcurrentManagedAccess, 0); print("concurrentManaged", v)
err, v = rt.cudaDeviceGetAttribute(rt.cudaDeviceAttr.cudaDevAttrHostRegisterSupported, 0); print("hostRegister", v)
# straddle probe: big buffer, register the middle page span, copy a range straddling its end
buf = np.zeros(1 << 20)
addr = buf.ctypes.data
pg = 4096
a = (addr + 10 * pg) & ~(pg - 1)
e = rt.cudaHostRegister(a, 4 * pg, rt.cudaHostRegisterMapped | rt.cudaHostRegisterPortable)
print("register", e)
off = (a - addr) // 8 + 4 * pg // 8 - 100  # starts inside the registered span, ends beyond
sub = buf[off: off + 1000]
t = torch.from_numpy(sub)
try:
    g = t.cuda(); torch.cuda.synchronize(); print("H2D straddle ok")
except Exception as ex:
    print("H2D straddle FAILED", ex)
try:
    g = torch.ones(1000, dtype=torch.float64, device="cuda")
    t.copy_(g); torch.cuda.synchronize(); print("D2H straddle ok")
except Exception as ex:
    print("D2H straddle FAILED", ex)
print(rt.cudaGetLastError())
