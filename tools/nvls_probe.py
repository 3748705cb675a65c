"""Probe multicast (NVLS) object creation with POSIX-FD handles on this box."""
from cuda.bindings import driver as d


def ck(r):
    return r if not isinstance(r, tuple) else (r[0], r[1] if len(r) == 2 else r[1:])


print(ck(d.cuInit(0)))
_, dev = ck(d.cuDeviceGet(0))
_, ctx = ck(d.cuDevicePrimaryCtxRetain(dev))
print(ck(d.cuCtxSetCurrent(ctx)))
FD = d.CUmemAllocationHandleType.CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR
ap = d.CUmemAllocationProp()
ap.type = d.CUmemAllocationType.CU_MEM_ALLOCATION_TYPE_PINNED
ap.location.type = d.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
ap.location.id = 0
ap.requestedHandleTypes = FD
err, h = ck(d.cuMemCreate(1 << 21, ap, 0))
print("memcreate fd", err)
print("export fd", ck(d.cuMemExportToShareableHandle(h, FD, 0)))
prop = d.CUmulticastObjectProp()
prop.numDevices = 2
prop.size = 1 << 21
prop.handleTypes = FD
err, mc = ck(d.cuMulticastCreate(prop))
print("mc create fd", err)
if err == d.CUresult.CUDA_SUCCESS:
    print("mc add dev", ck(d.cuMulticastAddDevice(mc, dev)))
    print("mc export", ck(d.cuMemExportToShareableHandle(mc, FD, 0)))
