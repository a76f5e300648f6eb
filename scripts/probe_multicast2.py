"""Probe (GPU box): which cuMulticastCreate properties the driver accepts."""
import cuda.bindings.driver as drv

print(drv.cuInit(0))
err, dev = drv.cuDeviceGet(0)
err, ctx = drv.cuDevicePrimaryCtxRetain(dev)
print("ctx", err, drv.cuCtxSetCurrent(ctx))
for attr in ("CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED", "CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED",
             "CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR_SUPPORTED"):
    print(attr, drv.cuDeviceGetAttribute(getattr(drv.CUdevice_attribute, attr), dev))
H = drv.CUmemAllocationHandleType
for ht in (0, H.CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, H.CU_MEM_HANDLE_TYPE_FABRIC):
    for nd in (1, 2):
        p = drv.CUmulticastObjectProp()
        p.numDevices = nd
        p.handleTypes = int(ht)
        p.size = 2 << 20
        e1, mg = drv.cuMulticastGetGranularity(p, drv.CUmulticastGranularity_flags.CU_MULTICAST_GRANULARITY_MINIMUM)
        e2, rg = drv.cuMulticastGetGranularity(p, drv.CUmulticastGranularity_flags.CU_MULTICAST_GRANULARITY_RECOMMENDED)
        p.size = max(int(mg or 0), int(rg or 0), 2 << 20)
        e3, mc = drv.cuMulticastCreate(p)
        print("handle", int(ht), "ndev", nd, "gran", e1, mg, e2, rg, "size", p.size, "create", e3, flush=True)
        if e3 == drv.CUresult.CUDA_SUCCESS:
            print("  add", drv.cuMulticastAddDevice(mc, dev))
            drv.cuMemRelease(mc)
