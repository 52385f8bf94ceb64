"""Probe which cuMulticast* step works on this box (single device)."""
from cuda.bindings import driver as drv

drv.cuInit(0)
err, dev = drv.cuDeviceGet(0)
err, ctx = drv.cuDevicePrimaryCtxRetain(dev)
drv.cuCtxSetCurrent(ctx)
print("devcount", drv.cuDeviceGetCount())
H = drv.CUmemAllocationHandleType
for nd in (1, 2, 4, 8):
    for name, ht in [("posix", H.CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR), ("fabric", H.CU_MEM_HANDLE_TYPE_FABRIC)]:
        for size in (2 << 20, 32 << 20, 512 << 20):
            mp = drv.CUmulticastObjectProp()
            mp.numDevices = nd
            mp.handleTypes = ht
            mp.size = size
            mp.flags = 0
            r2 = drv.cuMulticastCreate(mp)
            print(nd, name, size, "create", r2[0])
            if r2[0] == drv.CUresult.CUDA_SUCCESS:
                print("   add", drv.cuMulticastAddDevice(r2[1], dev))
