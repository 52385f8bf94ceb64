"""Test-only NVLS multicast buffer on ONE device (cuda-python driver API).

torch symmetric memory cannot export a multicast handle on the single-GPU test boxes
(no IMEX channel for fabric handles), so the multimem kernel is exercised here on a
multicast object of one device made in-process: cuMulticastCreate(numDevices=1),
cuMulticastAddDevice, one physical allocation bound to it, and two virtual mappings of
that allocation: the unicast one (plain loads / stores) and the multicast one (what
multimem.ld_reduce / multimem.st address).  With one device in the group the in-switch
sum has a single term, so the result must equal the unicast kernel's bit for bit."""
import torch
from cuda.bindings import driver as drv


def _ok(res):
    err = res[0] if isinstance(res, tuple) else res
    if err != drv.CUresult.CUDA_SUCCESS:
        raise RuntimeError(f"CUDA driver: {err}")
    return res[1] if isinstance(res, tuple) and len(res) == 2 else res[1:] if isinstance(res, tuple) else None


class _Cai:
    def __init__(self, ptr, n):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f4", "data": (ptr, False), "version": 3}


class MulticastBuffer:
    """n fp32 values; .tensor = the unicast view (a torch tensor), .mc = the multicast
    virtual address (int)."""

    def __init__(self, n, device=0):
        _ok(drv.cuInit(0))
        dev = _ok(drv.cuDeviceGet(device))
        if not _ok(drv.cuDeviceGetAttribute(drv.CUdevice_attribute.CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev)):
            raise RuntimeError("device has no multicast support")
        ht = drv.CUmemAllocationHandleType.CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR
        mp = drv.CUmulticastObjectProp()
        mp.numDevices = 1
        mp.handleTypes = ht
        mp.size = n * 4
        gran = _ok(drv.cuMulticastGetGranularity(
            mp, drv.CUmulticastGranularity_flags.CU_MULTICAST_GRANULARITY_RECOMMENDED))
        size = (n * 4 + gran - 1) // gran * gran
        mp.size = size
        self.mch = _ok(drv.cuMulticastCreate(mp))
        _ok(drv.cuMulticastAddDevice(self.mch, dev))
        ap = drv.CUmemAllocationProp()
        ap.type = drv.CUmemAllocationType.CU_MEM_ALLOCATION_TYPE_PINNED
        ap.location.type = drv.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
        ap.location.id = device
        ap.requestedHandleTypes = ht
        self.mem = _ok(drv.cuMemCreate(size, ap, 0))
        _ok(drv.cuMulticastBindMem(self.mch, 0, self.mem, 0, size, 0))
        acc = drv.CUmemAccessDesc()
        acc.location.type = drv.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
        acc.location.id = device
        acc.flags = drv.CUmemAccess_flags.CU_MEM_ACCESS_FLAGS_PROT_READWRITE
        self.uc = _ok(drv.cuMemAddressReserve(size, gran, 0, 0))
        _ok(drv.cuMemMap(self.uc, size, 0, self.mem, 0))
        _ok(drv.cuMemSetAccess(self.uc, size, [acc], 1))
        self.mcva = _ok(drv.cuMemAddressReserve(size, gran, 0, 0))
        _ok(drv.cuMemMap(self.mcva, size, 0, self.mch, 0))
        _ok(drv.cuMemSetAccess(self.mcva, size, [acc], 1))
        self.size, self.dev = size, dev
        self.tensor = torch.as_tensor(_Cai(int(self.uc), n), device=f"cuda:{device}")
        self.mc = int(self.mcva)

    def close(self):
        torch.cuda.synchronize()
        self.tensor = None
        _ok(drv.cuMemUnmap(self.mcva, self.size))
        _ok(drv.cuMemUnmap(self.uc, self.size))
        _ok(drv.cuMemAddressFree(self.mcva, self.size))
        _ok(drv.cuMemAddressFree(self.uc, self.size))
        _ok(drv.cuMulticastUnbind(self.mch, self.dev, 0, self.size))
        _ok(drv.cuMemRelease(self.mem))
        _ok(drv.cuMemRelease(self.mch))
