"""Test infrastructure: device buffers reachable through an NVLS multicast
object on ONE GPU (cuda-python driver API).  Each buffer is physical memory
from cuMemCreate, mapped twice -- at a unicast address (wrapped as a torch
tensor) and, through a one-device multicast object (cuMulticastCreate /
cuMulticastAddDevice / cuMulticastBindMem), at a multicast address on which
multimem.ld_reduce / multimem.st operate.  At world size 1 the multicast
"sum over ranks" is the buffer itself, so the multicast kernels can be
checked bit for bit against the plain ones.  (At world size > 1 torch
symmetric memory provides the same object spanning every rank.)"""
from cuda.bindings import driver as cu


def _ck(r):
    err = r[0] if isinstance(r, tuple) else r
    if err != cu.CUresult.CUDA_SUCCESS:
        raise RuntimeError(f"CUDA driver call failed: {err}")
    if isinstance(r, tuple):
        return r[1] if len(r) == 2 else r[1:]
    return None


def multicast_supported(dev: int = 0):
    """(ok, reason): the device attribute AND an actual one-device
    multicast object (a GPU can report support while the process has no
    access to the NVSwitch fabric, e.g. a one-GPU container: cuMulticastCreate
    then fails with CUDA_ERROR_INVALID_VALUE)."""
    import torch
    torch.cuda.init()
    _ck(cu.cuInit(0))
    d = _ck(cu.cuDeviceGet(dev))
    if not _ck(cu.cuDeviceGetAttribute(cu.CUdevice_attribute.CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, d)):
        return False, "CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED = 0"
    mp = cu.CUmulticastObjectProp()
    mp.numDevices = 1
    mp.handleTypes = cu.CUmemAllocationHandleType.CU_MEM_HANDLE_TYPE_NONE
    mp.size = 2 << 20
    err, h = cu.cuMulticastCreate(mp)
    if err != cu.CUresult.CUDA_SUCCESS:
        return False, f"cuMulticastCreate: {err} (no NVSwitch multicast access in this process)"
    cu.cuMemRelease(h)
    return True, ""


class _CAI:
    def __init__(self, ptr, n, typestr):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr, "data": (ptr, False), "version": 3}


class McBuffer:
    def __init__(self, nbytes: int, dev: int = 0):
        import torch
        torch.cuda.init()
        _ck(cu.cuInit(0))
        self.dev = _ck(cu.cuDeviceGet(dev))
        mp = cu.CUmulticastObjectProp()
        mp.numDevices = 1
        mp.handleTypes = cu.CUmemAllocationHandleType.CU_MEM_HANDLE_TYPE_NONE
        mp.size = nbytes
        g_mc = _ck(cu.cuMulticastGetGranularity(mp, cu.CUmulticastGranularity_flags.CU_MULTICAST_GRANULARITY_RECOMMENDED))
        ap = cu.CUmemAllocationProp()
        ap.type = cu.CUmemAllocationType.CU_MEM_ALLOCATION_TYPE_PINNED
        ap.location.type = cu.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
        ap.location.id = dev
        g_mem = _ck(cu.cuMemGetAllocationGranularity(ap, cu.CUmemAllocationGranularity_flags.CU_MEM_ALLOC_GRANULARITY_RECOMMENDED))
        g = max(int(g_mc), int(g_mem))
        self.size = (nbytes + g - 1) // g * g
        mp.size = self.size
        self.mc = _ck(cu.cuMulticastCreate(mp))
        _ck(cu.cuMulticastAddDevice(self.mc, self.dev))
        self.mem = _ck(cu.cuMemCreate(self.size, ap, 0))
        _ck(cu.cuMulticastBindMem(self.mc, 0, self.mem, 0, self.size, 0))
        acc = cu.CUmemAccessDesc()
        acc.location.type = cu.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
        acc.location.id = dev
        acc.flags = cu.CUmemAccess_flags.CU_MEM_ACCESS_FLAGS_PROT_READWRITE
        self.uva = int(_ck(cu.cuMemAddressReserve(self.size, g, 0, 0)))
        _ck(cu.cuMemMap(self.uva, self.size, 0, self.mem, 0))
        _ck(cu.cuMemSetAccess(self.uva, self.size, [acc], 1))
        self.mva = int(_ck(cu.cuMemAddressReserve(self.size, g, 0, 0)))
        _ck(cu.cuMemMap(self.mva, self.size, 0, self.mc, 0))
        _ck(cu.cuMemSetAccess(self.mva, self.size, [acc], 1))

    def tensor(self, n, dtype):
        import torch
        ts = {torch.float32: "<f4", torch.float16: "<f2", torch.bfloat16: "<V2"}[dtype]
        if dtype == torch.bfloat16:
            raise ValueError("bf16 not needed")
        t = torch.as_tensor(_CAI(self.uva, n, ts), device="cuda")
        t._mc_owner = self   # keep the mapping alive with the tensor
        return t


class McAllocator:
    """Trainer(alloc=...) hook: every buffer it hands out has a multicast
    twin; mc(t) returns the multicast address of tensor t's first element."""

    def __init__(self):
        self.bufs = []

    def __call__(self, n, dtype, device):
        import torch
        esz = torch.tensor([], dtype=dtype).element_size()
        b = McBuffer(n * esz)
        self.bufs.append(b)
        t = b.tensor(n, dtype)
        t.zero_()
        return t

    def mc(self, t) -> int:
        p = t.data_ptr()
        for b in self.bufs:
            if b.uva <= p < b.uva + b.size:
                return b.mva + (p - b.uva)
        raise KeyError("tensor not from this allocator")
