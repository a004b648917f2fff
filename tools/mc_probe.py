"""Which multicast-object setups does this GPU accept? (driver API, one device)"""
import torch
from cuda.bindings import driver as d

torch.zeros(1, device="cuda")
dev = d.cuDeviceGet(0)[1]
print("MULTICAST_SUPPORTED", d.cuDeviceGetAttribute(d.CUdevice_attribute.CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev))
for name in ("CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED", "CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR_SUPPORTED",
             "CU_DEVICE_ATTRIBUTE_VIRTUAL_MEMORY_MANAGEMENT_SUPPORTED"):
    a = getattr(d.CUdevice_attribute, name, None)
    if a is not None:
        print(name, d.cuDeviceGetAttribute(a, dev))
for hname in ("CU_MEM_HANDLE_TYPE_NONE", "CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR", "CU_MEM_HANDLE_TYPE_FABRIC"):
    for nd in (1, 2):
        prop = d.CUmulticastObjectProp()
        prop.numDevices = nd
        prop.handleTypes = getattr(d.CUmemAllocationHandleType, hname)
        prop.size = 2 << 20
        g = d.cuMulticastGetGranularity(prop, d.CUmulticastGranularity_flags.CU_MULTICAST_GRANULARITY_RECOMMENDED)
        prop.size = max(int(g[1]) if g[0] == d.CUresult.CUDA_SUCCESS else 0, 2 << 20)
        r = d.cuMulticastCreate(prop)
        msg = [hname, nd, "gran", g, "create", r[0]]
        if r[0] == d.CUresult.CUDA_SUCCESS:
            msg += ["add", d.cuMulticastAddDevice(r[1], dev)]
        print(*msg)
