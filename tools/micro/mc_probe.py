import torch
torch.cuda.init(); torch.zeros(1, device="cuda")
from cuda.bindings import driver as d
print("init", d.cuInit(0))
err, dev = d.cuDeviceGet(0)
for ht_name in ("CU_MEM_HANDLE_TYPE_NONE", "CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR", "CU_MEM_HANDLE_TYPE_FABRIC"):
    ht = getattr(d.CUmemAllocationHandleType, ht_name)
    p = d.CUmulticastObjectProp()
    p.numDevices = 1
    p.handleTypes = ht
    p.size = 2 << 20
    r = d.cuMulticastGetGranularity(p, d.CUmulticastGranularity_flags.CU_MULTICAST_GRANULARITY_RECOMMENDED)
    print(ht_name, "granularity", r)
    if r[0] == d.CUresult.CUDA_SUCCESS:
        p.size = max(r[1], 2 << 20)
    r2 = d.cuMulticastCreate(p)
    print(ht_name, "create", r2[0])
    if r2[0] == d.CUresult.CUDA_SUCCESS:
        print(ht_name, "add device", d.cuMulticastAddDevice(r2[1], dev))
