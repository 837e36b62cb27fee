"""Probe: torch symmetric memory and NVLink multicast on this box (world size 1)."""
import os
import torch
import torch.distributed as dist

os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29655")
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
import torch.distributed._symmetric_memory as symm_mem
from cuda.bindings import driver as drv

dev = torch.cuda.current_device()
print("multicast supported attr:", drv.cuDeviceGetAttribute(drv.CUdevice_attribute.CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev))
try:
    t = symm_mem.empty(1 << 20, dtype=torch.float32, device="cuda")
    h = symm_mem.rendezvous(t, dist.group.WORLD.group_name)
    print("rendezvous ok; multicast_ptr:", getattr(h, "multicast_ptr", None), "buffer_ptrs:", h.buffer_ptrs[:1])
except Exception as e:
    print("symm_mem failed:", type(e).__name__, e)
dist.destroy_process_group()
