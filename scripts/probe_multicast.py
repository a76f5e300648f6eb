"""Probe (GPU box): is NVLS multicast available to one process on one GPU?
Prints the driver's CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED and what torch's
symmetric memory rendezvous (world size 1, NCCL) returns for multicast_ptr."""
import os
import torch
import torch.distributed as dist

import cuda.bindings.driver as drv

drv.cuInit(0)
err, dev = drv.cuDeviceGet(0)
err, mc = drv.cuDeviceGetAttribute(drv.CUdevice_attribute.CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev)
print("driver multicast supported:", err, mc, flush=True)
os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29531")
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda:0"))
import torch.distributed._symmetric_memory as symm
try:
    t = symm.empty(1 << 20, dtype=torch.float64, device="cuda:0")
    h = symm.rendezvous(t, dist.group.WORLD)
    print("symm backend:", symm.get_backend(torch.device("cuda:0")) if hasattr(symm, "get_backend") else "?")
    print("multicast_ptr:", h.multicast_ptr, "buffer_ptrs:", h.buffer_ptrs, "world:", h.world_size, flush=True)
except Exception as e:   # report, do not fail the probe
    print("symmetric memory failed:", type(e).__name__, e, flush=True)
dist.destroy_process_group()
