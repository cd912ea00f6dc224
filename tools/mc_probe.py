"""NVLS multicast / symmetric-memory availability probe (measurement tool)."""
import os, torch, torch.distributed as dist
os.environ.setdefault("MASTER_ADDR", "127.0.0.1"); os.environ.setdefault("MASTER_PORT", "29533")
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
print("multicast supported attr:", torch.cuda.get_device_properties(0))
try:
    import torch.distributed._symmetric_memory as symm_mem
    t = symm_mem.empty(1024, dtype=torch.float32, device="cuda")
    h = symm_mem.rendezvous(t, dist.group.WORLD)
    print("symm handle:", type(h), "multicast_ptr:", getattr(h, "multicast_ptr", None))
    print("buffer ptrs:", getattr(h, "buffer_ptrs", None))
except Exception as e:
    print("symm_mem failed:", repr(e))
try:
    from cuda.bindings import driver as cu
    cu.cuInit(0)
    err, dev = cu.cuDeviceGet(0)
    err, v = cu.cuDeviceGetAttribute(cu.CUdevice_attribute.CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev)
    print("CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED:", err, v)
except Exception as e:
    print("cuda-python probe failed:", repr(e))
dist.destroy_process_group()
