"""Does this box support multicast (NVLS) objects through torch symmetric memory?"""
import os
import torch
import torch.distributed as dist

local = int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
try:
    import torch.distributed._symmetric_memory as symm
    t = symm.empty(1 << 20, dtype=torch.float32, device=f"cuda:{local}")
    h = symm.rendezvous(t, dist.group.WORLD.group_name)
    print(dist.get_rank(), "multicast", getattr(h, "has_multicast_support", None), "mc_ptr",
          hex(getattr(h, "multicast_ptr", 0) or 0), "buffers", [hex(p) for p in h.buffer_ptrs], flush=True)
    try:
        print(dist.get_rank(), "is_nvshmem", symm.is_nvshmem_available() if hasattr(symm, "is_nvshmem_available") else None)
    except Exception as ex:
        print("nvshmem query", repr(ex))
except Exception as ex:
    print(dist.get_rank(), "symm mem failed:", repr(ex)[:400], flush=True)
dist.barrier()
dist.destroy_process_group()
