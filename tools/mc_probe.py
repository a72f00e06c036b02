"""Dev tool: does torch symmetric memory give a multicast (NVLS) pointer on this box?"""
import os, sys
import torch
import torch.distributed as dist
rank = int(os.environ["RANK"]); ws = int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dist.init_process_group("nccl", device_id=torch.device("cuda", rank))
try:
    import torch.distributed._symmetric_memory as symm_mem
    t = symm_mem.empty((1024, 1024), dtype=torch.bfloat16, device=f"cuda:{rank}")
    hdl = symm_mem.rendezvous(t, dist.group.WORLD)
    mc = getattr(hdl, "multicast_ptr", None)
    print(rank, "symm ok", "buffer_ptrs", [hex(p) for p in hdl.buffer_ptrs][:2], "multicast_ptr", mc, flush=True)
except Exception as e:
    print(rank, "symm failed:", repr(e)[:300], flush=True)
dist.destroy_process_group()
