import os, torch, torch.distributed as dist
os.environ.setdefault("MASTER_ADDR","127.0.0.1"); os.environ.setdefault("MASTER_PORT","29533")
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda",0))
import torch.distributed._symmetric_memory as sm
t = sm.empty(4, 4, dtype=torch.int32, device="cuda:0")
h = sm.rendezvous(t, dist.group.WORLD)
print("symm ok", h.buffer_ptrs, t.data_ptr(), sm.get_backend(torch.device("cuda",0)) if hasattr(sm,"get_backend") else None)
dist.destroy_process_group()
