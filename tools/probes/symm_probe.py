import os, torch, torch.distributed as dist
import torch.distributed._symmetric_memory as sm
os.environ.setdefault("MASTER_ADDR", "127.0.0.1"); os.environ.setdefault("MASTER_PORT", "29555")
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda:0"))
t = sm.empty(1024, dtype=torch.uint8, device="cuda:0")
h = sm.rendezvous(t, dist.group.WORLD)
print("world", h.world_size, "rank", h.rank, "bufptrs", h.buffer_ptrs, "dev", hex(h.buffer_ptrs_dev), "sig", h.signal_pad_ptrs, hex(h.signal_pad_ptrs_dev), "sigsize", h.signal_pad_size)
dist.destroy_process_group()
