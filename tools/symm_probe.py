"""Probe torch symmetric memory on this box (dev tool): peer pointers,
multicast, device barrier. torchrun --nproc-per-node 2 tools/symm_probe.py"""
import os
import torch
import torch.distributed as dist
import torch.distributed._symmetric_memory as symm

rank = int(os.environ.get("RANK", 0)); world = int(os.environ.get("WORLD_SIZE", 1))
local = int(os.environ.get("LOCAL_RANK", 0)) % torch.cuda.device_count()
torch.cuda.set_device(local)
dist.init_process_group(os.environ.get("OPSC_DIST_BACKEND", "nccl"))
print(rank, "backend", symm.get_backend(torch.device("cuda", local)) if hasattr(symm, "get_backend") else None, flush=True)
try:
    t = symm.empty(16, dtype=torch.int64, device=f"cuda:{local}")
    h = symm.rendezvous(t, dist.group.WORLD.group_name)
    print(rank, "ptrs", [hex(p) for p in h.buffer_ptrs], "mc", hex(h.multicast_ptr) if hasattr(h, "multicast_ptr") else None,
          "signal", len(h.signal_pad_ptrs), flush=True)
    t.fill_(rank)
    h.barrier(channel=0)
    peer = h.get_buffer((rank + 1) % world, (16,), torch.int64)
    torch.cuda.synchronize()
    print(rank, "peer view", peer[:4].tolist(), flush=True)
    h.barrier(channel=0)
except Exception as e:
    import traceback; traceback.print_exc()
dist.destroy_process_group()
