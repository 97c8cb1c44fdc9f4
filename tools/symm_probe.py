"""Probe torch symmetric memory (peer pointers, NVLS multicast) under torchrun."""
import os

import torch
import torch.distributed as dist
import torch.distributed._symmetric_memory as symm

local = int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
r, w = dist.get_rank(), dist.get_world_size()
try:
    print(r, "backend", symm.get_backend(torch.device("cuda", local)), flush=True)
except Exception as e:
    print(r, "get_backend failed", e)
t = symm.empty(1 << 20, dtype=torch.bfloat16, device=f"cuda:{local}")
t.fill_(r + 1)
h = symm.rendezvous(t, dist.group.WORLD.group_name)
mc = getattr(h, "multicast_ptr", None)
print(r, "ptrs", [hex(p) for p in h.buffer_ptrs], "mc", hex(mc) if mc else mc,
      "has_mc", symm._SymmetricMemory.has_multicast_support(torch._C._autograd.DeviceType.CUDA, local)
      if hasattr(torch._C, "_autograd") else None,
      "signal_pad", h.signal_pad_size, flush=True)
h.barrier()
peer = h.get_buffer((r + 1) % w, (1 << 20,), torch.bfloat16)
print(r, "peer sum", peer.float().sum().item(), "expect", float(((r + 1) % w + 1) * (1 << 20)), flush=True)
torch.cuda.synchronize()
h.barrier()
dist.destroy_process_group()
