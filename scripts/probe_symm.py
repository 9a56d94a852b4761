# Probe: torch symmetric memory + NVLS multicast availability on this box.
import os, torch, torch.distributed as dist
import torch.distributed._symmetric_memory as symm_mem
local = int(os.environ.get("LOCAL_RANK", "0"))
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
try:
    print("backend", symm_mem.get_backend(torch.device("cuda", local)) if hasattr(symm_mem, "get_backend") else "?")
except Exception as e:
    print("get_backend err", e)
t = symm_mem.empty(1 << 20, dtype=torch.float32, device="cuda")
h = symm_mem.rendezvous(t, dist.group.WORLD.group_name)
print(dist.get_rank(), "multicast_ptr", hex(h.multicast_ptr) if h.multicast_ptr else h.multicast_ptr,
      "buffer_ptrs", [hex(p) for p in h.buffer_ptrs], "signal_pad_ptrs", [hex(p) for p in h.signal_pad_ptrs],
      "signal_pad_size", getattr(h, "signal_pad_size", None), "world", h.world_size, "rank", h.rank)
import subprocess
print(subprocess.run(["nvidia-smi", "-q", "-d", "FABRIC"], capture_output=True, text=True).stdout[-600:] if dist.get_rank() == 0 else "")
dist.barrier()
dist.destroy_process_group()
