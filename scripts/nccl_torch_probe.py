"""Probe: torch.distributed NCCL world of one (init, all_reduce), step-by-step prints."""
import os, time
import torch
import torch.distributed as dist
t0 = time.time()
log = lambda *a: print(f"[{time.time() - t0:7.2f}s]", *a, flush=True)
os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29533")
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
log("init ok")
t = torch.ones(4, device="cuda")
dist.all_reduce(t)
torch.cuda.synchronize()
log("all_reduce ok", t.tolist())
dist.destroy_process_group()
log("done")
