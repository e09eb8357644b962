"""NCCL allgather bandwidth vs message size on this box (torchrun, N ranks)."""
import json
import os

import torch
import torch.distributed as dist

ws = int(os.environ["WORLD_SIZE"]); rank = int(os.environ["RANK"])
torch.cuda.set_device(rank)
dist.init_process_group("nccl")
res = {}
for mb in [1, 4, 16, 34.6, 64, 128]:
    n = int(mb * 1e6)
    x = torch.empty(n, dtype=torch.uint8, device="cuda")
    y = torch.empty(n * ws, dtype=torch.uint8, device="cuda")
    for _ in range(5):
        dist.all_gather_into_tensor(y, x)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        dist.all_gather_into_tensor(y, x)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    res[mb] = {"us": round(ms * 1e3, 1), "busbw_GBps": round(n * (ws - 1) / (ms * 1e-3) / 1e9, 1)}
if rank == 0:
    print(json.dumps({"ws": ws, "env": {k: v for k, v in os.environ.items() if k.startswith("NCCL")}, "allgather": res}))
dist.destroy_process_group()
