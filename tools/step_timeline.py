"""Per-kernel timeline of tgb_step (events around every launch on its own stream).

    torchrun --nproc-per-node N --master-addr 127.0.0.1 tools/step_timeline.py \
        [workload] [exchange auto|fused|sharded|nccl] [pieces] [overlap 0|1]

Runs the product step (default schedule) on every rank, records 6 steps with
tgb_plan_enable_timing and prints, for the last step, every launch's start/end
(us from the step's first launch), per rank. Events add ~1-2 us per launch.
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_1705_07878_b200 as tg  # noqa: E402


def main():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if ws > 1:
        dist.init_process_group("gloo", rank=rank, world_size=ws)
    comm = tg.Comm(rank, ws) if ws > 1 else None
    wl = sys.argv[1] if len(sys.argv) > 1 else "vgg16"
    ex = sys.argv[2] if len(sys.argv) > 2 else "auto"
    pieces = int(sys.argv[3]) if len(sys.argv) > 3 else 0
    overlap = {"0": False, "1": True}.get(sys.argv[4]) if len(sys.argv) > 4 else None
    layers = tg.layersets.get(wl)
    sw = tg.SyncWorker([n for n, _ in layers], [s for _, s in layers], tg.CodecConfig(seed=42),
                       rank=rank, world_size=ws, comm=comm, device=dev, exchange=ex, pieces=pieces,
                       overlap=overlap)
    sw.grad_flat.normal_(0.0, 1e-3, generator=torch.Generator(device=dev).manual_seed(1000 + rank))
    for t in range(5):
        sw.step(t)
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    steps = 6
    sw.plan.enable_timing(64 * steps)
    per_step = []
    for k in range(steps):
        sw.step(100 + k)
        torch.cuda.synchronize()  # one step per record window: a clean per-step timeline
        if ws > 1:
            dist.barrier()
    recs = sw.plan.read_timing()
    sw.plan.enable_timing(0)
    sw.check()
    n_per = len(recs) // steps
    last = recs[-n_per:]
    t0 = min(r["start_ms"] for r in last)
    tl = [{"kernel": r["kernel"], "group": r["group"],
           "start_us": round((r["start_ms"] - t0) * 1e3, 1),
           "end_us": round((r["start_ms"] - t0 + r["ms"]) * 1e3, 1),
           "hbm_MB": round(r["hbm_bytes"] / 1e6, 1), "nvlink_MB": round(r["nvlink_bytes"] / 1e6, 1)}
          for r in last]
    span = max(x["end_us"] for x in tl)
    allr = [None] * ws
    if ws > 1:
        dist.all_gather_object(allr, {"rank": rank, "span_us": span, "timeline": tl})
    else:
        allr = [{"rank": 0, "span_us": span, "timeline": tl}]
    if rank == 0:
        print(json.dumps({"workload": wl, "n_gpus": ws, "exchange": sw.plan.exchange,
                          "pieces": pieces, "ranks": allr}), flush=True)
    if ws > 1:
        dist.barrier()
    sw.plan.close()
    if ws > 1:
        dist.barrier()
        comm.close()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
