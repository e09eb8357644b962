"""Single-layer size sweep (BASELINE.json configs[4]): one tensor of n fp32
elements, n = 2^10 .. 2^30, full tgb_step (encode + exchange + decode) per
worker, N = WORLD_SIZE GPUs (torchrun for N > 1; one process per GPU).

    python tools/size_sweep.py [--max-log2 30] [--step 2]
    torchrun --nproc-per-node 4 --master-addr 127.0.0.1 tools/size_sweep.py

Per size: K steps timed with CUDA events (K so that the timed region is >= 20 ms,
at least 5), max over ranks; aggregate elem/s = N * n * K / t; HBM roofline
fraction from the algorithmic bytes per element of the exchange actually used
(12.5 B at N = 1, 12 + 0.5 N allgather/fused, 12.5 + 2 w
sharded). Below ~2^23 elements the working set (12.5 B/elem) fits in the 126 MB
L2 and steps after the first hit in L2: fractions above 1 there are L2, not HBM.
Rank 0 prints one JSON line per size, then a summary line.
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_1705_07878_b200 as tg  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--min-log2", type=int, default=10)
    ap.add_argument("--max-log2", type=int, default=30)
    ap.add_argument("--step", type=int, default=2)
    args = ap.parse_args()
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if ws > 1:
        dist.init_process_group("gloo", rank=rank, world_size=ws)
    comm = tg.Comm(rank, ws) if ws > 1 else None
    try:
        with open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                               "MEASURED_PEAKS.json")) as f:
            hbm = float(json.load(f)["hbm_gbs"])
    except Exception:
        hbm = 6650.0
    st = torch.cuda.current_stream(dev)
    rows = []
    for lg in range(args.min_log2, args.max_log2 + 1, args.step):
        n = 1 << lg
        sw = tg.SyncWorker(["layer"], [[n]], tg.CodecConfig(seed=42), rank=rank, world_size=ws,
                           comm=comm, device=dev)
        info = tg._lib.PlanInfo()
        tg._lib.check(tg._lib.load().tgb_plan_get_info(sw.plan.h, tg.codec.C.byref(info)), "info")
        mode = tg._lib.EXCHANGE_NAMES[info.exchange]
        gen = torch.Generator(device=dev).manual_seed(1000 + rank)
        sw.grad_flat.normal_(0.0, 1e-3, generator=gen)
        for t in range(3):
            sw.step(t)
        torch.cuda.synchronize()
        # calibrate K on one step
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        sw.step(3)
        e1.record(st)
        torch.cuda.synchronize()
        one = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64)
        if ws > 1:
            dist.all_reduce(one, op=dist.ReduceOp.MAX)
        K = int(max(5, min(500, 20.0 / max(float(one[0]), 1e-3))))
        if ws > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0.record(st)
        for k in range(K):
            sw.step(10 + k)
        e1.record(st)
        torch.cuda.synchronize()
        sw.check()
        ms = torch.tensor([e0.elapsed_time(e1) / K], dtype=torch.float64)
        if ws > 1:
            dist.all_reduce(ms, op=dist.ReduceOp.MAX)
        ms = float(ms[0])
        w = (0.5 if ws <= 7 else 1.0) if mode == "sharded" else 0.0
        B = 12.5 if ws == 1 else (12.5 + 2 * w if mode == "sharded" else
                                  12.25 + 0.4 * ws if mode == "fused-r3" else 12.0 + 0.5 * ws)
        gbs = n * B / (ms * 1e-3) / 1e9
        row = {"log2_n": lg, "n": n, "n_gpus": ws, "exchange": mode, "steps": K,
               "us_per_step": ms * 1e3, "aggregate_elem_per_s": ws * n / (ms * 1e-3),
               "per_gpu_elem_per_s": n / (ms * 1e-3), "B_per_elem": B,
               "hbm_GBps_algorithmic": gbs, "roofline_frac": gbs / hbm,
               "l2_resident": n * B < 100e6}
        rows.append(row)
        if rank == 0:
            print(json.dumps(row), flush=True)
        if ws > 1:
            dist.barrier()
        sw.plan.close()
        if ws > 1:
            dist.barrier()
    if rank == 0:
        print(json.dumps({"summary": "size_sweep", "n_gpus": ws, "hbm_peak_GBps": hbm,
                          "rows": len(rows)}), flush=True)
    if comm is not None:
        comm.close()
    if ws > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
