"""Benchmark: fp32 gradient elements/s through ternarize + sync + decode.

Workload (BASELINE.json configs[3], the north-star target): the full VGG-16
gradient set (32 tensors, 138,357,544 fp32 elements per worker), one worker
per GPU, full encode (K1 clip/scaler, K2 ternarize+pack) + sync (N > 1: the
default exchange -- K2 stores codes into every peer over NVLink (fused, N <= 4)
or at the chunk owner, which sums them (sharded, N >= 5) -- or an NCCL
allgather with --exchange nccl) + decode (K3) per step. Synthetic
Gaussian gradients (sigma = 1e-3), seeded per rank. Inputs (553 MB per rank)
are larger than L2 (126 MB), so no L2 flush is needed between steps.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                  [--workload vgg16|alexnet|googlenet] [--exchange auto|fused|sharded|nccl]
                  [--schedule auto|single|groups] [--pull 0..8] [--pieces P] [--overlap -1|0|1]
                  [--no-e2e] [--no-cpu-baseline] [--no-kernel-timing]

N > 1: one process per GPU. Under torchrun (WORLD_SIZE set) this process is one
rank; without it, bench.py launches N ranks itself (torch.distributed.run on
127.0.0.1) and relays rank 0's line. gloo carries control (barriers,
max-over-ranks timing); the data moves over NVLink through libtgb (peer stores)
or NCCL.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "fp32 gradient elements/sec through ternarize+sync+decode; % of HBM roofline"
UNIT = "elem/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--workload", default="vgg16", choices=["vgg16", "alexnet", "googlenet"])
    ap.add_argument("--exchange", default="auto", choices=["auto", "fused", "sharded", "nccl"])
    ap.add_argument("--pieces", type=int, default=0, help="exchange pieces (0 = auto)")
    ap.add_argument("--overlap", type=int, default=-1, help="overlapped exchange: -1 auto, 0, 1")
    ap.add_argument("--schedule", default="auto", choices=["auto", "single", "groups"],
                    help="layer-group schedule (auto: dominant tensor || the rest)")
    ap.add_argument("--pull", type=int, default=0,
                    help="split exchange: eighths of the codes the decode pulls (0..8)")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--cpu-seconds", type=float, default=12.0,
                    help="CPU time budget of the in-line cpu_baseline (at least one full step)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-kernel-timing", action="store_true",
                    help="no per-launch events inside the timed region (A/B of their cost)")
    return ap.parse_args()


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return ws, rank, local


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled DURING the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.Q,
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 6:
                continue
            try:
                sm.append(float(f[0]))
                mx = float(f[1])
            except ValueError:
                continue
            for nme, v in zip(names, f[2:6]):
                if v.lower() == "active":
                    reasons.add(nme)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def workload_config(workload, n_tensors, n, N):
    """the `config` object of both arms' JSON lines (same workload, same keys)"""
    return {"workload": f"{workload} full gradient set ({n_tensors} tensors, {n} fp32 "
                        f"elements/worker), {N} worker(s), encode+sync+decode",
            "global_batch": None, "seq_len": None, "parallelism": f"dp{N}",
            "elements_per_worker": n,
            "codec": "c=2.5 per-tensor clip, sharing on, REF (post-hoc max) scalers, seed 42",
            "l2": f"inputs ({4 * n / 1e6:.0f} MB/rank) "
                  + ("> L2 (126 MB): no flush" if 4 * n > (126 << 20) else
                     "fit in L2 (126 MB): steps after the first read them from L2")}


def synth_host(ns, rank, pinned=True):
    """Per-rank synthetic gradients on the host (sigma 1e-3), flat & 16B-aligned."""
    import torch

    from paper_1705_07878_b200.layout import push_layout  # noqa: F401

    offs, pos = [], 0
    for n in ns:
        offs.append(pos)
        pos += (n + 3) // 4 * 4
    g = torch.Generator().manual_seed(1000 + rank)
    flat = torch.empty(pos, dtype=torch.float32, pin_memory=pinned)
    flat.normal_(0.0, 1e-3, generator=g)
    return flat, offs


# ------------------------------------------------------------------ CPU arm
def cpu_reference_run(layers, n_workers, steps, warmup, replicas, budget_s=None):
    """Time the reference as shipped (oracle/_ref: N worker threads encode_step +
    push -> ParameterServer::step fold + radix-packed pull -> N decode_pull, over
    InProcessHub; cluster.hpp:135-221, 283-297) on the FULL gradient set: every
    step processes every element of every tensor for every worker. `replicas`
    independent clusters (each N worker threads + 1 server thread) step
    concurrently from Python threads (ctypes releases the GIL) so every host core
    works; they share the input arrays (each cluster copies them). Throughput =
    all replicas' elements / wall time. With budget_s, as many steps as fit (at
    least one) instead of `steps`."""
    import threading as _th

    import numpy as np

    from oracle.oracle import Config, RefCluster, Reference

    names = [n for n, _ in layers]
    ns = [_numel(s) for _, s in layers]
    ref = Reference()
    grads = []
    for w in range(n_workers):
        rng = np.random.default_rng(1000 + w)
        grads.append([rng.standard_normal(n, dtype=np.float32) * np.float32(1e-3) for n in ns])
    clusters = [RefCluster(ref, names, grads, Config(seed=42)) for _ in range(replicas)]
    del grads
    barrier = _th.Barrier(replicas)

    def run(cl, t0, k, out):
        for t in range(t0, t0 + k):
            barrier.wait()  # replicas step together: one step = every replica's full step
            cl.step(t)
        out.append(k)

    def go(t0, k):
        done = []
        threads = [_th.Thread(target=run, args=(cl, t0, k, done)) for cl in clusters]
        w0 = time.perf_counter()
        for th in threads:
            th.start()
        for th in threads:
            th.join()
        return time.perf_counter() - w0

    if warmup:
        go(0, warmup)
    if budget_s is not None:  # one timed step, then as many more as the budget allows
        wall = go(warmup, 1)
        steps = 1
        extra = int(max(0.0, budget_s - wall) // max(wall, 1e-9))
        if extra:
            wall += go(warmup + 1, extra)
            steps += extra
    else:
        wall = go(warmup, steps)
    for cl in clusters:
        cl.close()
    elems = replicas * n_workers * sum(ns) * steps
    sample = (f"full {len(ns)}-tensor set ({sum(ns)} elements/worker, no truncation), "
              f"{n_workers} worker(s); {replicas} concurrent cluster replica(s) x ({n_workers} "
              f"worker threads + 1 server thread), each replica one full step per step; "
              f"{steps} timed steps in {wall:.1f} s after {warmup} warm-up step(s)")
    return elems, wall, steps, sample


def ref_replicas(n_workers):
    cores = os.cpu_count() or 1
    return max(1, cores // (n_workers + 1))


def _numel(shape):
    p = 1
    for d in shape:
        p *= int(d)
    return p if len(shape) else 0


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    from paper_1705_07878_b200 import layersets

    layers = layersets.get(args.workload)
    n_workers = max(args.gpus, ws)
    n = sum(_numel(s) for _, s in layers)
    reps = ref_replicas(n_workers)
    elems, wall, nsteps, sample = cpu_reference_run(layers, n_workers, args.steps, args.warmup,
                                                    reps)
    value = elems / wall
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * wall / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (Gaussian sigma=1e-3, seeded per worker, host-generated)",
        "impl": "reference",
        "config": workload_config(args.workload, len(layers), n, n_workers),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": reps * (n_workers + 1),
                         "kind": "reference", "sample": sample,
                         "host_cores_available": os.cpu_count()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "path": "oracle/_ref/libtgref.so: the reference's headers compiled unmodified "
                "(encode_step, ParameterServer::step, decode_pull over InProcessHub)",
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ GPU arm
def run_b200(args):
    import torch
    import torch.distributed as dist

    import paper_1705_07878_b200 as tg
    from paper_1705_07878_b200 import layersets

    ws, rank, local = dist_env()
    N = ws
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if ws > 1:
        dist.init_process_group("gloo", rank=rank, world_size=ws)
    comm = tg.Comm(rank, ws) if ws > 1 else None

    layers = layersets.get(args.workload)
    names = [n for n, _ in layers]
    shapes = [s for _, s in layers]
    cfg = tg.CodecConfig(seed=42)
    sw = tg.SyncWorker(names, shapes, cfg, rank=rank, world_size=ws, comm=comm, device=dev,
                       exchange=args.exchange, pieces=args.pieces,
                       overlap=None if args.overlap < 0 else bool(args.overlap),
                       pull=args.pull, schedule=args.schedule)
    ns = sw.ns
    n = sum(ns)
    plan = sw.plan
    mode = plan.exchange
    # algorithmic HBM bytes per element per GPU:
    #   N = 1 (K2 writes the decode): 4 (K1) + 4 (K2 read) + 0.25 (codes) + 4 (out) = 12.25;
    #   fused / allgather: B(N) = 12 + 0.5 N;
    #   sharded: 4 + 4 + 0.25 (codes land at owners) + 0.25 (K3a reads) + w (sums land)
    #            + w (K3b reads) + 4 = 12.5 + 2 w, w = 4 / radix_m bytes (base 2N+1 digits
    #            per u32 word: 0.4 B at N = 4, 0.57 B at N = 8)
    radix_m = {2: 13, 3: 11, 4: 10, 5: 9, 6: 8, 7: 8, 8: 7}.get(N, 0)
    sum_w = 4.0 / radix_m if mode == "sharded" else 0.0
    B_elem = (12.25 if N == 1 else 12.5 + 2 * sum_w if mode == "sharded" else 12.0 + 0.5 * N)
    host, _ = synth_host(ns, rank)
    sw.grad_flat[:host.numel()].copy_(host.to(dev, non_blocking=True))
    stream = torch.cuda.current_stream(dev)
    torch.cuda.synchronize(dev)

    def barrier():
        if ws > 1:
            dist.barrier()

    # per-stage events: K1 | K2 | sync | K3 (sequential stage API, one stream)
    def staged_step(t, ev=None):
        if ev is not None:
            ev[0].record(stream)
        plan.stats()
        if ev is not None:
            ev[1].record(stream)
        plan.ternarize_pack(t)
        if ev is not None:
            ev[2].record(stream)
        if N > 1:
            plan.sync(comm)  # fused path: device barrier (codes already pushed by K2)
        if ev is not None:
            ev[3].record(stream)
        plan.decode_average(None, N)
        if ev is not None:
            ev[4].record(stream)

    # the product step: tgb_step (two-group overlapped schedule; at N = 1 K2 also
    # writes the decoded output)
    def one_step(t):
        plan.step(t, comm)

    for t in range(args.warmup):
        one_step(t)
        staged_step(t)
    plan.raise_errors()
    torch.cuda.synchronize(dev)

    K = args.steps

    def soak(seconds, t0):
        # untimed steps around the timed region so nvidia-smi (100 ms period)
        # samples the clocks under this exact load. Every rank must run the SAME number
        # of steps (each step is a cross-rank exchange): the ranks agree after each batch
        # of 20 whether to run another (a rank-local clock test here let one rank
        # enqueue a batch its peers never joined -- every barrier then waits out its
        # ~10 s timeout)
        end = time.time() + seconds
        t = t0
        while True:
            for _ in range(20):
                one_step(t)
                t += 1
            torch.cuda.synchronize(dev)
            more = torch.tensor([1 if time.time() < end else 0], dtype=torch.int32)
            if ws > 1:
                dist.all_reduce(more, op=dist.ReduceOp.MAX)
            if not int(more.item()):
                break

    e_start = torch.cuda.Event(enable_timing=True)
    e_stop = torch.cuda.Event(enable_timing=True)
    live_timing = not args.no_kernel_timing
    with ClockSampler(local) as clk:
        soak(0.6, 10_000)
        barrier()
        torch.cuda.synchronize(dev)
        e_start.record(stream)
        for k in range(K):
            one_step(args.warmup + k)
        e_stop.record(stream)
        torch.cuda.synchronize(dev)
        barrier()
        soak(0.6, 20_000)
    plan.raise_errors()
    total_ms = e_start.elapsed_time(e_stop)

    # per-kernel breakdown (same kernels, launched sequentially with events between).
    # N = 1: on a second, ungrouped plan over the same gradients, so every kernel
    # covers the whole set in one launch; N > 1: the stage API of this plan.
    if N == 1:
        sw_b = tg.SyncWorker(names, shapes, cfg, device=dev, schedule="single")
        sw_b.grad_flat.copy_(sw.grad_flat)
        plan_b = sw_b.plan
    else:
        plan_b = plan

    def staged_step(t, ev=None):  # noqa: F811
        if ev is not None:
            ev[0].record(stream)
        plan_b.stats()
        if ev is not None:
            ev[1].record(stream)
        plan_b.ternarize_pack(t)
        if ev is not None:
            ev[2].record(stream)
        if N > 1:
            plan_b.sync(comm)
        if ev is not None:
            ev[3].record(stream)
        plan_b.decode_average(None, N)
        if ev is not None:
            ev[4].record(stream)

    for t in range(3):
        staged_step(40_000 + t)
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(5)] for _ in range(K)]
    barrier()
    torch.cuda.synchronize(dev)
    # attribution pass: the step's own kernels, one after another on one stream,
    # each bracketed by CUDA events on that stream (tgb_plan_enable_timing).
    # N = 1: tgb_step on the ungrouped plan (K1 + K2 with the fused decode);
    # N > 1: the stage API = the same K1 / K2 (peer stores) / barrier / K3 kernels.
    if live_timing:
        plan_b.enable_timing(64 * K)
    for k in range(K):
        staged_step(30_000 + k, evs[k])
    torch.cuda.synchronize(dev)
    if N == 1 and live_timing:
        plan_b.enable_timing(64 * K)
        for k in range(K):
            plan_b.step(50_000 + k)
        torch.cuda.synchronize(dev)
    live = plan_b.read_timing() if live_timing else []
    plan_b.enable_timing(0)
    # K1 and the L2 it starts with (N = 1): right after a step, the L2 holds up to 126 MB
    # of the previous decode's dirty output lines, written back while K1 streams the
    # gradients; after a 256 MB read the L2 is clean. Same kernel, same grid.
    k1_l2 = None
    if N == 1 and live_timing:
        flush = torch.empty(64 << 20, dtype=torch.float32, device=dev)

        def k1_after(prep):
            es = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                  for _ in range(K)]
            for k in range(K):
                prep(k)
                es[k][0].record(stream)
                plan_b.stats()
                es[k][1].record(stream)
            torch.cuda.synchronize(dev)
            return sum(x.elapsed_time(y) for x, y in es) / K

        hbm_peak = peaks()[0]
        ms_dirty = k1_after(lambda k: plan_b.step(60_000 + k))
        ms_clean = k1_after(lambda k: (plan_b.step(70_000 + k), flush.sum()))
        k1_l2 = {"after_step_ms": ms_dirty, "after_step_frac": 4.0 * n / (ms_dirty * 1e-3) / 1e9 / hbm_peak,
                 "clean_l2_ms": ms_clean, "clean_l2_frac": 4.0 * n / (ms_clean * 1e-3) / 1e9 / hbm_peak,
                 "note": "K1 alone (CUDA events), 4 B/elem read: right after a tgb_step (L2 full of "
                         "the decode's dirty output, written back under K1's loads) vs after a "
                         "256 MB read (clean L2)"}
        del flush
    barrier()
    plan.raise_errors()
    stage = [[e[i].elapsed_time(e[i + 1]) for e in evs] for i in range(4)]
    staged_total = evs[0][0].elapsed_time(evs[-1][4])
    if ws > 1:
        tt = torch.tensor([total_ms, staged_total] + [sum(s) for s in stage], dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        total_ms, staged_total = float(tt[0]), float(tt[1])
    ms_step = total_ms / K
    value = N * n * K / (total_ms * 1e-3)

    hbm, hbm_src = peaks()
    k1_ms = sum(stage[0]) / K
    k2_ms = sum(stage[1]) / K
    sync_ms = sum(stage[2]) / K
    k3_ms = sum(stage[3]) / K
    kb = {"K1_stats": (4.0 * n, k1_ms), "K2_ternarize_pack": (4.0 * n + n / 4.0, k2_ms),
          "K3_decode": ((sum_w if mode == "sharded" else N / 4.0) * n + 4.0 * n, k3_ms)}
    # live per-kernel timing of the attribution pass (events on each kernel's own
    # stream): aggregate per kernel over its launches (one per layer group); the
    # dominant kernel has the largest total time. Max over ranks of the totals.
    agg = {}
    for r in live:
        key = r["kernel"] + ("+decode" if N == 1 and r["kernel"].startswith("K2") else "")
        a = agg.setdefault(key, {"launches": 0, "ms": 0.0, "hbm_bytes": 0, "nvlink_bytes": 0,
                                 "elements": 0})
        a["launches"] += 1
        a["ms"] += r["ms"]
        a["hbm_bytes"] += r["hbm_bytes"]
        a["nvlink_bytes"] += r["nvlink_bytes"]
        a["elements"] += r["elements"]
    keys = sorted(agg)
    if ws > 1 and keys:
        tt = torch.tensor([agg[k]["ms"] for k in keys], dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        for k, v in zip(keys, tt.tolist()):
            agg[k]["ms"] = v
    kernels_live = {}
    for k in keys:
        a = agg[k]
        if a["ms"] <= 0:
            continue
        kernels_live[k] = {
            "launches_per_step": a["launches"] / K, "ms_per_launch": a["ms"] / a["launches"],
            "ms_per_step": a["ms"] / K,
            "hbm_bytes_per_launch": a["hbm_bytes"] / a["launches"],
            "nvlink_bytes_per_launch": a["nvlink_bytes"] / a["launches"],
            "GB/s": a["hbm_bytes"] / (a["ms"] * 1e-3) / 1e9,
            "frac": a["hbm_bytes"] / (a["ms"] * 1e-3) / 1e9 / hbm}
    if kernels_live:
        dom = max(kernels_live, key=lambda k: agg[k]["ms"])
        dom_bytes = kernels_live[dom]["hbm_bytes_per_launch"]
        dom_ms = kernels_live[dom]["ms_per_launch"]
        dom_src = ("live: CUDA events around each launch on its stream, attribution pass "
                   "(the step's kernels run sequentially: N=1 tgb_step ungrouped, N>1 stage API)")
    else:  # --no-kernel-timing: the sequential breakdown
        dom = max(kb, key=lambda k: kb[k][1])
        dom_bytes, dom_ms = kb[dom]
        dom_src = "sequential stage pass"
    achieved = dom_bytes / (dom_ms * 1e-3) / 1e9
    # NVLink view (N > 1): the kernel that moves the most bytes across NVLink, its
    # achieved rate vs the measured peer-copy bandwidth (B200_PROFILING.md: 770 GB/s
    # per direction; 900 nominal), and the whole step's NVLink bytes per rank
    roofline_nvlink = None
    nvl = {k: v for k, v in kernels_live.items() if v["nvlink_bytes_per_launch"] > 0}
    if nvl:
        kn = max(nvl, key=lambda k: nvl[k]["nvlink_bytes_per_launch"] * nvl[k]["launches_per_step"])
        v = nvl[kn]
        rate = v["nvlink_bytes_per_launch"] / (v["ms_per_launch"] * 1e-3) / 1e9
        step_nvl = sum(x["nvlink_bytes_per_launch"] * x["launches_per_step"]
                       for x in kernels_live.values())
        roofline_nvlink = {
            "kernel": kn, "achieved": rate, "peak": 770.0, "unit": "GB/s", "frac": rate / 770.0,
            "peak_source": "measured peer copy per direction (B200_PROFILING.md; 900 nominal)",
            "bytes_per_step_per_rank": step_nvl,
            "step_time_floor_ms": step_nvl / 770e9 * 1e3}
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        try:
            traffic = json.load(open(tpath)).get(args.workload, {}).get(f"n{N}", {}).get(dom)
        except Exception:
            traffic = None
    step_bytes = n * B_elem
    clocks = clk.summary()

    # ---- end to end through the public API with host buffers (pinned)
    e2e = None
    if not args.no_e2e:
        # tgb_step_host: per-layer pinned host gradients in, averaged gradients out,
        # every step; the next step's H2D overlaps this step's D2H (full-duplex PCIe)
        hin, hin_v, hout, hout_v = sw.host_buffers()
        hin[:host.numel()].copy_(host)
        KE = max(1, args.e2e_steps)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        for t in range(2):
            sw.step_host(t, hin_v, hout_v)
        barrier()
        torch.cuda.synchronize(dev)
        e0.record(stream)
        for t in range(KE):
            sw.step_host(100 + t, hin_v, hout_v)
        e1.record(stream)
        torch.cuda.synchronize(dev)
        barrier()
        sw.check()
        e2e_ms = e0.elapsed_time(e1)
        if ws > 1:
            tt = torch.tensor([e2e_ms], dtype=torch.float64)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            e2e_ms = float(tt[0])
        e2e = {"value": N * n * KE / (e2e_ms * 1e-3), "unit": UNIT,
               "h2d_bytes_per_step": 4 * n, "d2h_bytes_per_step": 4 * n,
               "steps": KE, "ms_per_step": e2e_ms / KE,
               "path": "SyncWorker.step_host -> tgb_step_host (C-ABI): pinned host gradients "
                       "in, averaged gradients out, every step; copy streams overlap step t's "
                       "D2H with step t+1's H2D"}

    cpu = None
    if rank == 0 and N == 1 and not args.no_cpu_baseline:
        try:
            reps = ref_replicas(1)
            elems, wall, _, sample = cpu_reference_run(layers, 1, 1, 0, reps,
                                                       budget_s=args.cpu_seconds)
            cpu = {"value": elems / wall, "unit": UNIT, "cores": 2 * reps,
                   "kind": "reference", "sample": sample,
                   "host_cores_available": os.cpu_count()}
        except Exception as ex:  # reported, never fatal for the GPU number
            cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "reference",
                   "sample": f"unavailable: {ex}"}

    groups = 2 if plan.grouped else 1
    # own kernels per tgb_step: N=1: K1 + K2(decode fused); fused: K1 + K2 + barrier + K3;
    # sharded: K1 + K2 + barrier + K3a + barrier + K3b; nccl: K1 + K2 + K3 (+ NCCL's own)
    launches_per_step = {"none": 2 * groups, "fused": 4 * groups, "sharded": 6,
                         "nccl": 3 * groups}[mode]
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": N, "steps": K,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32 (codes u8, sigma f64)",
            "data": "synthetic (Gaussian sigma=1e-3, seeded per rank, host-generated)",
            "config": workload_config(args.workload, len(ns), n, N),
            "roofline": {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": hbm,
                         "unit": "GB/s", "frac": achieved / hbm, "traffic": traffic,
                         "peak_source": hbm_src, "timing": dom_src,
                         "algorithmic_bytes_per_launch": dom_bytes, "ms_per_launch": dom_ms},
            "roofline_nvlink": roofline_nvlink,
            "kernels_live": kernels_live,
            "roofline_step": {"bytes_per_step": step_bytes,
                              "achieved": step_bytes / (ms_step * 1e-3) / 1e9,
                              "frac": step_bytes / (ms_step * 1e-3) / 1e9 / hbm,
                              "B_per_elem": B_elem},
            "stages_ms": {"K1_stats": k1_ms, "K2_ternarize_pack": k2_ms, "exchange": sync_ms,
                          "K3_decode": k3_ms, "sequential_step": staged_total / K,
                          "note": "per-kernel breakdown from a sequential pass; the headline "
                                  "ms_per_step is tgb_step (two-group overlap, N=1 fused decode)"},
            "k1_l2_state": k1_l2,
            "kernels_sequential": {k: {"ms": v[1], "GB/s": v[0] / (v[1] * 1e-3) / 1e9,
                            "frac": v[0] / (v[1] * 1e-3) / 1e9 / hbm} for k, v in kb.items()},
            "gpu_launches": launches_per_step * K,
            "gpu_launches_note": "own kernels per tgb_step (per layer group where the schedule "
                                 "has two): N=1 K1 + K2 (K2 also decodes); fused K1 + K2 + peer "
                                 "barrier + K3; sharded K1 + K2 + barrier + K3a (owner sums) + "
                                 "barrier + K3b; nccl K1 + K2 + K3",
            "exchange": {"fused": "fused NVLink peer stores in K2 + device barrier",
                         "sharded": "sharded: K2 stores codes at the chunk owner, owner sums N "
                                    "workers into radix-(2N+1) packed sums stored at every rank "
                                    "(NVLink), 2 device barriers",
                         "nccl": "NCCL allgather", "none": "none (N=1)"}[mode],
            "clocks": clocks,
            "e2e": e2e,
            "cpu_baseline": cpu,
        }
        if args.pull or args.pieces or args.overlap >= 0 or args.schedule != "auto":
            line["config"].update(pull=args.pull, pieces=args.pieces, overlap=args.overlap,
                                  schedule=args.schedule)
        print(json.dumps(line), flush=True)
    barrier()  # fused exchange: no rank frees a gather buffer a peer may still write
    sw.plan.close()
    barrier()
    if comm is not None:
        comm.close()
    if ws > 1:
        dist.destroy_process_group()
    return 0


def self_launch(args):
    """--gpus N > 1 without torchrun: launch N ranks of this script on 127.0.0.1
    (one process per GPU) and relay their output; rank 0 prints the line."""
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    args = parse()
    ws, _, _ = dist_env()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        return self_launch(args)
    if ws != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE {ws}", file=sys.stderr)
        return 2
    if args.impl == "reference":
        return run_reference(args)
    return run_b200(args)


if __name__ == "__main__":
    sys.exit(main())
