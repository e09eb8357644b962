"""Functional step latency of a LocalCluster (N workers as plans of one process on
cuda:0, tgb_local_step): K steps between events on a master stream that every
worker stream joins; host-issue bound for small sets (N plans x 6 launches per
step). BASELINE configs[2] asks GoogLeNet at N = 8; 8 GPUs are not available to
this repo's measurements, so this is the one-GPU functional figure.
    python tools/local_latency.py [workload] [N ...]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1705_07878_b200 as tg  # noqa: E402

dev = torch.device("cuda", 0)
wl = sys.argv[1] if len(sys.argv) > 1 else "googlenet"
Ns = [int(x) for x in sys.argv[2:]] or [2, 4, 8]
layers = tg.layersets.get(wl)
names, shapes = [n for n, _ in layers], [s for _, s in layers]
K = 50
for N in Ns:
    for ex in ("auto", "fused", "sharded"):
        cl = tg.LocalCluster(names, shapes, tg.CodecConfig(seed=42), N, dev, exchange=ex)
        for w in range(N):
            cl.grad_flat[w].normal_(0, 1e-3, generator=torch.Generator(device=dev).manual_seed(w))
        for t in range(3):
            cl.step(t)
        cl.synchronize()
        master = torch.cuda.current_stream(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(master)
        for k in range(K):
            cl.step(10 + k)
        for s in cl.streams:
            master.wait_stream(s)
        e1.record(master)
        torch.cuda.synchronize()
        cl.check()
        us = e0.elapsed_time(e1) * 1e3 / K
        print(json.dumps({"workload": wl, "N": N, "exchange": cl.exchange, "us_per_step": us,
                          "note": "N workers on ONE GPU (work x N), eager host issue"}),
              flush=True)
        cl.close()
