"""Small-workload probe: step time vs the sum of its kernels' durations (is the
step host/launch-bound?), N = 1. Prints one JSON line."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1705_07878_b200 as tg  # noqa: E402


def probe(names, shapes, dev, K=200):
    sw = tg.SyncWorker(names, shapes, tg.CodecConfig(seed=42), device=dev)
    sw.grad_flat.normal_(0, 1e-3)
    st = torch.cuda.current_stream(dev)
    for t in range(5):
        sw.step(t)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    h0 = time.perf_counter()
    e0.record(st)
    for k in range(K):
        sw.step(10 + k)
    e1.record(st)
    h1 = time.perf_counter()
    torch.cuda.synchronize()
    step_us = e0.elapsed_time(e1) * 1e3 / K
    host_us = (h1 - h0) * 1e6 / K
    sw.plan.enable_timing(16 * K)
    for k in range(K):
        sw.step(1000 + k)
    torch.cuda.synchronize()
    recs = sw.plan.read_timing()
    sw.plan.enable_timing(0)
    per = {}
    for r in recs:
        per[r["kernel"]] = per.get(r["kernel"], 0.0) + r["ms"] * 1e3 / K
    # synchronous single-step latency
    torch.cuda.synchronize()
    h0 = time.perf_counter()
    for k in range(20):
        sw.step(5000 + k)
        torch.cuda.synchronize()
    lat = (time.perf_counter() - h0) * 1e6 / 20
    sw.plan.close()
    return {"step_us": step_us, "host_enqueue_us": host_us, "kernel_us": per,
            "sync_step_latency_us": lat, "elements": sum(sw.ns)}


def main():
    dev = torch.device("cuda", 0)
    res = {}
    g = tg.layersets.get("googlenet")
    res["googlenet"] = probe([n for n, _ in g], [s for _, s in g], dev)
    res["layer_1M"] = probe(["g"], [[1000000]], dev)
    res["layer_1K"] = probe(["g"], [[1024]], dev)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
