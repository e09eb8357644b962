"""FixedSize(k) bucketing throughput probe, N = 1: VGG-16 step time and per-kernel
split for several bucket sizes k against PerTensor. Prints one JSON line."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1705_07878_b200 as tg  # noqa: E402


def probe(names, shapes, cfg, dev, K=20):
    sw = tg.SyncWorker(names, shapes, cfg, device=dev)
    sw.grad_flat.normal_(0, 1e-3)
    st = torch.cuda.current_stream(dev)
    for t in range(3):
        sw.step(t)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for k in range(K):
        sw.step(10 + k)
    e1.record(st)
    torch.cuda.synchronize()
    step_us = e0.elapsed_time(e1) * 1e3 / K
    sw.plan.enable_timing(16 * K)
    for k in range(K):
        sw.step(1000 + k)
    torch.cuda.synchronize()
    per = {}
    for r in sw.plan.read_timing():
        per[r["kernel"]] = round(per.get(r["kernel"], 0.0) + r["ms"] * 1e3 / K, 1)
    sw.plan.enable_timing(0)
    n = sum(sw.ns)
    sw.plan.close()
    return {"step_us": round(step_us, 1), "gelem_s": round(n / step_us / 1e3, 2), "kernel_us": per}


def main():
    dev = torch.device("cuda", 0)
    ks = [int(x) for x in (sys.argv[1:] or ["64", "256", "1000", "1024", "4096", "16384", "65536",
                                            str(1 << 20), str(1 << 24), "102760447"])]
    g = tg.layersets.get("vgg16")
    names, shapes = [a for a, _ in g], [s for _, s in g]
    res = {"per_tensor": probe(names, shapes, tg.CodecConfig(seed=42), dev)}
    for k in ks:
        cfg = tg.CodecConfig(seed=42, bucketing=tg.Bucketing.FixedSize, bucket_size=k)
        res[f"fixed_{k}"] = probe(names, shapes, cfg, dev)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
