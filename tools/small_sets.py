"""Step latency of the BASELINE gradient sets at N = 1 per schedule: the fused
K1+K2 persistent launch (default under 8 Mi elements) vs separate K1 and K2
launches, and the two-group schedule where it applies. CUDA events around K
steps (median of 5 runs); outputs checked bit-identical across schedules.
    python tools/small_sets.py [K]"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1705_07878_b200 as tg  # noqa: E402

dev = torch.device("cuda", 0)
K = int(sys.argv[1]) if len(sys.argv) > 1 else 200
sets = {w: tg.layersets.get(w) for w in ("googlenet", "alexnet", "vgg16")}
sets["layer_1M"] = [("g", [1 << 20])]
sets["layer_4M"] = [("g", [1 << 22])]
sets["layer_16M"] = [("g", [1 << 24])]
out = {}
for name, layers in sets.items():
    names, shapes = [n for n, _ in layers], [s for _, s in layers]
    n = sum(tg.layersets.numel(s) for s in shapes)
    res, ref = {}, None
    for sched in ("auto", "unfused", "fused12", "single"):
        sw = tg.SyncWorker(names, shapes, tg.CodecConfig(seed=42), device=dev, schedule=sched)
        sw.grad_flat.normal_(0, 1e-3, generator=torch.Generator(device=dev).manual_seed(1))
        st = torch.cuda.current_stream(dev)
        for t in range(5):
            sw.step(t)
        runs = []
        for r in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            for k in range(K):
                sw.step(100 + k)
            e1.record(st)
            torch.cuda.synchronize()
            runs.append(e0.elapsed_time(e1) * 1e3 / K)
        sw.step(7, check=True)
        o = sw.out_flat.clone()
        same = ref is None or torch.equal(o, ref)
        ref = o if ref is None else ref
        us = statistics.median(runs)
        res[sched] = {"us_per_step": us, "Gelem_s": n / us / 1e3, "k12": sw.plan.info.n_groups,
                      "same_output": bool(same), "groups": sw.plan.info.n_groups}
        sw.plan.close()
        del sw
    out[name] = {"elements": n, "schedules": res}
    print(json.dumps({name: out[name]}), flush=True)
