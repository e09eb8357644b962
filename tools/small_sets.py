"""Step latency of the BASELINE gradient sets at N = 1 per schedule, measured two
ways: eager (a host loop of plan.step, K steps between CUDA events: host/launch
overhead included) and graph (the same K steps captured once in a CUDA graph
and replayed: device time only). Schedules: auto (fused K1+K2 persistent launch
under 8 Mi elements, two-group split for VGG/AlexNet), unfused (K1 and K2
launches), fused12 (always one launch). Outputs checked bit-identical.
    python tools/small_sets.py [K]"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1705_07878_b200 as tg  # noqa: E402

dev = torch.device("cuda", 0)
K = int(sys.argv[1]) if len(sys.argv) > 1 else 50
sets = {w: tg.layersets.get(w) for w in ("googlenet", "alexnet", "vgg16")}
sets["layer_1M"] = [("g", [1 << 20])]
sets["layer_4M"] = [("g", [1 << 22])]
sets["layer_16M"] = [("g", [1 << 24])]
if len(sys.argv) > 2:
    sets = {k: v for k, v in sets.items() if k in sys.argv[2:]}


def timed(fn, reps=5):
    st = torch.cuda.current_stream(dev)
    runs = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        fn()
        e1.record(st)
        torch.cuda.synchronize()
        runs.append(e0.elapsed_time(e1) * 1e3 / K)
    return statistics.median(runs)


for name, layers in sets.items():
    names, shapes = [n for n, _ in layers], [s for _, s in layers]
    n = sum(tg.layersets.numel(s) for s in shapes)
    res, ref = {}, None
    for sched in ("auto", "fused12", "chunk4096", "chunk8192", "chunk16384"):
        sw = tg.SyncWorker(names, shapes, tg.CodecConfig(seed=42), device=dev,
                           schedule=sched if not sched.startswith("chunk") else "auto")
        if sched.startswith("chunk"):
            sw.plan.set_option(tg._lib.TGB_PLAN_OPT_CHUNK, int(sched[5:]))
        sw.grad_flat.normal_(0, 1e-3, generator=torch.Generator(device=dev).manual_seed(1))
        plan = sw.plan
        for t in range(5):
            plan.step(t)
        eager = timed(lambda: [plan.step(100 + k) for k in range(K)])
        side = torch.cuda.Stream(dev)
        side.wait_stream(torch.cuda.current_stream(dev))
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=side):
            for k in range(K):
                plan.step(200 + k)
        torch.cuda.synchronize()
        graph = timed(lambda: g.replay())
        sw.step(7, check=True)
        o = sw.out_flat.clone()
        same = ref is None or torch.equal(o, ref)
        ref = o if ref is None else ref
        res[sched] = {"eager_us": eager, "graph_us": graph, "Gelem_s_graph": n / graph / 1e3,
                      "groups": plan.info.n_groups, "same_output": bool(same)}
        del g
        plan.close()
        del sw
    print(json.dumps({name: {"elements": n, "schedules": res}}), flush=True)
