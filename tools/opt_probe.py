"""Fused decode -> optimizer vs step + separate optimizer kernel (VGG-16, 1 GPU).
    python tools/opt_probe.py [momentum|adam|vanilla]"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1705_07878_b200 as tg  # noqa: E402

dev = torch.device("cuda", 0)
rule = {"vanilla": 0, "momentum": 1, "adam": 2}[sys.argv[1] if len(sys.argv) > 1 else "momentum"]
layers = tg.layersets.get("vgg16")
names, shapes = [n for n, _ in layers], [s for _, s in layers]
ocfg = tg.OptimizerConfig(rule=tg.OptimizerRule(rule))
st = torch.cuda.current_stream(dev)
res = {}
for fused in (1, 0):
    w = tg.SyncWorker(names, shapes, tg.CodecConfig(seed=42), device=dev)
    w.plan.set_option(tg._lib.TGB_PLAN_OPT_FUSED_OPTIMIZER, fused)
    w.grad_flat.normal_(0, 1e-3, generator=torch.Generator(device=dev).manual_seed(1))
    pflat, params = tg.aligned_flat(w.ns, dev)
    w.bind_optimizer(ocfg, params)
    for t in range(3):
        w.step_apply(t, 0.1)
    ts = []
    for t in range(20):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        w.step_apply(10 + t, 0.1)
        e1.record(st)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    w.check()
    res[fused] = (statistics.median(ts), pflat.clone())
    print(f"rule {ocfg.rule.name} fused={fused}: {res[fused][0]*1e3:.1f} us/step", flush=True)
print("params identical fused vs unfused:", torch.equal(res[1][1], res[0][1]))
