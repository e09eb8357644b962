"""K1 (clip statistics) variants on the VGG-16 set, one GPU, CUDA events.
    python tools/k1_probe.py [variant ...]     (TGB_K1V values, default 0..6)"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1705_07878_b200 as tg  # noqa: E402

dev = torch.device("cuda", 0)
layers = tg.layersets.get("vgg16")
names, ns = [n for n, _ in layers], [tg.layersets.numel(s) for _, s in layers]
g, gv = tg.aligned_flat(ns, dev)
g.normal_(0, 1e-3, generator=torch.Generator(device=dev).manual_seed(3))
st = torch.cuda.current_stream(dev)
ref = None
for v in [int(x) for x in sys.argv[1:]] or list(range(7)):
    os.environ["TGB_K1V"] = str(v)
    os.environ["TGB_GROUPS"] = "0"
    plan = tg.Plan(names, ns, tg.CodecConfig(seed=42), device=dev)
    plan.bind(gv, None)
    for _ in range(3):
        plan.stats()
    ts = []
    for _ in range(20):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        plan.stats()
        e1.record(st)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    plan.raise_errors()
    sc = plan.scalers().clone()
    same = ref is None or torch.equal(sc, ref)
    ref = sc if ref is None else ref
    ms = statistics.median(ts)
    print(f"K1 variant {v}: {ms*1e3:7.1f} us  {4*sum(ns)/ms/1e6:7.1f} GB/s  scalers_equal={same}",
          flush=True)
    plan.close()
