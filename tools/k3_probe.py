"""K3 (decode) cost vs worker count on ONE GPU: a plan with n_workers = N whose
gather buffer holds N copies of this worker's push area (what the exchange
would deliver), timed with CUDA events.   python tools/k3_probe.py [N ...]"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1705_07878_b200 as tg  # noqa: E402

dev = torch.device("cuda", 0)
layers = tg.layersets.get("vgg16")
names, ns = [n for n, _ in layers], [tg.layersets.numel(s) for _, s in layers]
Ns = [int(x) for x in sys.argv[1:]] or [1, 2, 4, 8]
st = torch.cuda.current_stream(dev)
for N in Ns:
    os.environ["TGB_GROUPS"] = "0"
    plan = tg.Plan(names, ns, tg.CodecConfig(seed=42), worker=0, n_workers=max(N, 2), device=dev)
    g, gv = tg.aligned_flat(ns, dev)
    o, ov = tg.aligned_flat(ns, dev)
    g.normal_(0, 1e-3, generator=torch.Generator(device=dev).manual_seed(3))
    plan.bind(gv, ov)
    plan.encode(0)
    torch.cuda.synchronize()
    push, _ = plan.last_buffers()
    gathered = push.repeat(N)
    for _ in range(3):
        plan.decode_average(gathered, N)
    ts = []
    for _ in range(20):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        plan.decode_average(gathered, N)
        e1.record(st)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = statistics.median(ts)
    n = sum(ns)
    byts = n * (4 + N / 4)
    print(f"K3 N={N}: {ms*1e3:7.1f} us  {byts/ms/1e6:7.1f} GB/s ({byts/ms/1e6/6545.6:.2f} of peak)")
    plan.close()
