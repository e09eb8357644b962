"""A/B kernel timing on one GPU in one process (same box, same clocks).

Builds one SyncWorker per TGB_K12 mode (plan-creation-time switch), then
alternates timed blocks of steps and prints per-stage medians (ms).

    python tools/ab_bench.py [workload] [modes...]
"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1705_07878_b200 as tg  # noqa: E402
from paper_1705_07878_b200 import layersets  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "vgg16"
modes = sys.argv[2:] or ["persistent", "chunk"]
dev = torch.device("cuda", 0)
layers = layersets.get(wl)
workers = {}
for m in modes:
    # mode "A/B": K1 kernel A, K2 kernel B (persistent|chunk)
    parts = m.split("/")
    k1m, k2m = (parts + [m])[:2]
    os.environ["TGB_K1"], os.environ["TGB_K2"] = k1m, k2m
    os.environ["TGB_K2V"] = parts[2] if len(parts) > 2 else "0"
    os.environ["TGB_K1V"] = parts[3] if len(parts) > 3 else "0"
    os.environ["TGB_CHUNK"] = parts[4] if len(parts) > 4 else "32768"
    os.environ["TGB_CHUNK3"] = parts[5] if len(parts) > 5 else "16384"
    w = tg.SyncWorker([n for n, _ in layers], [s for _, s in layers], tg.CodecConfig(seed=42),
                      device=dev)
    g = torch.Generator(device=dev).manual_seed(1)
    w.grad_flat.normal_(0.0, 1e-3, generator=g)
    workers[m] = w
st = torch.cuda.current_stream(dev)
res = {m: [[], [], [], []] for m in modes}
n = sum(workers[modes[0]].ns)
for rnd in range(5):
    for m in modes:
        p = workers[m].plan
        for t in range(3):
            p.step(t)
        K = 20
        ev = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(K)]
        for k in range(K):
            ev[k][0].record(st)
            p.stats()
            ev[k][1].record(st)
            p.ternarize_pack(k)
            ev[k][2].record(st)
            p.decode_average(p.push, 1)
            ev[k][3].record(st)
        torch.cuda.synchronize()
        for k in range(K):
            for i in range(3):
                res[m][i].append(ev[k][i].elapsed_time(ev[k][i + 1]))
            res[m][3].append(ev[k][0].elapsed_time(ev[k][3]))
# codes identical across modes
ref = None
for m in modes:
    p = workers[m].plan
    p.step(123)
    torch.cuda.synchronize()
    c = p.push.clone()
    if ref is None:
        ref = c
    else:
        print("codes identical to", modes[0], ":", bool(torch.equal(ref, c)))
hbm = 6545.6
for m in modes:
    k1, k2, k3, tot = (statistics.median(x) for x in res[m])
    print(f"{m:12s} K1 {k1*1e3:7.1f}us ({4*n/k1/1e6/hbm:.2f})  K2 {k2*1e3:7.1f}us "
          f"({4.25*n/k2/1e6/hbm:.2f})  K3 {k3*1e3:7.1f}us ({4.25*n/k3/1e6/hbm:.2f})  "
          f"step {tot*1e3:7.1f}us ({12.5*n/tot/1e6/hbm:.2f})")
