"""Short driver for ncu: a few full VGG-16 steps (K1, K2, K3) on cuda:0.

    ncu --set full --clock-control none --import-source on \
        -k regex:"k1_stats|k2_ternarize|k3_decode" -s 3 -c 3 -o prof python tools/prof_step.py \
        [workload] [steps] [staged|ungrouped|k3n4]

  staged    : K1 | K2 | K3 stage API on one ungrouped plan
  ungrouped : tgb_step on an ungrouped plan (N = 1: K1 + K2 with the fused decode),
              i.e. the kernels bench.py's attribution pass times
  k3n4      : K3 of N = 4 workers (four unattached plans encode; K3 over their push
              areas back to back), the staged SWAR decode the fused exchange runs at N = 4
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1705_07878_b200 as tg  # noqa: E402
from paper_1705_07878_b200 import layersets  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "vgg16"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
mode = sys.argv[3] if len(sys.argv) > 3 else ""
staged = mode == "staged"  # K1 | K2 | K3 on one ungrouped plan
if mode == "k3n4":
    layers = layersets.get(wl)
    dev = torch.device("cuda", 0)
    names, ns = [n for n, _ in layers], [int(torch.Size(s).numel()) for _, s in layers]
    gf, gv = tg.aligned_flat(ns, dev)
    gf.normal_(0.0, 1e-3, generator=torch.Generator(device=dev).manual_seed(1))
    plans = []
    for w in range(4):
        p = tg.Plan(names, ns, tg.CodecConfig(seed=42), worker=w, n_workers=4, device=dev)
        p.bind(gv, None)
        p.encode(1)
        plans.append(p)
    gathered = torch.cat([p.push for p in plans])
    of, ov = tg.aligned_flat(ns, dev)
    plans[0].bind(gv, ov)
    for t in range(steps):
        plans[0].decode_average(gathered, 4)
    torch.cuda.synchronize()
    for p in plans:
        p.raise_errors()
    print("ok k3n4", wl, steps)
    sys.exit(0)
layers = layersets.get(wl)
dev = torch.device("cuda", 0)
w = tg.SyncWorker([n for n, _ in layers], [s for _, s in layers], tg.CodecConfig(seed=42),
                  device=dev, schedule="single" if mode in ("staged", "ungrouped") else "auto")
g = torch.Generator(device=dev).manual_seed(1)
w.grad_flat.normal_(0.0, 1e-3, generator=g)
for t in range(steps):
    if staged:
        w.plan.stats()
        w.plan.ternarize_pack(t)
        w.plan.decode_average(None, 1)
    else:
        w.step(t)
w.check()
torch.cuda.synchronize()
print("ok", wl, steps)
