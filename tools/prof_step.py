"""Short driver for ncu: a few full VGG-16 steps (K1, K2, K3) on cuda:0.

    ncu --set full --clock-control none --import-source on \
        -k regex:"k1_stats|k2_ternarize|k3_decode" -s 3 -c 3 -o prof python tools/prof_step.py \
        [workload] [steps] [staged]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1705_07878_b200 as tg  # noqa: E402
from paper_1705_07878_b200 import layersets  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "vgg16"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
staged = len(sys.argv) > 3 and sys.argv[3] == "staged"  # K1 | K2 | K3 on one ungrouped plan
if staged:
    os.environ["TGB_GROUPS"] = "0"
layers = layersets.get(wl)
dev = torch.device("cuda", 0)
w = tg.SyncWorker([n for n, _ in layers], [s for _, s in layers], tg.CodecConfig(seed=42),
                  device=dev)
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
