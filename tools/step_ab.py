"""A/B of whole-step schedules on one GPU: sequential vs two-group overlapped
(TGB_GROUPS). Times plan.step() (K1 -> K2 -> K3 for the whole set) with CUDA
events on the caller's stream; interleaved rounds, medians.

    python tools/step_ab.py [workload]
"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1705_07878_b200 as tg  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "vgg16"
modes = sys.argv[2:] or ["0", "1"]
dev = torch.device("cuda", 0)
layers = tg.layersets.get(wl)
ws = {}
for m in modes:
    parts = m.split("/")
    os.environ["TGB_GROUPS"] = parts[0]
    os.environ["TGB_GPRIO"] = parts[1] if len(parts) > 1 else "1"
    os.environ["TGB_FUSE1"] = parts[2] if len(parts) > 2 else "1"
    w = tg.SyncWorker([n for n, _ in layers], [s for _, s in layers], tg.CodecConfig(seed=42),
                      device=dev)
    w.grad_flat.normal_(0.0, 1e-3, generator=torch.Generator(device=dev).manual_seed(1))
    ws[m] = w
st = torch.cuda.current_stream(dev)
res = {m: [] for m in modes}
outs = {}
for rnd in range(6):
    for m in modes:
        w = ws[m]
        for t in range(3):
            w.step(t)
        K = 20
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for k in range(K):
            w.step(100 + k)
        e1.record(st)
        torch.cuda.synchronize()
        res[m].append(e0.elapsed_time(e1) / K)
        outs[m] = torch.cat([o.reshape(-1) for o in w.outs]).clone()
n = sum(ws[modes[0]].ns)
for m in modes:
    ms = statistics.median(res[m])
    print(f"GROUPS/PRIO/FUSE1={m}: step {ms*1e3:7.1f} us  {n/ms/1e6:8.1f} Gelem/s  "
          f"{12.5*n/ms/1e6/6545.6:.3f} of HBM roofline")
print("outputs identical:", all(torch.equal(outs[modes[0]], outs[m]) for m in modes))
