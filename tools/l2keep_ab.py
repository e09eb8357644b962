"""A/B of K1's L2 tail policy (TGB_K1KEEP, MB per K1 launch loaded with an L2
evict_last policy so that K2's last-to-first walk re-reads it from L2).

Each mode is "keep_mb:flush". flush=1 writes a 256 MB buffer between steps
(outside the timed region) so any reuse ACROSS steps is destroyed and only the
within-step K1 -> K2 reuse can show. Every step is timed alone with CUDA
events on the caller's stream; interleaved rounds, medians.

    python tools/l2keep_ab.py [workload] [modes...]
"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1705_07878_b200 as tg  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "vgg16"
modes = sys.argv[2:] or ["0:0", "0:1", "48:0", "48:1", "96:0", "96:1"]
dev = torch.device("cuda", 0)
layers = tg.layersets.get(wl)
ws = {}
for m in modes:
    keep = m.split(":")[0]
    if keep not in ws:
        os.environ["TGB_K1KEEP"] = keep
        w = tg.SyncWorker([n for n, _ in layers], [s for _, s in layers], tg.CodecConfig(seed=42),
                          device=dev)
        w.grad_flat.normal_(0.0, 1e-3, generator=torch.Generator(device=dev).manual_seed(1))
        ws[keep] = w
os.environ.pop("TGB_K1KEEP", None)
flushbuf = torch.empty(64 << 20, dtype=torch.float32, device=dev)
st = torch.cuda.current_stream(dev)
res = {m: [] for m in modes}
outs = {}
for rnd in range(6):
    for m in modes:
        keep, flush = m.split(":")
        w = ws[keep]
        for t in range(3):
            w.step(t)
        K = 20
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(K)]
        for k in range(K):
            if flush == "1":
                flushbuf.fill_(float(k))
            ev[k][0].record(st)
            w.step(100 + k)
            ev[k][1].record(st)
        torch.cuda.synchronize()
        res[m] += [a.elapsed_time(b) for a, b in ev]
        outs[keep] = torch.cat([o.reshape(-1) for o in w.outs]).clone()
n = sum(next(iter(ws.values())).ns)
for m in modes:
    ms = statistics.median(res[m])
    print(f"K1KEEP_MB:flush={m}: step {ms*1e3:7.1f} us  {n/ms/1e6:8.1f} Gelem/s  "
          f"{12.5*n/ms/1e6/6545.6:.3f} of HBM roofline")
ref = next(iter(outs.values()))
print("outputs identical:", all(torch.equal(ref, o) for o in outs.values()))
