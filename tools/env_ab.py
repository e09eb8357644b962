"""Generic A/B of plan-creation-time env switches on one GPU (whole step).

Each mode is "VAR=V[,VAR2=V2...][:flush]" ("-" = defaults); flush=1 writes a
256 MB buffer between steps (outside the timed region). Every step is timed
alone with CUDA events on the caller's stream; interleaved rounds, medians;
outputs compared bit-for-bit across modes.

    python tools/env_ab.py WORKLOAD MODE...     (WORKLOAD: a layer set or layer:N)
"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1705_07878_b200 as tg  # noqa: E402

wl = sys.argv[1]
modes = sys.argv[2:]
dev = torch.device("cuda", 0)
layers = [("layer", [int(wl[6:])])] if wl.startswith("layer:") else tg.layersets.get(wl)
ws = {}
for m in modes:
    envs = m.split(":")[0]
    if envs in ws:
        continue
    saved = dict(os.environ)
    if envs != "-":
        for kv in envs.split(","):
            k, v = kv.split("=")
            os.environ[k] = v
    w = tg.SyncWorker([n for n, _ in layers], [s for _, s in layers], tg.CodecConfig(seed=42),
                      device=dev)
    w.grad_flat.normal_(0.0, 1e-3, generator=torch.Generator(device=dev).manual_seed(1))
    ws[envs] = w
    os.environ.clear()
    os.environ.update(saved)
flushbuf = torch.empty(64 << 20, dtype=torch.float32, device=dev)
st = torch.cuda.current_stream(dev)
res = {m: [] for m in modes}
outs = {}
for rnd in range(6):
    for m in modes:
        envs, _, flush = m.partition(":")
        w = ws[envs]
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
        outs[envs] = torch.cat([o.reshape(-1) for o in w.outs]).clone()
n = sum(next(iter(ws.values())).ns)
for m in modes:
    ms = statistics.median(res[m])
    print(f"{wl} {m:28s}: step {ms*1e3:7.1f} us  {n/ms/1e6:8.1f} Gelem/s  "
          f"{12.5*n/ms/1e6/6545.6:.3f} of HBM roofline")
ref = next(iter(outs.values()))
print("outputs identical:", all(torch.equal(ref, o) for o in outs.values()))
