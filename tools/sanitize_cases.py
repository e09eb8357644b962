"""Small cases of every kernel family for compute-sanitizer (memcheck, racecheck,
synccheck), each checked against the oracle so a sanitizer run is also a parity
run:
  * N = 1 steps: PerTensor (K1 -> K2 + fused decode, K2 as K1's programmatic
    dependent), Global, FixedSize k = 256 (multi-bucket items + k1_bucket_slots)
    and k = 1000, a passthrough tensor, misaligned (non-16-B) gradient pointers;
  * the fused K1+K2 persistent launch (unless --no-k12: its spin-waits need every
    CTA co-resident, which a serialising tool does not give);
  * LocalCluster N = 2 and 3: fused and sharded exchanges (peer stores, barrier
    post/check, K3, K3a/K3b) against the reference's average;
  * the per-layer API (clip, scaler, ternarize, decode, average, histogram) and
    the wire format (serialize_push).
    compute-sanitizer --tool memcheck python tools/sanitize_cases.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1705_07878_b200 as tg  # noqa: E402
from oracle.oracle import Config, Reference, Restated  # noqa: E402

DEV = torch.device("cuda", 0)
R = Restated()
names = ["conv.weight", "conv.bias", "empty", "fc.weight", "fc.bias"]
sizes = [1728, 64, 0, 20003, 10]
grads = [R.normal(7, 0, "san/" + n, m, 1e-2) for n, m in zip(names, sizes)]
no_k12 = "--no-k12" in sys.argv
ok = True


def n1_case(cfg, ocfg, schedule="auto", pt=None):
    global ok
    sw = tg.SyncWorker(names, [[n] for n in sizes], cfg, device=DEV, schedule=schedule)
    for v, g in zip(sw.grads, grads):
        if g.size:
            v.copy_(torch.from_numpy(g).to(DEV))
    sw.step(3, check=True)
    (st, _), want = Reference().average_encoded(names, [grads], ocfg, 3, pt)
    got = torch.cat([o.cpu() for o in sw.outs]).numpy()
    same = st == 0 and np.array_equal(got.view(np.uint32), want.view(np.uint32))
    print("N=1", schedule, cfg.bucketing.name, cfg.bucket_size, "ok" if same else "MISMATCH",
          flush=True)
    ok &= bool(same)
    sw.plan.close()


F = tg.Bucketing.FixedSize
n1_case(tg.CodecConfig(seed=42), Config(seed=42))
n1_case(tg.CodecConfig(seed=42, bucketing=tg.Bucketing.Global), Config(seed=42, bucketing=1))
n1_case(tg.CodecConfig(seed=42, bucketing=F, bucket_size=256), Config(seed=42, bucketing=2,
                                                                         bucket_size=256))
n1_case(tg.CodecConfig(seed=42, bucketing=F, bucket_size=1000, passthrough={"conv.bias"}),
        Config(seed=42, bucketing=2, bucket_size=1000), pt=[0, 1, 0, 0, 0])
if not no_k12:
    n1_case(tg.CodecConfig(seed=42), Config(seed=42), schedule="fused12")

# misaligned gradient pointers (scalar paths)
plan = tg.Plan(["m"], [1001], tg.CodecConfig(seed=42), device=DEV)
buf = torch.zeros(1003, device=DEV)
g = buf[1:1002]
g.copy_(torch.from_numpy(R.normal(9, 0, "mis", 1001, 1e-2)).to(DEV))
out = torch.zeros(1001, device=DEV)
plan.bind([g], [out])
plan.step(1)
plan.raise_errors()
plan.close()

for N in (2, 3):
    for ex in ("fused", "sharded"):
        for cfg, ocfg in ((tg.CodecConfig(seed=42), Config(seed=42)),
                          (tg.CodecConfig(seed=42, bucketing=F, bucket_size=256),
                           Config(seed=42, bucketing=2, bucket_size=256))):
            cl = tg.LocalCluster(names, [[n] for n in sizes], cfg, N, DEV, exchange=ex)
            gw = [[R.normal(100 + w, 0, "san/" + n, m, 1e-2) for n, m in zip(names, sizes)]
                  for w in range(N)]
            for w in range(N):
                for v, gg in zip(cl.grads[w], gw[w]):
                    if gg.size:
                        v.copy_(torch.from_numpy(gg).to(DEV))
            for t in (4, 5):
                cl.step(t, check=True)
            (st, _), want = Reference().average_encoded(names, gw, ocfg, 5)
            got = torch.cat([o.cpu() for o in cl.outs[0]]).numpy()
            same = st == 0 and np.array_equal(got.view(np.uint32), want.view(np.uint32))
            print(f"LocalCluster N={N} {ex} k={cfg.bucket_size}", "ok" if same else "MISMATCH",
                  flush=True)
            ok &= bool(same)
            cl.close()

# per-layer API + wire
x = tg.GradTensor("fc.weight", [20003], torch.from_numpy(grads[3]).to(DEV))
c = tg.clip(x, 2.5)
s = tg.scaler(c)
blk = tg.ternarize("fc.weight", c.values, s, tg.RngStream(42, 3, "fc.weight", 0))
dec = tg.decode(blk)
res = tg.encode_step([x], tg.CodecConfig(seed=42), 3, 0)
avg = tg.average([res.encoded], 1, True)
h = tg.histogram(x.values, 16)
sw = tg.SyncWorker(names, [[n] for n in sizes], tg.CodecConfig(seed=42), device=DEV)
sw.step(1, check=True)
frame = sw.plan.serialize_push(1)
sw.plan.close()
torch.cuda.synchronize()
print("per-layer API + wire ok", len(frame), flush=True)
print("ALL OK" if ok else "SOME MISMATCH", flush=True)
sys.exit(0 if ok else 1)
