"""N-worker exchange parity on ONE GPU (LocalCluster / tgb_plan_attach_local).

    CUDA_DEVICE_MAX_CONNECTIONS=32 CUDA_MODULE_LOADING=EAGER python tools/local_cluster_check.py [N ...]

gpurun offers at most 4 GPUs, but the driver's scaling run goes to N = 8,
where tgb_step switches to the sharded exchange (owner-reduced 8-bit sums).
This runs N workers as N plans of one process on cuda:0, attached to each
other, each stepping on its own stream: the same K1/K2 peer stores, flag
barriers and K3 / K3a+K3b kernels as the multi-process path, minus NVLink.

Checks per N (default 2 3 4 5 8):
  * small tensor set x REF configs (shared/unshared, Global, FixedSize +
    passthrough), default schedule, forced fused (TGB_SHARD=0) and fused with
    radix-3 wire codes (TGB_R3=1, N >= 3): every worker
    holds bit-identical output equal to the reference's own average over the
    same N workers (oracle/_ref, codec.hpp:245-311);
  * full VGG-16 set at N = 8 (sharded, 8-bit sums), N = 5 (4-bit sums), and the
    fused exchange with 2-bit and radix-3 wire codes at N = 4 and 8:
    bit-identical on every worker and equal to K3 over the N unattached push
    areas laid out back to back (the NCCL-allgather path, itself pinned to
    the reference on the golden cases).
Prints one JSON line; exit 1 on any mismatch.
"""
import hashlib
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1705_07878_b200 as tg  # noqa: E402

DEV = torch.device("cuda", 0)


def exchange_of(plan):
    info = tg._lib.PlanInfo()
    tg._lib.check(tg._lib.load().tgb_plan_get_info(plan.h, tg.codec.C.byref(info)), "info")
    return tg._lib.EXCHANGE_NAMES[info.exchange]


def sha(t):
    return hashlib.sha256(t.cpu().numpy().tobytes()).hexdigest()


def small_checks(N, report):
    from oracle.oracle import Config, Reference, Restated

    R = Restated()
    ref = Reference()
    names = ["conv1.weight", "conv1.bias", "empty", "fc.weight", "fc.bias"]
    sizes = [1728, 64, 0, 40003, 10]
    P, G, F = tg.Bucketing.PerTensor, tg.Bucketing.Global, tg.Bucketing.FixedSize
    configs = [(True, P, 0, ()), (False, P, 0, ()), (True, G, 0, ()),
               (True, F, 1000, ("conv1.bias",)), (False, F, 7, ("fc.bias",))]
    for shard in ("default", "0", "0+r3"):
        for sharing, bucketing, k, pt_names in configs:
            if shard != "default":
                os.environ["TGB_SHARD"] = "0"
            if shard == "0+r3":
                os.environ["TGB_R3"] = "1"
            cfg = tg.CodecConfig(seed=42, scaler_sharing=sharing, bucketing=bucketing,
                                 bucket_size=k, passthrough=set(pt_names))
            cl = tg.LocalCluster(names, [[n] for n in sizes], cfg, N, DEV)
            os.environ.pop("TGB_SHARD", None)
            os.environ.pop("TGB_R3", None)
            grads = [[R.normal(100 + w, 0, "mp/" + n, m, 1e-2) for n, m in zip(names, sizes)]
                     for w in range(N)]
            for w in range(N):
                for v, g in zip(cl.grads[w], grads[w]):
                    if g.size:
                        v.copy_(torch.from_numpy(g).to(DEV))
            for t in (5, 6, 7):  # both gather-buffer parities before the checked step
                outs = cl.step(t)
            cl.synchronize()
            cl.check()
            flats = [torch.cat([o.cpu() for o in outs[w]]).numpy() for w in range(N)]
            same = all(np.array_equal(flats[0].view(np.uint32), f.view(np.uint32)) for f in flats)
            pt = [int(n in pt_names) for n in names]
            ocfg = Config(seed=42, scaler_sharing=sharing, bucketing=int(bucketing), bucket_size=k)
            (st, _), want = ref.average_encoded(names, grads, ocfg, 7, pt)
            ok = st == 0 and np.array_equal(want.view(np.uint32), flats[0].view(np.uint32))
            key = (f"N={N},shard={shard},sharing={sharing},bucketing={bucketing.name}{k or ''},"
                   f"passthrough={'+'.join(pt_names) or '-'}")
            report["checks"][key] = {"workers_identical": bool(same), "matches_reference": bool(ok),
                                     "exchange": exchange_of(cl.plans[0])}
            cl.close()


def vgg_check(N, report, shard="default"):
    layers = tg.layersets.get("vgg16")
    names, shapes = [n for n, _ in layers], [s for _, s in layers]
    cfg = tg.CodecConfig(seed=42)
    if shard != "default":
        os.environ["TGB_SHARD"] = "0"
    if shard == "0+r3":
        os.environ["TGB_R3"] = "1"
    cl = tg.LocalCluster(names, shapes, cfg, N, DEV)
    os.environ.pop("TGB_SHARD", None)
    os.environ.pop("TGB_R3", None)
    for w in range(N):
        g = torch.Generator(device=DEV).manual_seed(1000 + w)
        cl.grad_flat[w].normal_(0.0, 1e-3, generator=g)
    for t in (10, 11, 12):
        cl.step(t)
    cl.synchronize()
    cl.check()
    hs = {sha(cl.out_flat[w]) for w in range(N)}
    # the allgather path over the same inputs: N unattached plans encode, K3 over
    # their push areas back to back
    plans = []
    for w in range(N):
        p = tg.Plan(names, cl.ns, cfg, worker=w, n_workers=N, device=DEV)
        p.bind(cl.grads[w], None)
        p.encode(12)
        plans.append(p)
    torch.cuda.synchronize()
    gathered = torch.cat([p.push for p in plans])
    out_flat, outs = tg.aligned_flat(cl.ns, DEV)
    plans[0].bind(cl.grads[0], outs)
    plans[0].decode_average(gathered, N)
    torch.cuda.synchronize()
    for p in plans:
        p.raise_errors()
    same = len(hs) == 1
    ok = sha(out_flat) == sha(cl.out_flat[0])
    report["checks"][f"N={N},vgg16" + ("" if shard == "default" else f",shard={shard}")] = {"workers_identical": same, "matches_reference": ok,
                                        "exchange": exchange_of(cl.plans[0]),
                                        "elements_per_worker": sum(cl.ns)}
    for p in plans:
        p.close()
    cl.close()


def main():
    Ns = [int(x) for x in sys.argv[1:]] or [2, 3, 4, 5, 8]
    report = {"device": torch.cuda.get_device_name(0), "checks": {},
              "CUDA_DEVICE_MAX_CONNECTIONS": os.environ.get("CUDA_DEVICE_MAX_CONNECTIONS"),
              "CUDA_MODULE_LOADING": os.environ.get("CUDA_MODULE_LOADING")}
    for N in Ns:
        small_checks(N, report)
    for N in Ns:
        if N >= 5:
            vgg_check(N, report)
        if N in (4, 8):  # the fused exchange at full size, 2-bit and radix-3 wire codes
            vgg_check(N, report, shard="0")
            vgg_check(N, report, shard="0+r3")
    ok = all(v["workers_identical"] and v["matches_reference"] for v in report["checks"].values())
    report["ok"] = ok
    print(json.dumps(report), flush=True)
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
