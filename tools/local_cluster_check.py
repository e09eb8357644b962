"""N-worker exchange parity on ONE GPU (LocalCluster / tgb_local_step).

    python tools/local_cluster_check.py [N ...]        (default 2 3 4 5 6 7 8)

Runs N workers as N plans of one process on cuda:0, attached to each other
(tgb_plan_attach_local): the K1/K2 peer stores and the K3 / sharded K3a+K3b
kernels of the multi-process path, ordered by CUDA events between the plans'
streams. For every N, a small tensor set (incl. an empty tensor and ragged
sizes) x REF configs (shared / unshared scalers, Global, FixedSize with
passthrough tensors) x every exchange the product can select at that N (fused;
sharded for shared scalers): every worker must hold bit-identical output equal
to the reference's own average over the same N workers (oracle/_ref,
codec.hpp:245-311). PRESHARED (max-shared scalers before ternarize) against its own oracle.
Also checks LocalCluster's protocol validation: a skewed
iteration raises "server: iteration skew" and leaves the outputs untouched.
Prints one JSON line; exit 1 on any mismatch. (Full BASELINE gradient sets:
tests/test_baseline_parity.py.)
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1705_07878_b200 as tg  # noqa: E402

DEV = torch.device("cuda", 0)
NAMES = ["conv1.weight", "conv1.bias", "empty", "fc.weight", "fc.bias"]
SIZES = [1728, 64, 0, 40003, 10]


def small_checks(N, report):
    from oracle.oracle import Config, Reference, Restated

    R = Restated()
    ref = Reference()
    P, G, F = tg.Bucketing.PerTensor, tg.Bucketing.Global, tg.Bucketing.FixedSize
    configs = [(True, P, 0, ()), (False, P, 0, ()), (True, G, 0, ()),
               (True, F, 1000, ("conv1.bias",)), (False, F, 7, ("fc.bias",)),
               (True, F, 256, ("conv1.bias",)), (True, F, 64, ())]
    grads = [[R.normal(100 + w, 0, "mp/" + n, m, 1e-2) for n, m in zip(NAMES, SIZES)]
             for w in range(N)]
    # sharded3: 3 pieces of the K2 list; +ov: overlapped exchange (K2 publishes pieces)
    # +pull: split exchange (K3 reads 3/8 of the code items from the peers' areas);
    # +grp: the two-group schedule forced (PerTensor REF; sharded: one piece per group)
    for exchange in ("fused", "sharded", "sharded3", "fused+ov", "sharded+ov", "fused+pull",
                     "fused+grp", "sharded+grp"):
        for sharing, bucketing, k, pt_names in configs:
            if exchange.startswith("sharded") and not sharing:
                continue
            cfg = tg.CodecConfig(seed=42, scaler_sharing=sharing, bucketing=bucketing,
                                 bucket_size=k, passthrough=set(pt_names))
            cl = tg.LocalCluster(NAMES, [[n] for n in SIZES], cfg, N, DEV,
                                 exchange=exchange.split("+")[0][:7],
                                 pieces=3 if exchange in ("sharded3", "sharded+ov", "fused+ov") else 0,
                                 overlap=True if exchange.endswith("+ov") else None,
                                 pull=3 if exchange.endswith("+pull") else 0,
                                 schedule="groups" if exchange.endswith("+grp") else "auto")
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
            pt = [int(n in pt_names) for n in NAMES]
            ocfg = Config(seed=42, scaler_sharing=sharing, bucketing=int(bucketing), bucket_size=k)
            (st, _), want = ref.average_encoded(NAMES, grads, ocfg, 7, pt)
            ok = st == 0 and np.array_equal(want.view(np.uint32), flats[0].view(np.uint32))
            key = (f"N={N},exchange={exchange},sharing={sharing},bucketing={bucketing.name}"
                   f"{k or ''},passthrough={'+'.join(pt_names) or '-'}")
            report["checks"][key] = {"workers_identical": bool(same),
                                     "matches_reference": bool(ok), "exchange": cl.exchange}
            cl.close()


def preshared_checks(N, report):
    """PRESHARED (paper Eq. 4): each plan's own slots become the max over the N workers'
    local scalers before K2; against tools/mp_check.py's PRESHARED oracle"""
    import importlib.util

    from oracle.oracle import Config, Restated

    spec = importlib.util.spec_from_file_location(
        "mp_check", os.path.join(os.path.dirname(os.path.abspath(__file__)), "mp_check.py"))
    mp = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mp)
    R = Restated()
    F = tg.Bucketing.FixedSize
    grads = [[R.normal(100 + w, 0, "mp/" + n, m, 1e-2) for n, m in zip(NAMES, SIZES)]
             for w in range(N)]
    for exchange in ("fused", "sharded"):
        for bucketing, k, pt_names in ((tg.Bucketing.PerTensor, 0, ()),
                                       (F, 1000, ("conv1.bias",)), (F, 256, ())):
            cfg = tg.CodecConfig(seed=42, share_mode=tg.ShareMode.PRESHARED, bucketing=bucketing,
                                 bucket_size=k, passthrough=set(pt_names))
            cl = tg.LocalCluster(NAMES, [[n] for n in SIZES], cfg, N, DEV, exchange=exchange)
            for w in range(N):
                for v, g in zip(cl.grads[w], grads[w]):
                    if g.size:
                        v.copy_(torch.from_numpy(g).to(DEV))
            for t in (5, 6, 7):
                outs = cl.step(t)
            cl.synchronize()
            cl.check()
            flats = [torch.cat([o.cpu() for o in outs[w]]).numpy() for w in range(N)]
            same = all(np.array_equal(flats[0].view(np.uint32), f.view(np.uint32)) for f in flats)
            ocfg = Config(seed=42, bucketing=int(bucketing), bucket_size=k)
            ok = mp.preshared_oracle(R, NAMES, grads, flats[0], N, ocfg,
                                     [int(n in pt_names) for n in NAMES])
            key = f"N={N},exchange={exchange},PRESHARED,bucketing={bucketing.name}{k or ''}"
            report["checks"][key] = {"workers_identical": bool(same), "matches_reference": bool(ok),
                                     "exchange": cl.exchange}
            cl.close()


def skew_check(N, report):
    cl = tg.LocalCluster(NAMES, [[n] for n in SIZES], tg.CodecConfig(seed=42), N, DEV)
    for w in range(N):
        cl.grad_flat[w].normal_(0, 1e-2, generator=torch.Generator(device=DEV).manual_seed(w))
    cl.step(3, check=True)
    before = [f.clone() for f in cl.out_flat]
    cl.step([4] * (N - 1) + [5])  # the last worker is one iteration ahead
    cl.synchronize()
    msgs = []
    for p in cl.plans:
        try:
            p.raise_errors()
            msgs.append(None)
        except tg.ProtocolError as e:
            msgs.append(str(e))
    untouched = all(torch.equal(a, b) for a, b in zip(before, cl.out_flat))
    cl.step(6, check=True)  # recovers on the next agreeing step
    report["checks"][f"N={N},iteration_skew"] = {
        "workers_identical": untouched,
        "matches_reference": all(m is not None and m.startswith("server: iteration skew")
                                 for m in msgs),
        "messages": msgs, "exchange": cl.exchange}
    cl.close()


def main():
    Ns = [int(x) for x in sys.argv[1:]] or [2, 3, 4, 5, 6, 7, 8]
    report = {"device": torch.cuda.get_device_name(0), "checks": {}}
    for N in Ns:
        small_checks(N, report)
        preshared_checks(N, report)
        skew_check(N, report)
    ok = all(v["workers_identical"] and v["matches_reference"] for v in report["checks"].values())
    report["ok"] = ok
    print(json.dumps(report), flush=True)
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
