"""Multi-GPU parity + timing check (one process per GPU, torchrun).

    TGB_EXCHANGE=auto|fused|sharded|nccl torchrun --nproc-per-node N \
        --master-addr 127.0.0.1 --master-port 29511 tools/mp_check.py

Every rank encodes its own gradients (worker id = rank), the exchange
(NVLink peer stores, fused or sharded, or the NCCL allgather) moves
scalers + codes, every rank decodes. Checks:
  * all ranks hold bit-identical averaged gradients (the reference's
    "every worker decodes the same pull", cluster.hpp:153-161);
  * on the small tensor set, the result is bit-identical to the reference's
    average over the same N workers (oracle/_ref, cluster_test.cpp:157-195),
    for shared and unshared scalers and the PRESHARED mode's own oracle;
  * the full AlexNet and VGG-16 sets are bit-identical to the reference's own
    sync path (ParameterServer over InProcessHub, RefCluster) on the same inputs;
  * protocol validation: ranks stepping different iterations raise the
    reference's "server: iteration skew" ProtocolError (cluster.hpp:141-143) and
    leave the outputs untouched; ranks with different layer tables fail at
    attach with "server: block structure mismatch" (cluster.hpp:169-172).
Prints one JSON line from rank 0.
"""
import hashlib
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_1705_07878_b200 as tg  # noqa: E402

EXCHANGE = os.environ.get("TGB_EXCHANGE", "auto")
_OV = os.environ.get("TGB_OVERLAP")  # tool-level switch: "1" overlapped exchange, "0" off
OVERLAP = None if _OV is None else _OV == "1"
PULL = int(os.environ.get("TGB_PULL", "0"))  # tool-level switch: split exchange eighths


def ex_for(sharing):
    """the sharded exchange needs shared scalers (the owner sums integer codes)"""
    return "auto" if (EXCHANGE == "sharded" and not sharing) else EXCHANGE


def full_set_checks(report, rank, ws, comm, dev):
    """GoogLeNet, AlexNet and VGG-16 full sets vs the reference's own sync path (RefCluster)"""
    import numpy as np
    from oracle.oracle import Config, RefCluster, Reference

    for set_name in ("googlenet", "alexnet", "vgg16"):
        layers = tg.layersets.get(set_name)
        names, shapes = [n for n, _ in layers], [s for _, s in layers]
        ns = [tg.layersets.numel(s) for s in shapes]

        def grads_of(w):
            rng = np.random.default_rng(1000 + w)
            return [rng.standard_normal(n, dtype=np.float32) * np.float32(1e-3) for n in ns]

        sw = tg.SyncWorker(names, shapes, tg.CodecConfig(seed=42), rank=rank, world_size=ws,
                           comm=comm, device=dev, exchange=EXCHANGE, overlap=OVERLAP, pull=PULL)
        for v, g in zip(sw.grads, grads_of(rank)):
            v.copy_(torch.from_numpy(g).to(dev))
        for t in (10, 11, 12):
            sw.step(t)
        sw.check()
        torch.cuda.synchronize()
        flat = torch.cat([o.cpu() for o in sw.outs]).numpy()
        h = hashlib.sha256(flat.tobytes()).hexdigest()
        hs = [None] * ws
        dist.all_gather_object(hs, h)
        ok_ref = None
        if rank == 0:
            cl = RefCluster(Reference(), names, [grads_of(w) for w in range(ws)], Config(seed=42))
            cl.step(12)
            want = cl.output(0)
            cl.close()
            ok_ref = bool(np.array_equal(want.view(np.uint32), flat.view(np.uint32)))
        report["checks"][f"{set_name}_full_set"] = {"ranks_identical": len(set(hs)) == 1,
                                                    "matches_oracle": ok_ref,
                                                    "exchange": sw.plan.exchange}
        dist.barrier()
        sw.plan.close()


def protocol_checks(report, rank, ws, comm, dev):
    """iteration skew (cluster.hpp:141-143) and block-structure mismatch (:169-172)"""
    names = ["a.weight", "a.bias"]
    cfg = tg.CodecConfig(seed=42)
    sw = tg.SyncWorker(names, [[5000], [10]], cfg, rank=rank, world_size=ws, comm=comm,
                       device=dev, exchange=EXCHANGE)
    sw.grad_flat.normal_(0, 1e-2, generator=torch.Generator(device=dev).manual_seed(rank))
    sw.step(3, check=True)
    before = sw.out_flat.clone()
    msg = None
    if EXCHANGE != "nccl":  # the NCCL allgather carries no iteration
        sw.step(4 + (rank == 1))  # rank 1 is one iteration ahead
        try:
            sw.check()
        except tg.ProtocolError as e:
            msg = str(e)
        untouched = torch.equal(before, sw.out_flat)
        msgs = [None] * ws
        dist.all_gather_object(msgs, msg)
        report["checks"]["iteration_skew"] = {
            "ranks_identical": all(m is not None and "server: iteration skew" in m for m in msgs)
            and untouched, "matches_oracle": None, "messages": msgs}
        sw.step(9, check=True)  # the exchange recovers on the next agreeing step
    dist.barrier()
    sw.plan.close()
    if EXCHANGE == "nccl":
        return
    sizes = [[5000], [10 + (rank == ws - 1)]]  # the last rank's bias has one more element
    err = None
    try:
        bad = tg.SyncWorker(names, sizes, cfg, rank=rank, world_size=ws, comm=comm, device=dev,
                            exchange=EXCHANGE)
        bad.plan.close()
    except tg.ProtocolError as e:
        err = str(e)
    errs = [None] * ws
    dist.all_gather_object(errs, err)
    report["checks"]["block_structure_mismatch"] = {
        "ranks_identical": all(e is not None and "block structure mismatch" in e for e in errs),
        "matches_oracle": None, "messages": errs}
    dist.barrier()


def main():
    ws = int(os.environ["WORLD_SIZE"])
    rank = int(os.environ["RANK"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    comm = tg.Comm(rank, ws)
    from oracle.oracle import Config, Reference, Restated

    R = Restated()
    names = ["conv1.weight", "conv1.bias", "empty", "fc.weight", "fc.bias"]
    sizes = [1728, 64, 0, 40003, 10]
    report = {"world_size": ws, "exchange": EXCHANGE, "overlap": OVERLAP, "pull": PULL, "checks": {}}
    P, G, F = tg.Bucketing.PerTensor, tg.Bucketing.Global, tg.Bucketing.FixedSize
    configs = [  # (sharing, mode, bucketing, k, passthrough names)
        (True, tg.ShareMode.REF, P, 0, ()), (False, tg.ShareMode.REF, P, 0, ()),
        (True, tg.ShareMode.PRESHARED, P, 0, ()), (True, tg.ShareMode.REF, G, 0, ()),
        (True, tg.ShareMode.REF, F, 1000, ("conv1.bias",)),
        (False, tg.ShareMode.REF, F, 7, ("fc.bias",)),
        (True, tg.ShareMode.PRESHARED, F, 1000, ("conv1.bias",)),
    ]
    for sharing, mode, bucketing, k, pt_names in configs:
        cfg = tg.CodecConfig(seed=42, scaler_sharing=sharing, share_mode=mode,
                             bucketing=bucketing, bucket_size=k, passthrough=set(pt_names))
        pt = [int(n in pt_names) for n in names]
        sw = tg.SyncWorker(names, [[n] for n in sizes], cfg, rank=rank, world_size=ws, comm=comm,
                           device=dev, exchange=ex_for(sharing), overlap=OVERLAP, pull=PULL)
        grads = [R.normal(100 + rank, 0, "mp/" + n, k, 1e-2) for n, k in zip(names, sizes)]
        for v, g in zip(sw.grads, grads):
            if g.size:
                v.copy_(torch.from_numpy(g).to(dev))
        for t in (5, 6):  # exercise both gather-buffer parities before the checked step
            sw.step(t)
        out = sw.step(7)
        sw.check()
        torch.cuda.synchronize()
        flat = torch.cat([o.cpu() for o in out]).numpy()
        h = hashlib.sha256(flat.tobytes()).hexdigest()
        hs = [None] * ws
        dist.all_gather_object(hs, h)
        allg = [None] * ws
        dist.all_gather_object(allg, grads)
        key = f"sharing={sharing},mode={mode.name},bucketing={bucketing.name}{k or ''}," \
              f"passthrough={'+'.join(pt_names) or '-'}"
        ok_same = len(set(hs)) == 1
        ok_ref = None
        if rank == 0:
            ocfg = Config(seed=42, scaler_sharing=sharing, bucketing=int(bucketing), bucket_size=k)
            if mode == tg.ShareMode.REF:
                (st, msg), ref = Reference().average_encoded(names, allg, ocfg, 7, pt)
                ok_ref = st == 0 and np.array_equal(ref.view(np.uint32), flat.view(np.uint32))
            else:  # PRESHARED: every worker ternarizes with s = max_w s_w (paper Eq. 4)
                ok_ref = preshared_oracle(R, names, allg, flat, ws, ocfg, pt)
        report["checks"][key] = {"ranks_identical": ok_same, "matches_oracle": ok_ref,
                                 "exchange": sw.plan.exchange}
        dist.barrier()
        sw.plan.close()

    # fused decode -> optimizer (tgb_step_apply) == step + OptimizerState::apply, every rank
    for rule in (tg.OptimizerRule.Momentum, tg.OptimizerRule.Adam):
        ocfg = tg.OptimizerConfig(rule=rule, weight_decay=1e-4)
        cfg = tg.CodecConfig(seed=42)
        sw = tg.SyncWorker(names, [[n] for n in sizes], cfg, rank=rank, world_size=ws,
                           comm=comm, device=dev, exchange=ex_for(True), overlap=OVERLAP, pull=PULL)
        ref = tg.SyncWorker(names, [[n] for n in sizes], cfg, rank=rank, world_size=ws,
                            comm=comm, device=dev, exchange=ex_for(True), overlap=OVERLAP, pull=PULL)
        p0 = [torch.full((n,), 0.5, device=dev) for n in sizes]
        params = [x.clone() for x in p0]
        ref_params = [x.clone() for x in p0]
        sw.bind_optimizer(ocfg, params)
        ref_state = tg.OptimizerState(ocfg)
        for t, rate in enumerate([0.1, 0.05, 0.2]):
            grads = [R.normal(200 + rank + t, 0, "opt/" + nm, k, 1e-2) for nm, k in zip(names, sizes)]
            for v, r, g in zip(sw.grads, ref.grads, grads):
                if g.size:
                    v.copy_(torch.from_numpy(g).to(dev))
                    r.copy_(torch.from_numpy(g).to(dev))
            sw.step_apply(t, rate)
            ref_state.apply(ref_params, ref.step(t), rate)
        torch.cuda.synchronize()
        sw.check()
        same = all(torch.equal(a, b) for a, b in zip(params, ref_params))
        h = hashlib.sha256(torch.cat([x.cpu() for x in params]).numpy().tobytes()).hexdigest()
        hs = [None] * ws
        dist.all_gather_object(hs, h)
        report["checks"][f"step_apply,{rule.name}"] = {"ranks_identical": len(set(hs)) == 1,
                                                      "matches_oracle": same}
        dist.barrier()
        sw.plan.close()
        ref.plan.close()

    full_set_checks(report, rank, ws, comm, dev)
    protocol_checks(report, rank, ws, comm, dev)

    # timing: full VGG-16 step at this world size
    layers = tg.layersets.get("vgg16")
    sw = tg.SyncWorker([n for n, _ in layers], [s for _, s in layers], tg.CodecConfig(seed=42),
                       rank=rank, world_size=ws, comm=comm, device=dev, exchange=ex_for(True),
                       overlap=OVERLAP, pull=PULL)
    gen = torch.Generator(device=dev).manual_seed(1000 + rank)
    sw.grad_flat.normal_(0.0, 1e-3, generator=gen)
    st = torch.cuda.current_stream(dev)
    p = sw.plan
    for t in range(5):
        sw.step(t)
    torch.cuda.synchronize()
    K = 20
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(5)] for _ in range(K)]
    dist.barrier()
    for k in range(K):
        ev[k][0].record(st)
        p.stats()
        ev[k][1].record(st)
        p.ternarize_pack(k)
        ev[k][2].record(st)
        p.sync(comm)
        ev[k][3].record(st)
        p.decode_average(None, ws)
        ev[k][4].record(st)
    torch.cuda.synchronize()
    dist.barrier()
    sw.check()
    stage = [sorted(e[i].elapsed_time(e[i + 1]) for e in ev)[K // 2] for i in range(4)]
    staged = ev[0][0].elapsed_time(ev[-1][4]) / K
    # the product path: tgb_step (sharded / fused schedule)
    for t in range(3):
        sw.step(100 + t)
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for k in range(K):
        sw.step(200 + k)
    e1.record(st)
    torch.cuda.synchronize()
    dist.barrier()
    sw.check()
    tot = e0.elapsed_time(e1) / K
    t_all = torch.tensor([tot] + stage + [staged], dtype=torch.float64)
    dist.all_reduce(t_all, op=dist.ReduceOp.MAX)
    if rank == 0:
        n = sum(sw.ns)
        report["vgg16_exchange"] = p.exchange
        report["vgg16_ms_per_step_max_over_ranks"] = float(t_all[0])
        report["stage_ms_median_max_over_ranks"] = {
            k: float(v) for k, v in zip(["K1", "K2", "sync", "K3"], t_all[1:5])}
        report["staged_ms_per_step"] = float(t_all[5])
        report["aggregate_Gelem_s"] = ws * n / (float(t_all[0]) * 1e-3) / 1e9
        report["allgather_GBps_per_rank_in"] = (ws - 1) * p.info.push_bytes / (
            float(t_all[3]) * 1e-3) / 1e9
        report["note"] = ("vgg16_ms_per_step: tgb_step (the product schedule); stages: the "
                          "sequential stage API (K1 | K2 | exchange | K3) on the same plan")
        print(json.dumps(report), flush=True)
    dist.barrier()  # no rank frees memory a peer may still write
    sw.plan.close()
    dist.barrier()
    comm.close()
    dist.destroy_process_group()
    ok = all(v["ranks_identical"] and (v["matches_oracle"] in (True, None))
             for v in report["checks"].values())
    sys.exit(0 if ok else 1)


def preshared_oracle(R, names, allg, flat, ws, cfg, pt):
    """Oracle for PRESHARED: per block, s = max over workers of the local
    scalers; every worker ternarizes its clipped bucket with that s
    (ternarize(name, part, s, rng, off), codec.hpp:148, :229), then the
    shared-sum average; passthrough tensors take the fp64 mean."""
    from oracle.oracle import block_layout

    ns = [g.size for g in allg[0]]
    local = []
    for w in range(ws):
        st, _, sc, _, _ = R.encode_step(names, allg[w], cfg, 7, w, pt)
        if st:
            return False
        local.append(sc)
    lay = block_layout(ns, cfg, pt)
    outs, b = [], 0
    for li, name in enumerate(names):
        if pt[li]:
            outs.append(R.average_passthrough([allg[w][li] for w in range(ws)]))
            continue
        clipped = [R.clip(allg[w][li], cfg.clip_factor)[0] if ns[li] >= 2 else allg[w][li]
                   for w in range(ws)]
        while b < len(lay) and lay[b][0] == li:
            _, off, ln = lay[b]
            s = max(float(local[w][b]) for w in range(ws))
            codes = []
            for w in range(ws):
                st, cw = R.ternarize(clipped[w][off:off + ln], s, 42, 7, name, w, off)
                if st:
                    return False
                codes.append(cw)
            st, avg = R.average_block([s] * ws, codes, ln, True)
            outs.append(avg)
            b += 1
    ref = np.concatenate(outs)
    return bool(np.array_equal(ref.view(np.uint32), flat.view(np.uint32)))


if __name__ == "__main__":
    main()
