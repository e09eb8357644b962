"""World-size-2 host-logic tests on CPU (gloo), no GPU.

Covers the N > 1 control path around the kernels:
  * NCCL unique-id bootstrap through torch.distributed (what Comm does);
  * the push/gather layout (paper_1705_07878_b200/layout.py, the plan's
    tgb_plan_create layout): every rank packs its scalers + codes into a push
    buffer, the buffers are allgathered (gloo stands in for NCCL / the fused
    NVLink stores), each rank unpacks the gathered buffer and the oracle's
    decode of it equals the reference's average over both workers
    (cluster_test.cpp:157-195: decoded pull == average).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle.oracle import REF_SO, Config, Reference, Restated
from paper_1705_07878_b200.layout import pack_push, push_layout, unpack_gathered

NAMES = ["conv1.weight", "conv1.bias", "empty", "fc.weight", "fc.bias"]
SIZES = [1728, 64, 0, 40003, 10]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, ws, port, sharing, bucket, pt, q):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=ws)
        # 1. unique-id bootstrap (Comm.__init__ path, minus ncclCommInitRank)
        from paper_1705_07878_b200.plan import Comm

        buf = [Comm.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(buf, src=0)
        ids = [None] * ws
        dist.all_gather_object(ids, buf[0])
        assert len(buf[0]) == 128 and len(set(ids)) == 1

        # 2. encode (oracle stands in for K1/K2), pack, allgather, unpack, decode
        R = Restated()
        cfg = Config(seed=42, scaler_sharing=sharing, bucketing=2 if bucket else 0,
                     bucket_size=bucket)
        grads = [R.normal(100 + rank, 0, "mp/" + n, k, 1e-2) for n, k in zip(NAMES, SIZES)]
        st, blocks, scal, _, _ = R.encode_step(NAMES, grads, cfg, 7, rank, pt)
        assert st == 0
        lay = push_layout(SIZES, pt, cfg.bucketing, bucket)
        tern = iter(blocks)
        regions = [grads[b.layer].tobytes() if b.passthrough else bytes(next(tern))
                   for b in lay.blocks]
        mine = torch.frombuffer(bytearray(pack_push(lay, scal, regions)), dtype=torch.uint8)
        gathered = torch.empty(ws * lay.push_bytes, dtype=torch.uint8)
        dist.all_gather_into_tensor(gathered, mine)
        sc, rs = unpack_gathered(lay, bytes(gathered.numpy()), ws)
        out = []
        for i, b in enumerate(lay.blocks):  # K3 per block (codec.hpp:268-307)
            if b.passthrough:
                out.append(R.average_passthrough([np.frombuffer(rs[w][i], np.float32)
                                                  for w in range(ws)]))
                continue
            st, avg = R.average_block([sc[w][b.slot] for w in range(ws)],
                                      [np.frombuffer(rs[w][i], np.uint8) for w in range(ws)],
                                      b.n, sharing)
            assert st == 0
            out.append(avg)
        flat = np.concatenate(out)
        allg = [None] * ws
        dist.all_gather_object(allg, grads)
        if rank == 0 and os.path.exists(REF_SO):
            (st, msg), ref = Reference().average_encoded(NAMES, allg, cfg, 7, pt)
            assert st == 0, msg
            assert np.array_equal(ref.view(np.uint32), flat.view(np.uint32))
        hs = [None] * ws
        dist.all_gather_object(hs, flat.tobytes())
        assert len(set(hs)) == 1  # every rank decodes the same averaged gradient
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, repr(e)))


@pytest.mark.parametrize("sharing,bucket,pt", [
    (True, 0, None), (False, 0, None),
    (True, 1000, [0, 1, 0, 0, 0]),   # FixedSize buckets + a passthrough tensor
    (False, 7, [0, 0, 0, 0, 1]),     # k % 4 != 0
])
def test_two_rank_exchange_layout_gloo(sharing, bucket, pt):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    pt = pt or [0] * len(NAMES)
    ps = [ctx.Process(target=_worker, args=(r, 2, port, sharing, bucket, pt, q))
          for r in range(2)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=240) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    assert res == {0: "ok", 1: "ok"}, res
