"""BASELINE-config parity: the full gradient sets of BASELINE.json's configs,
stepped on the B200 and compared byte-for-byte with the reference's own sync
path run on the same inputs (oracle/_ref: N worker threads encode_step + push,
ParameterServer::step folds and broadcasts the radix-packed pull, every worker
decode_pulls; cluster.hpp:135-221, 283-297 -- the pin of cluster_test.cpp:157-195).

  * VGG-16 (138,357,544 elements) at N = 1 through SyncWorker (the bench path),
    and at N = 4 / 5 / 8 as LocalCluster workers on one GPU, with the fused
    exchange (codes to every worker) and the sharded exchange (owner sums,
    radix-(2N+1) packed) -- the N > 1 kernels of the multi-process path;
  * AlexNet (61,100,840 elements) at N = 2 (BASELINE configs[1]);
  * GoogLeNet (173 tensors, 6,624,904 elements) at N = 8 with scaler sharing
    (BASELINE configs[2]).

The clip bound is an fp64 sigma (SURVEY finding 7): a mismatch confined to a
tensor whose bound differs from the reference's is reported as "sigma-order",
any other byte difference as a kernel bug. Multi-GPU (one process per GPU)
versions of the same comparisons run in tools/mp_check.py (test_multi_gpu.py).
"""
import os

import numpy as np
import pytest
import torch

import paper_1705_07878_b200 as tg

pytestmark = pytest.mark.gpu

DEV = torch.device("cuda", 0) if torch.cuda.is_available() else None


def _grads(layers, n_workers, seed0=1000, sigma=1e-3):
    """[worker][tensor] float32 numpy gradients (Gaussian, seeded per worker)"""
    out = []
    for w in range(n_workers):
        rng = np.random.default_rng(seed0 + w)
        out.append([(rng.standard_normal(tg.layersets.numel(s), dtype=np.float32) *
                     np.float32(sigma)) for _, s in layers])
    return out


def _ref_output(reference, names, grads, t, cfg=None):
    from oracle.oracle import Config, RefCluster

    cl = RefCluster(reference, names, grads, cfg or Config(seed=42))
    try:
        cl.step(t)
        return cl.output(0)
    finally:
        cl.close()


def _compare(got_tensors, want_flat, names, ns):
    """byte comparison per tensor; returns a list of mismatching tensor names"""
    bad, pos = [], 0
    for name, n, g in zip(names, ns, got_tensors):
        w = want_flat[pos:pos + n]
        pos += n
        if not np.array_equal(g.view(np.uint32), w.view(np.uint32)):
            bad.append(name)
    return bad


def _to_device(dst_views, host_arrays):
    for v, g in zip(dst_views, host_arrays):
        if g.size:
            v.copy_(torch.from_numpy(g).to(DEV))


def _outputs(views):
    return [v.cpu().numpy() for v in views]


def _local_cluster_vs_reference(reference, set_name, n_workers, exchanges, t=12):
    layers = tg.layersets.get(set_name)
    names, shapes = [n for n, _ in layers], [s for _, s in layers]
    ns = [tg.layersets.numel(s) for s in shapes]
    grads = _grads(layers, n_workers)
    want = _ref_output(reference, names, grads, t)
    report = {}
    for ex in exchanges:
        cl = tg.LocalCluster(names, shapes, tg.CodecConfig(seed=42), n_workers, DEV, exchange=ex)
        for w in range(n_workers):
            _to_device(cl.grads[w], grads[w])
        for tt in (t - 2, t - 1, t):  # both gather-buffer parities before the checked step
            cl.step(tt)
        cl.synchronize()
        cl.check()
        outs = [_outputs(cl.outs[w]) for w in range(n_workers)]
        report[ex] = {
            "exchange": cl.exchange,
            "workers_identical": all(
                all(np.array_equal(a.view(np.uint32), b.view(np.uint32))
                    for a, b in zip(outs[0], outs[w])) for w in range(1, n_workers)),
            "mismatch": _compare(outs[0], want, names, ns),
        }
        cl.close()
        del cl
        torch.cuda.empty_cache()
    return report


@pytest.mark.timeout(900)
def test_vgg16_n1_full_set_bit_exact(reference):
    """BASELINE configs[3] at N = 1: the bench's own path (SyncWorker.step: K1 +
    K2 with the fused decode, two-group schedule) over the whole VGG-16 set."""
    layers = tg.layersets.get("vgg16")
    names, shapes = [n for n, _ in layers], [s for _, s in layers]
    ns = [tg.layersets.numel(s) for s in shapes]
    grads = _grads(layers, 1)
    want = _ref_output(reference, names, grads, 7)
    sw = tg.SyncWorker(names, shapes, tg.CodecConfig(seed=42), device=DEV)
    _to_device(sw.grads, grads[0])
    sw.step(7, check=True)
    bad = _compare(_outputs(sw.outs), want, names, ns)
    assert not bad, f"sigma-order or kernel mismatch in {bad}"
    assert sum(ns) == 138357544


@pytest.mark.timeout(900)
def test_alexnet_n2_bit_exact(reference):
    """BASELINE configs[1]: AlexNet, 2 workers, layer-wise clipping + ternarizing."""
    rep = _local_cluster_vs_reference(reference, "alexnet", 2, ["auto", "sharded"])
    for ex, r in rep.items():
        assert r["workers_identical"], ex
        assert not r["mismatch"], (ex, r)
    assert rep["auto"]["exchange"] == "fused"
    assert rep["sharded"]["exchange"] == "sharded"


@pytest.mark.timeout(900)
def test_googlenet_n8_bit_exact(reference):
    """BASELINE configs[2]: GoogLeNet (173 tensors), 8 workers with scaler sharing:
    the default (fused, for a small set) exchange and the sharded one."""
    rep = _local_cluster_vs_reference(reference, "googlenet", 8, ["auto", "sharded"])
    for ex, r in rep.items():
        assert r["workers_identical"], ex
        assert not r["mismatch"], (ex, r)
    assert rep["auto"]["exchange"] == "fused"  # a small set: sharded only from 16 Mi elements
    assert rep["sharded"]["exchange"] == "sharded"


@pytest.mark.timeout(1800)
@pytest.mark.parametrize("n_workers,exchanges", [(4, ["auto", "sharded"]), (5, ["auto"]),
                                                 (8, ["auto", "fused"])])
def test_vgg16_multiworker_bit_exact(reference, n_workers, exchanges):
    """BASELINE configs[3] at N = 4 / 5 / 8 (the 8-GPU scaling configuration) as
    LocalCluster workers: every exchange variant the product selects at that N."""
    if torch.cuda.get_device_properties(0).total_memory < (n_workers * 2 + 4) * (1 << 30):
        pytest.skip("not enough device memory for N VGG-16 workers on one GPU")
    rep = _local_cluster_vs_reference(reference, "vgg16", n_workers, exchanges)
    for ex, r in rep.items():
        assert r["workers_identical"], ex
        assert not r["mismatch"], (ex, r)
    assert rep["auto"]["exchange"] == ("fused" if n_workers <= 4 else "sharded")
