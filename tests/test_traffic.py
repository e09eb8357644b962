"""Traffic accounting (TrafficStats, cluster.hpp:62-74, 145-160) on CPU.

tgb_traffic_for_layers needs no device: the framed push / pull sizes of the
reference's wire format and their raw-fp32 equivalents, per worker and step.
Pinned against the reference itself (the frames its own ParameterServer path
produces for the same tensors, oracle/_ref RefCluster) and against its two
traffic gates: cluster_test.cpp:107-129 and acceptance criterion 5
(acceptance_test.cpp:153-180).
"""
import math

import numpy as np
import pytest

import paper_1705_07878_b200 as tg


def test_compression_ratio_acceptance_criterion_5():
    """n = 1e6: up ratio in [15.5, 16); pull with N = 4 sharing within 5 % of
    32 / log2(9) (acceptance_test.cpp:153-180)"""
    t = tg.TrafficStats.for_layers(["g"], [1000000], tg.CodecConfig(seed=5), 4)
    assert 15.5 <= t.up_reduction() < 16.0
    ideal = 32.0 / math.log2(9.0)
    assert abs(t.down_reduction() - ideal) / ideal <= 0.05


def test_float_mode_moves_traffic_at_ratio_one():
    """cluster_test.cpp:131-138: float_mode => every block raw fp32, ratio ~1"""
    cfg = tg.CodecConfig(seed=1, float_mode=True)
    t = tg.TrafficStats.for_layers(["w", "b"], [5000, 10], cfg, 3)
    assert t.up_reduction() == pytest.approx(1.0, rel=1e-6)
    assert t.down_reduction() == pytest.approx(1.0, rel=1e-6)


def test_accumulates_like_the_server():
    """ParameterServer::step adds every worker's push and every pull it sends
    (cluster.hpp:147-160): N workers x K steps of the per-worker terms"""
    one = tg.TrafficStats.for_layers(["g"], [4096], tg.CodecConfig(seed=5), 4)
    acc = tg.TrafficStats()
    for _ in range(3 * 4):
        acc += one
    assert acc.bytes_up == 12 * one.bytes_up and acc.float_bytes_down == 12 * one.float_bytes_down
    assert acc.up_reduction() == pytest.approx(one.up_reduction())


@pytest.mark.parametrize("bucketing,k,pt,sharing,N", [
    (tg.Bucketing.PerTensor, 0, (), True, 4),
    (tg.Bucketing.FixedSize, 7, ("fc.bias",), True, 3),
    (tg.Bucketing.Global, 0, (), False, 2),
    (tg.Bucketing.FixedSize, 1000, ("conv1.bias",), True, 8),
])
def test_sizes_equal_reference_frames(reference, restated, bucketing, k, pt, sharing, N):
    """bytes_up / bytes_down == the lengths of the push and pull frames the
    reference's own cluster exchanges for the same tensors (wire.hpp:41-53,
    codec.hpp:395-438, wire.hpp:113-145)"""
    from oracle.oracle import Config, RefCluster

    names = ["conv1.weight", "conv1.bias", "empty", "fc.weight", "fc.bias"]
    sizes = [1728, 64, 0, 40003, 10]
    grads = [[restated.normal(100 + w, 0, "tr/" + n, m, 1e-2) for n, m in zip(names, sizes)]
             for w in range(N)]
    cfg = tg.CodecConfig(seed=42, scaler_sharing=sharing, bucketing=bucketing, bucket_size=k,
                         passthrough=set(pt))
    mine = tg.TrafficStats.for_layers(names, sizes, cfg, N)
    ocfg = Config(seed=42, scaler_sharing=sharing, bucketing=int(bucketing), bucket_size=k)
    cl = RefCluster(reference, names, grads, ocfg, [int(n in pt) for n in names])
    try:
        cl.step(3)
        for w in range(N):
            assert len(cl.frame(w, 0)) == mine.bytes_up, w
            assert len(cl.frame(w, 1)) == mine.bytes_down, w
    finally:
        cl.close()
    # the raw-fp32 terms: header + per block (tag, name, n, 4n values)
    blocks = []
    for name, n in zip(names, sizes):
        if bucketing == tg.Bucketing.FixedSize and name not in pt and n:
            blocks += [(name, min(k, n - o)) for o in range(0, n, k)]
        else:
            blocks.append((name, n))
    flt = 18 + 2 + sum(1 + 2 + len(nm) + 4 + 4 * n for nm, n in blocks)
    assert mine.float_bytes_up == flt and mine.float_bytes_down == flt
    assert np.isfinite(mine.up_reduction())
