"""Pins the CPU oracle (tests are CPU-only, -m "not gpu").

1. Random123 / SURVEY Appendix B known-answer vectors.
2. The plain-C restatement (oracle/tg_oracle.c) against the golden fixtures
   generated from the reference itself (tests/golden/gen_golden.py).
3. The restatement against the compiled reference (oracle/_ref) on fresh
   random cases, mirroring the reference's own property tests
   (codec_test.cpp, wire_test.cpp, cluster_test.cpp:157-195).
"""
import hashlib
import math

import numpy as np
import pytest

from oracle.oracle import Config, RefCluster, block_layout
from tests.golden.check import check_codes, check_scalers, passthrough_of, restated_average
from tests.golden.recipes import make_input


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def cfg_of(d):
    return Config(clip_factor=d["clip_factor"], clipping_enabled=d["clipping_enabled"],
                  bucketing=d["bucketing"], bucket_size=d["bucket_size"],
                  scaler_sharing=d["scaler_sharing"], seed=d["seed"])


# ---------------------------------------------------------------- KATs
def test_philox_random123_kats(restated):
    # Random123 Philox4x32-10 known answers
    assert restated.philox([0] * 4, [0, 0]) == [0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8]
    assert restated.philox([0xFFFFFFFF] * 4, [0xFFFFFFFF] * 2) == [0x408F276D, 0x41C83B0E,
                                                                  0xA20BC7C6, 0x6D5451FD]
    assert restated.philox([0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344],
                           [0xA4093822, 0x299F31D0]) == [0xD16CFE09, 0x94FDCCEB, 0x5001E420,
                                                         0x24126EA1]


def test_fnv_and_stream_kats(restated, golden):
    assert restated.fnv1a64("fc.weight") == 0x79FB28A75603C7A0
    for k, v in golden["fnv1a64"].items():
        assert restated.fnv1a64(k) == v
    assert restated.bits(42, 0, "fc.weight", 0, range(8)) == [
        0xBA43FD1D, 0x6F3B9052, 0xC9184E86, 0xDE914761, 0x5D3296EA, 0xEDB6940C, 0x5297BCC7,
        0xEFD5AAE1]
    for c in golden["bits"]:
        got = restated.bits(c["seed"], c["t"], c["name"], c["worker"],
                            range(c["k0"], c["k0"] + len(c["out"])))
        assert got == c["out"]
    for c in golden["philox"]:
        assert restated.philox(c["ctr"], c["key"]) == c["out"]


def test_uniform_reaches_one():
    # SURVEY finding 6: float(0xFFFFFF80) rounds to 2^32, so uniform == 1.0f
    assert np.float32(0xFFFFFF80) * np.float32(2 ** -32) == np.float32(1.0)
    assert np.float32(0xFFFFFF7F) * np.float32(2 ** -32) < np.float32(1.0)


def test_appendix_b_encode_kats(restated):
    g = restated.normal(7, 0, "bench", 19)
    st, blocks, sc, bounds, _ = restated.encode_step(["g"], [g], Config(seed=7), 0, 0)
    assert st == 0
    assert bytes(blocks[0]).hex() == "2205580202"
    assert sc.view(np.uint32)[0] == 0x4007C496
    assert abs(float(bounds[0]) - 2.57596731) < 1e-6
    st, blocks, sc, _, _ = restated.encode_step(["g"], [g], Config(seed=7), 12345678901, 5)
    assert bytes(blocks[0]).hex() == "2224404012"
    fw = np.array([0.5, -0.25, 0.125, -1, 0, 0.75, -0.5, 0.3], np.float32)
    fb = np.array([0.1, -0.2, 0.05], np.float32)
    st, blocks, sc, _, _ = restated.encode_step(["fc.weight", "fc.bias"], [fw, fb],
                                                Config(seed=42, clipping_enabled=False), 0, 0)
    assert [bytes(b).hex() for b in blocks] == ["8020", "18"]
    assert list(sc.view(np.uint32)) == [0x3F800000, 0x3E4CCCCD]


# ------------------------------------------------------- golden fixtures
def test_restated_matches_golden_encode(restated, golden):
    for case in golden["encode"]:
        cfg = cfg_of(case["cfg"])
        names = [t["name"] for t in case["tensors"]]
        grads = [make_input(t["recipe"]) for t in case["tensors"]]
        for t, g in zip(case["tensors"], grads):
            assert sha(g) == t["input_sha256"], (case["name"], t["name"])
        st, blocks, sc, bounds, _ = restated.encode_step(names, grads, cfg, case["t"],
                                                         case["worker"], passthrough_of(case))
        assert st == case["status"], case["name"]
        check_scalers(case, sc)
        check_codes(case, blocks)
        assert bounds.tobytes().hex() == case["bounds_hex"], case["name"]


def test_restated_matches_golden_average(restated, golden):
    for case in golden["average"]:
        cfg = cfg_of(case["cfg"])
        names = [t["name"] for t in case["tensors"]]
        gw = [[make_input(dict(t["recipe"], worker=w)) for t in case["tensors"]]
              for w in range(case["N"])]
        flat = restated_average(restated, names, gw, cfg, case["t"], passthrough_of(case))
        assert sha(flat) == case["out_sha256"], case["name"]
        if "out_hex" in case:
            assert flat.tobytes().hex() == case["out_hex"]


# ------------------------------------------- restated vs compiled reference
@pytest.mark.parametrize("seed", [1, 2, 3])
def test_restated_vs_reference_random(restated, reference, seed):
    rng = np.random.default_rng(seed)
    for _ in range(10):
        n = int(rng.integers(0, 5000))
        scale = float(10.0 ** rng.uniform(-6, 1))
        g = (rng.standard_normal(n) * scale).astype(np.float32)
        if n and rng.random() < 0.3:
            g[rng.integers(0, n)] *= 1000
        t = int(rng.integers(0, 2 ** 40))
        w = int(rng.integers(0, 8))
        cfg = Config(seed=int(rng.integers(0, 2 ** 63)), clipping_enabled=bool(rng.random() < .8))
        st, b1, s1, _, _ = restated.encode_step(["x.weight"], [g], cfg, t, w)
        (st2, _), b2, s2 = reference.encode_step(["x.weight"], [g], cfg, t, w)
        assert st == st2 == 0
        assert s1.tobytes() == s2.tobytes()
        assert [bytes(x) for x in b1] == [bytes(x) for x in b2]
        assert math.isclose(restated.stddev(g), reference.stddev(g), rel_tol=0, abs_tol=0)


def test_restated_error_paths(restated, reference):
    g = np.array([0.5, -2.0, 0.25], np.float32)
    st, _ = restated.ternarize(g, 1.0, 1, 0, "t")
    (st2, msg), _ = reference.ternarize(g, 1.0, 1, 0, "t")
    assert st == 1 and st2 == 1 and "below max |g| in t" in msg
    st, _ = restated.ternarize(g, 0.0, 1, 0, "t")
    (st2, msg), _ = reference.ternarize(g, 0.0, 1, 0, "t")
    assert st == 2 and "s=0 but gradient has nonzero element" in msg
    st, _ = restated.decode(np.array([0b11], np.uint8), 1, 1.0)
    (st2, msg), _ = reference.decode(np.array([0b11], np.uint8), 1, 1.0)
    assert st == 4 and "corrupt ternary code 11" in msg
    bad = np.array([1.0, np.nan], np.float32)
    st, *_ = restated.encode_step(["b"], [bad], Config(), 0, 0)
    (st2, msg), *_ = reference.encode_step(["b"], [bad], Config(), 0, 0)
    assert st == 3 and "non-finite gradient b" in msg


def test_restated_rng_base_offsets(restated, reference):
    # ternarize(name, part, s, rng, off) draws indices off..off+n-1 (codec.hpp:167)
    g = restated.normal(5, 0, "gauss/off", 1001, 1e-3)
    s = restated.scaler(g)
    for off in (0, 1, 2, 3, 4, 4097):
        st, c1 = restated.ternarize(g, s, 9, 3, "w", 2, off)
        (st2, _), c2 = reference.ternarize(g, s, 9, 3, "w", 2, off)
        assert st == st2 == 0 and bytes(c1) == bytes(c2)


def test_pull_equals_average_reference(reference, restated):
    # cluster_test.cpp:157-195: decode_pull(aggregate) == average, bit-exact
    names = ["a.w", "a.b"]
    for N in (2, 3):
        for sharing in (True, False):
            gw = [[restated.normal(100 + w, 0, "p/a", 300, 1e-2),
                   restated.normal(200 + w, 0, "p/b", 7, 1e-1)] for w in range(N)]
            cfg = Config(seed=42, scaler_sharing=sharing)
            (st, _), avg = reference.average_encoded(names, gw, cfg, 0)
            assert st == 0
            cl = RefCluster(reference, names, gw, cfg)
            assert cl.step(0) >= 0
            for w in range(N):
                assert np.array_equal(cl.output(w).view(np.uint32), avg.view(np.uint32))
            cl.close()


def test_statistical_properties(restated):
    # codec_test.cpp:38-47 clip fraction ~ 2*Phi(-2.5); :106-120 unbiasedness
    g = restated.normal(11, 0, "gauss/g", 200000)
    c, bound = restated.clip(g, 2.5)
    frac = float(np.mean(c != g))
    assert abs(frac - 0.01242) < 0.002
    small = np.array([0.3, -0.6, 0.05, 0.9], np.float32)
    s = restated.scaler(small)
    acc = np.zeros(4)
    T = 4000
    for t in range(T):
        st, codes = restated.ternarize(small, s, 3, t, "mc")
        _, dec = restated.decode(codes, 4, s)
        acc += dec
    assert np.allclose(acc / T, small, atol=0.05)


def test_restated_histogram_vs_reference(restated, reference):
    rng = np.random.default_rng(5)
    cases = [np.zeros(0, np.float32), np.full(7, 0.25, np.float32),
             np.array([1, 2, 3, 4, 5], np.float32),
             (rng.standard_normal(3001) * 1e-3).astype(np.float32),
             np.array([-0.0, 0.0, 1e-30, -1e-30, 3.0], np.float32)]
    for v in cases:
        for bins in (1, 2, 7, 64):
            e, c = restated.histogram(v, bins)
            (st, _), re_, rc = reference.histogram(v, bins)
            assert st == 0
            assert e.tobytes() == re_.tobytes() and c.tobytes() == rc.tobytes(), (v.size, bins)


@pytest.mark.parametrize("rule", [0, 1, 2])
def test_restated_optimizer_vs_reference(restated, reference, rule):
    rng = np.random.default_rng(10 + rule)
    for wd in (0.0, 5e-4):
        w = rng.standard_normal(4099).astype(np.float32)
        gs = [(rng.standard_normal(4099) * 1e-2).astype(np.float32) for _ in range(5)]
        rates = [0.1, 0.05, 0.3, 1e-3, 0.2]
        (st, msg), ref = reference.optimizer_run(rule, w, gs, rates, weight_decay=wd)
        assert st == 0, msg
        got = restated.optimizer_run(rule, w, gs, rates, weight_decay=wd)
        assert got.tobytes() == ref.tobytes(), (rule, wd)
