"""GPU parity: the sm_100a path through the C-ABI vs the CPU oracle.

Bar (BASELINE.json north_star): ternary codes, packed bytes and scalers
bit-exact; decoded fp32 within 1e-6 relative (asserted bit-exact here).
Inputs are the golden fixtures (tests/golden, generated from the reference)
plus full-size layers checked through size-independent properties and
sampled bit-exact windows.
"""
import hashlib

import numpy as np
import pytest
import torch

import paper_1705_07878_b200 as tg
from oracle.oracle import Config
from tests.golden.check import check_codes, check_scalers, passthrough_of
from tests.golden.recipes import make_input

pytestmark = pytest.mark.gpu

DEV = torch.device("cuda", 0)


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def cfg_of(d, **kw):
    return tg.CodecConfig(clip_factor=d["clip_factor"], clipping_enabled=d["clipping_enabled"],
                          bucketing=tg.Bucketing(d["bucketing"]), bucket_size=d["bucket_size"],
                          scaler_sharing=d["scaler_sharing"], seed=d["seed"], **kw)


def to_dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).to(DEV)


def plan_encode(names, grads, cfg, t, worker, n_workers=1, passthrough=None):
    ns = [int(g.size) for g in grads]
    plan = tg.Plan(names, ns, cfg, worker=worker, n_workers=n_workers, device=DEV,
                   passthrough=passthrough)
    gflat, gviews = tg.aligned_flat(ns, DEV)
    oflat, oviews = tg.aligned_flat(ns, DEV)
    for v, g in zip(gviews, grads):
        v.copy_(to_dev(g))
    plan.bind(gviews, oviews)
    plan.encode(t)
    plan.raise_errors()
    torch.cuda.synchronize()
    scal = plan.scalers().cpu().numpy().copy()
    codes = [plan.block_region(b).cpu().numpy().copy() for b, bi in enumerate(plan.blocks)
             if not bi.flags & 1]
    bounds = plan.bounds.cpu().numpy().copy()
    return plan, scal, codes, bounds, (gflat, gviews, oflat, oviews)


def tensor_bounds(plan, bounds):
    """per-tensor clip bound from the per-block array (inf for passthrough)"""
    out = np.full(len(plan.ns), np.inf, np.float32)
    for b, bi in enumerate(plan.blocks):
        if not bi.flags & 1 and bi.offset == 0:
            out[bi.layer] = bounds[b]
    return out


# ----------------------------------------------------------------- rng
def test_rng_bits_kats(golden):
    for c in golden["bits"]:
        rs = tg.RngStream(c["seed"], c["t"], c["name"], c["worker"])
        got = rs.bits_range(c["k0"], len(c["out"]), DEV).cpu().numpy().view(np.uint32)
        assert [int(x) for x in got] == c["out"]
    rs = tg.RngStream(42, 0, "fc.weight", 0)
    assert rs.bits(0) == 0xBA43FD1D


# ------------------------------------------------------ encode_step golden
def test_encode_step_golden(golden):
    for case in golden["encode"]:
        cfg = cfg_of(case["cfg"])
        names = [t["name"] for t in case["tensors"]]
        grads = [make_input(t["recipe"]) for t in case["tensors"]]
        pt = passthrough_of(case)
        plan, scal, codes, bounds, _ = plan_encode(names, grads, cfg, case["t"], case["worker"],
                                                   passthrough=pt)
        check_scalers(case, scal)
        check_codes(case, codes)
        assert tensor_bounds(plan, bounds).tobytes().hex() == case["bounds_hex"], case["name"]
        # the reference-shaped API returns the same blocks; passthrough blocks verbatim
        cfg.passthrough = {n for n, p in zip(names, pt) if p}
        res = tg.encode_step([tg.GradTensor(n, [g.size], to_dev(g)) for n, g in zip(names, grads)],
                             cfg, case["t"], case["worker"])
        tern = [b for b in res.encoded.blocks if isinstance(b, tg.TernaryBlock)]
        check_codes(case, [b.codes.cpu().numpy() for b in tern])
        check_scalers(case, res.local_scalers)
        raw = [b for b in res.encoded.blocks if isinstance(b, tg.PassthroughBlock)]
        want = [g for g, p in zip(grads, pt) if p]
        assert len(raw) == len(want)
        for b, g in zip(raw, want):
            assert b.values.cpu().numpy().tobytes() == np.asarray(g, np.float32).tobytes()
        plan.close()


def test_encode_unaligned_inputs(golden, restated):
    # gradients at a non-16B-aligned address take the scalar path: same bytes
    case = next(c for c in golden["encode"] if c["name"] == "gauss_n1000")
    g = make_input(case["tensors"][0]["recipe"])
    buf = torch.zeros(g.size + 1, dtype=torch.float32, device=DEV)
    buf[1:].copy_(to_dev(g))
    plan = tg.Plan(["layer.w"], [g.size], cfg_of(case["cfg"]), worker=case["worker"], device=DEV)
    out = torch.zeros(g.size + 1, dtype=torch.float32, device=DEV)
    plan.bind([buf[1:]], [out[1:]])
    plan.step(case["t"])
    plan.raise_errors()
    assert sha(plan.layer_codes(0).cpu().numpy()) == case["codes_sha256"][0]
    st, dec = restated.decode(plan.layer_codes(0).cpu().numpy(), g.size,
                              float(plan.scalers()[0].item()))
    assert np.array_equal(out[1:].cpu().numpy().view(np.uint32), dec.view(np.uint32))


# --------------------------------------------------- per-layer functions
def test_layer_functions_vs_oracle(golden, restated):
    for case in golden["encode"]:
        if len(case["tensors"]) != 1 or case["tensors"][0]["n"] == 0:
            continue
        t0 = case["tensors"][0]
        g = make_input(t0["recipe"])
        cfg = case["cfg"]
        gt = tg.GradTensor(t0["name"], [g.size], to_dev(g))
        # clip (codec.hpp:117-124)
        if cfg["clipping_enabled"]:
            c_dev = tg.clip(gt, cfg["clip_factor"]).values.cpu().numpy()
            c_ref, b_ref = restated.clip(g, cfg["clip_factor"])
            assert np.array_equal(c_dev.view(np.uint32), c_ref.view(np.uint32)), case["name"]
            assert np.float32(tg.clip_bound(gt, cfg["clip_factor"])) == np.float32(b_ref)
            part = c_ref
        else:
            part = g
        # scaler (codec.hpp:128-134)
        s = tg.scaler(to_dev(part))
        assert np.float32(s) == np.float32(restated.scaler(part)), case["name"]
        # ternarize (codec.hpp:148-175)
        rng = tg.RngStream(cfg["seed"], case["t"], t0["name"], case["worker"])
        blk = tg.ternarize(t0["name"], to_dev(part), s, rng)
        st, ref_codes = restated.ternarize(part, s, cfg["seed"], case["t"], t0["name"],
                                           case["worker"])
        assert st == 0
        assert bytes(blk.codes.cpu().numpy()) == bytes(ref_codes), case["name"]
        # decode (codec.hpp:177-182)
        d = tg.decode(blk).values.cpu().numpy()
        _, dref = restated.decode(ref_codes, g.size, s)
        assert np.array_equal(d.view(np.uint32), dref.view(np.uint32)), case["name"]


@pytest.mark.parametrize("off", [0, 1, 2, 3, 4, 4097, 65536 + 2])
def test_ternarize_rng_base(restated, off):
    g = restated.normal(5, 0, "gauss/off", 40001, 1e-3)
    s = restated.scaler(g)
    blk = tg.ternarize("w", to_dev(g), s, tg.RngStream(9, 3, "w", 2), rng_base=off)
    st, ref = restated.ternarize(g, s, 9, 3, "w", 2, off)
    assert st == 0 and bytes(blk.codes.cpu().numpy()) == bytes(ref)


def test_uniform_one_edge(restated):
    # |g| == s gives p = 1; uniform can be exactly 1.0f (bits >= 0xFFFFFF80) => code 0.
    # Scan a stream for such a draw and check the device reproduces it.
    rs = tg.RngStream(1, 0, "edge", 0)
    bits = rs.bits_range(0, 1 << 26, DEV).cpu().numpy().view(np.uint32)
    hits = np.nonzero(bits >= 0xFFFFFF80)[0]
    assert hits.size > 0
    k = int(hits[0])
    n = k + 1
    g = np.full(n, 0.5, np.float32)
    blk = tg.ternarize("edge", to_dev(g), 0.5, tg.RngStream(1, 0, "edge", 0))
    st, ref = restated.ternarize(g, 0.5, 1, 0, "edge", 0)
    assert bytes(blk.codes.cpu().numpy()) == bytes(ref)
    assert blk.code_at(k) == 0 and blk.code_at(0 if k else 1) == 1


# ------------------------------------------------------------- errors
def test_error_messages():
    bad = tg.GradTensor("b.w", [3], to_dev(np.array([1.0, np.nan, 2.0], np.float32)))
    with pytest.raises(tg.CodecError, match="encode_step: non-finite gradient b.w"):
        tg.encode_step([bad], tg.CodecConfig(), 0, 0)
    g = to_dev(np.array([0.5, -2.0, 0.25], np.float32))
    with pytest.raises(tg.CodecError, match=r"ternarize: scaler 1.000000 below max \|g\| in t"):
        tg.ternarize("t", g, 1.0, tg.RngStream(1, 0, "t"))
    with pytest.raises(tg.CodecError, match="s=0 but gradient has nonzero element"):
        tg.ternarize("t", g, 0.0, tg.RngStream(1, 0, "t"))
    blk = tg.TernaryBlock("c", 4, 1.0, torch.tensor([0b01001100], dtype=torch.uint8, device=DEV))
    with pytest.raises(tg.CodecError, match="corrupt ternary code 11 in block c at element 1"):
        tg.decode(blk)
    with pytest.raises(ValueError, match="clip factor must be positive"):
        tg.encode_step([], tg.CodecConfig(clip_factor=0.0), 0, 0)
    # the plan keeps working after an error was reported
    ok = tg.GradTensor("b.w", [3], to_dev(np.array([1.0, -1.0, 2.0], np.float32)))
    tg.encode_step([ok], tg.CodecConfig(), 0, 0)


# ------------------------------------------------------------ average
def test_average_golden(golden):
    for case in golden["average"]:
        cfg = cfg_of(case["cfg"])
        names = [t["name"] for t in case["tensors"]]
        pt = passthrough_of(case)
        cfg.passthrough = {n for n, p in zip(names, pt) if p}
        N = case["N"]
        encs, pushes, plans = [], [], []
        for w in range(N):
            grads = [make_input(dict(t["recipe"], worker=w)) for t in case["tensors"]]
            res = tg.encode_step([tg.GradTensor(n, [g.size], to_dev(g))
                                  for n, g in zip(names, grads)], cfg, case["t"], w)
            encs.append(res.encoded)
            plan, _, _, _, bufs = plan_encode(names, grads, cfg, case["t"], w, n_workers=N,
                                              passthrough=pt)
            pushes.append(plan.push.clone())
            plans.append((plan, bufs))
        # reference-shaped average (codec.hpp:245-311)
        avg = tg.average(encs, N, cfg.scaler_sharing)
        flat = torch.cat([a.values for a in avg]).cpu().numpy() if avg else np.zeros(0, np.float32)
        assert sha(flat) == case["out_sha256"], case["name"]
        if "out_hex" in case:
            assert flat.tobytes().hex() == case["out_hex"]
        # plan decode over N push buffers laid out back to back (= the allgather result)
        plan, (gflat, gviews, oflat, oviews) = plans[0]
        gathered = torch.cat(pushes)
        plan.decode_average(gathered, N)
        plan.raise_errors()
        out = torch.cat([v for v in oviews]).cpu().numpy()
        assert sha(out) == case["out_sha256"], case["name"] + " (plan)"
        # the whole step at N = 1 (K2 writes the decoded output) equals average([enc])
        if N == 1:
            plan.step(case["t"])
            plan.raise_errors()
            out = torch.cat([v for v in oviews]).cpu().numpy()
            assert sha(out) == case["out_sha256"], case["name"] + " (step)"
        for p, _ in plans:
            p.close()


# ------------------------------------------------------- full-size layers
def _fc6_like(n, seed):
    g = torch.Generator(device=DEV)
    g.manual_seed(seed)
    return torch.randn(n, generator=g, device=DEV, dtype=torch.float32) * 1e-3


@pytest.mark.parametrize("n", [102760448, 37748736 + 3])
def test_full_size_layer_sampled_bit_exact(restated, n):
    """VGG-16 fc6 / AlexNet fc6(+pad) at full size: sigma, bound and scaler vs
    the oracle over the whole tensor; codes and decode bit-exact on sampled
    windows (the oracle's ternarize with rng_base=offset is exactly the
    reference's draw for that window, codec.hpp:167)."""
    name = "classifier.0.weight"
    x = _fc6_like(n, 1234)
    cfg = tg.CodecConfig(seed=42)
    plan = tg.Plan([name], [n], cfg, worker=0, device=DEV)
    out = torch.empty_like(x)
    plan.bind([x], [out])
    t = 77
    plan.step(t)
    plan.raise_errors()
    xh = x.cpu().numpy()
    bound_ref = np.float32(np.float64(np.float32(2.5)) * restated.stddev(xh))
    bound = plan.bounds.cpu().numpy()[0]
    assert bound == bound_ref, "sigma-order mismatch (see DESIGN.md K1)"
    s = np.float32(plan.scalers()[0].item())
    assert s == min(np.float32(np.abs(xh).max()), bound_ref)
    codes = plan.layer_codes(0).cpu().numpy()
    # no corrupt codes, decode is in {-s, 0, s}
    assert not np.any((codes & (codes >> 1)) & 0x55)
    oh = out.cpu().numpy()
    assert set(np.unique(oh).tolist()) <= {-float(s), 0.0, float(s)}
    rng = np.random.default_rng(n)
    for _ in range(24):
        off = int(rng.integers(0, n - 8192)) // 4 * 4
        ln = 8192 if off + 8192 <= n else n - off
        part = xh[off:off + ln]
        part = np.where(np.abs(part) > bound_ref, np.copysign(bound_ref, part), part).astype(
            np.float32)
        st, ref = restated.ternarize(part, s, 42, t, name, 0, off)
        assert st == 0
        assert bytes(codes[off // 4: off // 4 + (ln + 3) // 4]) == bytes(ref)
        _, dref = restated.decode(ref, ln, s)
        assert np.array_equal(oh[off:off + ln].view(np.uint32), dref.view(np.uint32))
    # tail window (padding bits)
    off = (n - 1000) // 4 * 4
    part = xh[off:]
    part = np.where(np.abs(part) > bound_ref, np.copysign(bound_ref, part), part).astype(np.float32)
    st, ref = restated.ternarize(part, s, 42, t, name, 0, off)
    assert bytes(codes[off // 4:]) == bytes(ref)
    # statistical: clip fraction ~ 2*Phi(-2.5), zero fraction ~ 1 - E|x|/s
    assert abs(float(np.mean(np.abs(xh) > bound_ref)) - 0.01242) < 0.001
    plan.close()


def test_vgg16_step_properties():
    """Whole VGG-16 gradient set, 1 worker: every layer's decode is s*code with
    s = min(max|g|, bound); deterministic across repeated steps."""
    layers = tg.layersets.get("vgg16")
    names = [n for n, _ in layers]
    shapes = [s for _, s in layers]
    w = tg.SyncWorker(names, shapes, tg.CodecConfig(seed=42), device=DEV)
    g = torch.Generator(device=DEV)
    g.manual_seed(7)
    w.grad_flat.copy_(torch.randn(w.grad_flat.numel(), generator=g, device=DEV) * 1e-3)
    a = [o.clone() for o in w.step(5)]
    w.check()
    b = w.step(5)
    for x, y in zip(a, b):
        assert torch.equal(x, y)
    sc = w.plan.scalers().cpu()
    for l, o in enumerate(a):
        vals = torch.unique(o.cpu())
        assert all(v in (-sc[l], 0.0, sc[l]) for v in vals.tolist())


@pytest.mark.parametrize("bucketing,k,pt", [(0, 0, None), (2, 6, [0, 0, 1, 0, 0, 1]),
                                             (2, 4096, None), (1, 0, [1, 0, 0, 0, 0, 0])])
def test_plan_layout_matches_host_restatement(bucketing, k, pt):
    from paper_1705_07878_b200.layout import push_layout

    ns = [5, 0, 16, 1000003, 4096, 7]
    cfg = tg.CodecConfig(bucketing=tg.Bucketing(bucketing), bucket_size=k)
    plan = tg.Plan([f"l{i}" for i in range(len(ns))], ns, cfg, device=DEV, passthrough=pt)
    lay = push_layout(ns, pt, bucketing, k)
    assert plan.code_offsets == lay.code_offsets
    assert plan.info.push_bytes == lay.push_bytes
    assert plan.info.code_bytes == lay.code_bytes
    assert plan.info.n_slots == lay.n_slots
    assert [(b.layer, b.offset, b.n, b.slot, b.region_offset) for b in plan.blocks] == \
        [(b.layer, b.offset, b.n, b.slot, b.region_offset) for b in lay.blocks]
    plan.close()


# ------------------------------------------- FixedSize / passthrough at size
@pytest.mark.parametrize("k", [64, 256, 300, 1000, 4096, 4097, (1 << 20) + 3, 3 << 20])
def test_fixed_size_large_vs_oracle(restated, k):
    names = ["fc.weight", "fc.bias", "conv.weight"]
    grads = [restated.normal(21, 0, "fx/" + n, m, 1e-3) for n, m in
             zip(names, [(1 << 22) + 5, 1001, 300000])]
    cfg = Config(seed=42, bucketing=2, bucket_size=k)
    st, blocks, sc, _, _ = restated.encode_step(names, grads, cfg, 11, 3)
    assert st == 0
    plan, scal, codes, _, _ = plan_encode(names, grads, cfg_of(cfg.__dict__), 11, 3)
    assert scal.tobytes() == np.asarray(sc, np.float32).tobytes()
    assert len(codes) == len(blocks)
    assert np.concatenate(codes).tobytes() == np.concatenate(blocks).tobytes()
    plan.close()


def test_passthrough_and_bucket_errors():
    nan = np.array([1.0, 2.0, np.nan, 4.0, 5.0], np.float32)
    ok = np.array([0.5, -0.25, 0.125], np.float32)
    cfg = tg.CodecConfig(passthrough={"p"})
    with pytest.raises(tg.CodecError, match="encode_step: non-finite gradient p"):
        tg.encode_step([tg.GradTensor("w", [3], to_dev(ok)), tg.GradTensor("p", [5], to_dev(nan))],
                       cfg, 0, 0)
    cfg = tg.CodecConfig(bucketing=tg.Bucketing.FixedSize, bucket_size=2)
    with pytest.raises(tg.CodecError, match="encode_step: non-finite gradient q"):
        tg.encode_step([tg.GradTensor("w", [3], to_dev(ok)), tg.GradTensor("q", [5], to_dev(nan))],
                       cfg, 0, 0)
    # a corrupt code in the 2nd bucket reports the element inside that bucket
    res = tg.encode_step([tg.GradTensor("w", [9], to_dev(np.arange(9, dtype=np.float32)))],
                         tg.CodecConfig(bucketing=tg.Bucketing.FixedSize, bucket_size=5), 0, 0)
    blk = res.encoded.blocks[1]
    blk.codes[0] = 0b00110000  # element 2 of the bucket
    with pytest.raises(tg.CodecError, match="corrupt ternary code 11 in block w at element 2"):
        tg.average([res.encoded], 1, True)


@pytest.mark.parametrize("schedule", ["auto", "groups"])
def test_step_host_matches_device_step(restated, schedule):
    # tgb_step_host (host buffers in/out, copy streams; "groups": the per-layer-group
    # pipelined H2D -> compute -> D2H) == tgb_step on device buffers
    names = ["conv.weight", "conv.bias", "fc.weight"]
    ns = [1728, 64, 40003]
    cfg = tg.CodecConfig(seed=42)
    w = tg.SyncWorker(names, [[n] for n in ns], cfg, device=DEV, schedule=schedule)
    assert w.plan.grouped == (schedule == "groups")
    hin, hin_v, hout, hout_v = w.host_buffers()
    ref = tg.SyncWorker(names, [[n] for n in ns], cfg, device=DEV)
    for t in range(3):
        grads = [restated.normal(7 + t, 0, "host/" + nm, n, 1e-3) for nm, n in zip(names, ns)]
        for v, g in zip(hin_v, grads):
            v.copy_(torch.from_numpy(g))
        w.step_host(t, hin_v, hout_v)
        for v, g in zip(ref.grads, grads):
            v.copy_(to_dev(g))
        outs = ref.step(t)
        torch.cuda.synchronize()
        w.check()
        for o, h in zip(outs, hout_v):
            assert o.cpu().numpy().tobytes() == h.numpy().tobytes()
    with pytest.raises(ValueError):
        w.step_host(9, [h[:1] for h in hin_v], hout_v)
    # back-to-back steps, no synchronisation between them: every step reads its own
    # inputs and writes its own outputs (the copy streams' events order the reuse)
    sets = [w.host_buffers() for _ in range(3)]
    for k, (_, iv, _, _) in enumerate(sets):
        for v, nm, n in zip(iv, names, ns):
            v.copy_(torch.from_numpy(restated.normal(50 + k, 0, "host/" + nm, n, 1e-3)))
    for k, (_, iv, _, ov) in enumerate(sets):
        w.step_host(20 + k, iv, ov)
    torch.cuda.synchronize()
    w.check()
    for k, (_, iv, _, ov) in enumerate(sets):
        for v, h in zip(ref.grads, iv):
            v.copy_(h.to(DEV))
        outs = ref.step(20 + k)
        torch.cuda.synchronize()
        for o, h in zip(outs, ov):
            assert o.cpu().numpy().tobytes() == h.numpy().tobytes(), k


def test_histogram_vs_reference(restated):
    from oracle.oracle import Reference

    R = Reference()
    rng = np.random.default_rng(6)
    cases = [np.zeros(0, np.float32), np.full(70001, 0.25, np.float32),
             (rng.standard_normal(1_000_003) * 1e-3).astype(np.float32),
             np.array([-0.0, 0.0, 1e-30, -1e-30, 3.0], np.float32),
             np.array([np.nan, 1.0, 2.0], np.float32), np.array([1.0, np.nan, 2.0], np.float32)]
    for v in cases:
        for bins in (1, 3, 64, 5000):
            h = tg.histogram(to_dev(v) if v.size else torch.zeros(0, device=DEV), bins)
            (st, _), e, c = R.histogram(v, bins)
            assert st == 0
            got_e = np.array([b.edge for b in h], np.float64)
            got_c = np.array([b.count for b in h], np.uint64)
            assert got_e.tobytes() == e.tobytes(), (v.size, bins)
            assert got_c.tobytes() == c.tobytes(), (v.size, bins)


def test_zero_fraction_telemetry():
    # Worker::zero_fraction (cluster.hpp:336-346) of the last encode, counted inside K2
    names = ["a", "b", "c", "p"]
    ns = [1000003, 17, 0, 33]
    rng = np.random.default_rng(8)
    grads = [(rng.standard_normal(n) * 1e-2).astype(np.float32) for n in ns]
    for cfg, pt in [(tg.CodecConfig(seed=1), None),
                    (tg.CodecConfig(seed=1, bucketing=tg.Bucketing.FixedSize, bucket_size=999),
                     [0, 0, 0, 1])]:
        plan, scal, codes, _, _ = plan_encode(names, grads, cfg, 3, 0, passthrough=pt)
        plan.enable_code_stats()
        plan.encode(3)
        zeros = total = 0
        for b, bi in enumerate(plan.blocks):
            if bi.flags & 1:
                continue
            cb = np.frombuffer(bytes(plan.block_region(b).cpu().numpy()), np.uint8)
            lanes = np.stack([(cb >> (2 * e)) & 3 for e in range(4)], 1).reshape(-1)[:bi.n]
            zeros += int((lanes == 0).sum())
            total += bi.n
        assert plan.code_stats() == (total - zeros, total)
        assert plan.zero_fraction() == zeros / total
        plan.close()


@pytest.mark.parametrize("rule", [0, 1, 2])
def test_optimizer_apply_vs_reference(rule):
    from oracle.oracle import Reference

    R = Reference()
    rng = np.random.default_rng(20 + rule)
    for wd in (0.0, 5e-4):
        ns = [70001, 5, 1]
        ws = [rng.standard_normal(n).astype(np.float32) for n in ns]
        gs = [[(rng.standard_normal(n) * 1e-2).astype(np.float32) for n in ns] for _ in range(4)]
        rates = [0.1, 0.05, 0.3, 1e-3]
        st = tg.OptimizerState(tg.OptimizerConfig(rule=tg.OptimizerRule(rule), weight_decay=wd))
        params = [to_dev(w) for w in ws]
        for k, r in enumerate(rates):
            st.apply(params, [to_dev(g) for g in gs[k]], r)
        for l in range(len(ns)):
            (s, msg), ref = R.optimizer_run(rule, ws[l], [gs[k][l] for k in range(4)], rates,
                                            weight_decay=wd)
            assert s == 0, msg
            assert params[l].cpu().numpy().tobytes() == ref.tobytes(), (rule, wd, l)


@pytest.mark.parametrize("rule,fused", [(1, 1), (1, 0), (2, 1), (0, 1)])
def test_step_apply_matches_step_then_optimizer(restated, rule, fused):
    # tgb_step_apply (fused: the decode kernel applies the optimizer, the averaged
    # gradient is never written) == tgb_step + OptimizerState::apply
    names = ["conv.weight", "conv.bias", "fc.weight", "p"]
    ns = [1728, 64, 40003, 33]
    cfg = tg.CodecConfig(seed=42, passthrough={"p"})
    ocfg = tg.OptimizerConfig(rule=tg.OptimizerRule(rule), weight_decay=1e-4)
    w = tg.SyncWorker(names, [[n] for n in ns], cfg, device=DEV)
    w.plan.set_option(tg._lib.TGB_PLAN_OPT_FUSED_OPTIMIZER, fused)
    p0 = [(np.arange(n, dtype=np.float32) % 7) * 0.01 for n in ns]
    params = [to_dev(p) for p in p0]
    w.bind_optimizer(ocfg, params)
    ref = tg.SyncWorker(names, [[n] for n in ns], cfg, device=DEV)
    ref_params = [to_dev(p) for p in p0]
    ref_state = tg.OptimizerState(ocfg)
    for t, rate in enumerate([0.1, 0.05, 0.2]):
        grads = [restated.normal(30 + t, 0, "opt/" + nm, n, 1e-3) for nm, n in zip(names, ns)]
        for v, r, g in zip(w.grads, ref.grads, grads):
            v.copy_(to_dev(g))
            r.copy_(to_dev(g))
        w.step_apply(t, rate)
        ref_state.apply(ref_params, ref.step(t), rate)
        torch.cuda.synchronize()
        w.check()
        for a, b in zip(params, ref_params):
            assert a.cpu().numpy().tobytes() == b.cpu().numpy().tobytes()


@pytest.mark.parametrize("bucketing,k,pt,sharing", [(0, 0, [0, 0, 0, 0], True),
                                                    (2, 5, [0, 1, 0, 0], True),
                                                    (0, 0, [0, 0, 0, 1], False)])
def test_wire_push_and_pull_match_reference(bucketing, k, pt, sharing):
    # interop with the reference's parameter server: our push frame is byte-identical to
    # frame(Message{Push, ...serialize_encoded}) and decoding its radix-packed pull frame
    # gives the workers' decode_pull bit-for-bit (cluster.hpp:283-297)
    from oracle.oracle import Config, Reference, RefCluster

    R = Reference()
    names = ["conv.weight", "conv.bias", "empty", "fc.weight"]
    ns = [1728, 64, 0, 40003]
    N, t = 3, 11
    rng = np.random.default_rng(3)
    gw = [[(rng.standard_normal(n) * 1e-2).astype(np.float32) for n in ns] for _ in range(N)]
    ocfg = Config(seed=42, bucketing=bucketing, bucket_size=k, scaler_sharing=sharing)
    c = RefCluster(R, names, gw, ocfg, passthrough=pt)
    c.step(t)
    want = c.output(0)
    cfg = tg.CodecConfig(seed=42, bucketing=tg.Bucketing(bucketing), bucket_size=k,
                         scaler_sharing=sharing,
                         passthrough={n for n, p in zip(names, pt) if p})
    for w in range(N):
        plan, _, _, _, (gflat, gviews, oflat, oviews) = plan_encode(names, gw[w], cfg, t, w,
                                                                     n_workers=N)
        assert plan.serialize_push(t) == c.frame(w, 0), w
        assert plan.decode_pull(c.frame(w, 1)) == t
        got = torch.cat([v for v in oviews]).cpu().numpy()
        assert got.tobytes() == want.tobytes(), w
        plan.close()


def test_wire_protocol_errors():
    from oracle.oracle import Config, Reference, RefCluster

    R = Reference()
    gw = [[np.full(9, 0.5, np.float32)] for _ in range(2)]
    c = RefCluster(R, ["w"], gw, Config(seed=1))
    c.step(0)
    pull = c.frame(0, 1)
    plan, _, _, _, _ = plan_encode(["w"], gw[0], tg.CodecConfig(seed=1), 0, 0, n_workers=2)
    with pytest.raises(tg.ProtocolError, match="bad magic"):
        plan.decode_pull(b"\x00" + pull[1:])
    with pytest.raises(tg.ProtocolError, match="worker: expected Pull"):
        plan.decode_pull(c.frame(0, 0))
    with pytest.raises(tg.ProtocolError, match="payload length mismatch"):
        plan.decode_pull(pull[:-1])
    bad = bytearray(pull)
    bad[-1] = 0xFF  # last radix word's top byte: digits beyond n are not zero
    with pytest.raises(tg.ProtocolError, match="nonzero radix remainder"):
        plan.decode_pull(bytes(bad))
    plan.close()


def test_live_kernel_timing_records():
    """tgb_plan_enable_timing: one record per launch with its algorithmic bytes
    (N = 1 step = K1 + K2 with the fused decode)."""
    names, ns = ["a.w", "b.w"], [1000, 40003]
    sw = tg.SyncWorker(names, [[n] for n in ns], tg.CodecConfig(seed=42), device=DEV,
                       schedule="unfused")
    sw.grad_flat.normal_(0.0, 1e-3)
    sw.step(0)
    sw.plan.enable_timing(16)
    for t in range(3):
        sw.step(1 + t)
    recs = sw.plan.read_timing()
    sw.plan.enable_timing(0)
    sw.check()
    kinds = [r["kernel"] for r in recs]
    assert kinds.count("K1_stats") == 3 * (2 if sw.plan.grouped else 1)
    n = sum(ns)
    k1 = sum(r["hbm_bytes"] for r in recs if r["kernel"] == "K1_stats")
    k2 = sum(r["hbm_bytes"] for r in recs if r["kernel"] == "K2_ternarize_pack")
    assert k1 == 3 * 4 * n
    assert k2 == 3 * (4 * n + 4 * n + (1000 + 3) // 4 + (40003 + 3) // 4) or \
        k2 == 3 * (4 * n + 4 * n + (n + 3) // 4)
    assert all(r["ms"] > 0 and r["start_ms"] >= 0 for r in recs)
    sw.plan.close()


def test_fused_k12_matches_separate_launches():
    """K1 + K2 as one persistent launch (k12_fused, opt-in schedule); its output,
    codes and scalers equal the two-launch schedule's, every bucketing mode,
    including replays of the same iteration (the ready flags reset per launch)"""
    names = ["conv.weight", "conv.bias", "empty", "fc.weight", "fc.bias", "p"]
    ns = [1728, 64, 0, 40003, 10, 77]
    for cfg in (tg.CodecConfig(seed=42, passthrough={"p"}),
                tg.CodecConfig(seed=42, bucketing=tg.Bucketing.Global),
                tg.CodecConfig(seed=42, bucketing=tg.Bucketing.FixedSize, bucket_size=300)):
        outs = {}
        for sched in ("fused12", "unfused"):
            sw = tg.SyncWorker(names, [[n] for n in ns], cfg, device=DEV, schedule=sched)
            sw.grad_flat.normal_(0.0, 1e-3, generator=torch.Generator(device=DEV).manual_seed(5))
            sw.plan.enable_timing(8)
            for t in (3, 3, 4):
                sw.step(t, check=True)
            kinds = {r["kernel"] for r in sw.plan.read_timing()}
            sw.plan.enable_timing(0)
            fixed = cfg.bucketing == tg.Bucketing.FixedSize  # (never fused: bucket slots)
            assert ("K12_fused" in kinds) == (sched == "fused12" and not fixed), kinds
            outs[sched] = (sw.out_flat.clone(), sw.plan.scalers().clone(),
                           torch.cat([sw.plan.block_region(b).view(torch.uint8).clone()
                                      for b in range(len(sw.plan.blocks))]))
            sw.plan.close()
        for a, b in zip(outs["fused12"], outs["unfused"]):
            assert torch.equal(a, b)


@pytest.mark.parametrize("k", [64, 256, 4096])
def test_fixed_size_multibucket_step_vs_oracle(restated, k):
    """FixedSize(k), k = 2^p: work items of whole buckets (K1 per-bucket maxima,
    k1_bucket_slots, per-bucket decision constants in K2, the N = 1 fused decode)
    == the oracle's encode_step + decode per bucket, incl. ragged last buckets"""
    names = ["fc.weight", "fc.bias", "conv.weight"]
    ns = [(1 << 20) + 67, 1001, 300003]
    grads = [restated.normal(23, 0, "mb/" + n, m, 1e-3) for n, m in zip(names, ns)]
    cfg = tg.CodecConfig(seed=42, bucketing=tg.Bucketing.FixedSize, bucket_size=k)
    sw = tg.SyncWorker(names, [[n] for n in ns], cfg, device=DEV)
    for v, g in zip(sw.grads, grads):
        v.copy_(to_dev(g))
    for t in (4, 5):
        sw.step(t, check=True)
    st, blocks, sc, _, _ = restated.encode_step(names, grads, Config(seed=42, bucketing=2,
                                                                     bucket_size=k), 5, 0)
    assert st == 0
    assert sw.plan.scalers().cpu().numpy().tobytes() == np.asarray(sc, np.float32).tobytes()
    want = np.concatenate([restated.decode(b, n_b, float(s))[1] for b, s, n_b in
                           zip(blocks, sc, [bi.n for bi in sw.plan.blocks])])
    got = np.concatenate([o.cpu().numpy() for o in sw.outs])
    assert got.view(np.uint32).tobytes() == want.view(np.uint32).tobytes()
    sw.plan.close()


def test_plan_audit_every_layout():
    """tgb_plan_audit over the layouts the tests and the bench build: block regions
    inside the push area, work items tiling their blocks (incl. multi-bucket items),
    sharded sums regions disjoint and inside the sums buffer, owners tiling pieces,
    barrier records inside the peer-exchange allocation (the class of bug a
    memcheck run would catch; compute-sanitizer is closed on the GPU pool)"""
    small = (["conv.weight", "conv.bias", "empty", "fc.weight", "fc.bias"],
             [1728, 64, 0, 40003, 10])
    g = tg.layersets.get("googlenet")
    sets = [small, ([n for n, _ in g], [tg.layersets.numel(s) for _, s in g])]
    cfgs = [tg.CodecConfig(seed=42), tg.CodecConfig(seed=42, bucketing=tg.Bucketing.Global),
            tg.CodecConfig(seed=42, scaler_sharing=False)] + \
        [tg.CodecConfig(seed=42, bucketing=tg.Bucketing.FixedSize, bucket_size=k,
                        passthrough={"conv.bias"}) for k in (7, 64, 256, 1000, 4096, 1 << 20)]
    n_checked = 0
    for names, ns in sets:
        for cfg in cfgs:
            for N, ex, pieces in ((1, "auto", 0), (2, "fused", 0), (3, "sharded", 2),
                                  (5, "sharded", 0), (8, "auto", 0), (8, "fused", 0)):
                if ex == "sharded" and not cfg.scaler_sharing:
                    continue
                plans = []
                for w in range(N):
                    p = tg.Plan(names, ns, cfg, worker=w, n_workers=N, device=DEV)
                    if N > 1 and ex != "auto":
                        p.set_exchange(ex)
                    if pieces:
                        p.set_pieces(pieces)
                    p.audit()
                    plans.append(p)
                if N > 1 and len(names) < 10:  # attach (IPC layout, barrier records)
                    flats = [tg.aligned_flat(ns, DEV) for _ in range(N)]
                    for p, (_, views) in zip(plans, flats):
                        p.bind(views, views)
                    tg.Plan.attach_local(plans)
                    for p in plans:
                        p.audit()
                n_checked += len(plans)
                for p in plans:
                    p.close()
    vgg = tg.layersets.get("vgg16")
    for cfg in (tg.CodecConfig(seed=42), tg.CodecConfig(seed=42, bucketing=tg.Bucketing.FixedSize,
                                                        bucket_size=256)):
        for N in (1, 4, 8):
            p = tg.Plan([n for n, _ in vgg], [tg.layersets.numel(s) for _, s in vgg], cfg,
                        worker=0, n_workers=N, device=DEV)
            p.audit()
            p.close()
    assert n_checked > 100
