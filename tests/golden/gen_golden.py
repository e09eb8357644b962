"""Generates tests/golden/golden.json from the REFERENCE itself.

Every expected output here comes from oracle/_ref/libtgref.so — the
reference headers (/root/reference/proj/include/terngrad) compiled unmodified
by oracle/Makefile. Run in the build container (where /root/reference
exists):  python tests/golden/gen_golden.py
Inputs are either stored verbatim (small cases, hex float32) or as a recipe
plus the sha256 of the input bytes (large cases).
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle.oracle import Config, Reference  # noqa: E402
from tests.golden.recipes import make_input  # noqa: E402

ref = Reference()


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def f32hex(a) -> str:
    return np.ascontiguousarray(a, dtype=np.float32).tobytes().hex()


def enc_case(name, tensors, cfg, t, worker, store_inputs=True, passthrough=None):
    names = [n for n, _ in tensors]
    grads = [make_input(r) for _, r in tensors]
    (st, msg), blocks, scal = ref.encode_step(names, grads, cfg, t, worker, passthrough)
    bounds = []  # clip bound per tensor; passthrough tensors are never clipped (codec.hpp:206)
    for i, g in enumerate(grads):
        if cfg.clipping_enabled and g.size >= 2 and not (passthrough and passthrough[i]):
            _, b = ref.clip(g, cfg.clip_factor)
        else:
            b = float("inf")
        bounds.append(float(np.float32(b)))
    case = {
        "name": name, "t": t, "worker": worker,
        "cfg": {"clip_factor": cfg.clip_factor, "clipping_enabled": cfg.clipping_enabled,
                "bucketing": cfg.bucketing, "bucket_size": cfg.bucket_size,
                "scaler_sharing": cfg.scaler_sharing, "seed": cfg.seed},
        "tensors": [{"name": n, "recipe": r, "n": int(g.size), "input_sha256": sha(g),
                     **({"input_hex": f32hex(g)} if store_inputs else {})}
                    for (n, r), g in zip(tensors, grads)],
        **({"passthrough": [int(x) for x in passthrough]} if passthrough else {}),
        "status": st, "error": msg,
        "bounds_hex": f32hex(np.array(bounds, dtype=np.float32)),
        "n_blocks": len(blocks),
    }
    if len(blocks) <= 64:
        case.update({"scalers_hex": f32hex(scal),
                     "codes": [bytes(b).hex() if store_inputs else None for b in blocks],
                     "codes_sha256": [sha(b) for b in blocks]})
    else:  # many buckets: digests of the concatenations keep the fixture small
        case.update({"scalers_sha256": sha(np.asarray(scal, np.float32)),
                     "codes_concat_sha256": sha(np.concatenate(blocks))})
    return case


def avg_case(name, tensors, cfg, t, N, store=True, passthrough=None):
    names = [n for n, _ in tensors]
    gw = [[make_input(dict(r, worker=w)) for _, r in tensors] for w in range(N)]
    (st, msg), out = ref.average_encoded(names, gw, cfg, t, passthrough)
    return {
        "name": name, "t": t, "N": N,
        "cfg": {"clip_factor": cfg.clip_factor, "clipping_enabled": cfg.clipping_enabled,
                "bucketing": cfg.bucketing, "bucket_size": cfg.bucket_size,
                "scaler_sharing": cfg.scaler_sharing, "seed": cfg.seed},
        "tensors": [{"name": n, "recipe": r, "n": int(gw[0][i].size)}
                    for i, (n, r) in enumerate(tensors)],
        **({"passthrough": [int(x) for x in passthrough]} if passthrough else {}),
        "status": st, "error": msg,
        "out_sha256": sha(out),
        **({"out_hex": f32hex(out)} if store else {}),
    }


def main():
    g = {}
    # --- KATs (rng.hpp) ---
    g["philox"] = []
    for ctr, key in [([0, 0, 0, 0], [0, 0]),
                     ([0xFFFFFFFF] * 4, [0xFFFFFFFF] * 2),
                     ([0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344], [0xA4093822, 0x299F31D0])]:
        g["philox"].append({"ctr": ctr, "key": key, "out": ref.philox(ctr, key)})
    g["fnv1a64"] = {n: ref.fnv1a64(n) for n in ["", "a", "fc.weight", "classifier.0.weight",
                                                 "features.0.bias"]}
    g["bits"] = []
    for seed, t, name, w, k0, n in [(42, 0, "fc.weight", 0, 0, 8),
                                    (7, 12345678901, "bench", 5, 1000, 16),
                                    (2**63 + 11, 2**40 + 3, "classifier.0.weight", 7, 2**33, 8)]:
        g["bits"].append({"seed": seed, "t": t, "name": name, "worker": w, "k0": k0,
                          "out": [int(x) for x in ref.bits(seed, t, name, w, k0, n)]})
    g["uniform_edges"] = {"0xffffff80": float(np.float32(np.float32(0xFFFFFF80) * np.float32(2**-32))),
                          "0xffffff7f": float(np.float32(np.float32(0xFFFFFF7F) * np.float32(2**-32)))}

    # --- encode_step cases ---
    enc = []
    bench = {"kind": "normal", "seed": 7, "t": 0, "name": "bench", "scale": 1.0}
    enc.append(enc_case("kat1_bench19", [("g", dict(bench, n=19))], Config(seed=7), 0, 0))
    enc.append(enc_case("kat2_bench19_t_w5", [("g", dict(bench, n=19))], Config(seed=7),
                        12345678901, 5))
    enc.append(enc_case("kat3_noclip",
                        [("fc.weight", {"kind": "list", "v": [0.5, -0.25, 0.125, -1, 0, 0.75, -0.5, 0.3]}),
                         ("fc.bias", {"kind": "list", "v": [0.1, -0.2, 0.05]})],
                        Config(seed=42, clipping_enabled=False), 0, 0))
    enc.append(enc_case("bench_1M", [("g", dict(bench, n=1000000))], Config(seed=7), 0, 0,
                        store_inputs=False))
    enc.append(enc_case("bench_1M_pad", [("g", dict(bench, n=1000003))], Config(seed=7), 3, 1,
                        store_inputs=False))
    small = [0, 1, 2, 3, 4, 5, 7, 15, 16, 17, 63, 1000]
    for n in small:
        enc.append(enc_case(f"gauss_n{n}", [("layer.w", {"kind": "normal", "seed": 11, "t": 0,
                                                          "name": f"gauss/{n}", "scale": 1e-3,
                                                          "n": n})],
                            Config(seed=42), 1, 2))
    edge = [
        ("zeros", {"kind": "const", "v": 0.0, "n": 37}),
        ("negzeros", {"kind": "signed_zeros", "n": 41}),
        ("constant", {"kind": "const", "v": 0.0123, "n": 50}),
        ("constant_neg", {"kind": "const", "v": -3.5, "n": 33}),
        ("outlier0", {"kind": "outlier", "pos": 0, "amp": 1e3, "n": 4099, "seed": 5}),
        ("outlier_mid", {"kind": "outlier", "pos": 2000, "amp": -7e2, "n": 4099, "seed": 6}),
        ("subnormal", {"kind": "subnormal", "n": 64, "seed": 9}),
        ("pm_max", {"kind": "pm_max", "n": 40}),
        ("tiny_scale", {"kind": "normal", "seed": 3, "t": 0, "name": "tiny", "scale": 1e-30,
                        "n": 513}),
        ("huge_scale", {"kind": "normal", "seed": 4, "t": 0, "name": "huge", "scale": 1e30,
                        "n": 513}),
        ("uniform", {"kind": "uniform", "seed": 12, "n": 2048}),
        ("mean_offset", {"kind": "normal", "seed": 13, "t": 0, "name": "off", "scale": 1e-3,
                         "offset": 0.5, "n": 3000}),
    ]
    for name, r in edge:
        enc.append(enc_case("edge_" + name, [(name, r)], Config(seed=42), 0, 0))
        enc.append(enc_case("edge_noclip_" + name, [(name, r)],
                            Config(seed=42, clipping_enabled=False), 5, 1))
    # multi-tensor + global bucketing
    multi = [("conv1.weight", {"kind": "normal", "seed": 21, "t": 0, "name": "m/a", "scale": 1e-2, "n": 1728}),
             ("conv1.bias", {"kind": "normal", "seed": 22, "t": 0, "name": "m/b", "scale": 1e-1, "n": 64}),
             ("empty", {"kind": "list", "v": []}),
             ("fc.weight", {"kind": "normal", "seed": 23, "t": 0, "name": "m/c", "scale": 3e-3, "n": 40003}),
             ("fc.bias", {"kind": "normal", "seed": 24, "t": 0, "name": "m/d", "scale": 1e-3, "n": 10})]
    enc.append(enc_case("multi_per_tensor", multi, Config(seed=42), 9, 3, store_inputs=False))
    enc.append(enc_case("multi_global", multi, Config(seed=42, bucketing=1), 9, 3,
                        store_inputs=False))
    enc.append(enc_case("multi_global_noclip", multi, Config(seed=42, bucketing=1,
                                                             clipping_enabled=False), 2, 0,
                        store_inputs=False))
    # FixedSize(k) buckets (codec.hpp:226-236): k % 4 != 0 shifts the RNG lanes
    # against the code bytes; k = 1 is the clip-equals-bucket case (codec_test 241-254)
    for k in (1, 3, 4, 5, 7, 64, 1000, 16385, 40000):
        enc.append(enc_case(f"fixed_k{k}", multi, Config(seed=42, bucketing=2, bucket_size=k),
                            6, 1, store_inputs=False))
    enc.append(enc_case("fixed_k13_noclip", multi, Config(seed=42, bucketing=2, bucket_size=13,
                                                          clipping_enabled=False), 1, 2,
                        store_inputs=False))
    # passthrough tensors (codec.hpp:206-209, 221-224), alone and with buckets / Global
    pt = [0, 1, 0, 0, 1]
    enc.append(enc_case("passthrough_per_tensor", multi, Config(seed=42), 2, 1,
                        store_inputs=False, passthrough=pt))
    enc.append(enc_case("passthrough_global", multi, Config(seed=42, bucketing=1), 2, 1,
                        store_inputs=False, passthrough=pt))
    enc.append(enc_case("passthrough_fixed_k6", multi, Config(seed=42, bucketing=2,
                                                              bucket_size=6), 2, 1,
                        store_inputs=False, passthrough=[1, 0, 0, 0, 0]))
    enc.append(enc_case("float_mode", multi, Config(seed=42), 2, 1, store_inputs=False,
                        passthrough=[1] * len(multi)))
    g["encode"] = enc

    # --- average across workers (inputs per worker from recipe + worker) ---
    avg = []
    for N in (1, 2, 3, 4, 8):
        for sharing in (True, False):
            avg.append(avg_case(f"avg_N{N}_{'shared' if sharing else 'unshared'}", multi,
                                Config(seed=42, scaler_sharing=sharing), 4, N, store=False))
    tiny = [("a.w", {"kind": "normal", "seed": 31, "t": 0, "name": "t/a", "scale": 1e-2, "n": 9}),
            ("a.b", {"kind": "list", "v": [0.5, -0.25, 0.125]})]
    for N in (2, 3):
        for sharing in (True, False):
            avg.append(avg_case(f"avg_tiny_N{N}_{'shared' if sharing else 'unshared'}", tiny,
                                Config(seed=42, scaler_sharing=sharing, clipping_enabled=False),
                                0, N, store=True))
    for N in (2, 3):
        for sharing in (True, False):
            sh = "shared" if sharing else "unshared"
            avg.append(avg_case(f"avg_fixed_k5_N{N}_{sh}", multi,
                                Config(seed=42, scaler_sharing=sharing, bucketing=2,
                                       bucket_size=5), 3, N, store=False))
            avg.append(avg_case(f"avg_fixed_k1000_N{N}_{sh}", multi,
                                Config(seed=42, scaler_sharing=sharing, bucketing=2,
                                       bucket_size=1000), 3, N, store=False))
            avg.append(avg_case(f"avg_passthrough_N{N}_{sh}", multi,
                                Config(seed=42, scaler_sharing=sharing), 3, N, store=False,
                                passthrough=[0, 1, 0, 0, 1]))
    avg.append(avg_case("avg_float_mode_N3", multi, Config(seed=42), 3, 3, store=False,
                        passthrough=[1] * len(multi)))
    avg.append(avg_case("avg_passthrough_fixed_k7_N2", multi,
                        Config(seed=42, bucketing=2, bucket_size=7), 3, 2, store=False,
                        passthrough=[0, 0, 0, 1, 0]))
    g["average"] = avg

    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(g, f, indent=1)
    print("wrote", len(enc), "encode cases,", len(avg), "average cases")


if __name__ == "__main__":
    main()
