"""Deterministic input recipes for the golden fixtures.

"normal" recipes use the reference's own RngStream::normal (rng.hpp:74-79),
evaluated by the plain-C restatement (oracle/_build) — pinned against the
reference by the input sha256 stored in golden.json.
"""
from __future__ import annotations

import numpy as np

_R = None


def _restated():
    global _R
    if _R is None:
        from oracle.oracle import Restated

        _R = Restated()
    return _R


def make_input(r: dict) -> np.ndarray:
    k = r["kind"]
    w = int(r.get("worker", 0))
    if k == "list":
        return np.array(r["v"], dtype=np.float32)
    n = int(r["n"])
    if k == "normal":
        v = _restated().normal(int(r["seed"]) + 1000 * w, int(r["t"]), r["name"], n,
                               float(r.get("scale", 1.0)))
        if "offset" in r:
            v = (v + np.float32(r["offset"])).astype(np.float32)
        return v
    if k == "const":
        return np.full(n, r["v"], dtype=np.float32)
    if k == "signed_zeros":
        v = np.zeros(n, dtype=np.float32)
        v[1::2] = -0.0
        return v
    rng = np.random.default_rng(int(r.get("seed", 0)) + 1000 * w)
    if k == "outlier":
        v = (rng.standard_normal(n) * 1e-3).astype(np.float32)
        v[int(r["pos"])] = np.float32(r["amp"])
        return v
    if k == "subnormal":
        m = rng.integers(1, 1 << 23, size=n, dtype=np.int64).astype(np.uint32)
        sign = (rng.integers(0, 2, size=n).astype(np.uint32) << 31)
        return (m | sign).view(np.float32)
    if k == "pm_max":
        v = np.full(n, 0.25, dtype=np.float32)  # every |x| equals max: p = 1 (codec_test 81-88)
        v[1::3] = np.float32(-0.25)
        v[2::5] = np.float32(0.125)
        return v
    if k == "uniform":
        return (rng.random(n, dtype=np.float32) * 2 - 1).astype(np.float32)
    raise ValueError(k)
