"""Comparison helpers for the golden fixtures (per-block hex/sha lists for
small cases, digests of the concatenations for many-bucket cases)."""
from __future__ import annotations

import hashlib

import numpy as np


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def passthrough_of(case):
    return case.get("passthrough") or [0] * len(case["tensors"])


def check_scalers(case, scal) -> None:
    scal = np.asarray(scal, np.float32)
    if "scalers_hex" in case:
        assert scal.tobytes().hex() == case["scalers_hex"], case["name"]
    else:
        assert sha(scal) == case["scalers_sha256"], case["name"]


def check_codes(case, blocks) -> None:
    """blocks: the ternary blocks' code bytes in canonical order"""
    assert len(blocks) == case["n_blocks"], case["name"]
    if "codes_sha256" in case:
        assert [sha(np.asarray(b, np.uint8)) for b in blocks] == case["codes_sha256"], case["name"]
    else:
        cat = np.concatenate([np.asarray(b, np.uint8) for b in blocks]) if blocks else \
            np.zeros(0, np.uint8)
        assert sha(cat) == case["codes_concat_sha256"], case["name"]


def restated_average(restated, names, grads_per_worker, cfg, t, passthrough=None):
    """average (codec.hpp:245-311) composed from the restated block functions:
    encode every worker, then per block the shared/unshared ternary average or
    the passthrough fp64 mean; flat output in canonical order."""
    from oracle.oracle import block_layout

    N = len(grads_per_worker)
    ns = [g.size for g in grads_per_worker[0]]
    passthrough = passthrough or [0] * len(ns)
    enc = []
    for w in range(N):
        st, blocks, sc, _, _ = restated.encode_step(names, grads_per_worker[w], cfg, t, w,
                                                    passthrough)
        assert st == 0
        enc.append((blocks, sc))
    lay = block_layout(ns, cfg, passthrough)
    out, b = [], 0
    for l, n in enumerate(ns):
        if passthrough[l]:
            out.append(restated.average_passthrough([gw[l] for gw in grads_per_worker]))
            continue
        while b < len(lay) and lay[b][0] == l:
            st, o = restated.average_block([e[1][b] for e in enc], [e[0][b] for e in enc],
                                           lay[b][2], cfg.scaler_sharing)
            assert st == 0
            out.append(o)
            b += 1
    return np.concatenate(out) if out else np.zeros(0, np.float32)
