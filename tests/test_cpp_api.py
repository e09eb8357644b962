"""The C++ host mirror (include/tgb/terngrad.hpp) over the C-ABI.

build/tgb_cpp_api_test (compiled by __graft_entry__.build from
tests/cpp/test_api.cpp) exercises encode_step / average / SyncWorker / clip /
scaler / ternarize / decode / CodecError on deterministic LCG inputs; this
test restates the LCG and checks every byte against the CPU oracle.
"""
import os
import struct
import subprocess
import tempfile

import numpy as np
import pytest
import torch

from oracle.oracle import Config
from tests.golden.check import restated_average

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "build", "tgb_cpp_api_test")
NAMES = ["conv.weight", "conv.bias", "fc.weight"]
SIZES = [1728, 64, 40003]


def lcg(seed, n, scale):
    x = np.uint64(seed)
    out = np.empty(n, np.float32)
    a, c = np.uint64(6364136223846793005), np.uint64(1442695040888963407)
    with np.errstate(over="ignore"):
        for k in range(n):
            x = x * a + c
            out[k] = (np.float32(int(x >> np.uint64(40))) * np.float32(2 ** -24) -
                      np.float32(0.5)) * np.float32(scale)
    return out


def read_sections(path):
    data = open(path, "rb").read()
    pos, out = 0, []
    while pos < len(data):
        (n,) = struct.unpack_from("<Q", data, pos)
        pos += 8
        out.append(data[pos:pos + n])
        pos += n
    return out


def test_cpp_binary_built():
    assert os.path.exists(BIN), "run __graft_entry__.build()"


@pytest.mark.skipif(torch.cuda.is_available(), reason="GPU present")
def test_cpp_api_fails_loudly_without_device():
    with tempfile.TemporaryDirectory() as d:
        r = subprocess.run([BIN, os.path.join(d, "o.bin")], capture_output=True, text=True,
                           timeout=120)
    assert r.returncode != 0


@pytest.mark.gpu
def test_cpp_api_matches_oracle(restated):
    with tempfile.TemporaryDirectory() as d:
        out = os.path.join(d, "o.bin")
        r = subprocess.run([BIN, out], capture_output=True, text=True, timeout=300)
        assert r.returncode == 0, r.stdout + r.stderr
        sec = read_sections(out)
    grads = [[lcg(1000 * (w + 1) + l, SIZES[l], 1e-2) for l in range(3)] for w in range(2)]
    cfg = Config(seed=42)
    i = 0
    enc = []
    for w in range(2):
        st, blocks, sc, _, _ = restated.encode_step(NAMES, grads[w], cfg, 3, w)
        assert sec[i] == sc.tobytes(); i += 1
        for b in blocks:
            assert sec[i] == bytes(b); i += 1
        enc.append((blocks, sc))
    for sharing in (True, False):
        for l in range(3):
            st, avg = restated.average_block([enc[w][1][l] for w in range(2)],
                                             [enc[w][0][l] for w in range(2)], SIZES[l], sharing)
            assert sec[i] == avg.tobytes(), (sharing, l); i += 1
    for l in range(3):  # SyncWorker N = 1 == decode(worker 0)
        st, dec = restated.decode(enc[0][0][l], SIZES[l], float(enc[0][1][l]))
        assert sec[i] == dec.tobytes(); i += 1
    g = grads[0][2]
    c, _ = restated.clip(g, 2.5)
    assert sec[i] == c.tobytes(); i += 1
    s = restated.scaler(c)
    assert sec[i] == np.float32(s).tobytes(); i += 1
    st, codes = restated.ternarize(c, s, 42, 3, "fc.weight", 0)
    assert sec[i] == bytes(codes); i += 1
    st, dec = restated.decode(codes, g.size, s)
    assert sec[i] == dec.tobytes(); i += 1
    msg = sec[i].decode()
    assert msg.startswith("ternarize: scaler 0.000000 below max |g| in fc.weight"), msg
    i += 1
    # FixedSize(1000) + passthrough conv.bias
    fx = Config(seed=42, bucketing=2, bucket_size=1000)
    pt = [0, 1, 0]
    for w in range(2):
        st, blocks, sc, _, _ = restated.encode_step(NAMES, grads[w], fx, 5, w, pt)
        assert st == 0
        assert sec[i] == sc.tobytes(); i += 1
        assert sec[i] == grads[w][1].tobytes(); i += 1
        assert sec[i] == b"".join(bytes(b) for b in blocks); i += 1
    for sharing in (True, False):
        fx.scaler_sharing = sharing
        flat = restated_average(restated, NAMES, grads, fx, 5, pt)
        assert sec[i] == flat.tobytes(), sharing; i += 1
    assert i == len(sec)
