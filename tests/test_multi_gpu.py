"""Multi-GPU parity.

* test_mp_check: tools/mp_check.py under torchrun, one process per GPU, for
  N in {2, 4, 8} that fit the visible GPUs and every exchange (fused NVLink
  stores, sharded owner sums, NCCL allgather, fused with 3/8 of the codes pulled
  by the decode): every rank holds bit-identical
  averaged gradients equal to the reference's average over the same workers
  (small sets: REF shared / unshared, Global, FixedSize + passthrough, PRESHARED
  against its own oracle; full AlexNet and VGG-16 sets against the reference's
  ParameterServer path), and the protocol checks (iteration skew, block
  structure mismatch) raise the reference's ProtocolError texts.
* test_local_cluster: N = 2..8 workers as plans of ONE process on cuda:0
  (tools/local_cluster_check.py) -- the same exchange kernels without NVLink.
"""
import json
import os
import subprocess
import sys

import pytest
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

pytestmark = [pytest.mark.gpu]

_NGPU = torch.cuda.device_count() if torch.cuda.is_available() else 0
_EXCHANGES = ("auto", "sharded", "nccl", "fused+pull")  # +pull: split exchange, 3/8 pulled
_CASES = [(n, ex) for n in (2, 4, 8) if n <= _NGPU for ex in _EXCHANGES]


@pytest.mark.multigpu
@pytest.mark.skipif(_NGPU < 2, reason="needs >= 2 GPUs")
@pytest.mark.parametrize("n,exchange", _CASES or [(2, "auto")])
def test_mp_check(n, exchange):
    env = dict(os.environ, TGB_EXCHANGE=exchange.split("+")[0],
               TGB_PULL="3" if exchange.endswith("+pull") else "0")
    port = 29600 + 10 * n + _EXCHANGES.index(exchange)
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        f"--nproc-per-node={n}", "--master-addr", "127.0.0.1",
                        "--master-port", str(port), os.path.join(ROOT, "tools", "mp_check.py")],
                       capture_output=True, text=True, timeout=1800, env=env, cwd=ROOT)
    line = [x for x in r.stdout.splitlines() if x.startswith("{")]
    assert r.returncode == 0 and line, r.stdout[-3000:] + r.stderr[-3000:]
    rep = json.loads(line[0])
    assert rep["world_size"] == n
    for k, v in rep["checks"].items():
        assert v["ranks_identical"], k
        assert v["matches_oracle"] in (True, None), k
    for k in ("googlenet_full_set", "alexnet_full_set", "vgg16_full_set"):
        assert rep["checks"][k]["matches_oracle"] is True, k
    if exchange != "nccl":
        assert "iteration_skew" in rep["checks"] and "block_structure_mismatch" in rep["checks"]


def test_local_cluster():
    """N = 2..8 workers of one process on cuda:0: fused and sharded exchanges
    bit-identical on every worker and equal to the reference's average; the
    iteration-skew check. No launch-environment settings are needed."""
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "local_cluster_check.py")],
                       capture_output=True, text=True, timeout=900, cwd=ROOT)
    line = [x for x in r.stdout.splitlines() if x.startswith("{")]
    assert line, r.stdout[-2000:] + r.stderr[-2000:]
    rep = json.loads(line[0])
    bad = {k: v for k, v in rep["checks"].items()
           if not (v["workers_identical"] and v["matches_reference"])}
    assert not bad and r.returncode == 0, bad
    assert rep["checks"]["N=8,exchange=sharded,sharing=True,bucketing=PerTensor,"
                         "passthrough=-"]["exchange"] == "sharded"
