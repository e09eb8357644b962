"""Multi-GPU parity (needs >= 2 GPUs; skipped on single-GPU boxes).

Runs tools/mp_check.py under torchrun for the fused NVLink exchange and the
NCCL-allgather exchange: every rank must hold bit-identical averaged
gradients equal to the reference's average over the same workers
(REF shared, unshared, and PRESHARED against its own oracle).
"""
import json
import os
import subprocess
import sys

import pytest
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

pytestmark = [pytest.mark.gpu, pytest.mark.multigpu]


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs >= 2 GPUs")
@pytest.mark.parametrize("exchange", ["fused", "nccl"])
def test_mp_check(exchange):
    n = min(4, torch.cuda.device_count())
    env = dict(os.environ, TGB_EXCHANGE=exchange)
    port = 29600 + (1 if exchange == "nccl" else 0)
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        f"--nproc-per-node={n}", "--master-addr", "127.0.0.1",
                        "--master-port", str(port), os.path.join(ROOT, "tools", "mp_check.py")],
                       capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)
    line = [x for x in r.stdout.splitlines() if x.startswith("{")]
    assert r.returncode == 0 and line, r.stdout[-2000:] + r.stderr[-2000:]
    rep = json.loads(line[0])
    assert rep["world_size"] == n
    for k, v in rep["checks"].items():
        assert v["ranks_identical"], k
        assert v["matches_oracle"], k
