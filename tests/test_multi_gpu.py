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


def test_local_cluster_n8_on_one_gpu():
    """N = 2/3/5/8 workers as plans of one process on cuda:0 (tgb_plan_attach_local):
    the fused and sharded exchange kernels (incl. N = 8's 8-bit sums) bit-identical
    on every worker and equal to the reference's average / the allgather path."""
    env = dict(os.environ, CUDA_DEVICE_MAX_CONNECTIONS="32", CUDA_MODULE_LOADING="EAGER")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "local_cluster_check.py")],
                       capture_output=True, text=True, timeout=900, env=env, cwd=ROOT)
    line = [x for x in r.stdout.splitlines() if x.startswith("{")]
    assert line, r.stdout[-2000:] + r.stderr[-2000:]
    rep = json.loads(line[0])
    bad = {k: v for k, v in rep["checks"].items()
           if not (v["workers_identical"] and v["matches_reference"])}
    assert not bad and r.returncode == 0, bad
    assert rep["checks"]["N=8,vgg16"]["exchange"] == "sharded"
