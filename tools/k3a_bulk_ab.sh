#!/bin/bash
# sharded exchange (TGB_SHARD_MIN=3) with TMA bulk stores (K2 codes to owners, K3a sums to
# every rank) vs 16-B SM stores; default fused N = 4; local cluster parity (N = 2..8)
for b in 1 0 1 0; do bash tools/mp_sweep.sh shbulk${b}_n4 4 TGB_SHARD_MIN=3 TGB_K2BULK=$b; done
bash tools/mp_sweep.sh default_n4 4
bash tools/mp_sweep.sh default_n3 3
CUDA_MODULE_LOADING=EAGER CUDA_DEVICE_MAX_CONNECTIONS=32 timeout 800 python tools/local_cluster_check.py > gpurun_out/lc.json 2> gpurun_out/lc.err
python -c "
import json;d=json.load(open('gpurun_out/lc.json'));print('local cluster ok', d['ok'], len(d['checks']))"
