#!/bin/bash
# TGB_K2BULK A/B: K2 code stores as TMA bulk copies vs 16-B SM stores (N = 2 / 4 mp_check, N = 1 bench)
for b in 1 0 1 0; do
  for np in 4 2; do bash tools/mp_sweep.sh bulk${b}_n$np $np TGB_K2BULK=$b; done
  TGB_K2BULK=$b python bench.py --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('bulk=$b N=1', round(d['ms_per_step']*1e3,1))"
done
CUDA_MODULE_LOADING=EAGER CUDA_DEVICE_MAX_CONNECTIONS=32 timeout 800 python tools/local_cluster_check.py > gpurun_out/lc.json 2> gpurun_out/lc.err
python -c "
import json;d=json.load(open('gpurun_out/lc.json'));print('local cluster ok', d['ok'], len(d['checks']))"
