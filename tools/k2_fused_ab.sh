#!/bin/bash
# K2 variant A/B (TGB_K2V): N = 1 bench (fused decode K2, live timing) and N = 2 / 4 mp_check
# (unfused K2 with peer stores)
for v in 3 4 6 3; do
  TGB_K2V=$v python bench.py --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels_live']
print('K2V=$v N=1 step', round(d['ms_per_step']*1e3,1), 'us; live K2+decode', round(k['K2_ternarize_pack+decode']['ms_per_launch']*1e3,1), 'us', round(k['K2_ternarize_pack+decode']['frac'],3))"
done
for v in 0 3 0 3; do for np in 2 4; do bash tools/mp_sweep.sh k2v${v}_n$np $np TGB_K2V=$v; done; done
