#!/bin/bash
# radix-3 wire codes A/B at N = 3 / 4 (mp_check parity + tgb_step time), then the GPU test suite
for r in 1 0 1 0; do for np in 4 3; do bash tools/mp_sweep.sh r3_${r}_n$np $np TGB_R3=$r; done; done
TGB_R3=1 torchrun --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29641 tools/step_timeline.py 2>/dev/null | grep "^{" > gpurun_out/tl4_r3.json
python -m pytest tests -m gpu -x -q 2>&1 | tail -2
