#!/bin/bash
# two-group schedule A/B at N = 2/4 (mp_check parity + tgb_step time): TGB_STAGGER x TGB_GPRIO x TGB_BSTREAM
for cfg in "0 1 0" "0 1 1" "1 1 1" "1 0 1" "2 1 1" "2 0 1"; do
  set -- $cfg
  for np in 2 4; do bash tools/mp_sweep.sh st$1_gp$2_bs$3_n$np $np TGB_STAGGER=$1 TGB_GPRIO=$2 TGB_BSTREAM=$3; done
done
