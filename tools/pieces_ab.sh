#!/bin/bash
# dominant-layer pieces A/B (TGB_PIECES x K3-piece stream priority TGB_P3PRIO), barriers on the
# greatest-priority stream; mp_check parity + tgb_step time at N = 2 / 4
for cfg in "1 1" "2 1" "4 1" "4 0" "8 0" "3 0"; do
  set -- $cfg
  for np in 4 2; do bash tools/mp_sweep.sh pc$1_p3$2_n$np $np TGB_PIECES=$1 TGB_P3PRIO=$2; done
done
