#!/bin/bash
# Same-box A/B of two builds of libtgb.so: the in-tree build (new) against
# build/libtgb_old.so (old), alternating, N = 1 bench.py kernel-only lines.
# usage: tools/lib_ab.sh [rounds] > gpurun_out/lib_ab.jsonl
R=${1:-3}
LIB=paper_1705_07878_b200/lib/libtgb.so
cp $LIB build/libtgb_new.so
for r in $(seq $R); do
  for v in ${ORDER:-new old}; do
    cp build/libtgb_$v.so $LIB
    line=$(python bench.py --steps 50 --warmup 5 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1)
    echo "{\"build\": \"$v\", \"round\": $r, \"line\": $line}"
  done
done
cp build/libtgb_new.so $LIB
