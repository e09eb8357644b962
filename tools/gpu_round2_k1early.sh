# K1: do the warps that exit before the ticket free their SM slot early? (timing probes)
LIB=paper_1705_07878_b200/lib/libtgb.so
cp $LIB build/libtgb_prod.so
for v in nofin early nowait; do
  cp build/libtgb_$v.so $LIB
  timeout 600 python tools/k1_sets.py > gpurun_out/r2p_k1_sets_$v.jsonl 2> gpurun_out/r2p_k1_sets_$v.err; echo $v rc=$?
done
cp build/libtgb_prod.so $LIB
for v in nofin early nowait; do echo $v; cat gpurun_out/r2p_k1_sets_$v.jsonl | python -c '
import sys, json
for l in sys.stdin:
    d = json.loads(l); print(d["set"], d["n_workers"], round(d["k1"]["clean"]["mean_us"], 1), round(d["k1"]["hot"]["mean_us"], 1))'; done
