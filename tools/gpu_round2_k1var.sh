# K1 fixed overhead: production vs no tensor merge vs no launch_dependents (same box)
LIB=paper_1705_07878_b200/lib/libtgb.so
cp $LIB build/libtgb_prod.so
tools/k1_variants quick > gpurun_out/r2l_k1_variants.log 2>&1
for v in prod nofin nodep; do
  cp build/libtgb_$v.so $LIB
  timeout 600 python tools/k1_sets.py > gpurun_out/r2l_k1_sets_$v.jsonl 2> gpurun_out/r2l_k1_sets_$v.err; echo $v rc=$?
done
cp build/libtgb_prod.so $LIB
grep "V0 prod" gpurun_out/r2l_k1_variants.log | tail -2
for v in prod nofin nodep; do echo $v; cat gpurun_out/r2l_k1_sets_$v.jsonl | python -c '
import sys, json
for l in sys.stdin:
    d = json.loads(l); print(d["set"], d["n_workers"], round(d["k1"]["clean"]["mean_us"], 1), round(d["k1"]["hot"]["mean_us"], 1))'; done
