# K1 layouts: production build vs a build without the per-tensor finalize (timing only)
LIB=paper_1705_07878_b200/lib/libtgb.so
cp $LIB build/libtgb_new.so
timeout 600 python tools/k1_sets.py > gpurun_out/r2i_k1_sets_prod.jsonl 2> gpurun_out/r2i_k1_sets_prod.err; echo prod rc=$?
cp build/libtgb_nofin.so $LIB
timeout 600 python tools/k1_sets.py > gpurun_out/r2i_k1_sets_nofin.jsonl 2> gpurun_out/r2i_k1_sets_nofin.err; echo nofin rc=$?
cp build/libtgb_new.so $LIB
for f in gpurun_out/r2i_k1_sets_*.jsonl; do echo $f; cat $f | python -c '
import sys, json
for l in sys.stdin:
    d = json.loads(l); print(d["set"], d["n_workers"], round(d["k1"]["clean"]["mean_us"], 1), round(d["k1"]["hot"]["mean_us"], 1))'; done
