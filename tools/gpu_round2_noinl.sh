# K1 moments loop as a separate (noinline) function: K1 layouts + bench A/B vs base
LIB=paper_1705_07878_b200/lib/libtgb.so
cp $LIB build/libtgb_prod.so
for v in base noinl; do
  cp build/libtgb_$v.so $LIB
  timeout 600 python tools/k1_sets.py > gpurun_out/r2v_k1_sets_$v.jsonl 2> gpurun_out/r2v_k1_sets_$v.err; echo $v rc=$?
done
cp build/libtgb_base.so build/libtgb_old.so; cp build/libtgb_noinl.so $LIB
ORDER="new old" timeout 900 bash tools/lib_ab.sh 2 > gpurun_out/r2v_lib_ab.jsonl 2> gpurun_out/r2v_lib_ab.err; echo ab rc=$?
cp build/libtgb_prod.so $LIB
for v in base noinl; do echo $v; cat gpurun_out/r2v_k1_sets_$v.jsonl | python -c '
import sys, json
for l in sys.stdin:
    d = json.loads(l); print(d["set"], d["n_workers"], round(d["k1"]["clean"]["mean_us"], 1), round(d["k1"]["hot"]["mean_us"], 1))'; done
python - <<'PY'
import json
for l in open("gpurun_out/r2v_lib_ab.jsonl"):
    d = json.loads(l); x = d["line"]
    print(d["build"], d["round"], round(x["ms_per_step"], 4), {k: round(v["ms_per_launch"], 4) for k, v in x["kernels_live"].items()}, round(x["k1_l2_state"]["clean_l2_ms"], 4), x["clocks"]["sm_mhz"])
PY
