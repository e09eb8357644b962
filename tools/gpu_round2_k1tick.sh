# K1 per-CTA ticket wait: base vs release-atomic ticket vs no merge vs fire-and-forget ticket
LIB=paper_1705_07878_b200/lib/libtgb.so
cp $LIB build/libtgb_prod.so
for v in base rel nofin nowait; do
  cp build/libtgb_$v.so $LIB
  timeout 600 python tools/k1_sets.py > gpurun_out/r2o_k1_sets_$v.jsonl 2> gpurun_out/r2o_k1_sets_$v.err; echo $v rc=$?
done
for r in 1 2; do
  for v in base rel; do
    cp build/libtgb_$v.so $LIB
    line=$(python bench.py --steps 50 --warmup 5 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1)
    echo "{\"build\": \"$v\", \"round\": $r, \"line\": $line}" >> gpurun_out/r2o_ab.jsonl
  done
done
cp build/libtgb_prod.so $LIB
for v in base rel nofin nowait; do echo $v; cat gpurun_out/r2o_k1_sets_$v.jsonl | python -c '
import sys, json
for l in sys.stdin:
    d = json.loads(l); print(d["set"], d["n_workers"], round(d["k1"]["clean"]["mean_us"], 1), round(d["k1"]["hot"]["mean_us"], 1))'; done
python - <<'PY'
import json
for l in open("gpurun_out/r2o_ab.jsonl"):
    d = json.loads(l); x = d["line"]
    print(d["build"], d["round"], round(x["ms_per_step"], 4), {k: round(v["ms_per_launch"], 4) for k, v in x["kernels_live"].items()}, round(x["k1_l2_state"]["clean_l2_ms"], 4), x["clocks"]["sm_mhz"])
PY
