# deferred K1 + k1_merge: GPU tests, K1 layouts, same-box A/B vs the in-kernel finalize
timeout 2400 python -m pytest tests -q -m gpu -x > gpurun_out/r2q_tests.log 2>&1; echo tests rc=$?
tail -n 3 gpurun_out/r2q_tests.log
timeout 600 python tools/k1_sets.py > gpurun_out/r2q_k1_sets.jsonl 2> gpurun_out/r2q_k1_sets.err; echo sets rc=$?
cat gpurun_out/r2q_k1_sets.jsonl | python -c '
import sys, json
for l in sys.stdin:
    d = json.loads(l); print(d["set"], d["n_workers"], round(d["k1"]["clean"]["mean_us"], 1), round(d["k1"]["hot"]["mean_us"], 1))'
cp build/libtgb_base.so build/libtgb_old.so
ORDER="new old" timeout 900 bash tools/lib_ab.sh 3 > gpurun_out/r2q_lib_ab.jsonl 2> gpurun_out/r2q_lib_ab.err; echo ab rc=$?
python - <<'PY'
import json
for l in open("gpurun_out/r2q_lib_ab.jsonl"):
    d = json.loads(l); x = d["line"]
    print(d["build"], d["round"], round(x["ms_per_step"], 4), {k: round(v["ms_per_launch"], 4) for k, v in x["kernels_live"].items()}, round(x["k1_l2_state"]["clean_l2_ms"], 4), x["clocks"]["sm_mhz"])
PY
timeout 600 python tools/fixed_probe.py > gpurun_out/r2q_fixed_probe.json 2> gpurun_out/r2q_fixed_probe.err; echo fixed rc=$?
timeout 600 python tools/small_sets.py > gpurun_out/r2q_small_sets.jsonl 2> gpurun_out/r2q_small_sets.err; echo small rc=$?
